"""CPU oracle for the GSGP hot path — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_2106_04034_b200`) imports this
package.  It may be used only by `tests/`, by `__graft_entry__.smoke()` (as
the checker) and by `bench.py` (the `cpu_baseline` leg and `--impl
reference`).  The product path has no CPU fallback: if the CUDA library is
missing it raises.

`restate` is a numpy restatement of the reference package `gsgp` 0.1.0
(`/root/reference/pkg/src/gsgp`), function by function, each citing the
reference file:line it follows.  It is pinned against golden vectors that
`tests/golden/make_golden.py` produced by importing the real reference in the
build container (`tests/test_oracle_golden.py`).

`engine32` restates, op for op, the arithmetic the B200 engine performs
(fp32 semantic storage, fp32 GSM update, fp64 SSE), so element-level kernel
outputs can be checked bit-exactly.
"""
