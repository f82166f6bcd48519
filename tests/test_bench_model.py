"""bench.py's derived numbers that do not need a GPU: the interpreter's
shared-memory wavefront model and the workload config labels."""

from __future__ import annotations

import types

import pytest

import bench


def _res(cfg, ins, ops):
    return types.SimpleNamespace(device={"interpreter": {"config": cfg}, "program_instructions": ins,
                                         "program_operands": ops})


def test_smem_wavefront_model_counts_operand_traffic():
    ins = {"population": 100, "pool": 50}
    ops = {"population": {"vector_loads": 80, "constant_loads": 20, "spill_stores": 10},
           "pool": {"vector_loads": 40, "constant_loads": 10, "spill_stores": 5}}
    N, t = 512 * 1000, 0.5
    s = bench.smem_roofline(_res(10, ins, ops), N, t)
    cpt = 4
    per_warp = 150 + cpt * (2 * 120 + 30 + 2 * 15)     # fetch + 2/case vector + 1/case const + 2/case store
    assert s["wavefronts"] == pytest.approx(per_warp * N / (32 * cpt))
    assert s["frac"] == pytest.approx(s["achieved"] / s["peak"])
    assert s["cases_per_thread"] == cpt
    # features left in HBM (cfg 2) or an unknown configuration: no shared-memory model
    assert bench.smem_roofline(_res(2, ins, ops), N, t) is None
    assert bench.smem_roofline(_res(8, ins, ops), N, t) is None


def test_l2_label_follows_the_semantics_bytes():
    for name, c in bench.CONFIGS.items():
        label = bench.workload_config(c)["l2"]
        big = 4 * c["m"] * (c["ntr"] + c["nte"]) > bench.L2_BYTES
        assert label.startswith("inputs larger than L2") == big, name
    assert bench.workload_config(bench.CONFIGS["c1"])["l2"].startswith("small")
    assert bench.workload_config(bench.CONFIGS["c4"])["l2"].startswith("inputs larger")
