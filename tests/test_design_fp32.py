"""CPU validation of the engine's fp32-storage design against the reference.

oracle/engine32.py restates the device arithmetic (fp32 semantic storage,
fp64 interpreter and SSE, fp32-overflow slots).  Run on the golden reference
runs it must reproduce the reference's elite/selection trace exactly and the
RMSE traces within the north-star tolerance (1e-5 relative) — the parity
contract the GPU engine is then held to in tests/test_gpu_run.py.
"""

from __future__ import annotations

import ast

import numpy as np
import pytest

from conftest import golden
from oracle import engine32, restate as R

RTOL = 1e-5


@pytest.mark.parametrize("name", ["tiny", "small", "plus", "g0", "accept", "c1", "c2s", "wide", "m1",
                                  "k1", "n1", "const", "funcs"])
def test_fp32_storage_reproduces_reference(name):
    g = golden(f"run_{name}")
    cfg = R.Cfg(**ast.literal_eval(str(g["cfg"][0])))
    out = engine32.run32(cfg, g["Xtr"], g["ytr"], g["Xte"], g["yte"])
    src = np.array([0 if e[0] == "parent" else 1 for e in out["elite"]], np.int8)
    assert np.array_equal(src, g["src"])
    assert [e[1] for e in out["elite"]] == g["idx"].tolist()
    assert [e[2] for e in out["elite"]] == g["slot"].tolist()
    np.testing.assert_allclose(out["train"], g["train"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(out["test"], g["test"], rtol=RTOL, atol=0)
    ref = g["elite_sem"]
    assert np.max(np.abs(out["elite_train_semantics"] - ref)) <= RTOL * np.max(np.abs(ref))
    assert out["overflow"] == int(g["overflow"][0])


def test_fp32_overflow_slots_are_needed_and_sufficient():
    """k=1024 genomes overflow fp32 in a few rows (SURVEY §7 hard part 3).  In
    the reference those values never change (|x| > FLT_MAX absorbs any
    |delta| <= 2), so the slot's fitness is constant; the engine keeps it.
    Golden run 'wide' has 5 such rows: with the mechanism the elite trace is
    the reference's, without it argmax ties among inf rows pick other slots."""
    g = golden("run_wide")
    cfg = R.Cfg(**ast.literal_eval(str(g["cfg"][0])))
    out = engine32.run32(cfg, g["Xtr"], g["ytr"], g["Xte"], g["yte"])
    assert sorted(np.nonzero(out["wide0"])[0].tolist()) == [181, 394, 513, 585, 921]
    assert [e[2] for e in out["elite"]] == g["slot"].tolist()
    plain = engine32.run32(cfg, g["Xtr"], g["ytr"], g["Xte"], g["yte"], wide_slots=False)
    assert [e[2] for e in plain["elite"]] != g["slot"].tolist()


def test_gsm_step32_rounding_order():
    P = np.array([[1.0]], np.float32)
    Q = np.array([[0.8], [0.3]], np.float32)
    o = engine32.gsm_step32(P, Q, np.array([0]), np.array([1]), np.array([0.1]))
    t = np.float32(np.float32(0.8) - np.float32(0.3)) * np.float32(0.1)
    assert o[0, 0] == np.float32(np.float32(1.0) + np.float32(t))
    assert abs(float(o[0, 0]) - 1.05) < 1e-6


@pytest.mark.parametrize("name", ["hugestep", "infstep"])
def test_fp32_storage_is_unsafe_for_huge_constant_steps(name):
    """gsgp/core.py:332-336 accepts any finite positive constant step.  With
    steps near FLT_MAX (1e38 plus-sign; 1e39 > FLT_MAX) plain fp32 storage
    overflows where the fp64 reference stays finite, and the survival slots
    diverge — which is why the engine stores such runs in fp64 (engine.cu:
    step * (1|2) * g >= 2^70).  The fp64 restatement is the reference."""
    g = golden(f"run_{name}")
    cfg = R.Cfg(**ast.literal_eval(str(g["cfg"][0])))
    with np.errstate(all="ignore"):
        out = engine32.run32(cfg, g["Xtr"], g["ytr"], g["Xte"], g["yte"])
    assert [e[2] for e in out["elite"]] != g["slot"].tolist()
    ref = R.run(cfg, g["Xtr"], g["ytr"], g["Xte"], g["yte"])
    assert [e[2] for e in ref["elite"]] == g["slot"].tolist()


@pytest.mark.parametrize("name", ["mid", "long"])
def test_fp32_storage_reproduces_reference_at_headline_shapes(name):
    """The fp32 design against the reference-generated headline-shape goldens
    (make_golden.py BIG_RUNS; data regenerated from the benchmark seeds)."""
    g = golden(f"big_{name}")
    ntr, l, s1, nte, s2 = (int(x) for x in g["data"])
    Xtr, ytr = R.benchmark_dataset(ntr, l, s1)
    Xte, yte = R.benchmark_dataset(nte, l, s2)
    out = engine32.run32(R.Cfg(**ast.literal_eval(str(g["cfg"][0]))), Xtr, ytr, Xte, yte)
    assert [e[2] for e in out["elite"]] == g["slot"].tolist()
    assert [e[1] for e in out["elite"]] == g["idx"].tolist()
    np.testing.assert_allclose(out["train"], g["train"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(out["test"], g["test"], rtol=RTOL, atol=0)
    ref = g["elite_sem_sample"]
    got = out["elite_train_semantics"][::int(g["sample_stride"][0])]
    assert np.max(np.abs(got - ref)) <= RTOL * np.max(np.abs(ref))
