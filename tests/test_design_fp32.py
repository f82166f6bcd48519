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
