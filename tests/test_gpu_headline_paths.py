"""Parity of the kernel configurations the benchmarks actually run.

The generation kernel claims work units (one 16 KB case tile of one
population row) in batches of 2..32, chosen from the work per CTA (C2 runs
batch 4, C3/C4/C5 batch 16), and the canonical SSE reduce has three shapes
chosen from the units per row: one load per lane (<= 32 units, C2 = 31),
a warp per row with 8 loads in flight (33..1024, C4 ~306, C5 ~611) and a
256-thread block per row (> 1024, C3 ~3053).  These tests run each of those
paths against

* reference-generated goldens at headline shapes (tests/golden/big_*.npz,
  make_golden.py BIG_RUNS: c2 = the C2 shape itself for 5 generations,
  mid = 123 units per row, long = 1124 units per row; data regenerated from
  the make_benchmark_dataset seeds): elite records and plans bit-exact,
  traces <= 1e-5 relative (fp32 storage) or 1e-12 (fp64 storage), sampled
  elite semantics <= 1e-5 relative;
* oracle/engine32.run32 (the engine's fp32 arithmetic restated): elite
  records identical, traces to 1e-12, elite semantics bit-identical;

for every forced claim batch, and check that the fused single-shard tail
equals the multi-shard (anchors -> digits -> finish) tail bit for bit.
(gsgp/fitness.py:28-51, gsgp/evolution.py:146-158.)
"""

from __future__ import annotations

import ast
import functools

import numpy as np
import pytest

from conftest import golden
from oracle import engine32, restate as R

pytestmark = pytest.mark.gpu

import paper_2106_04034_b200 as G  # noqa: E402

RTOL = 1e-5
TILE32 = 4096          # fp32 cases per 16 KB generation tile
TILE64 = 2048


def units_per_row(ntr: int, nte: int, tile: int) -> int:
    """make_layout (gsm.cu): train region padded to 32 cases, test tail merged
    into the train tail unit when both fit one tile."""
    pad = lambda x: (x + 31) // 32 * 32  # noqa: E731
    ntr_pad = pad(ntr)
    ttr = (ntr_pad + tile - 1) // tile
    tail_tr, tail_te = ntr_pad % tile, nte % tile
    if tail_tr and tail_te and tail_tr + pad(tail_te) <= tile:
        return ttr + (nte - tail_te) // tile
    return ttr + (pad(nte) + tile - 1) // tile


@functools.lru_cache(maxsize=None)
def _case(name: str):
    g = golden(f"big_{name}")
    ntr, l, s1, nte, s2 = (int(x) for x in g["data"])
    train = G.make_benchmark_dataset(ntr, l, seed=s1)
    test = G.make_benchmark_dataset(nte, l, seed=s2)
    kw = ast.literal_eval(str(g["cfg"][0]))
    return g, kw, train, test


@functools.lru_cache(maxsize=None)
def _engine32(name: str):
    g, kw, train, test = _case(name)
    return engine32.run32(R.Cfg(**kw), train.features, train.target, test.features, test.target)


def _check_golden(res, g, tol):
    ents = res.lineage.entries
    assert [0 if e.elite.source == "parent" else 1 for e in ents] == g["src"].tolist()
    assert [e.elite.index for e in ents] == g["idx"].tolist()
    assert [e.elite.slot for e in ents] == g["slot"].tolist()
    assert res.lineage.initial_elite.index == int(g["init"][0])
    for t, e in enumerate(ents):
        assert np.array_equal(e.plan.u, g["u"][t]) and np.array_equal(e.plan.v, g["v"][t])
        assert np.array_equal(e.plan.ms, g["ms"][t])
    np.testing.assert_allclose(res.train_fitness, g["train"], rtol=tol, atol=0)
    np.testing.assert_allclose(res.test_fitness, g["test"], rtol=tol, atol=0)
    ref = g["elite_sem_sample"]
    got = res.elite_train_semantics[::int(g["sample_stride"][0])]
    assert np.max(np.abs(got - ref)) <= tol * np.max(np.abs(ref))
    assert res.elite_slot == int(g["slot_final"][0])
    assert res.overflow_replacements == int(g["overflow"][0])


def test_golden_shapes_cover_every_reduce_path():
    """The three goldens land in the three reduce kernels (and C3 in the
    block-per-row one)."""
    got = {}
    for name in ("c2", "mid", "long"):
        ntr, _, _, nte, _ = (int(x) for x in golden(f"big_{name}")["data"])
        got[name] = units_per_row(ntr, nte, TILE32)
    assert got["c2"] <= 32 < got["mid"] <= 1024 < got["long"]
    assert units_per_row(10_000_000, 2_500_000, TILE32) > 1024          # C3
    assert 32 < units_per_row(1_000_000, 250_000, TILE32) <= 1024      # C4
    assert 32 < units_per_row(2_000_000, 500_000, TILE32) <= 1024      # C5


@pytest.mark.parametrize("batch", [None, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("name", ["c2", "mid", "long"])
def test_headline_shape_matches_reference_golden(name, batch, monkeypatch):
    if batch is not None:
        monkeypatch.setenv("GSGP_GSM_BATCH", str(batch))
    g, kw, train, test = _case(name)
    res = G.run_evolution(G.RunConfig(**kw), train, test)
    assert res.device["storage"] == "fp32"
    _check_golden(res, g, RTOL)


@pytest.mark.parametrize("name", ["c2", "mid", "long"])
def test_headline_shape_fp64_storage_matches_reference_tightly(name, monkeypatch):
    monkeypatch.setenv("GSGP_GSM_BATCH", "16")
    g, kw, train, test = _case(name)
    res = G.run_evolution(G.RunConfig(**kw), train, test, storage="fp64")
    _check_golden(res, g, 1e-12)


@pytest.mark.parametrize("batch", [2, 4, 16, 32])
@pytest.mark.parametrize("name", ["mid", "long"])
def test_headline_shape_bit_exact_vs_engine_restatement(name, batch, monkeypatch):
    monkeypatch.setenv("GSGP_GSM_BATCH", str(batch))
    g, kw, train, test = _case(name)
    o = _engine32(name)
    res = G.run_evolution(G.RunConfig(**kw), train, test)
    assert [(e.elite.source, e.elite.index, e.elite.slot) for e in res.lineage.entries] == \
        [e[:3] for e in o["elite"]]
    np.testing.assert_allclose(res.train_fitness, o["train"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(res.test_fitness, o["test"], rtol=1e-12, atol=0)
    assert np.array_equal(res.elite_train_semantics, o["elite_train_semantics"])


def _fingerprint(res):
    return ([(e.elite.source, e.elite.index, e.elite.slot) for e in res.lineage.entries],
            res.train_fitness.tobytes(), res.test_fitness.tobytes(), res.elite_train_semantics.tobytes())


@pytest.mark.parametrize("storage", ["fp32", "fp64"])
def test_wide_rows_fused_tail_equals_sharded_tail(storage, monkeypatch):
    """> 1024 units per row: the fused single-shard reduce (anchors from the
    GSM finalizer, block-per-row digit merge) gives the same bits as the
    multi-shard canon_exp -> canon_digits -> canon_finish path."""
    monkeypatch.setenv("GSGP_GSM_BATCH", "16")
    g, kw, train, test = _case("long")
    cfg = G.RunConfig(**kw)
    fused = _fingerprint(G.run_evolution(cfg, train, test, storage=storage))
    for shards in (2, 3):
        assert _fingerprint(G.run_evolution(cfg, train, test, storage=storage,
                                            virtual_shards=shards)) == fused
