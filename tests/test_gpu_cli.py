"""`gsgp-run -backend cuda` end to end on the B200 against the reference
CLI's own output for the same inputs (tests/golden/cli_ref)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2106_04034_b200 as G

pytestmark = pytest.mark.gpu

REF = GOLDEN / "cli_ref"


def _cli(tmp_path, *extra):
    out = tmp_path / "out"
    code = G.run_cli(["-train_file", str(REF / "train.txt"), "-test_file", str(REF / "test.txt"),
                      "-config", str(REF / "config.ini"), "-output_dir", str(out), "-backend", "cuda",
                      *extra])
    assert code == 0
    return out


def _split_sidecar(path):
    """(config lines without backend, plan lines, elite (src, idx, slot), fitness values)."""
    cfg, plans, elites, fits = [], [], [], []
    for line in path.read_text().splitlines():
        tok = line.split()
        if line.startswith(("init_elite ", "elite ")):
            elites.append(tuple(tok[1:4]))
            fits.append(float(tok[4]))
        elif line.startswith(("#", "gen ")):
            plans.append(line)
        elif "=" in line:
            if not line.startswith("backend"):
                cfg.append(line)
        else:
            plans.append(line)
    return cfg, plans, elites, np.array(fits)


@pytest.mark.parametrize("storage,rtol", [("fp32", 1e-5), ("fp64", 1e-12)])
def test_cli_matches_reference_cli(tmp_path, storage, rtol):
    out = _cli(tmp_path, "-storage", storage)
    for name in ("fitnesstrain.txt", "fitnesstest.txt"):
        ours = np.loadtxt(out / name)
        ref = np.loadtxt(REF / "out" / name)
        assert ours.shape == ref.shape == (2 * 13,)          # 2 runs x (g + 1) lines
        np.testing.assert_allclose(ours, ref, rtol=rtol, atol=0)
    for run in (0, 1):
        a = _split_sidecar(out / f"lineage_run{run:03d}.txt")
        b = _split_sidecar(REF / "out" / f"lineage_run{run:03d}.txt")
        assert a[0] == b[0]            # same effective config (incl. derived seed)
        assert a[1] == b[1]            # plan lines byte-identical (u, v, %.17g ms)
        assert a[2] == b[2]            # elite source / index / slot identical
        np.testing.assert_allclose(a[3], b[3], rtol=rtol, atol=0)
    assert (out / "timings.csv").read_text().splitlines()[0] == "m,n,k,backend,workers,stage,millis"


def test_replay_from_cli_sidecar_matches_reference_elite(tmp_path):
    out = _cli(tmp_path, "-storage", "fp64")
    cfg, log = G.read_lineage_sidecar(out / "lineage_run000.txt")
    train = G.load_dataset(REF / "train.txt")
    pop = G.create_population(cfg.population_size, cfg, 0, train.n_features)
    trees = G.create_population(cfg.random_trees, cfg, cfg.population_size, train.n_features)
    rep = G.replay_lineage(log, G.compute_semantics(pop, train, cfg),
                           G.compute_semantics(trees, train, cfg), cfg)
    fin = G.rmse(rep, train.target)
    assert fin == pytest.approx(log.final_elite().fitness, rel=1e-12)


def test_timed_run_and_sweep_on_device():
    rows = G.sweep([{"m": 64, "n": 500, "k": 31}, {"m": 0, "n": 10, "k": 3}], generations=3)
    stages = [r["stage"] for r in rows]
    assert stages[:4] == ["create_population", "compute_semantics", "generation", "total"]
    assert stages[-1] == "error"
    assert all(r["millis"] >= 0 for r in rows[:4])


def test_bench_cli_program_size_sweep(tmp_path):
    """gsgp-bench (gsgp/harness.py:130-152) on the device: one CSV row per
    stage and cell in the reference schema; ComputeSemantics time grows with
    program size (the paper's k sensitivity, pkg/tests/test_harness.py:62-68)."""
    import csv

    from paper_2106_04034_b200.harness import main
    out = tmp_path / "sweep.csv"
    assert main(["--m", "256", "--n", "400000", "--k", "127,1023,2047", "--out", str(out)]) == 0
    with open(out, newline="") as fh:
        rows = list(csv.DictReader(fh))
    assert len(rows) == 12 and {r["stage"] for r in rows} == {
        "create_population", "compute_semantics", "generation", "total"}
    sem = [float(r["millis"]) for r in rows if r["stage"] == "compute_semantics"]
    # the 2047-gene programs take longer than the 1023-gene ones; the first
    # (127-gene) cell can carry one-time costs (lazy kernel loading of the
    # interpreter configuration it selects, a trimmed block cache) and is
    # not compared
    assert sem[2] > sem[1]


def _cli_rank(rank, world, port, out_dir, q):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank), GSGP_SHARED_GPU="1")
    import paper_2106_04034_b200 as G2
    code = G2.run_cli(["-train_file", str(REF / "train.txt"), "-test_file", str(REF / "test.txt"),
                       "-config", str(REF / "config.ini"), "-output_dir", str(out_dir), "-backend", "cuda"])
    import torch.distributed as td
    if td.is_initialized():
        td.destroy_process_group()
    q.put((rank, code))


def test_cli_replicas_over_two_ranks_match_single_process(tmp_path):
    """gsgp-run under 2 ranks (runs as replicas, both ranks on this GPU):
    trace files in run order and sidecars identical to the one-process CLI."""
    import socket

    import torch.multiprocessing as mp
    one = _cli(tmp_path)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out2 = tmp_path / "rep"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cli_rank, args=(r, 2, port, out2, q)) for r in range(2)]
    for p in procs:
        p.start()
    codes = sorted(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    assert codes == [(0, 0), (1, 0)]
    for name in ("fitnesstrain.txt", "fitnesstest.txt", "lineage_run000.txt", "lineage_run001.txt"):
        assert (out2 / name).read_text() == (one / name).read_text(), name
