"""File-format compatibility with the reference CLI (tests/golden/cli_ref was
written by the reference's own `gsgp-run`).  CPU only; the end-to-end CLI run
on the device is in tests/test_gpu_cli.py."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2106_04034_b200 as G
from paper_2106_04034_b200 import io_cli

REF = GOLDEN / "cli_ref"


def test_reference_config_loads():
    cfg = G.load_config(REF / "config.ini")
    assert (cfg.population_size, cfg.random_trees, cfg.program_size, cfg.generations, cfg.runs,
            cfg.seed) == (24, 16, 31, 12, 2, 4242)
    assert cfg.mutation_step == "uniform"


def test_reference_dataset_loads_and_rewrites_byte_identical(tmp_path):
    ds = G.load_dataset(REF / "train.txt")
    assert ds.features.shape == (60, 3) and ds.target.shape == (60,)
    G.write_dataset(tmp_path / "t.txt", ds)
    assert (tmp_path / "t.txt").read_bytes() == (REF / "train.txt").read_bytes()


@pytest.mark.parametrize("run", [0, 1])
def test_reference_sidecar_round_trips_byte_identical(tmp_path, run):
    src = REF / "out" / f"lineage_run{run:03d}.txt"
    cfg, log = G.read_lineage_sidecar(src)
    assert log.generations == cfg.generations == 12
    assert all(len(e.plan) == cfg.population_size for e in log.entries)
    G.write_lineage_sidecar(tmp_path / "s.txt", cfg, log)
    assert (tmp_path / "s.txt").read_bytes() == src.read_bytes()


def test_config_errors(tmp_path):
    p = tmp_path / "c.ini"
    for text in ("tournament_size = 4\n", "population_size = many\n", "just words\n",
                 "backend = gpu\n"):
        p.write_text(text)
        with pytest.raises(G.ConfigError):
            G.load_config(p)
    p.write_text("; comment\n# comment\n[section]\nbackend = cuda\nmutation_step = 0.25\n")
    cfg = G.load_config(p)
    assert cfg.backend == "cuda" and cfg.mutation_step == 0.25
    assert "mutation_step = 0.25" in io_cli.config_lines(cfg)
    assert "backend = cuda" in io_cli.config_lines(cfg)


@pytest.mark.parametrize("text", ["1 2\n3\n", "1 x\n", "1 nan\n", "", "\n\n", "5\n6\n"])
def test_dataset_errors(tmp_path, text):
    p = tmp_path / "d.txt"
    p.write_text(text)
    with pytest.raises(G.DatasetFormatError):
        G.load_dataset(p)


def test_dataset_crlf_and_tabs(tmp_path):
    p = tmp_path / "d.txt"
    p.write_bytes(b"1\t2 3\r\n4 5\t6\r\n")
    ds = G.load_dataset(p)
    assert np.array_equal(ds.features, [[1, 2], [4, 5]]) and np.array_equal(ds.target, [3, 6])


def test_sidecar_truncation_and_corruption(tmp_path):
    text = (REF / "out" / "lineage_run000.txt").read_text().splitlines(keepends=True)
    p = tmp_path / "s.txt"
    p.write_text("".join(text[:-3]))            # truncated last plan block
    with pytest.raises(G.LineageError):
        G.read_lineage_sidecar(p)
    p.write_text("".join(text[:-1]))            # missing final elite
    with pytest.raises(G.LineageError):
        G.read_lineage_sidecar(p)
    p.write_text("".join(t.replace("gen 3", "gne 3") for t in text))
    with pytest.raises(G.LineageError):
        G.read_lineage_sidecar(p)
    p.write_text("# nothing\n")
    with pytest.raises(G.LineageError):
        G.read_lineage_sidecar(p)


def test_cli_rejects_gpu_backend_and_bad_files(tmp_path, capsys):
    code = G.run_cli(["-train_file", str(REF / "train.txt"), "-test_file", str(REF / "test.txt"),
                      "-backend", "gpu"])
    assert code != 0
    code = G.run_cli(["-train_file", str(tmp_path / "missing.txt"), "-test_file",
                      str(REF / "test.txt")])
    assert code == 1 and "error:" in capsys.readouterr().err
