"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/gsgp_b200.h declares, fails loudly without a device, and the
host-side mirror of the reference API validates like the reference."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden

HEADER = ROOT / "include" / "gsgp_b200.h"


def declared_symbols() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(gsgp_[a-z_0-9]+)\s*\(", text, re.M))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("gsgp_run", "gsgp_create_population", "gsgp_compute_semantics", "gsgp_gsm",
              "gsgp_build_mutation_plan", "gsgp_compute_fitness", "gsgp_survive",
              "gsgp_comm_init", "gsgp_rng_draw"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2106_04034_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert syms == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s
    assert b"sm_100a" in lib.gsgp_version()


def test_built_for_sm100a_only():
    import subprocess
    from paper_2106_04034_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_host_only_derive_seed_matches_reference():
    from paper_2106_04034_b200 import derive_seed
    g = golden("rng")
    for s, i, d in g["derive"]:
        assert derive_seed(int(s), int(i)) == int(d)


def test_shard_ranges_partition_the_cases():
    import ctypes as C
    from paper_2106_04034_b200 import _lib, dist
    lib = _lib.load()
    for n in (1, 7, 100, 12_287, 12_288, 50_000, 12_500_000):
        for count in (1, 2, 3, 8):
            spans = [dist.shard_range(n, count, i) for i in range(count)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            # interior boundaries sit on the canonical case grid, and the
            # split stays balanced to within one alignment block
            assert all(hi % dist.CASE_ALIGN == 0 for _, hi in spans[:-1])
            assert all(hi - lo <= -(-n // count) + dist.CASE_ALIGN for lo, hi in spans)
            for i, (lo, hi) in enumerate(spans):
                clo, chi = C.c_int64(), C.c_int64()
                lib.gsgp_shard_range(n, count, i, C.byref(clo), C.byref(chi))
                assert (clo.value, chi.value) == (lo, hi)


def test_compute_calls_fail_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2106_04034_b200 import GsgpError, rng_stream
    with pytest.raises(GsgpError, match="no CUDA device"):
        rng_stream(1, 0, 0)


def test_runconfig_mirrors_reference_validation():
    from paper_2106_04034_b200 import ConfigError, RunConfig
    RunConfig()
    RunConfig(backend="sequential")
    RunConfig(backend="threads", threads=4)
    for bad in (dict(backend="gpu"), dict(population_size=0), dict(generations=-1),
                dict(p_function=-1.0), dict(erc_low=2.0, erc_high=1.0), dict(division_eps=0.0),
                dict(gsm_sign="times"), dict(mutation_step="gaussian"), dict(mutation_step=-0.5),
                dict(threads=-1), dict(runs=0)):
        with pytest.raises(ConfigError):
            RunConfig(**bad)
    assert RunConfig(p_function=2, p_feature=1, p_constant=1).gene_probabilities == (0.5, 0.25, 0.25)


def test_dataset_validation():
    from paper_2106_04034_b200 import Dataset, DatasetFormatError
    Dataset(np.ones((3, 2)), np.ones(3))
    for X, y in ((np.ones(3), np.ones(3)), (np.ones((3, 2)), np.ones(2)),
                 (np.ones((0, 2)), np.ones(0)), (np.full((2, 2), np.nan), np.ones(2))):
        with pytest.raises(DatasetFormatError):
            Dataset(X, y)
