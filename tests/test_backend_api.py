"""The reference's backend plugin API for user closures
(paper_2106_04034_b200/backend.py vs gsgp/backend.py; cases follow
pkg/tests/test_backend.py).  None of the engine's operators use it."""

from __future__ import annotations

import threading

import numpy as np
import pytest

from paper_2106_04034_b200 import (
    ConfigError, CudaBackend, SequentialBackend, ThreadBackend, choose_chunk, get_backend,
)


@pytest.mark.parametrize("items,workers,expected", [(100, 4, 25), (10, 16, 1), (1, 1, 1), (7, 2, 4),
                                                    (8, 3, 3)])
def test_choose_chunk(items, workers, expected):
    assert choose_chunk(items, workers) == expected


def test_choose_chunk_rejects_nonpositive():
    for args in ((0, 4), (4, 0)):
        with pytest.raises(ConfigError):
            choose_chunk(*args)


@pytest.mark.parametrize("backend", [SequentialBackend(), ThreadBackend(1), ThreadBackend(8), CudaBackend()],
                         ids=lambda b: f"{b.name}{b.workers}")
def test_map_protocol(backend):
    with backend:
        out = np.full((5, 3), -1.0)
        backend.map_elements((5, 3), lambda i, j: i * 3 + j, out)
        assert out.ravel().tolist() == list(range(15))
        assert backend.map_rows(7, lambda i: i * i) == [i * i for i in range(7)]
        assert backend.map_rows(0, lambda i: i) == []
        seen, lock = [], threading.Lock()

        def block(lo, hi):
            with lock:
                seen.append((lo, hi))

        backend.map_row_blocks(23, block)
        cover = sorted(i for lo, hi in seen for i in range(lo, hi))
        assert cover == list(range(23))
        with pytest.raises(ConfigError):
            backend.map_elements((2, 2), lambda i, j: 0.0, np.zeros((3, 2)))


def test_get_backend_and_descriptors():
    assert get_backend("sequential").name == "sequential"
    b = get_backend("threads", 3)
    assert b.name == "threads" and b.workers == 3 and b.descriptor.workers == 3
    assert get_backend("threads", 0).workers >= 1
    assert get_backend("cuda").descriptor.name == "cuda"
    with pytest.raises(ConfigError):
        get_backend("gpu")
