"""Backend name registry (paper_2106_04034_b200/backend.py vs
gsgp/backend.py:133-138): "cuda" and the reference's names are accepted,
"gpu" and unknown names are rejected (pkg/tests/test_backend.py:128-129,
pkg/tests/test_core.py:41).  The reference's CPU thread pools are out of
scope: every name runs on the device."""

from __future__ import annotations

import pytest

from paper_2106_04034_b200 import ConfigError, RunConfig, get_backend


@pytest.mark.parametrize("name", ["cuda", "sequential", "threads"])
def test_registry_accepts_device_and_reference_names(name):
    d = get_backend(name, 4)
    assert d.name == "cuda" and d.workers == 1
    assert RunConfig(backend=name).backend == name


@pytest.mark.parametrize("name", ["gpu", "GPU", "", "thread"])
def test_registry_rejects_other_names(name):
    with pytest.raises(ConfigError):
        get_backend(name)
    with pytest.raises(ConfigError):
        RunConfig(backend=name)
