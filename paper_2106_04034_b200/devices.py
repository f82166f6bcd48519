"""Which GPUs one `run_evolution` call drives (single-process multi-GPU).

The reference's `run_evolution` uses every worker of the host through its
backend (gsgp/evolution.py:115, gsgp/backend.py:94-130: `threads=0` means all
cores).  The drop-in does the same with GPUs: `gsgp_init(n, ids)` makes the
next `gsgp_run` drive the listed devices from one host thread each, with the
fitness cases sharded by device and the per-generation canonical-SSE
collectives over NCCL (include/gsgp_b200.h).  Results are bit-identical to a
one-device run for any device count.

`devices` arguments accept:
  * ``"auto"`` (default) — every visible GPU the workload can use well: one
    device per 2 GiB of fp32 population semantics (m x cases x 4 bytes), so C3
    (51 GB) uses up to 8 GPUs while C1/C2 stay on one, where a generation is
    shorter than two collectives;
  * ``"all"`` — every visible GPU;
  * an int n — devices 0..n-1;
  * a sequence of device ids (a repeated id runs the threads on one GPU with a
    host exchange instead of NCCL: tests);
  * ``None`` — the current device only (also what "auto" resolves to inside a
    one-process-per-GPU job, `dist.init_from_torch`).
"""

from __future__ import annotations

import ctypes as C

from . import _lib
from ._lib import check
from .core import ConfigError

AUTO_BYTES_PER_DEVICE = 2 << 30

_active: tuple[int, ...] | None = None
_process_comm = False          # set by dist.init_from_torch / init_host_exchange


def visible_device_count() -> int:
    n, sms = C.c_int(0), C.c_int(0)
    name = C.create_string_buffer(128)
    check(_lib.load().gsgp_device_info(C.byref(n), C.byref(sms), name, 128))
    return n.value


def resolve(devices, population_size: int, n_cases: int) -> tuple[int, ...] | None:
    """The device tuple a run will use (None = the current device alone)."""
    if devices is None:
        return None
    if isinstance(devices, str):
        if devices not in ("auto", "all"):
            raise ConfigError("devices must be 'auto', 'all', an int, a list of ids or None")
        if _process_comm:
            return None
        count = visible_device_count()
        if devices == "all":
            n = count
        else:
            n = min(count, max(1, population_size * n_cases * 4 // AUTO_BYTES_PER_DEVICE))
        return tuple(range(n)) if n > 1 else None
    if isinstance(devices, int):
        if devices < 1:
            raise ConfigError("devices must be >= 1")
        ids = tuple(range(devices))
    else:
        ids = tuple(int(d) for d in devices)
        if not ids:
            raise ConfigError("devices must name at least one GPU")
    if _process_comm and len(ids) > 1:
        raise ConfigError("a one-process-per-GPU job (dist.init_from_torch) cannot also drive several "
                          "devices per process")
    return ids


def activate(ids: tuple[int, ...] | None) -> None:
    """Make `ids` the device set of the next gsgp_run (no-op if unchanged)."""
    global _active
    if ids == _active:
        return
    lib = _lib.load()
    if ids is None:
        check(lib.gsgp_finalize())
    else:
        arr = (C.c_int * len(ids))(*ids)
        check(lib.gsgp_init(len(ids), arr))
    _active = ids


def active() -> tuple[int, ...] | None:
    return _active


def reset() -> None:
    """Forget the device set (after gsgp_set_device or a failed run)."""
    global _active
    _active = None
