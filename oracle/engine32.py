"""Op-for-op restatement of the B200 engine's arithmetic (TEST INFRASTRUCTURE ONLY).

The engine stores semantics in fp32 but interprets genomes and accumulates
SSE in fp64.  This module restates exactly what the kernels
compute so that
  * element-level kernel outputs are checked bit-exactly (gsm_step32), and
  * the fp32-storage design itself is validated against the fp64 reference on
    CPU (run32 vs. the golden reference runs: identical elite records, traces
    within 1e-5) before any GPU is involved.

The SSE summation order here is numpy's, not the kernel's tiled order, so
SSE/RMSE agree with the device to ~1e-15 relative, not bitwise.
"""

from __future__ import annotations

import math

import numpy as np

from . import restate as R

FLT_MAX = float(np.finfo(np.float32).max)


def gsm_step32(P32: np.ndarray, Q32: np.ndarray, u, v, ms, sign: str = "minus") -> np.ndarray:
    """Engine GSM in fp32 with the reference's op order t=a-/+b; t*=ms;
    out=parent+t (gsgp/mutation.py:81-83), each step rounded to fp32."""
    a = Q32[u]
    b = Q32[v]
    t = (a - b) if sign == "minus" else (a + b)
    t = t * np.asarray(ms, np.float64).astype(np.float32)[:, None]
    return P32 + t


def sse(S, y) -> np.ndarray:
    d = S.astype(np.float64) - np.asarray(y, np.float64)
    with np.errstate(all="ignore"):
        return (d * d).sum(axis=1)


def rmse_from_sse(s, n) -> np.ndarray:
    with np.errstate(all="ignore"):
        v = np.sqrt(np.asarray(s, np.float64) / n)
    return np.where(np.isfinite(v), v, math.inf)


def init_state(s_pop_tr, s_pop_te, ytr, yte):
    """fp64 semantics -> fp32 storage, fp64 SSE, fp32-overflow ('wide') flags."""
    with np.errstate(over="ignore"):
        P_tr = s_pop_tr.astype(np.float32)
        P_te = s_pop_te.astype(np.float32)
    wide = (np.isinf(P_tr).any(axis=1) * 1) | (np.isinf(P_te).any(axis=1) * 2)
    F = rmse_from_sse(sse(s_pop_tr, ytr), s_pop_tr.shape[1])
    TS = sse(s_pop_te, yte)
    return P_tr, P_te, F, TS, wide.astype(np.int32)


def run32(cfg: R.Cfg, Xtr, ytr, Xte, yte, exchange=None, n_total=None, wide_slots=True):
    """The engine's run in fp32 storage.

    Sharded use (the multi-GPU protocol): each caller passes only
    its case slice, `n_total=(n_train, n_test)` of the whole dataset, and
    `exchange(name, array) -> array` summing an array over all shards (the
    NCCL allreduce of the engine).  Exchanged: per-row SSE (init and every
    generation), the fp32-overflow flags and the non-finite count."""
    m, r, g, l = cfg.m, cfg.r, cfg.g, Xtr.shape[1]
    kw = dict(p_function=cfg.p[0], p_feature=cfg.p[1], p_constant=cfg.p[2],
              erc_low=cfg.erc[0], erc_high=cfg.erc[1])
    pop = R.genomes(m, cfg.k, l, cfg.seed, 0, **kw)
    trees = R.genomes(r, cfg.k, l, cfg.seed, m, **kw)
    stacked = np.vstack([Xtr, Xte])
    ntr_l, nte_l = Xtr.shape[0], Xte.shape[0]
    ntr, nte = n_total if n_total else (ntr_l, nte_l)
    xch = exchange or (lambda name, arr: arr)
    s_pop, c1 = R.semantics(*pop, stacked, cfg.eps)
    s_tree, c2 = R.semantics(*trees, stacked, cfg.eps)
    with np.errstate(over="ignore"):
        P_tr = s_pop[:, :ntr_l].astype(np.float32)
        P_te = s_pop[:, ntr_l:].astype(np.float32)
    bits = np.stack([np.isinf(P_tr).any(axis=1), np.isinf(P_te).any(axis=1)], axis=1).astype(np.int64)
    bits = xch("wide", bits)
    wide = ((bits[:, 0] > 0) * 1 | (bits[:, 1] > 0) * 2).astype(np.int32)
    if not wide_slots:          # negative control: plain fp32 storage semantics
        wide[:] = 0
    # initial fitness from the STORED (fp32) semantics — the same values and
    # order a generation uses, so an offspring equal to its parent ties with
    # it exactly — except fp32-overflow slots, which keep the fp64 SSE
    s_st = xch("sse", np.stack([sse(P_tr, ytr), sse(P_te, yte)], axis=1))
    s64 = xch("sse", np.stack([sse(s_pop[:, :ntr_l], ytr), sse(s_pop[:, ntr_l:], yte)], axis=1))
    F = np.where(wide & 1, rmse_from_sse(s64[:, 0], ntr), rmse_from_sse(s_st[:, 0], ntr))
    TS = np.where(wide & 2, s64[:, 1], s_st[:, 1])
    overflow = int(xch("overflow", np.array([c1 + c2], np.int64))[0])
    Q = R.sigmoid(s_tree).astype(np.float32)
    Q_tr, Q_te = Q[:, :ntr_l], Q[:, ntr_l:]
    b0 = int(np.argmin(F))
    out = {"train": np.empty(g + 1), "test": np.empty(g + 1), "elite": [],
           "initial": ("initial", b0, b0, float(F[b0])), "overflow": overflow, "wide0": wide.copy(),
           "u": np.empty((g, m), np.int64), "v": np.empty((g, m), np.int64), "ms": np.empty((g, m))}
    out["train"][0] = F[b0]
    out["test"][0] = rmse_from_sse(TS[b0], nte)
    for gen in range(1, g + 1):
        u, v, ms = R.plan(m, r, cfg.seed, gen, cfg.mutation_step)
        O_tr = gsm_step32(P_tr, Q_tr, u, v, ms, cfg.sign)
        O_te = gsm_step32(P_te, Q_te, u, v, ms, cfg.sign)
        s = xch("sse", np.stack([sse(O_tr, ytr), sse(O_te, yte)], axis=1))
        s_tr, s_te = s[:, 0], s[:, 1]
        Fo = np.where(wide & 1, F, rmse_from_sse(s_tr, ntr))
        To = np.where(wide & 2, TS, s_te)
        src, idx, slot = R.survive(F, Fo)
        if src == "parent":
            O_tr[slot], O_te[slot] = P_tr[idx], P_te[idx]
            Fo[slot], To[slot] = F[idx], TS[idx]
            wide[slot] = wide[idx]
        P_tr, P_te, F, TS = O_tr, O_te, Fo, To
        out["u"][gen - 1], out["v"][gen - 1], out["ms"][gen - 1] = u, v, ms
        out["elite"].append((src, idx, slot, float(F[slot])))
        out["train"][gen] = F[slot]
        out["test"][gen] = rmse_from_sse(TS[slot], nte)
    final = out["elite"][-1] if g else out["initial"]
    out["slot"] = final[2]
    out["elite_train_semantics"] = P_tr[final[2]].astype(np.float64)
    out["wide"] = wide
    return out
