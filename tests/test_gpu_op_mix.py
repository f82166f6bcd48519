"""The compiled programs' op mix that bench.py's interpreter rooflines use
(k_compile's per-genome counts, summed by the engine into
RunResult.device["program_instructions" / "program_divisions" /
"program_operands"]) equals an independent restatement of the compiler's
emission rules (interp.cu k_compile: skip rule, constant folding,
Sethi-Ullman order, leaf pairs, spill + leaf-pair fusion) on the same
genomes (oracle.restate.genomes: population stream base 0, pool stream base m).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import restate as R

import paper_2106_04034_b200 as G

DIVS = {"DIV", "RDIV", "LDIV", "PDIV"}
OPS = ["ADD", "SUB", "MUL", "DIV"]


def compile_mix(tags, codes):
    """(instructions, divisions, per-case operand loads, constant loads,
    spill stores) of one genome, following interp.cu k_compile."""
    k = len(tags)
    fl, need, L, Rc = {}, {}, {}, {}
    stk, last = [], -1
    for j in range(k):
        t = tags[j]
        if t == R.FUNCTION:
            if len(stk) < 2:
                continue                       # skipped: operands unavailable
            r = stk.pop()
            l = stk.pop()
            L[j], Rc[j] = l, r
            stk.append(j)
            last = j
            if fl[l] == "c" and fl[r] == "c":
                fl[j] = "c"                    # folded to a constant
                continue
            la, lb = fl[l] in "cf", fl[r] in "cf"
            na = 0 if la else need[l]
            nb = 0 if lb else need[r]
            if la and lb:
                n = 0
            elif lb:
                n = na
            elif la:
                n = nb
            else:
                n = na + 1 if na == nb else max(na, nb)
            fl[j], need[j] = "n", min(n, 31)
        elif t == R.FEATURE:
            fl[j] = "f"
            stk.append(j)
        else:
            fl[j] = "c"
            stk.append(j)
    root = last if last >= 0 else (stk[-1] if stk else -1)
    out = []                                   # (kind, x class, y class or None)
    cls = lambda n: "C" if fl[n] == "c" else "V"   # noqa: E731
    if root < 0:
        out.append(("LOAD", "C", None))
    elif fl[root] in "cf":
        out.append(("LOAD", cls(root), None))
    else:
        pending = False
        work = [(root, 0)]
        rev = {"SUB": "RSUB", "DIV": "RDIV"}
        while work:
            n, st = work[-1]
            l, r = L[n], Rc[n]
            la, lb = fl[l] in "cf", fl[r] in "cf"
            left_first = (need[l] >= need[r]) if (not la and not lb) else (not la)
            op = OPS[codes[n]]
            if st == 0:
                if la and lb:
                    out.append((("P" if pending else "L") + op, cls(l), cls(r)))
                    pending = False
                    work.pop()
                else:
                    work[-1] = (n, 1)
                    work.append((l if left_first else r, 0))
            elif st == 1:
                if lb:
                    out.append((op, cls(r), None))
                    work.pop()
                elif la:
                    out.append((rev.get(op, op), cls(l), None))
                    work.pop()
                else:
                    pending = True
                    work[-1] = (n, 2)
                    work.append((r if left_first else l, 0))
            else:
                out.append((op, "V", None))     # spill-slot operand (per case)
                work.pop()
    ins = len(out)
    div = sum(kd in DIVS for kd, _, _ in out)
    vec = sum((x == "V") + (y == "V") for _, x, y in out)
    con = sum((x == "C") + (y == "C") for _, x, y in out)
    sto = sum(kd.startswith("P") for kd, _, _ in out)
    return ins, div, vec, con, sto


@pytest.mark.gpu
@pytest.mark.parametrize("k,l,probs", [(255, 5, (0.8, 0.14, 0.04)), (1024, 8, (0.8, 0.14, 0.04)),
                                       (127, 3, (0.6, 0.1, 0.3)), (64, 2, (0.5, 0.25, 0.25))])
def test_device_op_mix_equals_compiler_restatement(k, l, probs):
    m, r, seed = 24, 16, 5
    rng = np.random.default_rng(k)
    Xtr, Xte = rng.uniform(-1, 1, (700, l)), rng.uniform(-1, 1, (300, l))
    ytr, yte = rng.normal(size=700), rng.normal(size=300)
    cfg = G.RunConfig(population_size=m, random_trees=r, program_size=k, generations=0, seed=seed,
                      p_function=probs[0], p_feature=probs[1], p_constant=probs[2])
    res = G.run_evolution(cfg, G.Dataset(Xtr, ytr), G.Dataset(Xte, yte))
    kw = dict(p_function=probs[0], p_feature=probs[1], p_constant=probs[2])
    for side, (count, base) in {"population": (m, 0), "pool": (r, m)}.items():
        tags, codes, _ = R.genomes(count, k, l, seed, base, **kw)
        tot = np.zeros(5, np.int64)
        for i in range(count):
            tot += np.array(compile_mix(tags[i], codes[i]))
        ops = res.device["program_operands"][side]
        got = [res.device["program_instructions"][side], res.device["program_divisions"][side],
               ops["vector_loads"], ops["constant_loads"], ops["spill_stores"]]
        assert got == tot.tolist(), (side, got, tot.tolist())
