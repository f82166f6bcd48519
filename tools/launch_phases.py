"""Split an ncu launch list of `python bench.py` (tools/gpu_evidence.sh) into
its runs (C3 timed, C3 e2e, C2 secondary): per run the generation-kernel
launches, their mean time, the reduce+survive mean and the GSM share of the
generation-loop kernels (the bench's kernel_share_of_step, measured cold)."""
import csv, json, re, sys


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    seq = []
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3}[r[ui]]
        seq.append((re.sub(r'\(.*', '', r[ki]).replace('void ', '').replace('unnamed>::', ''),
                    float(r[vi].replace(',', '')) * scale))
    runs, cur = [], None
    for name, us in seq:
        if name.startswith('k_compile'):          # every run compiles its genomes first
            cur = {"gsm": [], "reduce": [], "interp": []}
            runs.append(cur)
        if cur is None:
            continue
        if re.match(r'k_gsm_tma<float, 0, 0(, 0)?>', name):   # engine generation kernel (minus sign)
            cur["gsm"].append(us)
        elif name.startswith('k_reduce_survive'):
            cur["reduce"].append(us)
        elif name.startswith('k_interpret'):
            cur["interp"].append(us)
    out = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none launch list of "
                     "`python bench.py` (cold, serialised launches)", "runs": []}
    for i, r in enumerate(runs):
        if not r["gsm"]:
            continue
        g, red = sum(r["gsm"]), sum(r["reduce"])
        out["runs"].append({"run": i, "gsm_launches": len(r["gsm"]),
                            "gsm_mean_us": round(g / len(r["gsm"]), 1),
                            "reduce_survive_mean_us": round(red / max(1, len(r["reduce"])), 2),
                            "gsm_share_of_loop_kernels": round(g / (g + red), 4),
                            "interpret_total_ms": round(sum(r["interp"]) / 1e3, 1),
                            "interpret_launches": len(r["interp"])})
    print(json.dumps(out, indent=1))


if __name__ == '__main__':
    main(sys.argv[1])
