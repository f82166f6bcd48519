"""Summarise ncu outputs for profiles/: launch-list shares and key raw metrics."""
import collections, csv, json, re, subprocess, sys

def launch_list(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) <= vi: continue
        name = re.sub(r'\(.*', '', r[ki]).replace('void ', '').replace('unnamed>::', '').strip()
        v = float(r[vi].replace(',', ''))
        scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3}[r[ui]]
        agg[name].append(v * scale)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append({"kernel": k, "launches": len(v), "total_us": round(sum(v), 1),
                    "mean_us": round(sum(v) / len(v), 2), "share": round(sum(v) / tot, 4)})
    return out

KEYS = r'^(gpu__time_duration.sum|dram__bytes_(read|write)\.sum|gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed|lts__t_sector_hit_rate.pct|lts__throughput.avg.pct_of_peak_sustained_elapsed|sm__throughput.avg.pct_of_peak_sustained_elapsed|sm__warps_active.avg.per_cycle_active|launch__registers_per_thread|launch__grid_size|launch__block_size|launch__shared_mem_per_block_dynamic|smsp__issue_active.avg.pct_of_peak_sustained_active|sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active|smsp__inst_executed.sum|smsp__average_warps_issue_stalled_(long_scoreboard|short_scoreboard|wait|barrier|math_pipe_throttle|no_instruction|branch_resolving|lg_throttle|mio_throttle)_per_issue_active.ratio)$'

def raw(rep):
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, u, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        item = {"kernel": re.sub(r'\(.*', '', d[h.index('Kernel Name')]).replace('void ', '')}
        for i, c in enumerate(h):
            if re.match(KEYS, c):
                item[c] = f"{d[i]} {u[i]}".strip()
        res.append(item)
    return res

if __name__ == '__main__':
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launch_list(path) if kind == 'launches' else raw(path), indent=1))
