"""Probe: sustained HBM copy bandwidth (torch D2D copy) under the power cap.

Copies a 16 GiB fp32 buffer back and forth for ~6 s and reports GB/s
(read + write bytes) per iteration with CUDA events, plus NVML power/clock
samples — the sustained counterpart of MEASURED_PEAKS.json's burst copy.
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

n = 4 << 30  # 4 Gi fp32 = 16 GiB
a = torch.empty(n, dtype=torch.float32, device="cuda").uniform_()
b = torch.empty_like(a)
smp = bench.ClockSampler(0, period=0.02)
smp.start()
res = []
t_end = time.perf_counter() + float(sys.argv[1] if len(sys.argv) > 1 else 6.0)
while time.perf_counter() < t_end:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    res.append(2 * 4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    a, b = b, a
summ = smp.summary()
k = len(res)
print(json.dumps({"copy_gbs_first": [round(x, 1) for x in res[:5]],
                  "copy_gbs_by_decile": [round(sum(c) / len(c), 1) for c in
                                         [res[i * k // 10:(i + 1) * k // 10] or res[-1:] for i in range(10)]],
                  "copy_gbs_best": max(res), "copy_gbs_last_half_mean": sum(res[k // 2:]) / len(res[k // 2:]),
                  "iterations": k, "clocks": summ}))
