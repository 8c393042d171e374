"""Time the cfg3 zoom workloads (per-call CUDA events, median and max) — quick A/B helper.
usage: python tools/zoom_time.py [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
pad = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # extra elements per row (row stride 4096 + pad)
dev = torch.device("cuda", 0)
x64 = torch.from_numpy(W.cfg3_batch(4096, 4096)).to(dev)
if pad:
    buf = torch.zeros((4096, 4096 + pad), dtype=torch.float64, device=dev)
    buf[:, :4096] = x64
    x64 = buf[:, :4096]
def f32_rows(x):
    if not pad:
        return x.float()
    b = torch.zeros((x.shape[0], 4096 + pad), dtype=torch.float32, device=dev)
    b[:, :4096] = x
    return b[:, :4096]


for prec, x in (("f64", x64), ("f32", f32_rows(x64))):
    for nf in (0, 2048):   # bench.py's cfg3 rows: D = 8, 65 taps, n_fft 512 (auto) and 2048
        p = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, sk.SKG_F32 if prec == "f32" else sk.SKG_F64, n_fft=nf,
                           decimation=8, num_taps=65)
        out = p.execute(x)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            p.execute(x, out=out)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"pad={pad} {prec} n_fft={p.n_fft}: median {np.median(ts):.4f} ms  min {min(ts):.4f}  max {max(ts):.4f}")
