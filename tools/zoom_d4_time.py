"""Time configs[4] zoom rows (101 taps, band 0.4-1.2 THz, D in {4, 16}) — A/B helper for the FIR
route against the frequency-domain route (SKG_ZOOM_NO_SPEC=1 disables the latter)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

tag = "fir" if os.environ.get("SKG_ZOOM_NO_SPEC") else "auto"
for prec, dt, s in (("f64", torch.float64, 8), ("f32", torch.float32, 4)):
    for n, D in ((1024, 4), (4096, 4), (16384, 4), (4096, 8), (4096, 16)):
        batch = (1 << 28) // (n * s)
        x = torch.from_numpy(W.sample_traces(64, n)).to(dt).cuda().repeat(batch // 64, 1)
        p = sk.ZoomPlanGPU(n, 0.4e12, 1.2e12, W.FS, sk.SKG_F64 if prec == "f64" else sk.SKG_F32, decimation=D)
        out = p.execute(x)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.execute(x, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"[{tag}] zoom {prec} N={n} D={D} batch={batch}: {float(np.median(ts)):.4f} ms")
