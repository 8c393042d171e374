"""Time the long zero-padded spectra (configs[4] FFT rows N=16384 -> L=65536, and L=32768/131072)
with per-call CUDA events; SKG_CLUSTER=1 selects the 8-CTA cluster kernel (default: four-step)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

tag = "cluster" if os.environ.get("SKG_CLUSTER") == "1" else "four-step"
for prec, dt, s in (("f64", torch.float64, 8), ("f32", torch.float32, 4)):
    for n, L in ((8192, 32768), (16384, 65536), (32768, 131072)):
        if prec == "f64" and L > 65536:
            continue
        batch = (1 << 30) // (n * s)
        x = torch.from_numpy(W.sample_traces(64, n)).to(dt).cuda().repeat(batch // 64, 1)
        out = sk.fft_spectrum_batch(x, L)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sk.fft_spectrum_batch(x, L, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        byts = x.shape[0] * (n * s + L * 2 * s)
        print(f"[{tag}] FFT {prec} N={n} L={L} batch={x.shape[0]}: {t:.3f} ms  {byts / t / 1e6:.0f} GB/s "
              f"({byts / t / 1e6 / 6540:.2f} of HBM)")
        del x, out
        torch.cuda.empty_cache()

for prec, dt, s in (("f64", torch.float64, 8), ("f32", torch.float32, 4)):
    for n, m in ((16384, 16384), (4096, 16384)):
        batch = 8192 if prec == "f64" else 16384
        x = torch.from_numpy(W.sample_traces(64, n)).to(dt).cuda().repeat(batch // 64, 1)
        a, w = W.cfg2_czt_params(m)
        p = sk.CztPlanGPU(n, a, w, m, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
        out = p.execute(x)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.execute(x, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"[{tag}] CZT {prec} N={n} M={m} L={p.conv_size} batch={batch}: {float(np.median(ts)):.3f} ms")
        del x, out
        torch.cuda.empty_cache()
