"""Time the long zero-padded spectra of the configs[4] sweep (FFT rows N = 16384 -> 65536 and
N = 65536 -> 262144, ~1 GiB batches, full layout) with per-call CUDA events. SKG_4STEP_REAL=0 selects
the complex four-step, SKG_4STEP_FUSED=0 the two-launch Hermitian path."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

tag = f"real={os.environ.get('SKG_4STEP_REAL', '1')} fused={os.environ.get('SKG_4STEP_FUSED', '1')}"
sizes = [(16384, 65536), (65536, 262144)]
if len(sys.argv) > 1:
    sizes = [(int(a) // 4, int(a)) for a in sys.argv[1:]]
for prec, dt, s in (("f64", torch.float64, 8), ("f32", torch.float32, 4)):
    for n, L in sizes:
        batch = (1 << 30) // (n * s)
        x = torch.from_numpy(W.sample_traces(64, n)).to(dt).cuda().repeat(batch // 64, 1)
        out = sk.fft_spectrum_batch(x, L)
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sk.fft_spectrum_batch(x, L, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        byts = x.shape[0] * (n * s + L * 2 * s)
        print(f"[{tag}] FFT {prec} N={n} L={L} batch={x.shape[0]}: {t:.3f} ms  {byts / t / 1e6:.0f} GB/s "
              f"({byts / t / 1e6 / 6459.3:.3f} of HBM)", flush=True)
        del x, out
        torch.cuda.empty_cache()
