"""Time the cfg4 cube workload (65536 px x 2048 fp32 -> FFT 8192 -> |H|, arg H) and the fp64/fp32
half-spectrum / band FFT rows with per-call CUDA events. usage: python tools/cube_time.py [reps]
(SKG_LIB_PATH selects an A/B build of the library)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402


def timeit(fn, reps, inner=10):
    """per-call device time: `inner` back-to-back calls between two events, so the host-side cost of
    a call (ctypes, tensor allocation) overlaps the previous call's kernel instead of idling the GPU"""
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(inner):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / inner)
    return float(np.median(ts)), float(min(ts))


reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
lib = os.environ.get("SKG_LIB_PATH", "default")
cube, ref = W.cfg4_cube(256, 256, 2048)
p = sk.TransferPlanGPU(ref, 8192, sk.SKG_F32)
xd = torch.from_numpy(cube).cuda()
mag = torch.empty((65536, 4097), dtype=torch.float32, device="cuda")
ph = torch.empty_like(mag)
med, mn = timeit(lambda: p.execute(xd, mag=mag, phase=ph), reps)
print(f"[{lib}] cube H fp32: median {med:.4f} ms min {mn:.4f}  ({65536 * 40968 / med / 1e6:.0f} GB/s)")
hs = sk.fft_spectrum_batch(xd, 8192, layout=sk.SKG_HALF)
med, mn = timeit(lambda: sk.fft_spectrum_batch(xd, 8192, layout=sk.SKG_HALF, out=hs), reps)
print(f"[{lib}] cube half spectrum only fp32: median {med:.4f} ms  ({65536 * (8192 + 4097 * 8) / med / 1e6:.0f} GB/s)")
del hs
x = torch.from_numpy(W.sample_traces(32768, 1024)).cuda()
for dt in (torch.float64, torch.float32):
    xx = x.to(dt)
    out = sk.fft_spectrum_batch(xx, 4096)
    med, mn = timeit(lambda: sk.fft_spectrum_batch(xx, 4096, out=out), reps)
    s = xx.element_size()
    print(f"[{lib}] spectrum full 1024->4096 {dt}: median {med:.4f} ms ({32768 * (1024 * s + 4096 * 2 * s) / med / 1e6:.0f} GB/s)")
    med, mn = timeit(lambda: sk.fft_spectrum_band_batch(xx, W.FS, 0.1e12, 3.0e12, 4096), reps)
    print(f"[{lib}] band 0.1-3 THz + dB {dt}: median {med:.4f} ms")
