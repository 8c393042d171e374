"""Run one hot-path workload a few times (for ncu / compute-sanitizer captures on the GPU box).
usage: python tools/prof.py {czt64,czt32,zoom64,zoom32,cube32,spec64,all} [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402


def run(name, steps):
    dev = torch.device("cuda", 0)
    if name.startswith("czt"):
        f32 = name.endswith("32")
        x = W.cfg2_batch(4096, 1024).astype(np.float32 if f32 else np.float64)
        a, w = W.cfg2_czt_params(2048)
        p = sk.CztPlanGPU(1024, a, w, 2048, sk.SKG_F32 if f32 else sk.SKG_F64)
        xd = torch.from_numpy(x).to(dev)
        fn = lambda: p.execute(xd)  # noqa: E731
    elif name.startswith("zoom"):
        f32 = name.endswith("32")
        x = W.cfg3_batch(4096, 4096).astype(np.float32 if f32 else np.float64)
        p = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, sk.SKG_F32 if f32 else sk.SKG_F64, decimation=8, num_taps=65)
        xd = torch.from_numpy(x).to(dev)
        fn = lambda: p.execute(xd)  # noqa: E731
    elif name == "cube32":
        cube, ref = W.cfg4_cube(256, 256, 2048)
        p = sk.TransferPlanGPU(ref, 8192, sk.SKG_F32)
        xd = torch.from_numpy(cube).to(dev)
        fn = lambda: p.execute(xd)  # noqa: E731
    elif name.startswith("spec4step"):
        f32 = name.endswith("32")
        x = W.sample_traces(2048, 16384).astype(np.float32 if f32 else np.float64)
        xd = torch.from_numpy(x).to(dev)
        fn = lambda: sk.fft_spectrum_batch(xd, 65536)  # noqa: E731
    elif name == "czt4step":
        x = W.sample_traces(1024, 16384)
        a, w = W.cfg2_czt_params(16384)
        p = sk.CztPlanGPU(16384, a, w, 16384, sk.SKG_F64)
        xd = torch.from_numpy(x).to(dev)
        fn = lambda: p.execute(xd)  # noqa: E731
    elif name.startswith("specL"):   # specL15_64: L = 2^15 fp64 spectra (cluster / four-step path)
        lgL, pr = name[5:].split("_")
        L = 1 << int(lgL)
        x = W.sample_traces(64, L // 4).astype(np.float32 if pr == "32" else np.float64)
        xd = torch.from_numpy(x).to(dev).repeat(32, 1)
        fn = lambda: sk.fft_spectrum_batch(xd, L)  # noqa: E731
    elif name == "spec64":
        x = W.sample_traces(32768, 1024)
        xd = torch.from_numpy(x).to(dev)
        fn = lambda: sk.fft_spectrum_batch(xd, 4096)  # noqa: E731
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
    print(name, "ok")


if __name__ == "__main__":
    which = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    for n in (["czt64", "czt32", "zoom64", "zoom32", "cube32", "spec64"] if which == "all" else [which]):
        run(n, steps)
