import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2108_03948_b200 as sk
from paper_2108_03948_b200 import workloads as W
for n, L in ((4096, 16384), (3000, 16384), (2048, 8192)):
    x = torch.from_numpy(W.sample_traces(64, n)).float().cuda().repeat((1 << 28) // (n * 64), 1)
    out = sk.fft_spectrum_batch(x, L); torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sk.fft_spectrum_batch(x, L, out=out); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(os.environ.get("SKG_LIB_PATH", "default")[-30:], n, L, x.shape[0], round(float(np.median(ts)), 4))
