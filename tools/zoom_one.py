"""One zoom call on a ~1 GiB batch (for ncu): python tools/zoom_one.py <f32|f64> <N> <D> [batch]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

prec, N, D = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
s = 8 if prec == "f64" else 4
batch = int(sys.argv[4]) if len(sys.argv) > 4 else (1 << 30) // (N * s)
dt = torch.float64 if prec == "f64" else torch.float32
x = torch.from_numpy(W.sample_traces(64, N)).to(dt).cuda().repeat(batch // 64 + 1, 1)[:batch]
plan = sk.ZoomPlanGPU(N, 0.4e12, 1.2e12, 20e12, sk.SKG_F64 if prec == "f64" else sk.SKG_F32, decimation=D)
print(f"N={N} D={D} taps={plan.num_taps} n_fft={plan.n_fft} bins={plan.bins} batch={batch}", flush=True)
out = plan.execute(x)
plan.execute(x, out=out)
torch.cuda.synchronize()
