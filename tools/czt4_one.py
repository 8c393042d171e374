"""One multi-pass CZT call (for ncu): python tools/czt4_one.py <f32|f64> <n> <m> <batch>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

prec, n, m, batch = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
dt = torch.float64 if prec == "f64" else torch.float32
x = torch.from_numpy(W.sample_traces(64, n)).to(dt).cuda().repeat(batch // 64, 1)
a, w = W.cfg2_czt_params(m)
p = sk.CztPlanGPU(n, a, w, m, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
out = p.execute(x)
p.execute(x, out=out)
torch.cuda.synchronize()
