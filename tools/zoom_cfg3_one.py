"""One cfg3 zoom call (for ncu): python tools/zoom_cfg3_one.py <f32|f64> <n_fft>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

prec, nf = sys.argv[1], int(sys.argv[2])
x = torch.from_numpy(W.cfg3_batch(4096, 4096)).cuda()
x = x if prec == "f64" else x.float()
p = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, sk.SKG_F32 if prec == "f32" else sk.SKG_F64, n_fft=nf, decimation=8,
                   num_taps=65)
out = p.execute(x)
p.execute(x, out=out)
torch.cuda.synchronize()
