"""One cfg4 cube call (for ncu): python tools/cube_one.py  (SKG_LIB_PATH selects an A/B build)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

cube, ref = W.cfg4_cube(256, 256, 2048)
tp = sk.TransferPlanGPU(ref, 8192, sk.SKG_F32)
cd = torch.from_numpy(cube).cuda()
mag = torch.empty((cube.shape[0], tp.bins), dtype=torch.float32, device="cuda")
ph = torch.empty_like(mag)
tp.execute(cd, mag, ph)
tp.execute(cd, mag, ph)
torch.cuda.synchronize()
