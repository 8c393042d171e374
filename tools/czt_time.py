"""Time the cfg2 CZT workload (N=1024, M=2048, 8192 traces; fp64 and fp32) with per-call CUDA events.
usage: python tools/czt_time.py [reps]   (env knobs such as SKG_CZT_SEGMENTS apply)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
x = torch.from_numpy(W.cfg2_batch(4096, 1024)).cuda()
a, w = W.cfg2_czt_params(2048)
for prec, xx in (("f64", x), ("f32", x.float())):
    p = sk.CztPlanGPU(1024, a, w, 2048, sk.SKG_F32 if prec == "f32" else sk.SKG_F64)
    out = p.execute(xx)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p.execute(xx, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"czt {prec} segments={os.environ.get('SKG_CZT_SEGMENTS', 'auto')} rt={'off' if os.environ.get('SKG_CZT_NO_RT') else 'on'}: "
          f"median {np.median(ts):.4f} ms  min {min(ts):.4f}")
