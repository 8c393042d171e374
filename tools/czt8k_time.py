"""Time configs[4] CZT rows whose convolution is one 8192-point CTA transform (fp32 / fp64) — A/B helper."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

for prec, dt in (("f32", torch.float32), ("f64", torch.float64)):
    for n, m in ((4096, 4096), (3000, 3000), (4096, 1024)):
        x = torch.from_numpy(W.sample_traces(64, n)).to(dt).cuda().repeat(8192 // 64, 1)
        a, w = W.cfg2_czt_params(m)
        p = sk.CztPlanGPU(n, a, w, m, sk.SKG_F32 if prec == "f32" else sk.SKG_F64)
        out = p.execute(x)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.execute(x, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(os.environ.get("SKG_LIB_PATH", "default")[-24:], prec, n, m, p.conv_size, round(float(np.median(ts)), 4))
