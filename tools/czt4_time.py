"""Time the multi-pass CZT rows of the configs[4] sweep (~1 GiB batches) with per-call CUDA events.
SKG_4STEP_FUSED=0 selects the three-launch path."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

tag = f"fused={os.environ.get('SKG_4STEP_FUSED', '1')}"
rows = [(3000, 12000), (4096, 16384), (16384, 4096), (16384, 16384), (16384, 65536), (65536, 16384), (65536, 65536),
        (65536, 262144)]
import os as _os
PRECS = [p for p in (("f64", torch.float64, 8), ("f32", torch.float32, 4)) if p[0] in _os.environ.get("SKG_PRECS", "f64,f32")]
for prec, dt, s in PRECS:
    for n, m in rows:
        batch = max(64, ((1 << 30) // (n * s)) // 64 * 64)
        x = torch.from_numpy(W.sample_traces(64, n)).to(dt).cuda().repeat(batch // 64, 1)
        a, w = W.cfg2_czt_params(m)
        p = sk.CztPlanGPU(n, a, w, m, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
        out = p.execute(x)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.execute(x, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"[{tag}] CZT {prec} N={n} M={m} L={p.conv_size} batch={batch}: {float(np.median(ts)):.3f} ms", flush=True)
        del x, out, p
        torch.cuda.empty_cache()
