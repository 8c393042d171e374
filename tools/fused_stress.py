"""Stress the one-launch four-step paths (k4_rfused, k4_czt_fused): many grid sizes x look-aheads x shapes,
each compared bit for bit with the multi-launch path. A hang shows as the outer `timeout` firing.
usage: timeout 900 python tools/fused_stress.py"""
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

caps = [0, 5, 37, 61, 148, 149, 296, 301, 443]
deltas = ["1", "4", "10", "25", "70"]
n_ok = 0
for prec, dt in (("f32", torch.float32), ("f64", torch.float64)):
    for L, b in ((65536, 330), (262144, 70)):
        n = L // 4 - 3
        x = torch.from_numpy(W.sample_traces(64, n)).to(dt).cuda().repeat(b // 64 + 1, 1)[:b].contiguous()
        os.environ["SKG_4STEP_FUSED"] = "0"
        ref = sk.fft_spectrum_batch(x, L)
        os.environ["SKG_4STEP_FUSED"] = "1"
        for cap, dx in itertools.product(caps, deltas):
            os.environ["SKG_4STEP_DELTA_X10"] = dx
            with sk.grid_cap(cap):
                got = sk.fft_spectrum_batch(x, L)
                torch.cuda.synchronize()
            assert torch.equal(got, ref), (prec, L, cap, dx)
            n_ok += 1
        print(f"fft {prec} L={L}: {len(caps) * len(deltas)} variants ok", flush=True)
        del x, ref, got
    for (n, m, b) in ((16384, 16384, 260), (3000, 12000, 400) if prec == "f64" else (30000, 30000, 200), (65536, 16384, 90)):
        x = torch.from_numpy(W.sample_traces(64, n)).to(dt).cuda().repeat(b // 64 + 1, 1)[:b].contiguous()
        a, w = W.cfg2_czt_params(m)
        p = sk.CztPlanGPU(n, a, w, m, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
        os.environ["SKG_4STEP_FUSED"] = "0"
        ref = p.execute(x)
        os.environ["SKG_4STEP_FUSED"] = "1"
        for cap, dx in itertools.product(caps, deltas):
            os.environ["SKG_4STEP_DELTA_X10"] = dx
            with sk.grid_cap(cap):
                got = p.execute(x)
                torch.cuda.synchronize()
            assert torch.equal(got, ref), (prec, n, m, cap, dx)
            n_ok += 1
        print(f"czt {prec} n={n} m={m}: {len(caps) * len(deltas)} variants ok", flush=True)
        del x, ref, got, p
print("all ok:", n_ok)
