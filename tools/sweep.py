"""configs[4] sweep on one B200: for N in {1000, 1024, 3000, 4096, 16384, 65536} — zero-padded FFT to
4*next_pow2(N), CZT with M in {N/4, N, 4N} over 0.1-3 THz ((M-1) W step), Zoom FFT with D in {4, 16}
over 0.4-1.2 THz — in fp64 and fp32, batch sized to ~1 GiB of input (capped so one
row stays within a few seconds). Each row: traces/s, achieved GB/s and TFLOP/s on the algorithmic
counts, fraction of the roof max(bytes/HBM, flops/FP peak), and a parity check of the
first, a middle and the last trace of the batch against the CPU oracle. Inputs are generated on the GPU (seeded pulse + noise)
and copied back for the check.

usage: python tools/sweep.py [--out profiles/r1_cfg5_sweep.json] [--quick]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2108_03948_b200 as sk  # noqa: E402
from bench import czt_counts, fp_peak_tflops, peaks, zoom_counts  # noqa: E402

FS = 20e12


def gen(B, n, dtype, seed):
    """a pulse(10 ps + d) + 0.25 a pulse(16 ps + d) + noise, generated on the device in fp64."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    d = torch.rand(B, 1, device="cuda", dtype=torch.float64, generator=g) * 3e-12 + 1e-12
    a = torch.rand(B, 1, device="cuda", dtype=torch.float64, generator=g) * 0.6 + 0.3
    t = torch.arange(n, device="cuda", dtype=torch.float64)[None, :] / FS
    x = torch.empty(B, n, device="cuda", dtype=dtype)
    step = max(1, (1 << 26) // n)
    for s in range(0, B, step):
        e = min(B, s + step)
        tt = t
        u1 = (tt - 10e-12 - d[s:e]) / 0.3e-12
        u2 = (tt - 16e-12 - d[s:e]) / 0.3e-12
        v = -(a[s:e] * math.exp(0.5)) * (u1 * torch.exp(-0.5 * u1 * u1) + 0.25 * u2 * torch.exp(-0.5 * u2 * u2))
        v += 1e-3 * torch.randn(e - s, n, device="cuda", dtype=torch.float64, generator=g)
        x[s:e] = v.to(dtype)
    return x


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


def check_rows(nb):
    """rows compared with the oracle: the first, a middle and the last of the batch actually run (the
    persistent kernels' later waves included)"""
    return sorted({0, nb // 2, nb - 1})


def parity(got, want, f32):
    got, want = np.asarray(got, np.complex128), np.asarray(want, np.complex128)
    if f32:
        return max(np.linalg.norm(g - w) / np.linalg.norm(w) for g, w in zip(got, want))
    return max(np.max(np.abs(g - w)) / np.max(np.abs(w)) for g, w in zip(got, want))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_cfg5_sweep.json"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--max-seconds", type=float, default=1.5, help="cap on one batch's kernel time")
    ap.add_argument("--ns", default="", help="comma list of N to run (default: all)")
    ap.add_argument("--kinds", default="fft,czt,zoom")
    ap.add_argument("--precs", default="f64,f32")
    args = ap.parse_args()
    pk = peaks()
    fp = {"f64": fp_peak_tflops(torch.float64), "f32": fp_peak_tflops(torch.float32)}
    rows = []
    Ns = [1000, 1024, 3000, 4096, 16384, 65536] if not args.quick else [1000, 4096]
    if args.ns:
        Ns = [int(v) for v in args.ns.split(",")]
    kinds = set(args.kinds.split(","))
    for prec in args.precs.split(","):
        dt = torch.float64 if prec == "f64" else torch.float32
        s = 8 if prec == "f64" else 4
        P = sk.SKG_F64 if prec == "f64" else sk.SKG_F32
        for N in Ns:
            B = (1 << 30) // (N * s)
            x = gen(B, N, dt, seed=N)
            jobs = []
            L = 4 * O.next_pow2(N)
            if "fft" in kinds:
                jobs.append(("fft", {"L": L}))
            if "czt" in kinds:
                for M in (N // 4, N, 4 * N):
                    jobs.append(("czt", {"M": M}))
            if "zoom" in kinds:
                for D in (4, 16):
                    jobs.append(("zoom", {"D": D}))
            for kind, kw in jobs:
                torch.cuda.empty_cache()
                if kind == "fft":
                    L = kw["L"]
                    fl = 2.5 * L * math.log2(L)
                    by = N * s + L * 2 * s
                    nb = B
                    out = torch.empty((nb, L), dtype=torch.complex128 if prec == "f64" else torch.complex64,
                                      device="cuda")
                    fn = lambda: sk.fft_spectrum_batch(x[:nb], L, out=out)  # noqa: E731
                    t1 = timeit(fn, 1, 1)
                    if t1 > args.max_seconds:
                        nb = max(64, int(nb * args.max_seconds / t1))
                        out = out[:nb]
                        fn = lambda: sk.fft_spectrum_batch(x[:nb], L, out=out)  # noqa: E731
                    t = timeit(fn)
                    rr = check_rows(nb)
                    want = O.fft_spectrum_batch(x[rr].double().cpu().numpy(), L)
                    err = parity(out[rr].cpu().numpy(), want, prec == "f32")
                    label = f"FFT N={N} L={L}"
                elif kind == "czt":
                    M = kw["M"]
                    a, w = complex(np.exp(2j * np.pi * 0.1e12 / FS)), complex(np.exp(-2j * np.pi * (2.9e12 / (M - 1)) / FS))
                    plan = sk.CztPlanGPU(N, a, w, M, P)
                    c = czt_counts(N, M, s)
                    fl, by = c["flops"], c["bytes"]
                    nb = B
                    if nb * M * 2 * s > 24e9:
                        nb = int(24e9 / (M * 2 * s))
                    out = torch.empty((nb, M), dtype=torch.complex128 if prec == "f64" else torch.complex64,
                                      device="cuda")
                    fn = lambda: plan.execute(x[:nb], out=out)  # noqa: E731
                    t1 = timeit(fn, 1, 1)
                    if t1 > args.max_seconds:
                        nb = max(16, int(nb * args.max_seconds / t1))
                        out = out[:nb]
                        fn = lambda: plan.execute(x[:nb], out=out)  # noqa: E731
                    t = timeit(fn)
                    rr = check_rows(nb)
                    want = O.CztPlan(N, a, w, M).batch_real(x[rr].double().cpu().numpy())
                    err = parity(out[rr].cpu().numpy(), want, prec == "f32")
                    label = f"CZT N={N} M={M} L={c['L']}"
                    del plan
                else:
                    D = kw["D"]
                    plan = sk.ZoomPlanGPU(N, 0.4e12, 1.2e12, FS, P, decimation=D)
                    c = zoom_counts(N, D, plan.num_taps, plan.n_fft, plan.bins, s)
                    fl, by = c["flops"], c["bytes"]
                    nb = B
                    out = torch.empty((nb, plan.bins), dtype=torch.complex128 if prec == "f64" else torch.complex64,
                                      device="cuda")
                    fn = lambda: plan.execute(x[:nb], out=out)  # noqa: E731
                    t1 = timeit(fn, 1, 1)
                    if t1 > args.max_seconds:
                        nb = max(64, int(nb * args.max_seconds / t1))
                        out = out[:nb]
                        fn = lambda: plan.execute(x[:nb], out=out)  # noqa: E731
                    t = timeit(fn)
                    ref = O.ZoomPlan(N, 0.4e12, 1.2e12, FS, decimation=D)
                    rr = check_rows(nb)
                    err = parity(out[rr].cpu().numpy(), [ref(r)[0] for r in x[rr].double().cpu().numpy()],
                                 prec == "f32")
                    label = f"ZOOM N={N} D={D} n_fft={plan.n_fft} bins={plan.bins}"
                    del plan
                del out
                roof_t = max(by * nb / (pk["hbm_gbs"] * 1e9), fl * nb / (fp[prec] * 1e12))
                bound = "HBM" if by * nb / (pk["hbm_gbs"] * 1e9) >= fl * nb / (fp[prec] * 1e12) else "FP"
                row = {"prec": prec, "row": label, "batch": nb, "seconds": t, "traces_per_s": nb / t,
                       "gbs": by * nb / t / 1e9, "tflops": fl * nb / t / 1e12, "bound": bound,
                       "roof_frac": roof_t / t, "parity": err,
                       "parity_ok": bool(err <= (1e-5 if prec == "f32" else 1e-10)), "parity_rows": rr}
                rows.append(row)
                print(json.dumps(row), flush=True)
            del x
    meta = {"hbm_gbs": pk["hbm_gbs"], "fp64_peak_tflops": fp["f64"], "fp32_peak_tflops": fp["f32"],
            "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "device": sk.device_info()}
    with open(args.out, "w") as f:
        json.dump({"meta": meta, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
