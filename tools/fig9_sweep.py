"""The reference's resolution sweep (run_bench, bench.cpp:230-291 — the paper's Fig. 9: transform
time against target bin spacing) with a GPU method beside the CPU one.

Grid and sizes are bench_sizes (bench.cpp:45-60) restated: the 500-sample pulse at 10 THz, spacing
20 GHz down to 5 GHz in 0.5 GHz steps; record_len = record_len_for_step(fs, spacing), FFT length
next_pow2(record_len), CZT m matched to the FFT's spacing over 0.5-2 THz, zoom decimation
floor(fs / (2 band)). Per point and method:
  * gpu_call_us   — one trace, device-resident, plan reused (CUDA events around the call);
  * gpu_batch_us  — per-trace time of a 4096-trace batch (the throughput view);
  * ref_us        — the compiled reference on one host thread, plan reused (skr_* shim), when
                    oracle/_ref is built (test / baseline infrastructure only).
usage: python tools/fig9_sweep.py [out.json]"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

FS, TRACE_LEN, F1, F2 = 10e12, 500, 0.5e12, 2.0e12


def record_len_for_step(fs, step):   # resolution.cpp:18-26
    q = fs / step
    qr = round(q)
    return int(qr) if abs(q - qr) <= 1e-9 * q else int(math.ceil(q))


def sizes(res):   # bench.cpp:45-60
    rl = record_len_for_step(FS, res)
    m = max(1, int(round((F2 - F1) / FS * rl)))   # czt_len_for_matched_resolution
    d = max(1, int(math.floor(FS / (2.0 * (F2 - F1)))))
    return rl, 1 << (rl - 1).bit_length(), m, d


def ev_time(fn, reps=20, inner=1):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(inner):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / inner)
    return float(np.median(ts)) * 1e3   # us


def main(out_path):
    pulse = W.thz_pulse(TRACE_LEN, fs=FS)
    R = None
    try:
        import ctypes as C

        import oracle as O
        R = O.ref()
    except Exception:
        pass
    rows = []
    B = 4096
    for i in range(31):
        res = 20e9 - 0.5e9 * i
        rl, L, m, d = sizes(res)
        x1 = np.zeros(rl)
        x1[:TRACE_LEN] = pulse
        row = {"resolution_hz": res, "record_len": rl, "fft_len": L, "czt_m": m, "zoom_decimation": d}
        dev1 = torch.from_numpy(x1[None]).cuda()
        devB = dev1.repeat(B, 1)
        # fft / ifft: complex FFT of the zero-padded record (bench_one: FftPlan on a padded buffer)
        c1 = torch.zeros((1, L), dtype=torch.complex128, device="cuda")
        c1[0, :rl] = dev1[0]
        cB = c1.repeat(B, 1)
        o1, oB = torch.empty_like(c1), torch.empty_like(cB)
        row["fft_gpu_call_us"] = ev_time(lambda: sk.fft_batch(c1, out=o1))
        row["fft_gpu_batch_us"] = ev_time(lambda: sk.fft_batch(cB, out=oB), reps=5) / B
        row["ifft_gpu_call_us"] = ev_time(lambda: sk.fft_batch(c1, inverse=True, out=o1))
        row["ifft_gpu_batch_us"] = ev_time(lambda: sk.fft_batch(cB, inverse=True, out=oB), reps=5) / B
        # czt: the padded record over the band at matched spacing (czt_params_for_band, m bins)
        a, w = sk.czt_params_for_band(F1, F2, FS, m)
        cp = sk.CztPlanGPU(rl, a, w, m)
        z1 = torch.empty((1, m), dtype=torch.complex128, device="cuda")
        zB = torch.empty((B, m), dtype=torch.complex128, device="cuda")
        row["czt_gpu_call_us"] = ev_time(lambda: cp.execute(dev1, out=z1))
        row["czt_gpu_batch_us"] = ev_time(lambda: cp.execute(devB, out=zB), reps=5) / B
        # zoom: the padded record, decimation from the band
        zp = sk.ZoomPlanGPU(rl, F1, F2, FS, decimation=d)
        q1 = torch.empty((1, zp.bins), dtype=torch.complex128, device="cuda")
        qB = torch.empty((B, zp.bins), dtype=torch.complex128, device="cuda")
        row["zoom_gpu_call_us"] = ev_time(lambda: zp.execute(dev1, out=q1))
        row["zoom_gpu_batch_us"] = ev_time(lambda: zp.execute(devB, out=qB), reps=5) / B
        if R is not None:
            xr = np.ascontiguousarray(np.tile(x1, (64, 1)))
            t = R.skr_fft_batch(L, O._p(xr), rl, 64, 1, None)
            row["fft_ref_us"] = t / 64 * 1e6
            h = R.skr_czt_plan_create(rl, a.real, a.imag, w.real, w.imag, m)
            row["czt_ref_us"] = R.skr_czt_batch(h, O._p(xr), rl, 64, 1, None) / 64 * 1e6
            R.skr_czt_plan_free(h)
            hz = R.skr_zoom_plan_create(rl, F1, F2, FS, 0.0, 0, d, 0.0, 0, 1, 0, 1)
            nb, f0, df = C.c_size_t(), C.c_double(), C.c_double()
            row["zoom_ref_us"] = R.skr_zoom_batch(hz, O._p(xr), rl, FS, 64, 1, None, C.byref(nb), C.byref(f0),
                                                  C.byref(df)) / 64 * 1e6
            R.skr_zoom_plan_free(hz)
        rows.append(row)
        print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row.items()}, flush=True)
    meta = {"what": "run_bench resolution sweep (bench.cpp:230-291) with a GPU method", "fs_hz": FS,
            "trace_len": TRACE_LEN, "band_hz": [F1, F2], "batch_for_throughput": B,
            "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    with open(out_path, "w") as f:
        json.dump({"meta": meta, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "fig9_sweep.json"))
