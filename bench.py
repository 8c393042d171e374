"""bench.py — batched FFT / CZT / Zoom FFT throughput on B200 (BASELINE.json metric).

Headline workload (configs[1]): Bluestein CZT of 4096 THz-TDS trace pairs (8192 real traces,
N=1024, M=2048 over 0.1-3 THz, L=4096), fp64, inputs resident in HBM. A "step" is one pass of the
fused CZT kernel over the whole batch. Traces are independent, so N GPUs run weak-scaled batches
with no data-path collective. Extra keys report the other configs (fp32 CZT, cfg3 zoom,
cfg4 H cube, cfg1 latency) measured the same way.

  python bench.py [--gpus N --steps K --warmup W]          our CUDA path
  python bench.py --impl reference [...]                    the reference CPU path (oracle/_ref)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "traces/sec & achieved HBM GB/s (% of roofline) for batched FFT / CZT / Zoom FFT"
UNIT = "traces/s"


def _profile_version(path):
    """(round, version) from a profiles/ file name: r2v3_... -> (2, 3); r1_... -> (1, 0)."""
    import re
    m = re.match(r"r(\d+)(?:v(\d+))?", os.path.basename(path))
    return (int(m.group(1)), int(m.group(2) or 0)) if m else (-1, -1)


def ncu_traffic(kernel_prefix):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the named kernel from the newest
    (highest round, then version) committed ncu --set full summary in profiles/ (None when absent)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_full*.json")), key=_profile_version)
    best = None
    for f in files:
        try:
            with open(f) as fh:
                for d in json.load(fh)["launches"]:
                    if d["kernel"].startswith(kernel_prefix) and "dram_bytes" in d:
                        best = {"bytes": d["dram_bytes"], "source": os.path.relpath(f, ROOT)}
        except Exception:
            pass
    return best


def peaks():
    p = {"hbm_gbs": 6540.2, "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p["hbm_gbs"] = float(m["hbm_gbs"])
        p["source"] = "MEASURED_PEAKS.json"
    except Exception:
        pass
    return p


# ---- algorithmic counts ----------------------------------------------------------
def czt_counts(n, m, s):
    L = 1 << math.ceil(math.log2(n + m - 1))
    return {"bytes": n * s + m * 2 * s, "flops": 2 * 5 * L * math.log2(L) + 6 * (n + L + m), "L": L}


def zoom_counts(n, D, T, n_fft, nb, s):
    usable = (n // D) * D
    blk = usable // D
    return {"bytes": n * s + nb * 2 * s,
            "flops": 2 * usable + 4 * T * blk + 5 * n_fft * math.log2(n_fft) + 8 * nb}


def h_counts(n, L, s):
    return {"bytes": n * s + (L // 2 + 1) * 2 * s, "flops": 2.5 * L * math.log2(L) + 6 * (L // 2 + 1)}


class ClockSampler:
    """SM clock + throttle reasons polled through NVML every ~2 ms during the timed region
    (the recipe's nvidia-smi clocks line, at a rate that resolves sub-second regions)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0, period=0.002):
        self.index, self.period, self.sm, self.reasons, self.stop = index, period, [], 0, False
        self.smax = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:   # pragma: no cover
            self.err = str(e)
            self.N = None
        return self

    def _run(self):
        N = self.N
        while not self.stop:
            try:
                self.sm.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                self.reasons |= N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self.stop = True
        if getattr(self, "N", None):
            self.t.join(timeout=2)

    def summary(self):
        rs = sorted(k for k, bit in self.REASONS.items() if self.reasons & bit)
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.smax,
                "reasons": rs, "samples": len(self.sm), "source": "nvml"}


def dist_init(args=None, backend="nccl"):
    """One process per GPU (torchrun env). NCCL logs at INFO into a per-rank file (stdout carries
    only the JSON line); there is no collective on the data path, only barrier + max-over-ranks."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args is not None and args.gpus > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/skg_nccl.rank{rank}.%p.log")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    elif backend == "nccl" and torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world, device="cuda"):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_device(fn, steps, warmup, world, flush=None):
    """W untimed steps, then K steps bracketed by barrier + synchronize; CUDA events on the
    launching (current) stream; returns the max-over-ranks seconds for the K steps and the
    per-step event times."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(st)
    for a, b in evs:
        if flush is not None:
            flush()
        a.record(st)
        fn()
        b.record(st)
    t1.record(st)
    torch.cuda.synchronize()
    barrier(world)
    per = [a.elapsed_time(b) * 1e-3 for a, b in evs]
    kernel_total = max_over_ranks(sum(per), world)
    return kernel_total, per


def fp_peak_tflops(dtype):
    """In-run measured CUDA-core FMA peak: cuBLAS {D,S}GEMM 8192^3 (TF32 off), best of 5 —
    the same method MEASURED_PEAKS.json uses for bf16 (there is no fp64/fp32 entry there)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    n = 8192 if dtype == torch.float32 else 4096
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return 2 * n ** 3 / best / 1e12


# ---- CPU baseline (the reference on this host's cores) -----------------------------------------
def cpu_model():
    """The reference's bench_environment() line (bench.cpp:100-129) when the reference is built,
    else /proc/cpuinfo's model name (what that function reads)."""
    try:
        import oracle
        R = oracle.ref()
        if R is not None:
            return R.skr_bench_environment().decode()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return "cpu: " + line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown cpu"


def _measure_cpu(run, total, seconds, threads):
    """run(count, threads) -> wall seconds; grows the sample until it takes >= seconds / 2 (or the
    whole workload). Returns (units/s, count, seconds)."""
    run(min(total, threads), threads)   # warm-up: page in, start threads
    cnt = min(total, 2 * threads)
    dt = run(cnt, threads)
    while dt < seconds / 2 and cnt < total:
        cnt = min(total, max(cnt * 2, int(cnt * seconds / 2 / max(dt, 1e-4))))
        dt = run(cnt, threads)
    return cnt / dt, cnt, dt


def cpu_baseline(run, total, what, seconds, kind, unit=UNIT):
    """The reference CPU path at all host threads and at one thread."""
    T = os.cpu_count() or 1
    v, c, dt = _measure_cpu(run, total, seconds, T)
    v1, c1, dt1 = _measure_cpu(run, total, seconds / 2, 1)
    return {"value": v, "unit": unit, "cores": T, "kind": kind, "value_t1": v1, "cores_t1": 1,
            "cpu_model": cpu_model(),
            "sample": f"{what}: {c} units on {T} threads in {dt:.2f} s; {c1} units on 1 thread in {dt1:.2f} s"}


def ref_runners(x_czt=None, czt=None, x_zoom=None, zoom=None, x_px=None, px=None):
    """run(count, threads) closures over the compiled reference (oracle/_ref: CztPlan::execute,
    zoom_fft, FftPlan::forward + restated H, plan reuse, shared plan) — or the C port when the
    reference was not built. Returns (dict of closures, kind)."""
    import oracle
    R = oracle.ref()
    kind = "reference" if R is not None else "port"
    runs = {}
    if czt is not None:
        n, a, w, m = czt
        xs = np.ascontiguousarray(x_czt, dtype=np.float64)
        if R is not None:
            p = R.skr_czt_plan_create(n, a.real, a.imag, w.real, w.imag, m)
            runs["czt"] = lambda cnt, th: R.skr_czt_batch(p, oracle._p(xs), n, cnt, th, None)
        else:
            plan = oracle.CztPlan(n, a, w, m)
            runs["czt"] = lambda cnt, th: oracle.port().sko_bench_czt(plan._h, oracle._p(xs), n, cnt, th, None)
        runs["_keep_czt"] = xs
    if zoom is not None:
        n, f1, f2, fs, d, taps, n_fft = zoom
        xz = np.ascontiguousarray(x_zoom, dtype=np.float64)
        if R is not None:
            zp = R.skr_zoom_plan_create(n, f1, f2, fs, 0.0, 0, d, 0.0, taps, 1, 0, 1)
            if n_fft:
                R.skr_zoom_plan_set_n_fft(zp, n_fft)
            runs["zoom"] = lambda cnt, th: R.skr_zoom_batch(zp, oracle._p(xz), n, fs, cnt, th, None, None, None, None)
        else:
            op = oracle.ZoomPlan(n, f1, f2, fs, decimation=d, num_taps=taps, **({"n_fft": n_fft} if n_fft else {}))
            runs["zoom"] = lambda cnt, th: op.batch(xz[:cnt], th)
        runs["_keep_zoom"] = xz
    if px is not None and R is not None:
        L, ref = px
        xp = np.ascontiguousarray(x_px, dtype=np.float64)
        rf = np.ascontiguousarray(ref, dtype=np.float64)
        runs["px"] = lambda cnt, th: R.skr_transfer_batch(L, oracle._p(rf), oracle._p(xp), xp.shape[1], cnt, th,
                                                          None, None)
        runs["_keep_px"] = (xp, rf)
    return runs, kind


def dt_name(prec):
    return "double" if prec == "f64" else "float"


def roofline_entry(bytes_per, flops_per, units, kern_s, hbm_gbs, fp_tflops, fp_name, kernel, traffic_prefix):
    """roof time = max(bytes / HBM, flops / FP peak); frac = roof time / measured time,
    reported in the bound's units."""
    t_hbm = bytes_per * units / (hbm_gbs * 1e9)
    t_fp = flops_per * units / (fp_tflops * 1e12)
    tr = ncu_traffic(traffic_prefix) if traffic_prefix else None
    if t_hbm >= t_fp:
        ach, peak, unit, bound = bytes_per * units / kern_s / 1e9, hbm_gbs, "GB/s", "hbm"
    else:
        ach, peak, unit, bound = flops_per * units / kern_s / 1e12, fp_tflops, "TFLOP/s", fp_name
    return {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
            "traffic": (tr or {}).get("bytes"), "traffic_source": (tr or {}).get("source"),
            "kernel": kernel, "kernel_ms": kern_s * 1e3, "bytes_per_unit": bytes_per, "flops_per_unit": flops_per,
            "units_per_launch": units, "hbm_frac": bytes_per * units / kern_s / 1e9 / hbm_gbs,
            "fp_frac": flops_per * units / kern_s / 1e12 / fp_tflops}


# ---- the headline workload, shared by both arms -----------------------------------------------
def headline_config(world):
    return {"workload": "cfg2: Bluestein CZT of 4096 THz-TDS trace pairs = 8192 real traces, N=1024, "
                        "M=2048 over 0.1-3 THz ((M-1) W step), L=4096, fp64",
            "global_batch": 8192 * world, "per_gpu_batch": 8192,
            "parallelism": f"dp{world} (independent traces, weak-scaled, no collective)",
            "l2": "inputs 64 MiB + outputs 256 MiB per step > 126 MB L2 (no flush needed)"}


# ---- our path ---------------------------------------------------------------------------------
def bench_ours(args):
    import torch

    import paper_2108_03948_b200 as sk
    from paper_2108_03948_b200 import workloads as W
    rank, world, local = dist_init(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pk = peaks()
    info = sk.device_info()
    K, Wm = args.steps, args.warmup

    # ---- headline: cfg2 CZT fp64 -----------------------------------------------------------
    x_host = W.cfg2_batch(args.pairs, 1024).astype(np.float64)      # 8192 x 1024 (ref, sample pairs)
    B = x_host.shape[0]
    a, w = W.cfg2_czt_params(2048)
    plan = sk.CztPlanGPU(1024, a, w, 2048, sk.SKG_F64)
    xd = torch.from_numpy(x_host).to(dev)
    out = torch.empty((B, 2048), dtype=torch.complex128, device=dev)
    fn = lambda: plan.execute(xd, out=out)  # noqa: E731
    fn()
    torch.cuda.synchronize()
    l0 = sk.launch_count()
    fn()
    per_step_launches = sk.launch_count() - l0
    with ClockSampler(local) as clk:
        total, per = time_device(fn, K, Wm, world)
    ms = total / K * 1e3
    value = world * B * K / total
    c = czt_counts(1024, 2048, 8)
    fp64_peak = fp_peak_tflops(torch.float64)
    kern_s = float(np.mean(per))
    # S=2 blocks of the L=4096 plan at L'=2048, one shared forward FFT, tables + parked spectrum in TMEM
    kname = "k_czt_tm<double, 11"
    roof = roofline_entry(c["bytes"], c["flops"], B, kern_s, pk["hbm_gbs"], fp64_peak, "fp64", kname, kname)
    roof["peak_source"] = "in-run cuBLAS DGEMM 4096^3 (MEASURED_PEAKS.json has no fp64 entry)"
    roof["hbm_peak_source"] = pk["source"]

    # ---- e2e: pinned host rows through the C ABI's host-buffer call (skg_czt_execute_host:
    # chunked H2D / kernel / D2H on the library's streams), every step ---------------------------
    xh = torch.from_numpy(x_host).pin_memory()
    oh = torch.empty((B, 2048), dtype=torch.complex128).pin_memory()
    e2e_fn = lambda: plan.execute_host(xh, out=oh)  # noqa: E731
    for _ in range(2):
        e2e_fn()
    l0 = sk.launch_count()
    e2e_fn()
    e2e_launches = sk.launch_count() - l0
    barrier(world)
    ke = max(2, K // 2)
    t0 = time.perf_counter()
    for _ in range(ke):
        e2e_fn()
    e2e_dt = max_over_ranks(time.perf_counter() - t0, world)
    e2e_val = world * B * ke / e2e_dt
    # every e2e row against the CPU oracle (the C restatement pinned to the reference at 0 ulp)
    e2e_err = None
    if not args.no_cpu:
        import oracle as O
        want = O.CztPlan(1024, a, w, 2048).batch_real(x_host, threads=os.cpu_count() or 4)
        got = oh.numpy()
        e2e_err = float(np.max(np.max(np.abs(got - want), axis=1) / np.max(np.abs(want), axis=1)))

    extra = {}
    if not args.quick and world == 1:   # single-GPU characterisation (the scaled metric is the headline)
        extra = bench_extras(args, sk, W, dev, world, pk, fp64_peak)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": Wm,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded THz-TDS pulse pairs, SURVEY §8d)",
        "config": headline_config(world),
        "roofline": roof,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(B * 1024 * 8),
                "d2h_bytes_per_step": int(B * 2048 * 16), "api": "skg_czt_execute_host (pinned host rows)",
                "launches_per_step": int(e2e_launches), "max_rel_err_vs_oracle_all_rows": e2e_err},
        "gpu_launches": int(per_step_launches * K),
        "clocks": clk.summary(),
        "device": info,
    }
    if world > 1:
        line["nccl_log"] = os.environ.get("NCCL_DEBUG_FILE")
    if extra:
        line["extra"] = extra
    if rank == 0 and world == 1 and not args.no_cpu:
        runs, kind = ref_runners(x_czt=x_host, czt=(1024, a, w, 2048))
        line["cpu_baseline"] = cpu_baseline(runs["czt"], B, "cfg2 traces, CztPlan::execute plan reuse, shared plan",
                                            args.cpu_seconds, kind)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def bench_extras(args, sk, W, dev, world, pk, fp64_peak):
    import torch
    res = {}
    K = max(3, args.steps // 2)
    Wm = 3
    fp32_peak = fp_peak_tflops(torch.float32)
    peak_of = {"f64": (fp64_peak, "fp64"), "f32": (fp32_peak, "fp32")}
    # cfg2 fp32
    x = W.cfg2_batch(args.pairs, 1024)
    a, w = W.cfg2_czt_params(2048)
    p32 = sk.CztPlanGPU(1024, a, w, 2048, sk.SKG_F32)
    xd = torch.from_numpy(x.astype(np.float32)).to(dev)
    out = torch.empty((x.shape[0], 2048), dtype=torch.complex64, device=dev)
    t, per = time_device(lambda: p32.execute(xd, out=out), K, Wm, world)
    c = czt_counts(1024, 2048, 4)
    ks = float(np.mean(per))
    res["cfg2_czt_f32"] = {"traces_per_s": x.shape[0] * K / t,
                           "roofline": roofline_entry(c["bytes"], c["flops"], x.shape[0], ks, pk["hbm_gbs"],
                                                      fp32_peak, "fp32", "k_czt_tm<float, 11", "k_czt_tm<float, 11"),
                           "fp32_peak_source": "in-run cuBLAS SGEMM 8192^3, TF32 off"}
    del xd, out
    cpu = {}
    # cfg3 zoom (reference sizing n_fft 512, and the 2048 text variant), fp64 + fp32
    x3 = W.cfg3_batch(4096, 4096)
    if not args.no_cpu:
        for nf in (0, 2048):
            runs, kind = ref_runners(x_zoom=x3, zoom=(4096, 0.4e12, 1.2e12, W.FS, 8, 65, nf))
            cpu[nf] = cpu_baseline(runs["zoom"], x3.shape[0], f"cfg3 records, zoom_fft plan reuse (n_fft "
                                   f"{nf or 512})", args.cpu_seconds / 2, kind)
    for prec, dt, s in (("f64", torch.float64, 8), ("f32", torch.float32, 4)):
        xd = torch.from_numpy(x3).to(dt).to(dev)
        for nf in (0, 2048):
            zp = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, sk.SKG_F64 if prec == "f64" else sk.SKG_F32, n_fft=nf,
                                decimation=8, num_taps=65)
            out = torch.empty((4096, zp.bins), dtype=torch.complex128 if prec == "f64" else torch.complex64,
                              device=dev)
            l0 = sk.launch_count()
            zp.execute(xd, out=out)
            nl = sk.launch_count() - l0
            t, per = time_device(lambda: zp.execute(xd, out=out), K, Wm, world)
            ks = float(np.mean(per))
            cc = zoom_counts(4096, 8, 65, zp.n_fft, zp.bins, s)
            e = {"traces_per_s": 4096 * K / t, "launches_per_call": nl,
                 "roofline": roofline_entry(cc["bytes"], cc["flops"], 4096, ks, pk["hbm_gbs"], peak_of[prec][0],
                                            peak_of[prec][1], "zoom call",
                                            f"unnamed>::k_zoom_{'rfir_fft' if nf else 'pcfir'}<{dt_name(prec)}, 8, 65")}
            if nf in cpu:
                e["cpu_baseline"] = cpu[nf]
            res[f"cfg3_zoom_nfft{zp.n_fft}_{prec}"] = e
        del xd
    # cfg4 cube: 65536 px x 2048 fp32 -> |H|, arg H on 4097 bins
    cube, ref = W.cfg4_cube(256, 256, 2048)
    tp = sk.TransferPlanGPU(ref, 8192, sk.SKG_F32)
    cd = torch.from_numpy(cube).to(dev)
    mag = torch.empty((cube.shape[0], tp.bins), dtype=torch.float32, device=dev)
    ph = torch.empty_like(mag)
    t, per = time_device(lambda: tp.execute(cd, mag, ph), K, Wm, world)
    ks = float(np.mean(per))
    hc = h_counts(2048, 8192, 4)
    e = {"pixels_per_s": cube.shape[0] * K / t,
         "roofline": roofline_entry(hc["bytes"], hc["flops"], cube.shape[0], ks, pk["hbm_gbs"], fp32_peak, "fp32",
                                    "k_fft_r2c<float, 12", "k_fft_r2c<float, 12")}
    if not args.no_cpu:
        runs, kind = ref_runners(x_px=cube[:8192], px=(8192, ref))
        if "px" in runs:
            e["cpu_baseline"] = cpu_baseline(runs["px"], 8192, "cfg4 pixels, FftPlan(8192)::forward + restated H "
                                             "(reference FFT, fp64)", args.cpu_seconds / 2, kind, unit="pixels/s")
    res["cfg4_cube_H_f32"] = e
    del cd, mag, ph
    # cfg5 long zero-padded spectra (N = 16384 -> 65536 bins, full layout): the Hermitian-half four-step in
    # one cooperative launch, work rows in an L2-resident ring (0.5 GiB of traces in, 4 GiB of spectra out)
    n5, L5 = 16384, 65536
    for prec, dt, s in (("f64", torch.float64, 8), ("f32", torch.float32, 4)):
        b5 = (1 << 29) // (n5 * s)
        x5 = torch.from_numpy(W.sample_traces(64, n5)).to(dt).to(dev).repeat(b5 // 64, 1)
        out = torch.empty((b5, L5), dtype=torch.complex128 if prec == "f64" else torch.complex64, device=dev)
        l0 = sk.launch_count()
        sk.fft_spectrum_batch(x5, L5, out=out)
        nl = sk.launch_count() - l0
        t, per = time_device(lambda: sk.fft_spectrum_batch(x5, L5, out=out), K, Wm, world)
        ks = float(np.mean(per))
        res[f"cfg5_fft65536_{prec}"] = {
            "traces_per_s": b5 * K / t, "launches_per_call": nl,
            "roofline": roofline_entry(n5 * s + L5 * 2 * s, 2.5 * L5 * math.log2(L5), b5, ks, pk["hbm_gbs"],
                                       peak_of[prec][0], peak_of[prec][1], f"k4_rfused<{dt_name(prec)}, 8",
                                       f"k4_rfused<{dt_name(prec)}, 8")}
        del x5, out
    # SURVEY §8f rows 1-2, files -> files: 1024 cfg2 traces (N=1024 fp64) as reference-format CSV
    # (written once, untimed); a step = batched ingest -> fused band FFT 4096 (0.1-3 THz) -> batched
    # reference-format CSV writer. Host wall clock (file I/O and parsing are the work here).
    res["csv_pipeline_f64"] = bench_csv_pipeline(args, sk, W, dev)
    # the two-tone resolvability sweep as a batched caller (THz scale: fs 20 THz,
    # n 1024, band 0.1-3 THz, m 2048 -> padded FFT 14124 via Bluestein, 999 separations)
    res["resolvability_scan_thz"] = bench_scan(args, sk, W)
    # cfg1 latency: one pair, fp64, FFT 4096 + H (device-resident) and through the C ABI (host)
    r1, s1 = W.cfg1_pair()
    tp1 = sk.TransferPlanGPU(r1, 4096, sk.SKG_F64)
    sd = torch.from_numpy(s1[None]).to(dev)
    t, per = time_device(lambda: tp1.execute(sd), 20, 5, world)
    sk.fft_spectrum(s1, W.FS, 4096)   # first call: per-thread staging buffers, tables
    torch.cuda.synchronize()
    calls = []
    for _ in range(30):
        t0 = time.perf_counter()
        sk.fft_spectrum(s1, W.FS, 4096)
        calls.append(time.perf_counter() - t0)
    res["cfg1_pair_f64"] = {"device_us_per_pair_H": float(np.median(per)) * 1e6,
                            "c_abi_us_per_fft_spectrum": float(np.median(calls)) * 1e6,
                            "c_abi_us_per_fft_spectrum_max": float(np.max(calls)) * 1e6}
    return res


def bench_csv_pipeline(args, sk, W, dev, nfiles=1024):
    import tempfile

    import torch
    x = W.cfg2_batch(nfiles // 2, 1024)
    with tempfile.TemporaryDirectory() as td:
        ins = [os.path.join(td, f"t{i:05d}.csv") for i in range(nfiles)]
        outs = [os.path.join(td, f"s{i:05d}.csv") for i in range(nfiles)]
        for p, r in zip(ins, x):
            sk.trace_write_csv(r, W.FS, 0.0, p)

        def step():
            d, fs, _ = sk.traces_read_csv(ins, 1024, device=dev)
            bins, _, f0, df = sk.fft_spectrum_band_batch(d, fs[0], 0.1e12, 3.0e12, 4096, db=False)
            sk.spectra_write_csv(outs, bins, f0, df)
            return bins.shape[1]

        nb = step()
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out_bytes = sum(os.path.getsize(p) for p in outs)
        in_bytes = sum(os.path.getsize(p) for p in ins)
        res = {"files_per_s": nfiles / float(np.median(ts)), "ms_per_step": float(np.median(ts)) * 1e3,
               "bins_per_file": nb, "csv_in_mb": in_bytes / 1e6, "csv_out_mb": out_bytes / 1e6,
               "host_threads": os.cpu_count()}
        if not args.no_cpu:
            try:
                import oracle as O
                from concurrent.futures import ThreadPoolExecutor
                if O.ref() is not None:
                    refo = [p + ".ref" for p in outs]
                    with ThreadPoolExecutor(os.cpu_count()) as ex:
                        t0 = time.perf_counter()
                        list(ex.map(lambda i: O.ref_csv_chain(ins[i], refo[i], 4096, 0.1e12, 3.0e12), range(nfiles)))
                        tr = time.perf_counter() - t0
                    worst = 0.0
                    for a, b in zip(outs[:16], refo[:16]):   # parsed back: bins of the GPU path vs the reference
                        ga, gb = np.loadtxt(a, delimiter=",", skiprows=1), np.loadtxt(b, delimiter=",", skiprows=1)
                        za, zb = ga[:, 1] + 1j * ga[:, 2], gb[:, 1] + 1j * gb[:, 2]
                        worst = max(worst, float(np.max(np.abs(za - zb)) / np.max(np.abs(zb))))
                        assert np.array_equal(ga[:, 0], gb[:, 0])
                    res["reference_files_per_s"] = nfiles / tr
                    res["reference_kind"] = ("compiled reference: sk_trace_read_csv -> sk_fft_spectrum -> "
                                             f"sk_spectrum_slice_band -> sk_spectrum_write_csv, {os.cpu_count()} threads")
                    res["parity_max_rel_vs_reference"] = worst
            except Exception as e:   # the reference arm is a report, not a gate
                res["reference_error"] = str(e)[:200]
    return res


def bench_scan(args, sk, W):
    import torch
    cfg = dict(W.SCAN_CASES["thz"], center_hz=1.5e12, sep_start_hz=1e9, sep_stop_hz=500e9, sep_step_hz=0.5e9)
    got = sk.resolvability_scan(**cfg)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got = sk.resolvability_scan(**cfg)
        ts.append(time.perf_counter() - t0)
    S = got["separations_hz"].size
    res = {"separations": S, "fft_len": got["fft_len"], "separations_per_s": S / float(np.median(ts)),
           "ms_per_sweep": float(np.median(ts)) * 1e3, "min_resolved_fft_hz": got["min_resolved_fft_hz"],
           "min_resolved_czt_hz": got["min_resolved_czt_hz"]}
    if not args.no_cpu:
        try:
            import ctypes as C

            import oracle as O
            R = O.ref()
            if R is not None:   # the reference's own sweep (single thread, as it runs) on a bounded subset
                sub = dict(cfg, sep_stop_hz=cfg["sep_start_hz"] + 19 * cfg["sep_step_hz"])
                c = sk.scan_config(**sub)
                R.sk_resolvability_scan.argtypes = [C.POINTER(sk.SkScanConfig), C.POINTER(C.c_void_p)]
                R.sk_resolvability_curve_free.argtypes = [C.c_void_p]
                h = C.c_void_p()
                t0 = time.perf_counter()
                assert R.sk_resolvability_scan(C.byref(c), C.byref(h)) == 0
                tr = time.perf_counter() - t0
                R.sk_resolvability_curve_free(h)
                res["reference_separations_per_s"] = 20 / tr
                res["reference_kind"] = "compiled reference sk_resolvability_scan, 1 thread, 20 separations"
        except Exception as e:
            res["reference_error"] = str(e)[:200]
    return res


# ---- reference arm ----------------------------------------------------------------------------
def bench_reference(args):
    """The reference's own CPU implementation of the path (oracle/_ref: the unmodified reference
    compiled from its sources; CztPlan::execute with plan reuse, as its bench harness runs it,
    bench.cpp:194-204) on all host threads, on the same config as our arm. Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from paper_2108_03948_b200 import workloads as W
    threads = os.cpu_count() or 1
    x = W.cfg2_batch(args.pairs, 1024)
    a, w = W.cfg2_czt_params(2048)
    runs, kind = ref_runners(x_czt=x, czt=(1024, a, w, 2048))
    run = runs["czt"]
    # one step = the whole 8192-trace batch when that takes <= ref_step_s, else a bounded sample
    dt = run(threads, threads)
    per_trace = dt / threads
    cnt = int(min(len(x), max(threads, args.ref_step_s / max(per_trace, 1e-9) * threads)))
    for _ in range(args.warmup):
        run(cnt, threads)
    tot = 0.0
    for _ in range(args.steps):
        tot += run(cnt, threads)
    value = cnt * args.steps / tot
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded THz-TDS pulse pairs, SURVEY §8d)",
            "config": headline_config(world),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                             "sample": f"{cnt} of the {len(x)} cfg2 traces per step, CztPlan::execute plan reuse, "
                                       f"shared plan, {threads} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run with N ranks
    (one process per GPU, 127.0.0.1 rendezvous), as the driver launches it."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def selftest_dist(args):
    """CPU check of the multi-rank plumbing (gloo): launcher, rank / world discovery, barrier,
    max-over-ranks timing and the rank-0-only JSON line — what --gpus N runs around the kernels."""
    rank, world, _ = dist_init(args, backend="gloo")
    per = [0.001 * (rank + 1)] * args.steps
    total = max_over_ranks(sum(per), world, device="cpu")
    barrier(world)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": world * 8192 * args.steps / total, "unit": UNIT,
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "selftest": "gloo",
                          "max_over_ranks_s": total, "config": headline_config(world)}), flush=True)
    import torch.distributed as dist
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pairs", type=int, default=4096)
    ap.add_argument("--quick", action="store_true", help="headline only")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=4.0)
    ap.add_argument("--ref-step-s", type=float, default=3.0)
    ap.add_argument("--selftest-dist", action="store_true", help="CPU (gloo) check of the multi-rank plumbing")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    if args.selftest_dist:
        selftest_dist(args)
    elif args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
