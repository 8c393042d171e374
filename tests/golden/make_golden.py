"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Run in the build container (needs /root/reference and `make -C oracle ref`):
    python tests/golden/make_golden.py
Every output array here is produced by the unmodified reference C++ (oracle/_ref/libskref.so:
its own sk_* C ABI plus the plan-reuse shim), never by our code. Inputs are seeded. The
fixtures pin (a) the oracle restatement (tests/test_oracle.py) and (b) the GPU path
(tests/test_gpu_*.py) at sizes that stay small in git.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2108_03948_b200 import workloads as W  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
R = oracle.ref()
if R is None:
    raise SystemExit("oracle/_ref/libskref.so missing: run `make -C oracle ref` first")
P = oracle._p


def ref_fft(x, inverse=False):
    re, im = np.ascontiguousarray(x.real), np.ascontiguousarray(x.imag)
    rc = (R.sk_ifft if inverse else R.sk_fft)(P(re), P(im), re.size)
    assert rc == 0, R.sk_last_error()
    return re + 1j * im


def ref_czt(x, a, w, m):
    x = np.asarray(x, np.complex128)
    re, im = np.ascontiguousarray(x.real), np.ascontiguousarray(x.imag)
    orr, oi = np.zeros(m), np.zeros(m)
    rc = R.sk_czt(P(re), P(im), x.size, a.real, a.imag, w.real, w.imag, m, P(orr), P(oi))
    assert rc == 0, R.sk_last_error()
    return orr + 1j * oi


def ref_dft_naive(x):
    re, im = np.ascontiguousarray(x.real), np.ascontiguousarray(x.imag)
    orr, oi = np.zeros(x.size), np.zeros(x.size)
    assert R.sk_dft_naive(P(re), P(im), x.size, P(orr), P(oi)) == 0
    return orr + 1j * oi


def ref_fft_spectrum(samples, fs, length):
    s = np.ascontiguousarray(samples, np.float64)
    t = C.c_void_p()
    assert R.sk_trace_create(P(s), s.size, fs, 0.0, C.byref(t)) == 0
    sp = C.c_void_p()
    assert R.sk_fft_spectrum(t, length, C.byref(sp)) == 0, R.sk_last_error()
    n = R.sk_spectrum_size(sp)
    re, im = np.zeros(n), np.zeros(n)
    R.sk_spectrum_copy_data(sp, P(re), P(im))
    f0, df = R.sk_spectrum_f_start(sp), R.sk_spectrum_f_step(sp)
    R.sk_spectrum_free(sp)
    R.sk_trace_free(t)
    return re + 1j * im, f0, df


def ref_band(samples, fs, length, lo, hi):
    """sk_fft_spectrum -> sk_spectrum_slice_band -> per-bin sk_spectrum_magnitude_db (the CLI's
    half-spectrum / band rows, spectral_kit.cpp:143-148, and the CSV dB column, spectra.cpp:63-72)."""
    R.sk_spectrum_slice_band.argtypes = [C.c_void_p, C.c_double, C.c_double, C.POINTER(C.c_void_p)]
    R.sk_spectrum_magnitude_db.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_double)]
    s = np.ascontiguousarray(samples, np.float64)
    t = C.c_void_p()
    assert R.sk_trace_create(P(s), s.size, fs, 0.0, C.byref(t)) == 0
    sp = C.c_void_p()
    assert R.sk_fft_spectrum(t, length, C.byref(sp)) == 0, R.sk_last_error()
    band = C.c_void_p()
    assert R.sk_spectrum_slice_band(sp, lo, hi, C.byref(band)) == 0, R.sk_last_error()
    n = R.sk_spectrum_size(band)
    re, im = np.zeros(n), np.zeros(n)
    R.sk_spectrum_copy_data(band, P(re), P(im))
    db = np.zeros(n)
    v = C.c_double()
    for k in range(n):
        assert R.sk_spectrum_magnitude_db(band, k, C.byref(v)) == 0
        db[k] = v.value
    f0, df = R.sk_spectrum_f_start(band), R.sk_spectrum_f_step(band)
    for h in (band, sp):
        R.sk_spectrum_free(h)
    R.sk_trace_free(t)
    return re + 1j * im, db, f0, df


CSV_CASES = {
    # name: file body (bytes) — read through sk_trace_read_csv (signals.cpp:125-170)
    "crlf_blank_ws": b"\r\n  0.0 ,\t1.5\r\n\r\n1e-13, -2.25 \r\n 2e-13,3\r\n   \r\n3e-13,4.5e-3\r\n",
    "header_notrail": b"time_s,amplitude\n0,1\n0.5,2\n1.0,3\n1.5,4",
    "jitter_ok": b"0,1\n1.0000001,2\n2,3\n3.0000002,4\n4,5\n",
    "malformed": b"t,x\n0,1\n1,2\n\n1.5;2\n2,3\n",
    "three_cols": b"t,x\n0,1,2\n",
    "bad_number": b"0,1\n1,2x\n",
    "nonuniform": b"0,1\n1,2\n2,3\n3.5,4\n4.5,5\n",
    "decreasing": b"3,1\n2,2\n1,3\n",
    "one_sample": b"time_s,amplitude\n0,1\n",
    "header_only": b"time_s,amplitude\n",
    "empty": b"",
    "nan_sample": b"0,1\n1,nan\n2,3\n",
    "plus_sign": b"0,+1\n1,2\n",
    "two_headers": b"a,b\nc,d\n0,1\n",
}


def ref_trace_read_csv(path):
    R.sk_trace_read_csv.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    R.sk_trace_size.restype = C.c_size_t
    R.sk_trace_size.argtypes = [C.c_void_p]
    R.sk_trace_sample_rate.restype = C.c_double
    R.sk_trace_sample_rate.argtypes = [C.c_void_p]
    R.sk_trace_t0.restype = C.c_double
    R.sk_trace_t0.argtypes = [C.c_void_p]
    R.sk_trace_samples.restype = C.POINTER(C.c_double)
    R.sk_trace_samples.argtypes = [C.c_void_p]
    t = C.c_void_p()
    rc = R.sk_trace_read_csv(path.encode(), C.byref(t))
    if rc != 0:
        return rc, R.sk_last_error().decode(), None, 0.0, 0.0
    n = R.sk_trace_size(t)
    x = np.array([R.sk_trace_samples(t)[i] for i in range(n)])
    fs, t0 = R.sk_trace_sample_rate(t), R.sk_trace_t0(t)
    R.sk_trace_free(t)
    return 0, "", x, fs, t0


SPEC_CSV_CASES = {
    "three_fields": b"frequency_hz,re,im,magnitude_db\n0,1,2,3\n1,1,2\n",
    "five_fields": b"0,1,2,3\n1,1,2,3,4\n",
    "nonuniform": b"0,1,0,0\n1,1,0,0\n2.5,1,0,0\n3.5,1,0,0\n",
    "decreasing": b"2,1,0,0\n1,1,0,0\n",
    "single": b"frequency_hz,re,im,magnitude_db\n5e12,1.5,-2,4\n",
    "header_only": b"frequency_hz,re,im,magnitude_db\n",
    "crlf_ws": b"\r\n 0 , 1 ,\t2, 0\r\n1e9,3,4,0\r\n\r\n2e9,5,6,0",
    "jitter": b"0,1,0,0\n1.0000000001,2,0,0\n2,3,0,0\n",
}


def ref_spectrum_read_csv(path):
    R.sk_spectrum_read_csv.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    R.sk_spectrum_source_n.restype = C.c_size_t
    R.sk_spectrum_source_n.argtypes = [C.c_void_p]
    h = C.c_void_p()
    rc = R.sk_spectrum_read_csv(path.encode(), C.byref(h))
    if rc != 0:
        return rc, R.sk_last_error().decode(), None, 0.0, 0.0, 0
    n = R.sk_spectrum_size(h)
    re, im = np.zeros(n), np.zeros(n)
    R.sk_spectrum_copy_data(h, P(re), P(im))
    out = (0, "", re + 1j * im, R.sk_spectrum_f_start(h), R.sk_spectrum_f_step(h), R.sk_spectrum_source_n(h))
    R.sk_spectrum_free(h)
    return out


def ref_write_csv(kind, path, data, a, b):
    """sk_trace_write_csv (kind 'trace': data samples, a fs, b t0) or sk_spectrum_write_csv
    (kind 'spectrum': data complex bins, a f_start, b f_step); returns the file bytes"""
    if kind == "trace":
        s = np.ascontiguousarray(data, np.float64)
        h = C.c_void_p()
        assert R.sk_trace_create(P(s), s.size, a, b, C.byref(h)) == 0
        R.sk_trace_write_csv.argtypes = [C.c_void_p, C.c_char_p]
        assert R.sk_trace_write_csv(h, path.encode()) == 0
        R.sk_trace_free(h)
    else:
        re, im = np.ascontiguousarray(data.real), np.ascontiguousarray(data.imag)
        h = C.c_void_p()
        R.sk_spectrum_create.argtypes = [oracle.dp, oracle.dp, C.c_size_t, C.c_double, C.c_double,
                                         C.POINTER(C.c_void_p)]
        assert R.sk_spectrum_create(P(re), P(im), re.size, a, b, C.byref(h)) == 0
        R.sk_spectrum_write_csv.argtypes = [C.c_void_p, C.c_char_p]
        assert R.sk_spectrum_write_csv(h, path.encode()) == 0
        R.sk_spectrum_free(h)
    with open(path, "rb") as f:
        return f.read()


SCAN_CASES = W.SCAN_CASES


def ref_scan(**kw):
    import paper_2108_03948_b200 as sk
    R.sk_scan_config_defaults.argtypes = [C.POINTER(sk.SkScanConfig)]
    R.sk_resolvability_scan.argtypes = [C.POINTER(sk.SkScanConfig), C.POINTER(C.c_void_p)]
    R.sk_resolvability_curve_size.restype = C.c_size_t
    R.sk_resolvability_curve_size.argtypes = [C.c_void_p]
    R.sk_resolvability_curve_point.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_double),
                                               C.POINTER(sk.SkDipMetric), C.POINTER(sk.SkDipMetric)]
    R.sk_resolvability_min_fft.restype = R.sk_resolvability_min_czt.restype = C.c_double
    R.sk_resolvability_min_fft.argtypes = R.sk_resolvability_min_czt.argtypes = [C.c_void_p]
    R.sk_resolvability_curve_free.argtypes = [C.c_void_p]
    c = sk.SkScanConfig()
    R.sk_scan_config_defaults(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    h = C.c_void_p()
    assert R.sk_resolvability_scan(C.byref(c), C.byref(h)) == 0, R.sk_last_error()
    out = sk.read_curve(R, h)
    R.sk_resolvability_curve_free(h)
    return out


def ref_zoom(samples, fs, f1, f2, taps=None, n_fft=None, **kw):
    o = dict(center_hz=0.0, center_set=0, decimation=0, cutoff_hz=0.0, num_taps=0, circular=1,
             trim_transient=0, pad_pow2=1)
    o.update(kw)
    x = np.ascontiguousarray(np.atleast_2d(samples), np.float64)
    n = x.shape[1]
    p = R.skr_zoom_plan_create(n, f1, f2, fs, o["center_hz"], o["center_set"], o["decimation"],
                               o["cutoff_hz"], o["num_taps"], o["circular"], o["trim_transient"],
                               o["pad_pow2"])
    assert p
    if taps is not None:
        t = np.ascontiguousarray(taps, np.float64)
        R.skr_zoom_plan_set_taps(p, P(t), t.size)
    if n_fft is not None:
        assert R.skr_zoom_plan_set_n_fft(p, n_fft) == 0
    nb, f0, df = C.c_size_t(), C.c_double(), C.c_double()
    R.skr_zoom_batch(p, P(x), n, fs, 0, 1, None, C.byref(nb), C.byref(f0), C.byref(df))
    out = np.zeros((x.shape[0], nb.value), np.complex128)
    R.skr_zoom_batch(p, P(x), n, fs, x.shape[0], 1, P(out.view(np.float64)), C.byref(nb), C.byref(f0),
                     C.byref(df))
    R.skr_zoom_plan_free(p)
    return out, f0.value, df.value


def main():
    rng = np.random.default_rng(101)
    # --- FFT: random complex inputs, every power of two 1..4096 plus the reference KAT ------
    fft = {}
    for lg in range(0, 13):
        n = 1 << lg
        x = rng.uniform(-1, 1, (2, n)) + 1j * rng.uniform(-1, 1, (2, n))
        fft[f"x{n}"] = x
        fft[f"X{n}"] = np.stack([ref_fft(r) for r in x])
        fft[f"i{n}"] = np.stack([ref_fft(r, inverse=True) for r in x])
    fft["kat_x"] = np.array([1, 2, 3, 4], np.complex128)
    fft["kat_X"] = ref_fft(fft["kat_x"])
    x = rng.uniform(-1, 1, 12) + 1j * rng.uniform(-1, 1, 12)
    fft["naive_x"], fft["naive_X"] = x, ref_dft_naive(x)
    np.savez_compressed(os.path.join(OUT, "fft.npz"), **fft)

    # --- CZT: cfg2-shape trace, random band configs, off-circle spiral, full circle ----------
    czt = {}
    a, w = W.cfg2_czt_params(2048)
    x = W.cfg2_batch(2, 1024)[[0, 2]]   # one reference and one sample trace
    czt["cfg2_x"], czt["cfg2_a"], czt["cfg2_w"] = x, a, w
    czt["cfg2_X"] = np.stack([ref_czt(r, a, w, 2048) for r in x])
    cases = []
    crng = np.random.default_rng(303)
    for i in range(24):
        n = int(crng.integers(2, 700))
        m = int(crng.integers(2, 700))
        f1 = crng.uniform(0, 3500)
        f2 = crng.uniform(f1 + 10, 4000)
        ab, wb = oracle.czt_params_for_band(f1, f2, 8000.0, m)
        xx = crng.uniform(-1, 1, n) + 1j * crng.uniform(-1, 1, n)
        czt[f"r{i}_x"], czt[f"r{i}_X"] = xx, ref_czt(xx, ab, wb, m)
        cases.append((n, m, ab.real, ab.imag, wb.real, wb.imag))
    czt["rand_params"] = np.array(cases)
    sa, sw = 1.05 * np.exp(0.3j), 0.995 * np.exp(-0.11j)
    xx = np.random.default_rng(5).uniform(-1, 1, 20) + 1j * np.random.default_rng(6).uniform(-1, 1, 20)
    czt["spiral_x"], czt["spiral_a"], czt["spiral_w"] = xx, sa, sw
    czt["spiral_X"] = ref_czt(xx, sa, sw, 24)
    np.savez_compressed(os.path.join(OUT, "czt.npz"), **czt)

    # --- spectra: cfg1 pair at 4096, the 500-sample pulse (pow2 pad and exact 500) ----------
    sp = {}
    ref, sample = W.cfg1_pair()
    sp["cfg1_ref"], sp["cfg1_sample"] = ref, sample
    sp["cfg1_Xr"], f0, df = ref_fft_spectrum(ref, W.FS, 4096)
    sp["cfg1_Xs"], _, _ = ref_fft_spectrum(sample, W.FS, 4096)
    sp["cfg1_df"] = df
    pulse = W.thz_pulse(500, fs=10e12)
    sp["pulse500"] = pulse
    sp["pulse500_X512"], _, _ = ref_fft_spectrum(pulse, 10e12, 0)
    sp["pulse500_X500"], _, _ = ref_fft_spectrum(pulse, 10e12, 500)
    np.savez_compressed(os.path.join(OUT, "spectra.npz"), **sp)

    # --- band slice + dB column: cfg1 sample at 4096, the 500-sample pulse ------
    bd = {}
    bands = {"thz": (0.1e12, 3.0e12), "half": (0.0, W.FS / 2), "nyq": (9.0e12, 12.0e12), "edge": (
        sp["cfg1_df"] * 100, sp["cfg1_df"] * 140), "top": (19.9e12, 25e12)}
    bd["x"] = sample
    for name, (lo, hi) in bands.items():
        bd[f"{name}_band"] = np.array([lo, hi])
        bd[f"{name}_X"], bd[f"{name}_db"], bd[f"{name}_f0"], bd[f"{name}_df"] = ref_band(sample, W.FS, 4096, lo, hi)
    bd["p500_X"], bd["p500_db"], bd["p500_f0"], bd["p500_df"] = ref_band(pulse, 10e12, 500, 0.5e12, 2.0e12)
    bd["zeros_X"], bd["zeros_db"], _, _ = ref_band(np.zeros(64), W.FS, 64, 0.0, 5e12)
    np.savez_compressed(os.path.join(OUT, "band.npz"), **bd)

    # --- CSV ingest / writers: reference parse results and file bytes --------
    import tempfile
    cv = {}
    with tempfile.TemporaryDirectory() as td:
        for name, body in CSV_CASES.items():
            path = os.path.join(td, name + ".csv")
            with open(path, "wb") as f:
                f.write(body)
            rc, msg, x, fs, t0 = ref_trace_read_csv(path)
            cv[f"in_{name}"] = np.frombuffer(body, np.uint8)
            cv[f"rc_{name}"] = rc
            cv[f"msg_{name}"] = msg.replace(path, "<PATH>")
            if rc == 0:
                cv[f"x_{name}"], cv[f"fs_{name}"], cv[f"t0_{name}"] = x, fs, t0
        rc, msg, _, _, _ = ref_trace_read_csv(os.path.join(td, "missing.csv"))
        cv["rc_missing"], cv["msg_missing"] = rc, msg.replace(td, "<DIR>")
        tr = sample[:300]
        cv["w_trace_x"] = tr
        cv["w_trace"] = np.frombuffer(ref_write_csv("trace", os.path.join(td, "t.csv"), tr, W.FS, 1.25e-12), np.uint8)
        cv["w_spec_X"], cv["w_spec_f0"], cv["w_spec_df"] = bd["thz_X"], bd["thz_f0"], bd["thz_df"]
        cv["w_spec"] = np.frombuffer(ref_write_csv("spectrum", os.path.join(td, "s.csv"), bd["thz_X"], bd["thz_f0"],
                                                   bd["thz_df"]), np.uint8)
        odd = np.array([0.0, -0.0 + 1e-300j, 1e-16, -1.0 - 0.0j, 3.14159e200 + 1e-320j, 2.5e-8 - 7e8j, 0.1 + 0.2j])
        cv["w_odd_X"] = odd
        cv["w_odd"] = np.frombuffer(ref_write_csv("spectrum", os.path.join(td, "o.csv"), odd, -5.0, 1.0 / 3.0),
                                    np.uint8)
        for name, body in dict(SPEC_CSV_CASES, written=bytes(cv["w_spec"])).items():
            path = os.path.join(td, "sp_" + name + ".csv")
            with open(path, "wb") as f:
                f.write(body)
            rc, msg, X, f0, df, sn = ref_spectrum_read_csv(path)
            cv[f"sin_{name}"] = np.frombuffer(body, np.uint8)
            cv[f"src_{name}"], cv[f"smsg_{name}"] = rc, msg.replace(path, "<PATH>")
            if rc == 0:
                cv[f"sX_{name}"], cv[f"sf0_{name}"], cv[f"sdf_{name}"], cv[f"sn_{name}"] = X, f0, df, sn
        # spectrum JSON (spectra.cpp:161-183): the band spectrum, the odd values, and random bit patterns
        R.sk_spectrum_write_json.argtypes = [C.c_void_p, C.c_char_p]

        def ref_json(bins, f0, df):
            re, im = np.ascontiguousarray(np.real(bins)), np.ascontiguousarray(np.imag(bins))
            h = C.c_void_p()
            assert R.sk_spectrum_create(P(re), P(im), re.size, f0, df, C.byref(h)) == 0
            path = os.path.join(td, "s.json")
            assert R.sk_spectrum_write_json(h, path.encode()) == 0
            R.sk_spectrum_free(h)
            with open(path, "rb") as f:
                return np.frombuffer(f.read(), np.uint8)
        cv["j_spec"] = ref_json(bd["thz_X"], float(bd["thz_f0"]), float(bd["thz_df"]))
        cv["j_odd"] = ref_json(odd, -5.0, 1.0 / 3.0)
        rj = np.random.default_rng(11)
        bits = rj.integers(0, 2**63, 3000, dtype=np.uint64) | (rj.integers(0, 2, 3000, dtype=np.uint64) << np.uint64(63))
        rv = bits.view(np.float64)
        rv = rv[np.isfinite(rv)]
        rv = rv[: rv.size // 2 * 2]
        cv["j_rand_X"] = rv[0::2] + 1j * rv[1::2]
        cv["j_rand"] = ref_json(cv["j_rand_X"], 0.0, 4882812500.0)
        rt_path = os.path.join(td, "t.csv")   # the written trace read back by the reference
        rc, _, x, fs, t0 = ref_trace_read_csv(rt_path)
        cv["rt_x"], cv["rt_fs"], cv["rt_t0"] = x, fs, t0
    np.savez_compressed(os.path.join(OUT, "csv.npz"), **cv)

    # --- resolvability sweep: the reference's own curves -------------------------
    rs = {}
    for name, kw in SCAN_CASES.items():
        rs[f"{name}_sep"], rs[f"{name}_fft"], rs[f"{name}_czt"], rs[f"{name}_minfft"], rs[f"{name}_minczt"] = \
            ref_scan(**kw)
    # the reference's curve JSON / CSV files for the default sweep (layout pins for the writers)
    import paper_2108_03948_b200 as sk
    R.sk_resolvability_write_json.argtypes = [C.c_void_p, C.c_char_p]
    R.sk_resolvability_write_csv.argtypes = [C.c_void_p, C.c_char_p]
    c = sk.SkScanConfig()
    R.sk_scan_config_defaults(C.byref(c))
    h = C.c_void_p()
    assert R.sk_resolvability_scan(C.byref(c), C.byref(h)) == 0
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        for ext, fn in (("json", R.sk_resolvability_write_json), ("csv", R.sk_resolvability_write_csv)):
            path = os.path.join(td, "curve." + ext)
            assert fn(h, path.encode()) == 0
            with open(path, "rb") as f:
                rs[f"default_{ext}"] = np.frombuffer(f.read(), np.uint8)
    R.sk_resolvability_curve_free(h)
    # dip_metric on a reference spectrum (fft of a two-tone record), incl. the insufficient-resolution case
    np.savez_compressed(os.path.join(OUT, "scan.npz"), **rs)

    # --- zoom: cfg3 reference sizing (65 taps, n_fft 512), the 2048 variant, 500-sample plans ----
    zm = {}
    x3 = W.cfg3_batch(3, 4096)
    zm["cfg3_x"] = x3
    zm["cfg3_Z512"], zm["cfg3_f0_512"], zm["cfg3_df_512"] = ref_zoom(x3, W.FS, 0.4e12, 1.2e12, decimation=8,
                                                                      num_taps=65)
    zm["cfg3_Z2048"], zm["cfg3_f0_2048"], zm["cfg3_df_2048"] = ref_zoom(x3, W.FS, 0.4e12, 1.2e12, decimation=8,
                                                                        num_taps=65, n_fft=2048)
    p500 = W.thz_pulse(500, fs=10e12)
    zm["p500"] = p500
    zm["p500_default"], zm["p500_default_f0"], _ = ref_zoom(p500, 10e12, 0.5e12, 2.0e12)
    zm["p500_lin_trim"], zm["p500_lin_trim_f0"], _ = ref_zoom(p500, 10e12, 0.5e12, 2.0e12, decimation=4,
                                                              circular=0, trim_transient=1)
    zm["p500_d2"], _, _ = ref_zoom(p500, 10e12, 0.5e12, 2.0e12, decimation=2)
    np.savez_compressed(os.path.join(OUT, "zoom.npz"), **zm)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
