"""paper_2108_03948_b200 — B200-native batched FFT / CZT / Zoom FFT for THz-TDS traces.

The product is the C-ABI shared library ``lib/libspectralkit_b200.so`` (CUDA C++ for sm_100a,
sources in ``csrc/``). This module is the Python mirror of the reference's transform API
(/root/reference/proj/include/spectralkit.h and src/*.hpp) over that C ABI:

* single-trace, host-memory calls with the reference's names and semantics
  (``fft``, ``ifft``, ``czt``, ``fft_spectrum``, ``czt_spectrum``, ``ZoomPlan`` ...), each one a
  host->device->host round trip through the ``sk_*`` entry points;
* batched, device-resident calls on torch CUDA tensors (``fft_batch``, ``fft_spectrum_batch``,
  ``CztPlanGPU``, ``TransferPlanGPU``, ``ZoomPlanGPU``) through the ``skg_*`` extension, enqueued on
  the current torch stream.

Errors raise :class:`SkError` carrying the ``sk_status`` code and ``sk_last_error()`` text
(the reference maps C++ exceptions to the same codes, capi.cpp:48-78). There is no CPU fallback:
if the shared library is missing or no GPU is present the calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SKG_LIB_PATH") or os.path.join(HERE, "lib", "libspectralkit_b200.so")

SK_OK, SK_ERR_INVALID_ARGUMENT, SK_ERR_INTERNAL = 0, 1, 6
SKG_F64, SKG_F32 = 0, 1
SKG_FULL, SKG_HALF = 0, 1

_lib = None
dp = C.POINTER(C.c_double)
sz = C.c_size_t
vp = C.c_void_p


class SkError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[{status}] {message}")
        self.status = status
        self.message = message


class SkDipMetric(C.Structure):
    """sk_dip_metric (spectralkit.h two-tone analysis; analysis.hpp:15-24)."""
    _fields_ = [("resolved", C.c_int), ("dip_db", C.c_double), ("f_peak_a_hz", C.c_double),
                ("peak_a_db", C.c_double), ("f_peak_b_hz", C.c_double), ("peak_b_db", C.c_double),
                ("f_valley_hz", C.c_double), ("valley_db", C.c_double)]

    def astuple(self):
        return tuple(float(getattr(self, f)) for f, _ in self._fields_)


class SkScanConfig(C.Structure):
    """sk_scan_config (analysis.hpp:31-41)."""
    _fields_ = [("sample_rate_hz", C.c_double), ("n", C.c_size_t), ("f1_hz", C.c_double), ("f2_hz", C.c_double),
                ("m", C.c_size_t), ("center_hz", C.c_double), ("sep_start_hz", C.c_double),
                ("sep_stop_hz", C.c_double), ("sep_step_hz", C.c_double)]


class SkZoomOptions(C.Structure):
    """sk_zoom_options (spectralkit.h:170-179 layout)."""
    _fields_ = [("center_hz", C.c_double), ("center_set", C.c_int), ("decimation", sz),
                ("cutoff_hz", C.c_double), ("num_taps", sz), ("circular", C.c_int),
                ("trim_transient", C.c_int), ("pad_pow2", C.c_int)]


class SkgZoomExt(C.Structure):
    _fields_ = [("n_fft", sz), ("taps", dp), ("num_taps", sz)]


def _declare(L):
    st = C.c_int
    sig = {
        "sk_status_name": (C.c_char_p, [st]),
        "sk_last_error": (C.c_char_p, []),
        "sk_version": (C.c_char_p, []),
        "sk_fft": (st, [dp, dp, sz]),
        "sk_ifft": (st, [dp, dp, sz]),
        "sk_dft_naive": (st, [dp, dp, sz, dp, dp]),
        "sk_czt": (st, [dp, dp, sz, C.c_double, C.c_double, C.c_double, C.c_double, sz, dp, dp]),
        "sk_czt_direct": (st, [dp, dp, sz, C.c_double, C.c_double, C.c_double, C.c_double, sz, dp, dp]),
        "sk_czt_params_for_band": (st, [C.c_double, C.c_double, C.c_double, sz, dp, dp, dp, dp]),
        "sk_next_pow2": (sz, [sz]),
        "sk_trace_create": (st, [dp, sz, C.c_double, C.c_double, C.POINTER(vp)]),
        "sk_trace_free": (None, [vp]),
        "sk_trace_size": (sz, [vp]),
        "sk_trace_sample_rate": (C.c_double, [vp]),
        "sk_trace_t0": (C.c_double, [vp]),
        "sk_trace_samples": (dp, [vp]),
        "sk_fft_spectrum": (st, [vp, sz, C.POINTER(vp)]),
        "sk_czt_spectrum": (st, [vp, C.c_double, C.c_double, sz, C.POINTER(vp)]),
        "sk_spectrum_create": (st, [dp, dp, sz, C.c_double, C.c_double, C.POINTER(vp)]),
        "sk_spectrum_free": (None, [vp]),
        "sk_spectrum_size": (sz, [vp]),
        "sk_spectrum_f_start": (C.c_double, [vp]),
        "sk_spectrum_f_step": (C.c_double, [vp]),
        "sk_spectrum_frequency": (C.c_double, [vp, sz]),
        "sk_spectrum_source_n": (sz, [vp]),
        "sk_spectrum_bin": (st, [vp, sz, dp, dp]),
        "sk_spectrum_magnitude_db": (st, [vp, sz, dp]),
        "sk_spectrum_copy_data": (st, [vp, dp, dp]),
        "sk_spectrum_slice_band": (st, [vp, C.c_double, C.c_double, C.POINTER(vp)]),
        "sk_zoom_options_defaults": (None, [C.POINTER(SkZoomOptions)]),
        "sk_zoom_plan_create": (st, [sz, C.c_double, C.c_double, C.c_double, C.POINTER(SkZoomOptions),
                                     C.POINTER(vp)]),
        "sk_zoom_plan_free": (None, [vp]),
        "sk_zoom_plan_decimation": (sz, [vp]),
        "sk_zoom_plan_n_fft": (sz, [vp]),
        "sk_zoom_plan_filter_len": (sz, [vp]),
        "sk_zoom_plan_f_step": (C.c_double, [vp]),
        "sk_zoom_spectrum": (st, [vp, vp, C.POINTER(vp)]),
        "skg_device_info": (st, [C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(sz), C.POINTER(sz)]),
        "skg_launch_count": (C.c_uint64, []),
        "skg_debug_set_grid_cap": (None, [C.c_uint]),
        "skg_synchronize": (st, [vp]),
        "skg_fft_batch": (st, [sz, C.c_int, C.c_int, vp, sz, vp, sz, sz, vp]),
        "skg_fft_spectrum_batch": (st, [sz, sz, C.c_int, C.c_int, vp, sz, sz, vp, sz, vp]),
        "skg_band_bins": (st, [sz, C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(sz), C.POINTER(sz), dp]),
        "skg_fft_spectrum_band_batch": (st, [sz, sz, C.c_int, sz, sz, vp, sz, sz, vp, sz, vp, sz, vp]),
        "skg_band_db_batch": (st, [C.c_int, vp, sz, sz, sz, sz, vp, sz, vp, sz, vp]),
        "sk_trace_read_csv": (st, [C.c_char_p, C.POINTER(vp)]),
        "sk_trace_write_csv": (st, [vp, C.c_char_p]),
        "sk_spectrum_write_csv": (st, [vp, C.c_char_p]),
        "skg_traces_read_csv": (st, [C.POINTER(C.c_char_p), sz, sz, C.c_int, vp, sz, dp, dp, C.c_int, vp]),
        "skg_spectra_write_csv": (st, [C.POINTER(C.c_char_p), sz, C.c_int, vp, sz, sz, dp, C.c_double, C.c_int,
                                       vp]),
        "sk_spectrum_read_csv": (st, [C.c_char_p, C.POINTER(vp)]),
        "sk_spectrum_write_json": (st, [vp, C.c_char_p]),
        "sk_resolvability_write_csv": (st, [vp, C.c_char_p]),
        "sk_resolvability_write_json": (st, [vp, C.c_char_p]),
        "sk_fft_resolution": (st, [C.c_double, sz, dp]),
        "sk_record_len_for_step": (st, [C.c_double, C.c_double, C.POINTER(sz)]),
        "sk_zeros_for_resolution": (st, [C.c_double, sz, C.c_double, C.POINTER(sz)]),
        "sk_czt_len_for_matched_resolution": (st, [C.c_double, C.c_double, C.c_double, sz, C.POINTER(sz)]),
        "sk_dip_metric_compute": (st, [vp, C.c_double, C.c_double, C.POINTER(SkDipMetric)]),
        "sk_scan_config_defaults": (None, [C.POINTER(SkScanConfig)]),
        "sk_resolvability_scan": (st, [C.POINTER(SkScanConfig), C.POINTER(vp)]),
        "sk_resolvability_curve_free": (None, [vp]),
        "sk_resolvability_curve_size": (sz, [vp]),
        "sk_resolvability_curve_point": (st, [vp, sz, dp, C.POINTER(SkDipMetric), C.POINTER(SkDipMetric)]),
        "sk_resolvability_min_fft": (C.c_double, [vp]),
        "sk_resolvability_min_czt": (C.c_double, [vp]),
        "skg_resolvability_fft_len": (sz, [vp]),
        "skg_czt_plan_create": (st, [sz, C.c_double, C.c_double, C.c_double, C.c_double, sz, C.c_int,
                                     C.POINTER(vp)]),
        "skg_czt_plan_free": (None, [vp]),
        "skg_czt_plan_conv_size": (sz, [vp]),
        "skg_czt_execute": (st, [vp, vp, C.c_int, sz, sz, vp, sz, vp]),
        "skg_transfer_plan_create": (st, [dp, sz, sz, C.c_int, C.POINTER(vp)]),
        "skg_transfer_plan_free": (None, [vp]),
        "skg_transfer_plan_bins": (sz, [vp]),
        "skg_transfer_plan_reference": (st, [vp, dp]),
        "skg_transfer_execute": (st, [vp, vp, sz, sz, vp, vp, sz, vp, sz, vp]),
        "skg_zoom_plan_create": (st, [sz, C.c_double, C.c_double, C.c_double, C.POINTER(SkZoomOptions),
                                      C.POINTER(SkgZoomExt), C.c_int, C.POINTER(vp)]),
        "skg_zoom_plan_free": (None, [vp]),
        "skg_zoom_plan_info": (st, [vp, C.POINTER(sz), dp, dp, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz)]),
        "skg_zoom_execute": (st, [vp, vp, sz, sz, vp, sz, vp]),
        "skg_czt_execute_host": (st, [vp, vp, C.c_int, sz, sz, vp, sz, sz]),
        "skg_fft_spectrum_host": (st, [sz, sz, C.c_int, C.c_int, vp, sz, sz, vp, sz, sz]),
        "skg_zoom_execute_host": (st, [vp, vp, sz, sz, vp, sz, sz]),
        "skg_transfer_execute_host": (st, [vp, vp, sz, sz, vp, vp, sz, sz]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


def lib():
    """Load the CUDA shared library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C csrc)")
        _lib = _declare(C.CDLL(LIB_PATH))
    return _lib


def exported_symbols():
    """Names declared SK_API in include/*.h (used by the export test)."""
    import re
    names = []
    inc = os.path.join(os.path.dirname(HERE), "include")
    for fn in sorted(os.listdir(inc)):
        if fn.endswith(".h"):
            src = open(os.path.join(inc, fn)).read()
            names += re.findall(r"SK_API\s+[\w\s\*]+?\b(sk\w+)\s*\(", src)
    return names


def _chk(status):
    if status != SK_OK:
        raise SkError(status, lib().sk_last_error().decode())


def _p(a):
    return a.ctypes.data_as(dp)


def last_error() -> str:
    return lib().sk_last_error().decode()


def launch_count() -> int:
    return int(lib().skg_launch_count())


class grid_cap:
    """Context manager over the skg_debug_set_grid_cap test hook: persistent grids capped at
    `cap` CTAs, so every CTA loops over many units (later waves, prefetch, slot reuse)."""

    def __init__(self, cap):
        self.cap = int(cap)

    def __enter__(self):
        lib().skg_debug_set_grid_cap(self.cap)
        return self

    def __exit__(self, *exc):
        lib().skg_debug_set_grid_cap(0)
        return False


def device_info():
    d, s = C.c_int(), C.c_int()
    smem, l2 = sz(), sz()
    _chk(lib().skg_device_info(C.byref(d), C.byref(s), C.byref(smem), C.byref(l2)))
    return {"device": d.value, "sm_count": s.value, "smem_optin": smem.value, "l2_bytes": l2.value}


# ---- single-trace host API (reference C ABI semantics) ---------------------------------------

def _split(x):
    x = np.asarray(x, dtype=np.complex128)
    return np.ascontiguousarray(x.real), np.ascontiguousarray(x.imag)


def fft(x):
    """sk_fft: forward, unnormalised, n power of two (numerics.cpp:102-120)."""
    re, im = _split(x)
    _chk(lib().sk_fft(_p(re), _p(im), re.size))
    return re + 1j * im


def ifft(x):
    re, im = _split(x)
    _chk(lib().sk_ifft(_p(re), _p(im), re.size))
    return re + 1j * im


def dft_naive(x):
    re, im = _split(x)
    orr, oi = np.empty_like(re), np.empty_like(im)
    _chk(lib().sk_dft_naive(_p(re), _p(im), re.size, _p(orr), _p(oi)))
    return orr + 1j * oi


def czt(x, a, w, m):
    """sk_czt: X[k] = sum_n x[n] a^-n w^(kn), k < m (Bluestein on the GPU)."""
    re, im = _split(x)
    orr, oi = np.empty(m), np.empty(m)
    a, w = complex(a), complex(w)
    _chk(lib().sk_czt(_p(re), _p(im), re.size, a.real, a.imag, w.real, w.imag, m, _p(orr), _p(oi)))
    return orr + 1j * oi


def czt_direct(x, a, w, m):
    re, im = _split(x)
    orr, oi = np.empty(m), np.empty(m)
    a, w = complex(a), complex(w)
    _chk(lib().sk_czt_direct(_p(re), _p(im), re.size, a.real, a.imag, w.real, w.imag, m, _p(orr), _p(oi)))
    return orr + 1j * oi


def czt_params_for_band(f1, f2, fs, m):
    v = [C.c_double() for _ in range(4)]
    _chk(lib().sk_czt_params_for_band(f1, f2, fs, m, *[C.byref(t) for t in v]))
    return complex(v[0].value, v[1].value), complex(v[2].value, v[3].value)


def next_pow2(n: int) -> int:
    return int(lib().sk_next_pow2(n))


@dataclass
class Spectrum:
    bins: np.ndarray
    f_start_hz: float
    f_step_hz: float
    source_n: int

    def frequency(self, k):
        return self.f_start_hz + k * self.f_step_hz


def _release(fn, h):
    """free a native handle; quiet at interpreter teardown (module globals may already be gone)"""
    try:
        getattr(lib(), fn)(h)
    except Exception:
        pass


class Trace:
    """Owning wrapper of sk_trace (samples, fs, t0)."""

    def __init__(self, samples, sample_rate_hz, t0_s=0.0):
        s = np.ascontiguousarray(samples, dtype=np.float64)
        h = vp()
        _chk(lib().sk_trace_create(_p(s), s.size, sample_rate_hz, t0_s, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def __len__(self):
        return int(lib().sk_trace_size(self._h))

    @property
    def sample_rate_hz(self):
        return float(lib().sk_trace_sample_rate(self._h))

    def __del__(self, _rel=_release):
        if getattr(self, "_h", None):
            _rel("sk_trace_free", self._h)
            self._h = None


def trace_read_csv(path):
    """sk_trace_read_csv (signals.cpp:125-170): (samples, sample_rate_hz, t0_s)."""
    h = vp()
    _chk(lib().sk_trace_read_csv(os.fsencode(path), C.byref(h)))
    L = lib()
    try:
        n = int(L.sk_trace_size(h))
        x = np.ctypeslib.as_array(L.sk_trace_samples(h), shape=(n,)).copy() if n else np.empty(0)
        return x, float(L.sk_trace_sample_rate(h)), float(L.sk_trace_t0(h))
    finally:
        L.sk_trace_free(h)


def trace_write_csv(samples, sample_rate_hz, t0_s, path):
    """sk_trace_write_csv (signals.cpp:178-189)."""
    t = Trace(samples, sample_rate_hz, t0_s)
    _chk(lib().sk_trace_write_csv(t.handle, os.fsencode(path)))


def spectrum_write_csv(bins, f_start_hz, f_step_hz, path):
    """sk_spectrum_write_csv (spectra.cpp:63-78): reference-format CSV of a spectrum."""
    b = np.ascontiguousarray(bins, np.complex128)
    re, im = np.ascontiguousarray(b.real), np.ascontiguousarray(b.imag)
    h = vp()
    _chk(lib().sk_spectrum_create(_p(re), _p(im), b.size, f_start_hz, f_step_hz, C.byref(h)))
    try:
        _chk(lib().sk_spectrum_write_csv(h, os.fsencode(path)))
    finally:
        lib().sk_spectrum_free(h)


def spectrum_write_json(bins, f_start_hz, f_step_hz, path):
    """sk_spectrum_write_json (spectra.cpp:161-183): the reference's JSON, byte for byte."""
    b = np.ascontiguousarray(bins, np.complex128)
    re, im = np.ascontiguousarray(b.real), np.ascontiguousarray(b.imag)
    h = vp()
    _chk(lib().sk_spectrum_create(_p(re), _p(im), b.size, f_start_hz, f_step_hz, C.byref(h)))
    try:
        _chk(lib().sk_spectrum_write_json(h, os.fsencode(path)))
    finally:
        lib().sk_spectrum_free(h)


def _paths(paths):
    arr = (C.c_char_p * len(paths))(*[os.fsencode(p) for p in paths])
    return arr


def traces_read_csv(paths, n, dtype=None, device="cuda", threads=0):
    """Batched ingest (skg_traces_read_csv): every file parsed like sk_trace_read_csv, in parallel,
    into one (len(paths), n) device tensor. Returns (traces, fs[], t0[])."""
    torch = _torch()
    dtype = dtype or torch.float64
    out = torch.empty((len(paths), n), dtype=dtype, device=device)
    fs, t0 = np.zeros(len(paths)), np.zeros(len(paths))
    prec = SKG_F64 if dtype == torch.float64 else SKG_F32
    _chk(lib().skg_traces_read_csv(_paths(paths), len(paths), n, prec, vp(out.data_ptr()), n, _p(fs), _p(t0),
                                   threads, _stream()))
    return out, fs, t0


def spectra_write_csv(paths, bins, f_start_hz, f_step_hz, threads=0):
    """Batched writer (skg_spectra_write_csv): one reference-format CSV per row of a complex device
    tensor; f_start_hz scalar or per row."""
    bins, b, s = _rows(bins)
    f0 = np.ascontiguousarray(np.broadcast_to(np.asarray(f_start_hz, np.float64), (b,)))
    _chk(lib().skg_spectra_write_csv(_paths(paths), b, _prec(bins), vp(bins.data_ptr()), s, bins.shape[-1], _p(f0),
                                     f_step_hz, threads, _stream()))


def scan_config(**kw) -> SkScanConfig:
    c = SkScanConfig()
    lib().sk_scan_config_defaults(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def read_curve(L, h, fft_len_fn=None):
    """(separations, fft metrics S x 8, czt metrics S x 8, min_fft, min_czt) of a curve handle through
    the sk_resolvability_* accessors of library L (ours or the reference's: same ABI)."""
    S = int(L.sk_resolvability_curve_size(h))
    sep, fm, cm = np.zeros(S), np.zeros((S, 8)), np.zeros((S, 8))
    a, b, v = SkDipMetric(), SkDipMetric(), C.c_double()
    for i in range(S):
        _chk(L.sk_resolvability_curve_point(h, i, C.byref(v), C.byref(a), C.byref(b)))
        sep[i], fm[i], cm[i] = v.value, a.astuple(), b.astuple()
    return sep, fm, cm, float(L.sk_resolvability_min_fft(h)), float(L.sk_resolvability_min_czt(h))


def spectrum_read_csv(path) -> "Spectrum":
    """sk_spectrum_read_csv (spectra.cpp:94-156)."""
    h = vp()
    _chk(lib().sk_spectrum_read_csv(os.fsencode(path), C.byref(h)))
    return _take_spectrum(h)


def fft_resolution(fs, n):
    v = C.c_double()
    _chk(lib().sk_fft_resolution(fs, n, C.byref(v)))
    return v.value


def record_len_for_step(fs, step):
    v = sz()
    _chk(lib().sk_record_len_for_step(fs, step, C.byref(v)))
    return v.value


def zeros_for_resolution(fs, n, step):
    v = sz()
    _chk(lib().sk_zeros_for_resolution(fs, n, step, C.byref(v)))
    return v.value


def czt_len_for_matched_resolution(f1, f2, fs, n_fft):
    v = sz()
    _chk(lib().sk_czt_len_for_matched_resolution(f1, f2, fs, n_fft, C.byref(v)))
    return v.value


def resolvability_scan(csv_path=None, json_path=None, **cfg):
    """sk_resolvability_scan (analysis.cpp:99-195) on the GPU: dict with separations_hz, fft / czt
    metric rows (resolved, dip_db, f_peak_a, peak_a_db, f_peak_b, peak_b_db, f_valley, valley_db),
    min_resolved_fft_hz / _czt_hz (NaN when none) and fft_len; csv_path: also write the curve
    (sk_resolvability_write_csv)."""
    c = scan_config(**cfg)
    h = vp()
    _chk(lib().sk_resolvability_scan(C.byref(c), C.byref(h)))
    try:
        if csv_path is not None:
            _chk(lib().sk_resolvability_write_csv(h, os.fsencode(csv_path)))
        if json_path is not None:
            _chk(lib().sk_resolvability_write_json(h, os.fsencode(json_path)))
        sep, fm, cm, mf, mc = read_curve(lib(), h)
        return {"separations_hz": sep, "fft": fm, "czt": cm, "min_resolved_fft_hz": mf, "min_resolved_czt_hz": mc,
                "fft_len": int(lib().skg_resolvability_fft_len(h))}
    finally:
        lib().sk_resolvability_curve_free(h)


def dip_metric(bins, f_start_hz, f_step_hz, f_a_hz, f_b_hz):
    """sk_dip_metric_compute (analysis.cpp:30-97) on a host spectrum."""
    b = np.ascontiguousarray(bins, np.complex128)
    re, im = np.ascontiguousarray(b.real), np.ascontiguousarray(b.imag)
    h = vp()
    _chk(lib().sk_spectrum_create(_p(re), _p(im), b.size, f_start_hz, f_step_hz, C.byref(h)))
    try:
        m = SkDipMetric()
        _chk(lib().sk_dip_metric_compute(h, f_a_hz, f_b_hz, C.byref(m)))
        return m.astuple()
    finally:
        lib().sk_spectrum_free(h)


def _take_spectrum(h) -> Spectrum:
    L = lib()
    n = int(L.sk_spectrum_size(h))
    re, im = np.empty(n), np.empty(n)
    _chk(L.sk_spectrum_copy_data(h, _p(re), _p(im)))
    s = Spectrum(re + 1j * im, float(L.sk_spectrum_f_start(h)), float(L.sk_spectrum_f_step(h)),
                 int(L.sk_spectrum_source_n(h)))
    L.sk_spectrum_free(h)
    return s


def fft_spectrum(samples, sample_rate_hz, transform_len=0) -> Spectrum:
    """sk_fft_spectrum: full [0, fs) spectrum of a real trace (spectra.cpp:21-38)."""
    t = Trace(samples, sample_rate_hz)
    h = vp()
    _chk(lib().sk_fft_spectrum(t.handle, transform_len, C.byref(h)))
    return _take_spectrum(h)


def czt_spectrum(samples, sample_rate_hz, f1, f2, m) -> Spectrum:
    t = Trace(samples, sample_rate_hz)
    h = vp()
    _chk(lib().sk_czt_spectrum(t.handle, f1, f2, m, C.byref(h)))
    return _take_spectrum(h)


def slice_band(spec: Spectrum, f_lo, f_hi) -> Spectrum:
    re, im = _split(spec.bins)
    h = vp()
    _chk(lib().sk_spectrum_create(_p(re), _p(im), re.size, spec.f_start_hz, spec.f_step_hz, C.byref(h)))
    out = vp()
    st = lib().sk_spectrum_slice_band(h, f_lo, f_hi, C.byref(out))
    lib().sk_spectrum_free(h)
    _chk(st)
    s = _take_spectrum(out)
    s.source_n = spec.source_n
    return s


def zoom_options(**kw) -> SkZoomOptions:
    o = SkZoomOptions()
    lib().sk_zoom_options_defaults(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
        if k == "center_hz":
            o.center_set = 1
    return o


class ZoomPlan:
    """sk_zoom_plan (make_zoom_plan, zoomfft.cpp:106-181)."""

    def __init__(self, input_len, f1, f2, fs, **opts):
        o = zoom_options(**opts)
        h = vp()
        _chk(lib().sk_zoom_plan_create(input_len, f1, f2, fs, C.byref(o), C.byref(h)))
        self._h = h
        self.fs = fs

    @property
    def decimation(self):
        return int(lib().sk_zoom_plan_decimation(self._h))

    @property
    def n_fft(self):
        return int(lib().sk_zoom_plan_n_fft(self._h))

    @property
    def filter_len(self):
        return int(lib().sk_zoom_plan_filter_len(self._h))

    @property
    def f_step_hz(self):
        return float(lib().sk_zoom_plan_f_step(self._h))

    def spectrum(self, samples, fs=None) -> Spectrum:
        t = Trace(samples, self.fs if fs is None else fs)
        h = vp()
        _chk(lib().sk_zoom_spectrum(self._h, t.handle, C.byref(h)))
        return _take_spectrum(h)

    def __del__(self, _rel=_release):
        if getattr(self, "_h", None):
            _rel("sk_zoom_plan_free", self._h)
            self._h = None


# ---- batched device API (torch CUDA tensors) -------------------------------------------------

def _torch():
    import torch
    return torch


def _stream():
    torch = _torch()
    return vp(torch.cuda.current_stream().cuda_stream)


def _prec(t):
    torch = _torch()
    if t.dtype in (torch.float64, torch.complex128):
        return SKG_F64
    if t.dtype in (torch.float32, torch.complex64):
        return SKG_F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _cdtype(prec):
    torch = _torch()
    return torch.complex128 if prec == SKG_F64 else torch.complex64


def _rows(x):
    """(batch, row stride) of a 1-D or 2-D tensor with unit inner stride."""
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if x.dim() != 2 or x.stride(-1) != 1:
        raise ValueError(f"expected 1-D or 2-D rows with unit inner stride, got shape {tuple(x.shape)} "
                         f"stride {tuple(x.stride())}")
    return x, x.shape[0], x.stride(0)


def _check_in(x, n, precision, what, complex_ok=False):
    """Input rows for a plan: CUDA, the plan's precision, n samples per row (the C side reads
    n * row-stride elements: a wrong dtype or row length would read past the buffer)."""
    if not x.is_cuda:
        raise ValueError(f"{what}: input must be a CUDA tensor")
    if x.is_complex() and not complex_ok:
        raise TypeError(f"{what}: input must be real, got {x.dtype}")
    if _prec(x) != precision:
        raise TypeError(f"{what}: input dtype {x.dtype} does not match the plan precision "
                        f"({'fp64' if precision == SKG_F64 else 'fp32'})")
    if x.shape[-1] != n:
        raise ValueError(f"{what}: rows hold {x.shape[-1]} samples, the plan expects {n}")


def _check_out(out, rows, cols, dtype, device, what):
    """Caller-supplied output rows: right dtype, device, >= rows x cols, unit inner stride."""
    if out.dtype != dtype:
        raise TypeError(f"{what}: output dtype {out.dtype}, expected {dtype}")
    if out.device != device:
        raise ValueError(f"{what}: output on {out.device}, input on {device}")
    o = out.unsqueeze(0) if out.dim() == 1 else out
    if o.dim() != 2 or o.shape[0] < rows or o.shape[1] < cols or o.stride(-1) != 1:
        raise ValueError(f"{what}: output must be ({rows}, >= {cols}) rows with unit inner stride, "
                         f"got shape {tuple(out.shape)} stride {tuple(out.stride())}")
    return o


def fft_batch(x, inverse=False, out=None):
    """Complex FFT of each row of a complex CUDA tensor (skg_fft_batch)."""
    x, b, s = _rows(x)
    prec = _prec(x)
    if not x.is_complex():
        raise TypeError(f"fft_batch: complex rows expected, got {x.dtype}")
    out = torch_empty_like_rows(x) if out is None else out
    o = _check_out(out, b, x.shape[-1], x.dtype, x.device, "fft_batch")
    _chk(lib().skg_fft_batch(x.shape[-1], int(inverse), prec, vp(x.data_ptr()), s, vp(o.data_ptr()),
                             o.stride(0), b, _stream()))
    return out


def torch_empty_like_rows(x):
    torch = _torch()
    return torch.empty(x.shape, dtype=x.dtype, device=x.device)


def fft_spectrum_batch(x, transform_len=0, layout=SKG_FULL, out=None):
    """Zero-padded spectra of real trace rows (skg_fft_spectrum_batch)."""
    torch = _torch()
    x, b, s = _rows(x)
    prec = _prec(x)
    n = x.shape[-1]
    L = transform_len or next_pow2(n)
    nb = L if layout == SKG_FULL else L // 2 + 1
    if x.is_complex():
        raise TypeError(f"fft_spectrum_batch: real trace rows expected, got {x.dtype}")
    if out is None:
        out = torch.empty((b, nb), dtype=_cdtype(prec), device=x.device)
    o = _check_out(out, b, nb, _cdtype(prec), x.device, "fft_spectrum_batch")
    _chk(lib().skg_fft_spectrum_batch(n, L, prec, layout, vp(x.data_ptr()), s, b, vp(o.data_ptr()),
                                      o.stride(0), _stream()))
    return out


def _np_cdtype(prec):
    return np.complex128 if prec == SKG_F64 else np.complex64


def _host_rows(x, n, precision, what, complex_ok=False):
    """(array, batch, row stride in elements, data pointer, is_complex) of host rows: a numpy array
    or a CPU torch tensor (pinned or pageable) of the plan precision, unit inner stride."""
    if hasattr(x, "is_cuda"):
        if x.is_cuda:
            raise ValueError(f"{what}: host rows expected, got a CUDA tensor (use execute)")
        t = x.unsqueeze(0) if x.dim() == 1 else x
        if t.dim() != 2 or t.stride(-1) != 1:
            raise ValueError(f"{what}: 1-D or 2-D rows with unit inner stride expected")
        if t.is_complex() and not complex_ok:
            raise TypeError(f"{what}: real rows expected")
        if _prec(t) != precision:
            raise TypeError(f"{what}: dtype {t.dtype} does not match the plan precision")
        if t.shape[-1] != n:
            raise ValueError(f"{what}: rows hold {t.shape[-1]} samples, the plan expects {n}")
        return t, t.shape[0], t.stride(0), vp(t.data_ptr()), t.is_complex()
    a = np.asarray(x)
    a = a[None] if a.ndim == 1 else a
    if a.ndim != 2 or a.strides[-1] != a.itemsize:
        raise ValueError(f"{what}: 1-D or 2-D rows with unit inner stride expected")
    is_c = np.iscomplexobj(a)
    if is_c and not complex_ok:
        raise TypeError(f"{what}: real rows expected")
    want = {SKG_F64: (np.float64, np.complex128), SKG_F32: (np.float32, np.complex64)}[precision]
    if a.dtype not in want:
        raise TypeError(f"{what}: dtype {a.dtype} does not match the plan precision")
    if a.shape[-1] != n:
        raise ValueError(f"{what}: rows hold {a.shape[-1]} samples, the plan expects {n}")
    return a, a.shape[0], a.strides[0] // a.itemsize, vp(a.ctypes.data), is_c


def _host_out(out, rows, cols, dtype, what):
    if out is None:
        return np.empty((rows, cols), dtype)
    if hasattr(out, "is_cuda"):
        import torch
        td = {np.complex128: torch.complex128, np.complex64: torch.complex64, np.float64: torch.float64,
              np.float32: torch.float32}[np.dtype(dtype).type]
        if out.is_cuda or out.dtype != td:
            raise TypeError(f"{what}: host output of dtype {td} expected")
        o = out.unsqueeze(0) if out.dim() == 1 else out
        if o.dim() != 2 or o.shape[0] < rows or o.shape[1] < cols or o.stride(-1) != 1:
            raise ValueError(f"{what}: output must be ({rows}, >= {cols}) rows with unit inner stride")
        return out
    o = out[None] if out.ndim == 1 else out
    if out.dtype != dtype or o.ndim != 2 or o.shape[0] < rows or o.shape[1] < cols or o.strides[-1] != o.itemsize:
        raise ValueError(f"{what}: output must be ({rows}, >= {cols}) {np.dtype(dtype)} rows with unit inner stride")
    return out


def _host_ptr(a):
    return vp(a.data_ptr()) if hasattr(a, "data_ptr") else vp(a.ctypes.data)


def _host_stride(a):
    if hasattr(a, "is_cuda"):
        return a.stride(0) if a.dim() == 2 else a.shape[-1]
    return a.strides[0] // a.itemsize if a.ndim == 2 else a.shape[-1]


def fft_spectrum_host(x, transform_len=0, layout=SKG_FULL, precision=None, out=None, chunk=0):
    """Zero-padded spectra of host trace rows through the library pipeline (skg_fft_spectrum_host)."""
    a = x if hasattr(x, "is_cuda") else np.asarray(x)
    dt = a.dtype
    prec = precision if precision is not None else (SKG_F32 if str(dt) in ("float32", "torch.float32") else SKG_F64)
    n = a.shape[-1]
    x2, b, s, ptr, _ = _host_rows(a, n, prec, "fft_spectrum_host")
    L = transform_len or next_pow2(n)
    nb = L if layout == SKG_FULL else L // 2 + 1
    out = _host_out(out, b, nb, _np_cdtype(prec), "fft_spectrum_host")
    _chk(lib().skg_fft_spectrum_host(n, L, prec, layout, ptr, s, b, _host_ptr(out), _host_stride(out), chunk))
    return out


def band_bins(spectrum_size, f_start_hz, f_step_hz, f_lo_hz, f_hi_hz):
    """(k_lo, count, band f_start) of slice_band on a spectrum of spectrum_size bins (skg_band_bins,
    spectra.cpp:40-61)."""
    k, c, f = sz(), sz(), C.c_double()
    _chk(lib().skg_band_bins(spectrum_size, f_start_hz, f_step_hz, f_lo_hz, f_hi_hz, C.byref(k), C.byref(c),
                             C.byref(f)))
    return k.value, c.value, f.value


def fft_spectrum_band_batch(x, sample_rate_hz, f_lo_hz, f_hi_hz, transform_len=0, bins=True, db=True):
    """Band-sliced zero-padded spectra of real trace rows with the magnitude_db column, fused into the
    FFT store (skg_fft_spectrum_band_batch). Returns (bins or None, db or None, f_start_hz, f_step_hz)."""
    torch = _torch()
    x, b, s = _rows(x)
    prec = _prec(x)
    n = x.shape[-1]
    L = transform_len or next_pow2(n)
    step = sample_rate_hz / L
    k_lo, cnt, f0 = band_bins(L, 0.0, step, f_lo_hz, f_hi_hz)
    ob = torch.empty((b, cnt), dtype=_cdtype(prec), device=x.device) if bins else None
    od = torch.empty((b, cnt), dtype=x.dtype, device=x.device) if db else None
    _chk(lib().skg_fft_spectrum_band_batch(n, L, prec, k_lo, cnt, vp(x.data_ptr()), s, b,
                                           vp(ob.data_ptr()) if ob is not None else None, cnt,
                                           vp(od.data_ptr()) if od is not None else None, cnt, _stream()))
    return ob, od, f0, step


def band_db_batch(spectra, k_lo, count, bins=True, db=True):
    """Band slice [k_lo, k_lo + count) and magnitude_db of complex rows on the device
    (skg_band_db_batch)."""
    torch = _torch()
    spectra, b, s = _rows(spectra)
    prec = _prec(spectra)
    real = torch.float64 if prec == SKG_F64 else torch.float32
    ob = torch.empty((b, count), dtype=spectra.dtype, device=spectra.device) if bins else None
    od = torch.empty((b, count), dtype=real, device=spectra.device) if db else None
    _chk(lib().skg_band_db_batch(prec, vp(spectra.data_ptr()), s, k_lo, count, b,
                                 vp(ob.data_ptr()) if ob is not None else None, count,
                                 vp(od.data_ptr()) if od is not None else None, count, _stream()))
    return ob, od


class CztPlanGPU:
    """Batched Bluestein CZT plan (CztPlan, czt.cpp:85-137) on device tables."""

    def __init__(self, n, a, w, m, precision=SKG_F64):
        a, w = complex(a), complex(w)
        h = vp()
        _chk(lib().skg_czt_plan_create(n, a.real, a.imag, w.real, w.imag, m, precision, C.byref(h)))
        self._h, self.n, self.m, self.precision = h, n, m, precision

    @property
    def conv_size(self):
        return int(lib().skg_czt_plan_conv_size(self._h))

    def execute(self, x, out=None):
        torch = _torch()
        x, b, s = _rows(x)
        _check_in(x, self.n, self.precision, "CztPlanGPU.execute", complex_ok=True)
        is_c = x.is_complex()
        if out is None:
            out = torch.empty((b, self.m), dtype=_cdtype(self.precision), device=x.device)
        o = _check_out(out, b, self.m, _cdtype(self.precision), x.device, "CztPlanGPU.execute")
        _chk(lib().skg_czt_execute(self._h, vp(x.data_ptr()), int(is_c), s, b, vp(o.data_ptr()),
                                   o.stride(0), _stream()))
        return out

    def execute_host(self, x, out=None, chunk=0):
        """Host rows in, host rows out through the library's chunked pipeline (skg_czt_execute_host).
        x: numpy array or CPU tensor (pinned or pageable) of the plan's precision."""
        x2, b, s, ptr, is_c = _host_rows(x, self.n, self.precision, "CztPlanGPU.execute_host", complex_ok=True)
        out = _host_out(out, b, self.m, _np_cdtype(self.precision), "CztPlanGPU.execute_host")
        _chk(lib().skg_czt_execute_host(self._h, ptr, int(is_c), s, b, _host_ptr(out), _host_stride(out), chunk))
        return out

    def __del__(self, _rel=_release):
        if getattr(self, "_h", None):
            _rel("skg_czt_plan_free", self._h)
            self._h = None


class TransferPlanGPU:
    """H(f) = X_sample / X_ref fused into the FFT store epilogue (skg_transfer_*)."""

    def __init__(self, ref_samples, transform_len=0, precision=SKG_F64):
        r = np.ascontiguousarray(ref_samples, dtype=np.float64)
        h = vp()
        _chk(lib().skg_transfer_plan_create(_p(r), r.size, transform_len, precision, C.byref(h)))
        self._h, self.n, self.precision = h, r.size, precision
        self.bins = int(lib().skg_transfer_plan_bins(h))

    def reference_spectrum(self):
        out = np.empty(self.bins, np.complex128)
        _chk(lib().skg_transfer_plan_reference(self._h, _p(out.view(np.float64))))
        return out

    def execute(self, x, mag=None, phase=None, h=None):
        torch = _torch()
        x, b, s = _rows(x)
        _check_in(x, self.n, self.precision, "TransferPlanGPU.execute")
        rd = torch.float64 if self.precision == SKG_F64 else torch.float32
        if mag is None:
            mag = torch.empty((b, self.bins), dtype=rd, device=x.device)
        if phase is None:
            phase = torch.empty((b, self.bins), dtype=rd, device=x.device)
        m2 = _check_out(mag, b, self.bins, rd, x.device, "TransferPlanGPU.execute (|H|)")
        p2 = _check_out(phase, b, self.bins, rd, x.device, "TransferPlanGPU.execute (arg H)")
        if m2.stride(0) != p2.stride(0):
            raise ValueError("TransferPlanGPU.execute: |H| and arg H rows must share one stride")
        h2 = None if h is None else _check_out(h, b, self.bins, _cdtype(self.precision), x.device,
                                               "TransferPlanGPU.execute (H)")
        _chk(lib().skg_transfer_execute(self._h, vp(x.data_ptr()), s, b, vp(m2.data_ptr()),
                                        vp(p2.data_ptr()), m2.stride(0),
                                        vp(h2.data_ptr()) if h2 is not None else None,
                                        h2.stride(0) if h2 is not None else 0, _stream()))
        return mag, phase

    def execute_host(self, x, mag=None, phase=None, chunk=0):
        x2, b, s, ptr, _ = _host_rows(x, self.n, self.precision, "TransferPlanGPU.execute_host")
        rd = np.float64 if self.precision == SKG_F64 else np.float32
        mag = _host_out(mag, b, self.bins, rd, "TransferPlanGPU.execute_host")
        phase = _host_out(phase, b, self.bins, rd, "TransferPlanGPU.execute_host")
        if _host_stride(mag) != _host_stride(phase):
            raise ValueError("TransferPlanGPU.execute_host: |H| and arg H rows must share one stride")
        _chk(lib().skg_transfer_execute_host(self._h, ptr, s, b, _host_ptr(mag), _host_ptr(phase), _host_stride(mag),
                                             chunk))
        return mag, phase

    def __del__(self, _rel=_release):
        if getattr(self, "_h", None):
            _rel("skg_transfer_plan_free", self._h)
            self._h = None


class ZoomPlanGPU:
    """Batched fused Zoom FFT plan (make_zoom_plan + zoom_fft) with optional n_fft / taps overrides."""

    def __init__(self, input_len, f1, f2, fs, precision=SKG_F64, n_fft=0, taps=None, **opts):
        o = zoom_options(**opts)
        ext = SkgZoomExt()
        ext.n_fft = n_fft
        self._taps = None
        if taps is not None:
            self._taps = np.ascontiguousarray(taps, dtype=np.float64)
            ext.taps = _p(self._taps)
            ext.num_taps = self._taps.size
        h = vp()
        _chk(lib().skg_zoom_plan_create(input_len, f1, f2, fs, C.byref(o), C.byref(ext), precision, C.byref(h)))
        self._h, self.precision, self.input_len = h, precision, input_len
        nb, nf, d, nt = sz(), sz(), sz(), sz()
        f0, df = C.c_double(), C.c_double()
        _chk(lib().skg_zoom_plan_info(h, C.byref(nb), C.byref(f0), C.byref(df), C.byref(nf), C.byref(d),
                                      C.byref(nt)))
        self.bins, self.f_start_hz, self.f_step_hz = nb.value, f0.value, df.value
        self.n_fft, self.decimation, self.num_taps = nf.value, d.value, nt.value

    def execute(self, x, out=None):
        torch = _torch()
        x, b, s = _rows(x)
        _check_in(x, self.input_len, self.precision, "ZoomPlanGPU.execute")
        if out is None:
            out = torch.empty((b, self.bins), dtype=_cdtype(self.precision), device=x.device)
        o = _check_out(out, b, self.bins, _cdtype(self.precision), x.device, "ZoomPlanGPU.execute")
        _chk(lib().skg_zoom_execute(self._h, vp(x.data_ptr()), s, b, vp(o.data_ptr()), o.stride(0),
                                    _stream()))
        return out

    def execute_host(self, x, out=None, chunk=0):
        x2, b, s, ptr, _ = _host_rows(x, self.input_len, self.precision, "ZoomPlanGPU.execute_host")
        out = _host_out(out, b, self.bins, _np_cdtype(self.precision), "ZoomPlanGPU.execute_host")
        _chk(lib().skg_zoom_execute_host(self._h, ptr, s, b, _host_ptr(out), _host_stride(out), chunk))
        return out

    def __del__(self, _rel=_release):
        if getattr(self, "_h", None):
            _rel("skg_zoom_plan_free", self._h)
            self._h = None
