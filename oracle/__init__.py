"""oracle — TEST INFRASTRUCTURE (the parity checker, never the product).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package. It wraps two CPU libraries with ctypes:

* ``libskoracle.so`` — our plain-C restatement of the reference transform path
  (oracle/skoracle.c; every function cites /root/reference/proj/src file:line).
* ``_ref/libskref.so`` — the UNMODIFIED reference sources compiled by oracle/Makefile
  (``make -C oracle ref``) plus a plan-reuse shim (oracle/ref_shim.cpp). Present wherever it
  was built in the build container (it travels to the GPU box as an untracked build artefact);
  ``ref()`` returns None when it is absent.

Complex arrays are numpy complex128 (interleaved re/im, the std::complex<double> layout).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_PORT_PATH = os.path.join(HERE, "libskoracle.so")
_REF_PATH = os.path.join(HERE, "_ref", "libskref.so")

_port = None
_ref = None
_ref_tried = False

dp = C.POINTER(C.c_double)
sz = C.c_size_t


def _p(a):
    return a.ctypes.data_as(dp)


def build_port() -> str:
    """Compile the C restatement (gcc only; works on the GPU box too)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    return _PORT_PATH


class SkZoomOptions(C.Structure):
    _fields_ = [("center_hz", C.c_double), ("center_set", C.c_int), ("decimation", sz),
                ("cutoff_hz", C.c_double), ("num_taps", sz), ("circular", C.c_int),
                ("trim_transient", C.c_int), ("pad_pow2", C.c_int)]


def port():
    global _port
    if _port is None:
        if not os.path.exists(_PORT_PATH):
            build_port()
        L = C.CDLL(_PORT_PATH)
        L.sko_last_error.restype = C.c_char_p
        L.sko_next_pow2.restype = sz
        L.sko_next_pow2.argtypes = [sz]
        L.sko_fft_plan_create.restype = C.c_void_p
        L.sko_fft_plan_create.argtypes = [sz]
        L.sko_fft_plan_free.argtypes = [C.c_void_p]
        L.sko_fft_plan_run.argtypes = [C.c_void_p, dp, sz, C.c_int]
        L.sko_fft.argtypes = [dp, sz, C.c_int, dp]
        L.sko_dft_naive.argtypes = [dp, sz, dp]
        L.sko_czt_params_for_band.argtypes = [C.c_double, C.c_double, C.c_double, sz, dp, dp]
        L.sko_czt_plan_create.restype = C.c_void_p
        L.sko_czt_plan_create.argtypes = [dp, dp, sz]
        L.sko_czt_plan_create.argtypes = [sz, dp, dp, sz]
        L.sko_czt_plan_free.argtypes = [C.c_void_p]
        L.sko_czt_plan_conv_size.restype = sz
        L.sko_czt_plan_conv_size.argtypes = [C.c_void_p]
        L.sko_czt_execute.argtypes = [C.c_void_p, dp, dp, dp]
        L.sko_czt.argtypes = [dp, sz, dp, dp, sz, dp]
        L.sko_czt_direct.argtypes = [dp, sz, dp, dp, sz, dp]
        L.sko_dft_any.argtypes = [dp, sz, dp]
        L.sko_fft_spectrum.argtypes = [dp, sz, C.c_double, sz, C.POINTER(sz), dp]
        L.sko_slice_band.argtypes = [sz, C.c_double, C.c_double, C.c_double, C.c_double,
                                     C.POINTER(sz), C.POINTER(sz)]
        L.sko_magnitude_db.argtypes = [dp, sz, dp]
        L.sko_design_lowpass.argtypes = [C.c_double, C.c_double, sz, dp]
        L.sko_zoom_options_defaults.argtypes = [C.POINTER(SkZoomOptions)]
        L.sko_zoom_plan_create.restype = C.c_void_p
        L.sko_zoom_plan_create.argtypes = [sz, C.c_double, C.c_double, C.c_double,
                                           C.POINTER(SkZoomOptions)]
        L.sko_zoom_plan_free.argtypes = [C.c_void_p]
        L.sko_zoom_plan_info.argtypes = [C.c_void_p, C.POINTER(sz), dp]
        L.sko_zoom_plan_set_taps.argtypes = [C.c_void_p, dp, sz]
        L.sko_zoom_plan_set_n_fft.argtypes = [C.c_void_p, sz]
        L.sko_zoom_fft.argtypes = [C.c_void_p, dp, sz, C.c_double, C.POINTER(sz), dp, dp, dp]
        L.sko_transfer.argtypes = [dp, dp, sz, dp, dp, dp]
        L.sko_bench_czt.restype = C.c_double
        L.sko_bench_czt.argtypes = [C.c_void_p, dp, sz, sz, C.c_int, dp]
        L.sko_bench_fft_spectrum.restype = C.c_double
        L.sko_bench_fft_spectrum.argtypes = [sz, dp, sz, sz, C.c_int, dp]
        L.sko_bench_zoom.restype = C.c_double
        L.sko_bench_zoom.argtypes = [C.c_void_p, dp, sz, C.c_double, sz, C.c_int]
        L.sko_batch_zoom.restype = C.c_double
        L.sko_batch_zoom.argtypes = [C.c_void_p, dp, sz, C.c_double, sz, C.c_int, dp]
        _port = L
    return _port


def ref():
    """The reference itself (compiled from its sources), or None when not built here."""
    global _ref, _ref_tried
    if not _ref_tried:
        _ref_tried = True
        if os.path.exists(_REF_PATH):
            L = C.CDLL(_REF_PATH)
            L.sk_last_error.restype = C.c_char_p
            L.sk_fft.argtypes = [dp, dp, sz]
            L.sk_ifft.argtypes = [dp, dp, sz]
            L.sk_dft_naive.argtypes = [dp, dp, sz, dp, dp]
            L.sk_czt.argtypes = [dp, dp, sz, C.c_double, C.c_double, C.c_double, C.c_double,
                                 sz, dp, dp]
            L.sk_czt_direct.argtypes = L.sk_czt.argtypes
            L.sk_trace_create.argtypes = [dp, sz, C.c_double, C.c_double, C.POINTER(C.c_void_p)]
            L.sk_trace_free.argtypes = [C.c_void_p]
            L.sk_fft_spectrum.argtypes = [C.c_void_p, sz, C.POINTER(C.c_void_p)]
            L.sk_spectrum_size.restype = sz
            L.sk_spectrum_size.argtypes = [C.c_void_p]
            L.sk_spectrum_f_start.restype = C.c_double
            L.sk_spectrum_f_start.argtypes = [C.c_void_p]
            L.sk_spectrum_f_step.restype = C.c_double
            L.sk_spectrum_f_step.argtypes = [C.c_void_p]
            L.sk_spectrum_copy_data.argtypes = [C.c_void_p, dp, dp]
            L.sk_spectrum_free.argtypes = [C.c_void_p]
            L.skr_czt_plan_create.restype = C.c_void_p
            L.skr_czt_plan_create.argtypes = [sz, C.c_double, C.c_double, C.c_double, C.c_double, sz]
            L.skr_czt_plan_free.argtypes = [C.c_void_p]
            L.skr_czt_batch.restype = C.c_double
            L.skr_czt_batch.argtypes = [C.c_void_p, dp, sz, sz, C.c_int, dp]
            L.skr_fft_batch.restype = C.c_double
            L.skr_fft_batch.argtypes = [sz, dp, sz, sz, C.c_int, dp]
            L.skr_zoom_plan_create.restype = C.c_void_p
            L.skr_zoom_plan_create.argtypes = [sz, C.c_double, C.c_double, C.c_double, C.c_double,
                                               C.c_int, sz, C.c_double, sz, C.c_int, C.c_int, C.c_int]
            L.skr_zoom_plan_free.argtypes = [C.c_void_p]
            L.skr_zoom_plan_set_n_fft.argtypes = [C.c_void_p, sz]
            L.skr_zoom_plan_set_taps.argtypes = [C.c_void_p, dp, sz]
            L.skr_bench_environment.restype = C.c_char_p
            L.skr_transfer_batch.restype = C.c_double
            L.skr_transfer_batch.argtypes = [sz, dp, dp, sz, sz, C.c_int, dp, dp]
            L.skr_zoom_batch.restype = C.c_double
            L.skr_zoom_batch.argtypes = [C.c_void_p, dp, sz, C.c_double, sz, C.c_int, dp,
                                         C.POINTER(sz), dp, dp]
            _ref = L
    return _ref


def ref_csv_chain(in_path, out_path, transform_len, f_lo, f_hi):
    """The reference's own file-to-file chain for one trace (the CLI `transform` path,
    spectral_kit.cpp:109-186): sk_trace_read_csv -> sk_fft_spectrum -> sk_spectrum_slice_band ->
    sk_spectrum_write_csv. Test / cpu_baseline infrastructure only."""
    R = ref()
    if not getattr(R, "_csv_sigs", False):
        R.sk_trace_read_csv.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        R.sk_spectrum_slice_band.argtypes = [C.c_void_p, C.c_double, C.c_double, C.POINTER(C.c_void_p)]
        R.sk_spectrum_write_csv.argtypes = [C.c_void_p, C.c_char_p]
        R._csv_sigs = True
    t, s, b = C.c_void_p(), C.c_void_p(), C.c_void_p()
    rc = R.sk_trace_read_csv(os.fsencode(in_path), C.byref(t))
    rc = rc or R.sk_fft_spectrum(t, transform_len, C.byref(s))
    rc = rc or R.sk_spectrum_slice_band(s, f_lo, f_hi, C.byref(b))
    rc = rc or R.sk_spectrum_write_csv(b, os.fsencode(out_path))
    for h, fr in ((b, R.sk_spectrum_free), (s, R.sk_spectrum_free), (t, R.sk_trace_free)):
        if h.value:
            fr(h)
    if rc:
        raise OracleError(R.sk_last_error().decode())


class OracleError(ValueError):
    pass


def _chk(rc):
    if rc != 0:
        raise OracleError(port().sko_last_error().decode())


def c128(x):
    return np.ascontiguousarray(x, dtype=np.complex128)


def f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


# ---- restatement (port) entry points ---------------------------------------------------

def next_pow2(n: int) -> int:
    return int(port().sko_next_pow2(n))


def cis_cycles(q: float, t: float) -> complex:
    out = np.zeros(2)
    port().sko_cis_cycles(C.c_double(q), C.c_double(t), _p(out))
    return complex(out[0], out[1])


def fft(x, inverse=False):
    x = c128(x)
    out = np.empty_like(x)
    _chk(port().sko_fft(_p(x.view(np.float64)), x.size, int(inverse), _p(out.view(np.float64))))
    return out


def ifft(x):
    return fft(x, inverse=True)


def fft_plan_forward(x):
    """FftPlan(n).forward on a copy (numerics.cpp:73-100)."""
    x = c128(x).copy()
    p = port().sko_fft_plan_create(x.size)
    if not p:
        raise OracleError(port().sko_last_error().decode())
    port().sko_fft_plan_run(p, _p(x.view(np.float64)), x.size, 0)
    port().sko_fft_plan_free(p)
    return x


def dft_naive(x):
    x = c128(x)
    out = np.empty_like(x)
    _chk(port().sko_dft_naive(_p(x.view(np.float64)), x.size, _p(out.view(np.float64))))
    return out


def czt_params_for_band(f1, f2, fs, m):
    a = np.zeros(2)
    w = np.zeros(2)
    _chk(port().sko_czt_params_for_band(f1, f2, fs, m, _p(a), _p(w)))
    return complex(a[0], a[1]), complex(w[0], w[1])


def czt(x, a, w, m):
    x = c128(x)
    out = np.empty(m, np.complex128)
    av = np.array([a.real, a.imag])
    wv = np.array([w.real, w.imag])
    _chk(port().sko_czt(_p(x.view(np.float64)), x.size, _p(av), _p(wv), m, _p(out.view(np.float64))))
    return out


def czt_direct(x, a, w, m):
    x = c128(x)
    out = np.empty(m, np.complex128)
    av = np.array([a.real, a.imag])
    wv = np.array([w.real, w.imag])
    _chk(port().sko_czt_direct(_p(x.view(np.float64)), x.size, _p(av), _p(wv), m,
                               _p(out.view(np.float64))))
    return out


class CztPlan:
    """Plan-reuse CZT (czt.cpp:85-137) over real or complex traces, batch helper for tests."""

    def __init__(self, n, a, w, m):
        self.n, self.m = n, m
        av = np.array([complex(a).real, complex(a).imag])
        wv = np.array([complex(w).real, complex(w).imag])
        self._h = port().sko_czt_plan_create(n, _p(av), _p(wv), m)
        if not self._h:
            raise OracleError(port().sko_last_error().decode())
        self.L = int(port().sko_czt_plan_conv_size(self._h))

    def execute(self, x):
        x = c128(x)
        out = np.empty(self.m, np.complex128)
        port().sko_czt_execute(self._h, _p(x.view(np.float64)), None, _p(out.view(np.float64)))
        return out

    def batch_real(self, x_real, threads=1):
        x_real = f64(x_real)
        count = x_real.shape[0]
        out = np.empty((count, self.m), np.complex128)
        port().sko_bench_czt(self._h, _p(x_real), self.n, count, threads, _p(out.view(np.float64)))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            port().sko_czt_plan_free(self._h)
            self._h = None


def dft_any(x):
    x = c128(x)
    out = np.empty_like(x)
    _chk(port().sko_dft_any(_p(x.view(np.float64)), x.size, _p(out.view(np.float64))))
    return out


def fft_spectrum(samples, fs, transform_len=0):
    """Returns (bins, f_start, f_step, source_n) like spectra.cpp:21-38."""
    s = f64(samples)
    ln = sz(0)
    _chk(port().sko_fft_spectrum(_p(s), s.size, fs, transform_len, C.byref(ln), None))
    out = np.empty(ln.value, np.complex128)
    _chk(port().sko_fft_spectrum(_p(s), s.size, fs, transform_len, C.byref(ln),
                                 _p(out.view(np.float64))))
    return out, 0.0, fs / ln.value, ln.value


def fft_spectrum_batch(x_real, L, threads=1):
    """fft_spectrum of each row (bench helper: power-of-two L; other lengths go through the
    per-trace fft_spectrum, i.e. dft_any's chirp route)."""
    x_real = f64(x_real)
    count, n = x_real.shape
    if L & (L - 1):
        return np.stack([fft_spectrum(r, 1.0, L)[0] for r in x_real])
    out = np.empty((count, L), np.complex128)
    port().sko_bench_fft_spectrum(L, _p(x_real), n, count, threads, _p(out.view(np.float64)))
    return out


def slice_band(n_bins, f_start, f_step, lo, hi):
    a, c = sz(0), sz(0)
    _chk(port().sko_slice_band(n_bins, f_start, f_step, lo, hi, C.byref(a), C.byref(c)))
    return a.value, c.value


def magnitude_db(bins):
    """types.cpp:13-18 per bin."""
    v = c128(bins)
    out = np.empty(v.size)
    port().sko_magnitude_db(_p(v.view(np.float64)), v.size, _p(out))
    return out


def design_lowpass(cutoff, fs, taps):
    out = np.empty(max(taps, 1))
    _chk(port().sko_design_lowpass(cutoff, fs, taps, _p(out)))
    return out


def zoom_options(**kw) -> SkZoomOptions:
    o = SkZoomOptions()
    port().sko_zoom_options_defaults(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
        if k == "center_hz":
            o.center_set = 1
    return o


class ZoomPlan:
    """make_zoom_plan + zoom_fft restated (zoomfft.cpp:106-239)."""

    def __init__(self, n, f1, f2, fs, taps=None, n_fft=None, **opts):
        o = zoom_options(**opts)
        self._h = port().sko_zoom_plan_create(n, f1, f2, fs, C.byref(o))
        if not self._h:
            raise OracleError(port().sko_last_error().decode())
        if taps is not None:
            t = f64(taps)
            _chk(port().sko_zoom_plan_set_taps(self._h, _p(t), t.size))
        if n_fft is not None:
            _chk(port().sko_zoom_plan_set_n_fft(self._h, n_fft))
        self.fs = fs
        self.n = n
        info = (sz * 6)()
        d = np.zeros(4)
        port().sko_zoom_plan_info(self._h, info, _p(d))
        (self.decimation, self.n_taps, self.usable_len, self.decimated_len, self.n_fft,
         self.trim_samples) = [int(v) for v in info]
        self.center, self.cutoff, self.group_delay, self.f_step = [float(v) for v in d]

    def __call__(self, samples, fs=None):
        s = f64(samples)
        fs = self.fs if fs is None else fs
        nb, f0, df = sz(0), C.c_double(0), C.c_double(0)
        _chk(port().sko_zoom_fft(self._h, _p(s), s.size, fs, C.byref(nb), C.byref(f0), C.byref(df), None))
        out = np.empty(nb.value, np.complex128)
        _chk(port().sko_zoom_fft(self._h, _p(s), s.size, fs, C.byref(nb), C.byref(f0), C.byref(df),
                                 _p(out.view(np.float64))))
        return out, f0.value, df.value

    def batch(self, x_real, threads=1):
        x_real = f64(x_real)
        return port().sko_bench_zoom(self._h, _p(x_real), self.n, self.fs, x_real.shape[0], threads)

    def batch_out(self, x_real, threads=1):
        """zoom_fft of every row (threaded), the band bins of each row."""
        x_real = f64(x_real)
        nb = self(x_real[0])[0].size
        out = np.empty((x_real.shape[0], nb), np.complex128)
        port().sko_batch_zoom(self._h, _p(x_real), self.n, self.fs, x_real.shape[0], threads,
                              _p(out.view(np.float64)))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            port().sko_zoom_plan_free(self._h)
            self._h = None


def transfer(xs, xr):
    xs, xr = c128(xs), c128(xr)
    h = np.empty_like(xs)
    mag = np.empty(xs.size)
    ph = np.empty(xs.size)
    port().sko_transfer(_p(xs.view(np.float64)), _p(xr.view(np.float64)), xs.size,
                        _p(h.view(np.float64)), _p(mag), _p(ph))
    return h, mag, ph
