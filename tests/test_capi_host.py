"""C-ABI checks that need no GPU: the library loads, exports every SK_API symbol that
include/*.h declares, and the host-side logic (validation, sizing, error mapping, handle
getters) behaves like the reference's C ABI (capi.cpp, test_capi.cpp). GPU-executing calls are
expected to fail LOUDLY here (SK_ERR_INTERNAL, "no CUDA device") — never to fall back to a CPU."""
import ctypes as C
import subprocess

import numpy as np
import pytest

import paper_2108_03948_b200 as sk

torch = pytest.importorskip("torch")
HAS_GPU = torch.cuda.is_available()


def test_library_exports_every_declared_symbol():
    L = sk.lib()
    names = sk.exported_symbols()
    assert len(names) >= 50
    for n in names:
        assert hasattr(L, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", sk.LIB_PATH], capture_output=True, text=True).stdout
    dyn = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(names) <= dyn
    # hidden visibility: nothing but the C ABI and the spectral:: C++ API leaks out
    assert all(s.startswith("sk") or s.startswith("_ZN8spectral") or s.startswith("_ZNK8spectral") for s in dyn)


def test_status_strings_and_version():   # test_capi.cpp:32-39
    L = sk.lib()
    assert L.sk_status_name(0) == b"ok"
    assert L.sk_status_name(1) == b"invalid argument"
    assert L.sk_status_name(5) == b"insufficient resolution"
    assert len(L.sk_version()) > 0


def test_next_pow2_and_band_params():   # test_capi.cpp:121-125, test_czt.cpp:48-54
    assert sk.next_pow2(500) == 512 and sk.next_pow2(512) == 512 and sk.next_pow2(0) == 1
    a, w = sk.czt_params_for_band(100.0, 1000.0, 8000.0, 128)
    assert abs(a - np.exp(2j * np.pi * 100 / 8000)) < 1e-15
    assert abs(w - np.exp(-2j * np.pi * 900 / (128 * 8000))) < 1e-15
    for bad in ((100.0, 50.0, 8000.0, 16), (0.0, 9000.0, 8000.0, 16), (0.0, 4000.0, 8000.0, 1)):
        with pytest.raises(sk.SkError) as e:
            sk.czt_params_for_band(*bad)
        assert e.value.status == sk.SK_ERR_INVALID_ARGUMENT


def test_argument_errors_before_device_work():   # test_capi.cpp:68-74, numerics.cpp:104-108
    with pytest.raises(sk.SkError) as e:
        sk.fft(np.zeros(12))
    assert e.value.status == sk.SK_ERR_INVALID_ARGUMENT and "pad" in e.value.message and "16" in e.value.message
    with pytest.raises(sk.SkError) as e:
        sk.fft(np.zeros(6))
    assert "8" in e.value.message
    with pytest.raises(sk.SkError):
        sk.fft(np.zeros(0))
    L = sk.lib()
    im = np.zeros(4)
    assert L.sk_fft(None, im.ctypes.data_as(sk.dp), 4) == sk.SK_ERR_INVALID_ARGUMENT
    assert b"null" in L.sk_last_error()
    with pytest.raises(sk.SkError) as e:
        sk.czt(np.ones(8), 0.0, 1.0, 4)   # a = 0 (test_capi.cpp:117-118)
    assert e.value.status == sk.SK_ERR_INVALID_ARGUMENT
    with pytest.raises(sk.SkError):
        sk.czt(np.ones(8), 1.0, 1.0, 0)   # m = 0


def test_trace_and_spectrum_handles():
    t = sk.Trace(np.arange(5.0), 10.0, 0.5)
    assert len(t) == 5 and t.sample_rate_hz == 10.0
    L = sk.lib()
    assert L.sk_trace_size(None) == 0 and L.sk_spectrum_size(None) == 0
    for bad in ([], [1.0, np.nan]):
        with pytest.raises(sk.SkError):
            sk.Trace(np.array(bad, dtype=float), 10.0)
    with pytest.raises(sk.SkError):
        sk.Trace([1.0, 2.0], 0.0)


def test_slice_band_host():   # test_spectra.cpp:61-87
    s = sk.Spectrum(np.arange(11, dtype=complex), 0.0, 10.0, 64)
    cut = sk.slice_band(s, 20.0, 50.0)
    assert cut.bins.size == 4 and cut.f_start_hz == 20.0 and cut.bins[0] == 2 and cut.bins[3] == 5
    assert cut.source_n == 64
    assert sk.slice_band(s, -100.0, 1e9).bins.size == 11
    small = sk.Spectrum(np.ones(5, dtype=complex), 0.0, 10.0, 5)
    for lo, hi in ((42.0, 47.0), (50.0, 40.0), (500.0, 600.0)):
        with pytest.raises(sk.SkError):
            sk.slice_band(small, lo, hi)


def test_zoom_plan_host_logic():   # test_capi.cpp:333-363, test_zoomfft.cpp:65-87, 158-179
    o = sk.zoom_options()
    assert (o.circular, o.pad_pow2, o.decimation) == (1, 1, 0)
    p = sk.ZoomPlan(500, 0.5e12, 2.0e12, 10e12)
    assert (p.decimation, p.n_fft, p.filter_len) == (3, 256, 101)
    assert abs(p.f_step_hz - 10e12 / (3 * 256)) < 1e-3
    u = sk.ZoomPlan(256, 32.0, 96.0, 256.0, decimation=1)
    assert (u.filter_len, u.n_fft) == (1, 256)
    for args, kw in (((500, 2.0e12, 0.5e12, 10e12), {}), ((500, 0.5e12, 6.0e12, 10e12), {}),
                     ((500, 0.5e12, 2.0e12, 10e12), {"decimation": 50}),
                     ((4, 0.5e12, 2.0e12, 10e12), {"decimation": 4}),
                     ((60, 0.5e12, 2.0e12, 10e12), {"decimation": 2}),
                     ((4096, 0.4e12, 1.2e12, 20e12), {"decimation": 8, "num_taps": 64})):
        with pytest.raises(sk.SkError) as e:
            sk.ZoomPlan(*args, **kw)
        assert e.value.status == sk.SK_ERR_INVALID_ARGUMENT


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure mode")
def test_gpu_calls_fail_loudly_without_a_device():
    with pytest.raises(sk.SkError) as e:
        sk.fft(np.ones(8))
    assert e.value.status == sk.SK_ERR_INTERNAL and "CUDA" in e.value.message
    with pytest.raises(sk.SkError) as e:
        sk.fft_spectrum(np.ones(8), 10.0)
    assert e.value.status == sk.SK_ERR_INTERNAL
    p = sk.ZoomPlan(500, 0.5e12, 2.0e12, 10e12)
    with pytest.raises(sk.SkError) as e:
        p.spectrum(np.ones(500))
    assert e.value.status == sk.SK_ERR_INTERNAL
