"""Pin the CPU oracle (oracle/skoracle.c) before trusting it as the parity checker.

(1) The reference's own known-answer tests and property tests, restated
    (test_numerics.cpp, test_czt.cpp, test_zoomfft.cpp, test_spectra.cpp, acceptance.cpp).
(2) Golden vectors produced by the reference itself (tests/golden/*.npz, tests/golden/make_golden.py).
(3) When oracle/_ref (the compiled reference) is present, a differential run on fresh inputs.
"""
import numpy as np
import pytest

import oracle as O
from helpers import rel_max, rel_max_rows
from paper_2108_03948_b200 import workloads as W


# ---- (1) reference KATs, restated -----------------------------------------------------------

def test_pow2_helpers():   # test_numerics.cpp:41-55
    assert [O.next_pow2(n) for n in (1, 2, 3, 500, 1024, 1025)] == [1, 2, 4, 512, 1024, 2048]
    assert O.next_pow2(0) == 0   # error path (reference throws)


def test_four_point_kat():   # test_numerics.cpp:66-74
    X = O.fft([1, 2, 3, 4])
    np.testing.assert_allclose(X, [10, -2 + 2j, -2, -2 - 2j], atol=1e-12)
    np.testing.assert_allclose(O.dft_naive([1, 2, 3, 4]), [10, -2 + 2j, -2, -2 - 2j], atol=1e-12)


def test_impulse_constant_tone():   # test_numerics.cpp:76-96
    n = 16
    d = np.zeros(n, complex)
    d[0] = 1
    np.testing.assert_allclose(O.fft(d), np.ones(n), atol=1e-12)
    c = O.fft(np.ones(n))
    assert abs(c[0] - n) < 1e-12 and np.max(np.abs(c[1:])) < 1e-12
    tone = np.array([O.cis_cycles(5 / n, i) for i in range(n)])
    want = np.zeros(n)
    want[5] = n
    np.testing.assert_allclose(O.dft_naive(tone), want, atol=1e-9)


def test_fft_vs_naive_all_pow2():   # acceptance.cpp:76-92 (reduced rep count)
    rng = np.random.default_rng(101)
    for lg in range(1, 11):
        n = 1 << lg
        x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        assert rel_max(O.fft(x), O.dft_naive(x)) <= 1e-10


def test_fft_errors():   # test_numerics.cpp:108-126
    with pytest.raises(O.OracleError, match=r"pad.*8"):
        O.fft(np.ones(6))
    with pytest.raises(O.OracleError):
        O.fft(np.ones(0))


def test_properties():   # acceptance.cpp:337-372 (Parseval, round trip, superposition)
    rng = np.random.default_rng(707)
    for _ in range(50):
        n = 1 << int(rng.integers(2, 11))
        x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        X = O.fft(x)
        assert abs(np.sum(np.abs(X) ** 2) / n - np.sum(np.abs(x) ** 2)) / np.sum(np.abs(x) ** 2) <= 1e-10
        assert rel_max(O.ifft(X), x) <= 1e-10
        y = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        a, b = complex(*rng.uniform(-2, 2, 2)), complex(*rng.uniform(-2, 2, 2))
        assert rel_max(O.fft(a * x + b * y), a * X + b * O.fft(y)) <= 1e-10


def test_cis_cycles():   # test_numerics.cpp:176-199
    assert abs(O.cis_cycles(0.25, 1.0) - 1j) < 1e-15
    v = O.cis_cycles(0.25, 4.0e15 + 1.0)
    assert abs(v.real) < 1e-12 and abs(v.imag - 1) < 1e-12


def test_czt_full_circle_is_dft():   # acceptance.cpp:96-112
    rng = np.random.default_rng(202)
    for n in (7, 16, 100, 128, 500):
        x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        w = O.cis_cycles(-1.0 / n, 1.0)
        assert rel_max(O.czt(x, 1.0, w, n), O.dft_naive(x)) <= 1e-9


def test_czt_vs_direct_random_bands():   # acceptance.cpp:116-132 / test_czt.cpp:66-80 (reduced)
    rng = np.random.default_rng(303)
    for _ in range(20):
        n, m = int(rng.integers(2, 300)), int(rng.integers(2, 300))
        f1 = rng.uniform(0, 3500)
        a, w = O.czt_params_for_band(f1, rng.uniform(f1 + 10, 4000), 8000.0, m)
        x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        assert rel_max(O.czt(x, a, w, m), O.czt_direct(x, a, w, m)) <= 1e-9


def test_czt_band_params():   # test_czt.cpp:48-54
    a, w = O.czt_params_for_band(100.0, 1000.0, 8000.0, 128)
    assert abs(a - np.exp(2j * np.pi * 100 / 8000)) < 1e-15
    assert abs(w - np.exp(-2j * np.pi * 900 / (128 * 8000))) < 1e-15


def test_zoom_plan_sizing():   # test_zoomfft.cpp:65-87, 110-140
    p = O.ZoomPlan(500, 0.5e12, 2.0e12, 10e12)
    assert (p.decimation, p.n_taps, p.usable_len, p.decimated_len, p.n_fft) == (3, 101, 498, 166, 256)
    assert abs(p.group_delay - 50) < 1e-12
    assert abs(p.cutoff - 0.5 * (0.75e12 + 10e12 / 6)) < 1e-3
    q = O.ZoomPlan(500, 0.5e12, 2.0e12, 10e12, decimation=4, pad_pow2=0)
    assert (q.usable_len, q.decimated_len, q.n_fft) == (500, 125, 125)
    z, f0, df = q(W.thz_pulse(500, fs=10e12))
    assert z.size == 75 and abs(f0 - (1.25e12 - 37 * 20e9)) < 1.0
    r = O.ZoomPlan(500, 0.5e12, 2.0e12, 10e12, decimation=4, circular=0, trim_transient=1)
    assert (r.trim_samples, r.decimated_len, r.n_fft) == (25, 100, 128)
    with pytest.raises(O.OracleError, match="odd"):
        O.design_lowpass(1000.0, 8000.0, 30)
    with pytest.raises(O.OracleError, match="decimation too large"):
        O.ZoomPlan(4096, 0.1e12, 3e12, 20e12, decimation=16, num_taps=101)


def test_zoom_degenerate_equals_sliced_fft():   # test_zoomfft.cpp:89-108
    rng = np.random.default_rng(17)
    x = rng.uniform(-1, 1, 256)
    z, f0, df = O.ZoomPlan(256, 32.0, 96.0, 256.0, decimation=1)(x)
    X, _, step, _ = O.fft_spectrum(x, 256.0, 256)
    k0, cnt = O.slice_band(256, 0.0, step, 32.0, 96.0)
    assert cnt == z.size and abs(f0 - k0 * step) < 1e-9
    assert rel_max(z, X[k0:k0 + cnt]) < 1e-10


# ---- (2) golden vectors from the reference ----------------------------------------------

def test_golden_fft(golden):
    g = golden("fft")
    for lg in range(0, 13):
        n = 1 << lg
        x = g[f"x{n}"]
        assert rel_max_rows([O.fft(r) for r in x], g[f"X{n}"]) <= 1e-14
        assert rel_max_rows([O.ifft(r) for r in x], g[f"i{n}"]) <= 1e-14
    assert rel_max(O.fft(g["kat_x"]), g["kat_X"]) == 0.0
    assert rel_max(O.dft_naive(g["naive_x"]), g["naive_X"]) <= 1e-14


def test_golden_czt(golden):
    g = golden("czt")
    a, w = complex(g["cfg2_a"]), complex(g["cfg2_w"])
    assert rel_max_rows([O.czt(r, a, w, 2048) for r in g["cfg2_x"]], g["cfg2_X"]) <= 1e-14
    for i, (n, m, ar, ai, wr, wi) in enumerate(g["rand_params"]):
        got = O.czt(g[f"r{i}_x"], complex(ar, ai), complex(wr, wi), int(m))
        assert rel_max(got, g[f"r{i}_X"]) <= 1e-14
    got = O.czt(g["spiral_x"], complex(g["spiral_a"]), complex(g["spiral_w"]), 24)
    assert rel_max(got, g["spiral_X"]) <= 1e-14


def test_golden_spectra(golden):
    g = golden("spectra")
    Xr, f0, df, n = O.fft_spectrum(g["cfg1_ref"], W.FS, 4096)
    assert n == 4096 and f0 == 0.0 and abs(df - float(g["cfg1_df"])) < 1e-6
    assert rel_max(Xr, g["cfg1_Xr"]) <= 1e-14
    assert rel_max(O.fft_spectrum(g["cfg1_sample"], W.FS, 4096)[0], g["cfg1_Xs"]) <= 1e-14
    assert rel_max(O.fft_spectrum(g["pulse500"], 10e12, 0)[0], g["pulse500_X512"]) <= 1e-14
    assert rel_max(O.fft_spectrum(g["pulse500"], 10e12, 500)[0], g["pulse500_X500"]) <= 1e-14


def test_golden_zoom(golden):
    g = golden("zoom")
    p = O.ZoomPlan(4096, 0.4e12, 1.2e12, W.FS, decimation=8, num_taps=65)
    rows = [p(r)[0] for r in g["cfg3_x"]]
    assert rel_max_rows(rows, g["cfg3_Z512"]) <= 1e-14
    assert abs(p(g["cfg3_x"][0])[1] - float(g["cfg3_f0_512"])) < 1e-3
    p2 = O.ZoomPlan(4096, 0.4e12, 1.2e12, W.FS, decimation=8, num_taps=65, n_fft=2048)
    assert rel_max_rows([p2(r)[0] for r in g["cfg3_x"]], g["cfg3_Z2048"]) <= 1e-14
    assert rel_max(O.ZoomPlan(500, 0.5e12, 2e12, 10e12)(g["p500"])[0], g["p500_default"][0]) <= 1e-14
    lt = O.ZoomPlan(500, 0.5e12, 2e12, 10e12, decimation=4, circular=0, trim_transient=1)
    assert rel_max(lt(g["p500"])[0], g["p500_lin_trim"][0]) <= 1e-14
    assert rel_max(O.ZoomPlan(500, 0.5e12, 2e12, 10e12, decimation=2)(g["p500"])[0], g["p500_d2"][0]) <= 1e-14


# ---- (3) differential against the compiled reference, when present --------------------------

@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built in this environment")
def test_differential_vs_reference():
    import ctypes as C
    R = O.ref()
    rng = np.random.default_rng(9)
    for n in (1024, 8192, 65536):
        x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        re, im = x.real.copy(), x.imag.copy()
        assert R.sk_fft(O._p(re), O._p(im), n) == 0
        assert rel_max(O.fft(x), re + 1j * im) == 0.0
    for n, m in ((1024, 2048), (3000, 750), (333, 4001)):
        a, w = W.cfg2_czt_params(m)
        x = rng.uniform(-1, 1, n)
        p = R.skr_czt_plan_create(n, a.real, a.imag, w.real, w.imag, m)
        out = np.zeros(m, np.complex128)
        R.skr_czt_batch(p, O._p(np.ascontiguousarray(x)), n, 1, 1, O._p(out.view(np.float64)))
        R.skr_czt_plan_free(p)
        assert rel_max(O.czt(x, a, w, m), out) == 0.0


def test_golden_band_db(golden):
    """slice_band + magnitude_db against the reference's own sk_spectrum_slice_band
    and sk_spectrum_magnitude_db outputs: bin selection exact, band axis exact, dB bit-exact on the
    reference's bins (same formula, hypot + log10)."""
    g = golden("band")
    for name in ("thz", "half", "nyq", "edge", "top"):
        lo, hi = g[f"{name}_band"]
        X, _, step, _ = O.fft_spectrum(g["x"], W.FS, 4096)
        k0, cnt = O.slice_band(4096, 0.0, step, lo, hi)
        assert cnt == g[f"{name}_X"].size and k0 * step == g[f"{name}_f0"] and step == g[f"{name}_df"]
        assert rel_max(X[k0:k0 + cnt], g[f"{name}_X"]) <= 1e-14
        assert np.max(np.abs(O.magnitude_db(g[f"{name}_X"]) - g[f"{name}_db"])) <= 1e-12
    assert np.all(O.magnitude_db(g["zeros_X"]) == -300.0) and np.all(g["zeros_db"] == -300.0)
    with pytest.raises(O.OracleError, match="inverted"):
        O.slice_band(16, 0.0, 1.0, 5.0, 4.0)
    with pytest.raises(O.OracleError, match="no bins"):
        O.slice_band(16, 0.0, 1.0, 4.2, 4.8)
