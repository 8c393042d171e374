"""GPU parity: complex FFT, zero-padded real spectra and the direct DFT route, through the C ABI.
Oracle = tests/golden (produced by the reference) and the pinned CPU restatement (oracle/)."""
import numpy as np
import pytest

import oracle as O
import paper_2108_03948_b200 as sk
from helpers import TOL_F32, TOL_F64, rel_l2_rows, rel_max, rel_max_rows
from paper_2108_03948_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda"


def test_golden_fft_all_pow2_through_sk_fft(golden):   # acceptance.cpp:76-92 sizes
    g = golden("fft")
    for lg in range(0, 13):
        n = 1 << lg
        for r, want, iwant in zip(g[f"x{n}"], g[f"X{n}"], g[f"i{n}"]):
            assert rel_max(sk.fft(r), want) <= TOL_F64
            assert rel_max(sk.ifft(r), iwant) <= TOL_F64
    np.testing.assert_allclose(sk.fft(g["kat_x"]), [10, -2 + 2j, -2, -2 - 2j], atol=1e-12)


def test_impulse_and_round_trip():   # test_capi.cpp:43-66
    d = np.zeros(4)
    d[0] = 1
    np.testing.assert_allclose(sk.fft(d), np.ones(4), atol=1e-15)
    x = np.random.default_rng(11).uniform(-1, 1, 8) + 1j * np.random.default_rng(12).uniform(-1, 1, 8)
    np.testing.assert_allclose(sk.ifft(sk.fft(x)), x, rtol=0, atol=1e-12)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_batched_c2c_all_sizes(prec):
    rng = np.random.default_rng(5)
    top = 13 if prec == "f64" else 14
    for lg in range(0, top + 1):
        n = 1 << lg
        b = 37
        x = rng.uniform(-1, 1, (b, n)) + 1j * rng.uniform(-1, 1, (b, n))
        dt = torch.complex128 if prec == "f64" else torch.complex64
        xd = torch.from_numpy(x).to(dt).to(DEV)
        xin = xd.cpu().numpy().astype(np.complex128)   # the rounded inputs the GPU sees
        want = np.stack([O.fft(r) for r in xin])
        got = sk.fft_batch(xd).cpu().numpy()
        back = sk.fft_batch(torch.from_numpy(got).to(DEV), inverse=True).cpu().numpy()
        if prec == "f64":
            assert rel_max_rows(got, want) <= TOL_F64, n
            assert rel_max_rows(back, xin) <= TOL_F64, n
        else:
            assert rel_l2_rows(got, want) <= TOL_F32, n
            assert rel_l2_rows(back, xin) <= TOL_F32, n


def test_properties_large_batch():   # Parseval / linearity, acceptance.cpp:337-372, at batch scale
    rng = np.random.default_rng(707)
    n, b = 4096, 1024
    x = torch.from_numpy(rng.uniform(-1, 1, (b, n)) + 1j * rng.uniform(-1, 1, (b, n))).to(DEV)
    y = torch.from_numpy(rng.uniform(-1, 1, (b, n)) + 1j * rng.uniform(-1, 1, (b, n))).to(DEV)
    X, Y = sk.fft_batch(x), sk.fft_batch(y)
    ex = (x.abs() ** 2).sum(1)
    eX = (X.abs() ** 2).sum(1) / n
    assert float(((eX - ex).abs() / ex).max()) <= 1e-10
    a, bb = 0.7 - 1.3j, -2.1 + 0.4j
    M = sk.fft_batch(a * x + bb * y)
    err = ((M - (a * X + bb * Y)).abs().amax(1) / (a * X + bb * Y).abs().amax(1)).max()
    assert float(err) <= 1e-10
    xr = sk.fft_batch(X, inverse=True)
    assert float(((xr - x).abs().amax(1) / x.abs().amax(1)).max()) <= 1e-10


def test_in_place_and_strided_rows():
    rng = np.random.default_rng(3)
    big = torch.from_numpy(rng.uniform(-1, 1, (10, 300)) + 0j).to(DEV)
    view = big[:, 10:266]   # strided rows, 256 points each
    want = np.stack([O.fft(r) for r in view.cpu().numpy()])
    out = torch.empty((10, 256), dtype=torch.complex128, device=DEV)
    sk.fft_batch(view, out=out)
    assert rel_max_rows(out.cpu().numpy(), want) <= TOL_F64


def test_golden_fft_spectrum_through_c_abi(golden):   # spectra.cpp:21-38, test_spectra.cpp:36-59
    g = golden("spectra")
    s = sk.fft_spectrum(g["cfg1_ref"], W.FS, 4096)
    assert s.bins.size == 4096 and s.source_n == 4096 and s.f_start_hz == 0.0
    assert abs(s.f_step_hz - float(g["cfg1_df"])) < 1e-6
    assert rel_max(s.bins, g["cfg1_Xr"]) <= TOL_F64
    assert rel_max(sk.fft_spectrum(g["cfg1_sample"], W.FS, 4096).bins, g["cfg1_Xs"]) <= TOL_F64
    s512 = sk.fft_spectrum(g["pulse500"], 10e12)
    assert s512.bins.size == 512 and rel_max(s512.bins, g["pulse500_X512"]) <= TOL_F64
    assert abs(s512.bins[0].real - g["pulse500"].sum()) < 1e-9
    s500 = sk.fft_spectrum(g["pulse500"], 10e12, 500)   # exact non-pow2 length: chirp route
    assert s500.bins.size == 500 and rel_max(s500.bins, g["pulse500_X500"]) <= TOL_F64
    imp = np.zeros(500)
    imp[0] = 1
    np.testing.assert_allclose(np.abs(sk.fft_spectrum(imp, 10e12, 500).bins), 1.0, atol=1e-9)
    with pytest.raises(sk.SkError):
        sk.fft_spectrum(imp, 10e12, 499)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n,L", [(1, 1), (2, 2), (3, 4), (5, 8), (100, 128), (1000, 4096), (1024, 4096),
                                 (2048, 8192), (3000, 16384), (4096, 16384), (1000, 1000), (777, 1200)])
def test_batched_spectrum_vs_oracle(prec, n, L):
    if prec == "f64" and L > 16384:
        pytest.skip("multi-pass sizes covered elsewhere")
    x = W.sample_traces(9, n) if n >= 1000 else np.random.default_rng(n).uniform(-1, 1, (9, n))
    dt = torch.float64 if prec == "f64" else torch.float32
    xd = torch.from_numpy(x).to(dt).to(DEV)
    xin = xd.cpu().double().numpy()
    want = np.stack([O.fft_spectrum(r, 1.0, L)[0] for r in xin])
    got = sk.fft_spectrum_batch(xd, L).cpu().numpy()
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64
    else:
        assert rel_l2_rows(got, want) <= TOL_F32
    if L & (L - 1) == 0 and L >= 2:
        half = sk.fft_spectrum_batch(xd, L, layout=sk.SKG_HALF).cpu().numpy()
        np.testing.assert_array_equal(half, got[:, : L // 2 + 1])


def test_dft_naive_route(golden):
    g = golden("fft")
    assert rel_max(sk.dft_naive(g["naive_x"]), g["naive_X"]) <= 1e-12
    x = np.random.default_rng(1).uniform(-1, 1, 1000) + 0j
    assert rel_max(sk.dft_naive(x), O.dft_naive(x)) <= 1e-12
