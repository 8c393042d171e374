"""GPU parity: band slice + magnitude_db — slice_band (spectra.cpp:40-61) and
magnitude_db (types.cpp:13-18) fused into the zero-padded FFT's store (single-CTA route) or run as
one pass over complex rows on the device (chirp / multi-pass routes, CZT and zoom outputs).
Golden vectors: tests/golden/band.npz, produced by the reference's own sk_fft_spectrum ->
sk_spectrum_slice_band -> sk_spectrum_magnitude_db. Tolerances: fp64 bins max|d|/max|X| <= 1e-10
(the dB column to 1e-8 dB where |X| >= 1e-6 max|X|, i.e. the bins' 1e-10 relative error through
20 log10); fp32 relative L2 <= 1e-5 for the bins, the dB column to 1e-4 dB against the same bins."""
import numpy as np
import pytest

import oracle as O
import paper_2108_03948_b200 as sk
from helpers import TOL_F32, TOL_F64, rel_l2, rel_max
from paper_2108_03948_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda"


def _db_ok(db, want_db, X):
    m = np.abs(X) >= 1e-6 * np.max(np.abs(X))
    return np.max(np.abs(db[m] - want_db[m])) <= 1e-8 and np.all(db[~m] <= want_db[m].max())


@pytest.mark.parametrize("name", ["thz", "half", "nyq", "edge", "top"])
def test_golden_bands_fp64(golden, name):
    g = golden("band")
    lo, hi = g[f"{name}_band"]
    x = torch.from_numpy(g["x"][None]).to(DEV)
    bins, db, f0, df = sk.fft_spectrum_band_batch(x, W.FS, lo, hi, 4096)
    want = g[f"{name}_X"]
    assert bins.shape[1] == want.size and f0 == g[f"{name}_f0"] and df == g[f"{name}_df"]
    assert rel_max(bins.cpu().numpy()[0], want) <= TOL_F64
    assert _db_ok(db.cpu().numpy()[0], g[f"{name}_db"], want)


def test_golden_nonpow2_and_floor(golden):
    """exact length 500 (chirp route, then the band pass) and an all-zero trace (-300 dB floor)."""
    g = golden("band")
    p500 = W.thz_pulse(500, fs=10e12)
    bins, db, f0, _ = sk.fft_spectrum_band_batch(torch.from_numpy(p500[None]).to(DEV), 10e12, 0.5e12, 2.0e12, 500)
    assert f0 == g["p500_f0"] and rel_max(bins.cpu().numpy()[0], g["p500_X"]) <= TOL_F64
    assert _db_ok(db.cpu().numpy()[0], g["p500_db"], g["p500_X"])
    z = torch.zeros((3, 64), dtype=torch.float64, device=DEV)
    _, db, _, _ = sk.fft_spectrum_band_batch(z, W.FS, 0.0, 5e12, 64, bins=False)
    assert db.shape[1] == g["zeros_db"].size and torch.all(db == -300.0)


@pytest.mark.parametrize("n,L", [(1024, 4096), (2048, 8192), (1000, 4096), (16384, 65536), (3000, 3000)])
def test_batch_vs_oracle(n, L):
    """fp64 and fp32 batches on every route: single-CTA fused (4096, 8192), multi-pass (65536),
    chirp (3000); bins only, dB only, both."""
    x = W.sample_traces(6, n)
    lo, hi = 0.1e12, 3.0e12
    step = W.FS / L
    k0, cnt = O.slice_band(L, 0.0, step, lo, hi)
    want = np.stack([O.fft_spectrum(r, W.FS, L)[0][k0:k0 + cnt] for r in x])
    want_db = np.stack([O.magnitude_db(r) for r in want])
    for dt in (torch.float64, torch.float32):
        xd = torch.from_numpy(x).to(DEV, dt)
        bins, db, f0, _ = sk.fft_spectrum_band_batch(xd, W.FS, lo, hi, L)
        assert bins.shape == (6, cnt) and f0 == k0 * step
        b, d = bins.cpu().numpy(), db.cpu().numpy()
        if dt == torch.float64:
            assert max(rel_max(b[i], want[i]) for i in range(6)) <= TOL_F64
            assert all(_db_ok(d[i], want_db[i], want[i]) for i in range(6))
        else:
            want32 = np.stack([O.fft_spectrum(r.astype(np.float32).astype(np.float64), W.FS, L)[0][k0:k0 + cnt]
                               for r in x])
            assert max(rel_l2(b[i], want32[i]) for i in range(6)) <= TOL_F32
            # the dB column is 20 log10 of the bins: its own arithmetic (fp32 log10 of |X|^2) is checked
            # against the same bins to 1e-4 dB; against the oracle it inherits the bins' fp32 error
            # amplified by 8.7 dB per unit relative error on weak bins, so the L2 bound there is 10x
            assert max(np.max(np.abs(d[i] - O.magnitude_db(b[i].astype(np.complex128)))) for i in range(6)) <= 1e-4
            assert max(np.linalg.norm(d[i] - O.magnitude_db(want32[i])) / np.linalg.norm(O.magnitude_db(want32[i]))
                       for i in range(6)) <= 10 * TOL_F32
        b_only, none, _, _ = sk.fft_spectrum_band_batch(xd, W.FS, lo, hi, L, db=False)
        assert none is None and torch.equal(b_only, bins)
        none, d_only, _, _ = sk.fft_spectrum_band_batch(xd, W.FS, lo, hi, L, bins=False)
        assert none is None and torch.equal(d_only, db)


def test_band_db_on_czt_output():
    """the standalone pass over CZT rows (configs[1] geometry): slice of bins 100..1899 + dB."""
    x = W.cfg2_batch(2, 1024)
    a, w = W.cfg2_czt_params(2048)
    out = sk.CztPlanGPU(1024, a, w, 2048).execute(torch.from_numpy(x).to(DEV))
    bins, db = sk.band_db_batch(out, 100, 1800)
    want = O.CztPlan(1024, a, w, 2048).batch_real(x)[:, 100:1900]
    assert max(rel_max(bins.cpu().numpy()[i], want[i]) for i in range(4)) <= TOL_F64
    assert all(_db_ok(db.cpu().numpy()[i], O.magnitude_db(want[i]), want[i]) for i in range(4))


def test_errors():
    x = torch.zeros((1, 64), dtype=torch.float64, device=DEV)
    with pytest.raises(sk.SkError, match="inverted"):
        sk.fft_spectrum_band_batch(x, W.FS, 2e12, 1e12, 64)
    # slice_band's slack is 0.5 * f_step * 1e-9 in HERTZ applied to bin indices (spectra.cpp:44-48): at
    # fs = 20 THz it spans ~156 bins, so an empty band needs a small step to exist at all (restated as is)
    assert sk.band_bins(64, 0.0, W.FS / 64, 1.001e12, 1.002e12) == (0, 64, 0.0)
    with pytest.raises(sk.SkError, match="no bins"):
        sk.fft_spectrum_band_batch(x, 1.0, 0.2001, 0.2002, 64)
    with pytest.raises(sk.SkError):
        sk.band_db_batch(torch.zeros((1, 8), dtype=torch.complex128, device=DEV), 0, 0)
