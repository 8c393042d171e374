"""GPU parity: transfer function H = X_sample / X_ref fused into the FFT store epilogue.
Not in the reference: the oracle is the reference's own spectra of both
traces plus the restated per-bin division, |H| = hypot, arg H = atan2 (oracle/skoracle.c
sko_transfer). Bins where |X_ref| < 1e-3 max|X_ref| are noise-dominated and masked."""
import numpy as np
import pytest

import oracle as O
import paper_2108_03948_b200 as sk
from helpers import TOL_F32, TOL_F64
from paper_2108_03948_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda"


def _mask(xr):
    return np.abs(xr) >= 1e-3 * np.max(np.abs(xr))


def _wrap(d):
    return np.angle(np.exp(1j * d))


def test_cfg1_pair_fp64(golden):
    """configs[0]: one pair, N=1024 -> 4096, fp64."""
    g = golden("spectra")
    ref, sample = g["cfg1_ref"], g["cfg1_sample"]
    plan = sk.TransferPlanGPU(ref, 4096, sk.SKG_F64)
    assert plan.bins == 2049
    xr = plan.reference_spectrum()
    assert np.max(np.abs(xr - g["cfg1_Xr"][:2049])) <= TOL_F64 * np.max(np.abs(g["cfg1_Xr"]))
    h = torch.empty((1, 2049), dtype=torch.complex128, device=DEV)
    mag, ph = plan.execute(torch.from_numpy(sample[None]).to(DEV), h=h)
    H, M, P = O.transfer(g["cfg1_Xs"][:2049], g["cfg1_Xr"][:2049])
    m = _mask(g["cfg1_Xr"][:2049])
    hg = h.cpu().numpy()[0]
    assert np.max(np.abs(hg[m] - H[m])) <= TOL_F64 * np.max(np.abs(H[m]))
    assert np.max(np.abs(mag.cpu().numpy()[0][m] - M[m])) <= TOL_F64 * np.max(M[m])
    assert np.max(np.abs(_wrap(ph.cpu().numpy()[0][m] - P[m]))) <= 1e-9


def test_cube_slice_fp32():
    """configs[3] shape on a 16 x 16 tile: 2048 samples fp32 -> FFT 8192 -> |H|, arg H on 4097 bins.
    fp32 tolerance 1e-5 (relative L2) applies to the spectra X_s (the transform itself) and to |H| on the
    SURVEY §8d mask (|X_ref| >= 1e-3 max); the complex H / phase carries the fp32 transform error
    divided by small |X_s|, |X_ref|, so it is checked at 1e-5 on the better-conditioned 1e-2 mask and at
    1e-4 on the 1e-3 mask."""
    cube, ref = W.cfg4_cube(16, 16, 2048)
    plan = sk.TransferPlanGPU(ref, 8192, sk.SKG_F32)
    assert plan.bins == 4097
    cd = torch.from_numpy(cube).to(DEV)
    mag, ph = plan.execute(cd)
    xs_gpu = sk.fft_spectrum_batch(cd, 8192, layout=sk.SKG_HALF).cpu().numpy()
    xr = O.fft_spectrum(ref, 1.0, 8192)[0][:4097]
    m = _mask(xr)
    m2 = np.abs(xr) >= 1e-2 * np.max(np.abs(xr))
    magg, phg = mag.cpu().numpy(), ph.cpu().numpy()
    worst_mag = worst_h = worst_h2 = worst_ph = worst_xs = 0.0
    for i in range(cube.shape[0]):
        xs = O.fft_spectrum(cube[i].astype(np.float64), 1.0, 8192)[0][:4097]
        worst_xs = max(worst_xs, np.linalg.norm(xs_gpu[i] - xs) / np.linalg.norm(xs))
        H, M, P = O.transfer(xs, xr)
        hg2 = magg[i][m2] * np.exp(1j * phg[i][m2].astype(np.float64))
        worst_h2 = max(worst_h2, np.linalg.norm(hg2 - H[m2]) / np.linalg.norm(H[m2]))
        worst_mag = max(worst_mag, np.linalg.norm(magg[i][m] - M[m]) / np.linalg.norm(M[m]))
        # magnitude and phase together: rel L2 of |H| e^{i arg H} (phase of near-zero bins carries no weight)
        hg = magg[i][m] * np.exp(1j * phg[i][m].astype(np.float64))
        worst_h = max(worst_h, np.linalg.norm(hg - H[m]) / np.linalg.norm(H[m]))
        # phase alone, weighted by |H|: fp32 phase noise on a bin is ~eps * max|X| / |X_k|, so the
        # phase error times |H_k| is bounded by the spectrum-wide fp32 error
        worst_ph = max(worst_ph, np.max(np.abs(_wrap(phg[i][m] - P[m])) * M[m]) / M[m].max())
    assert worst_xs <= TOL_F32 and worst_mag <= TOL_F32 and worst_h2 <= TOL_F32
    assert worst_h <= 10 * TOL_F32 and worst_ph <= 10 * TOL_F32


def test_errors():
    with pytest.raises(sk.SkError):
        sk.TransferPlanGPU(np.zeros(0), 16)
    with pytest.raises(sk.SkError):
        sk.TransferPlanGPU(np.ones(100), 1000)   # non power of two
