"""GPU parity: the two-tone resolvability sweep (analysis.cpp:99-195) as a batched
caller — every separation's padded-FFT route and band-CZT route run as two batched launches, the valley
test on host threads. Against the REFERENCE's own sk_resolvability_scan curves (tests/golden/scan.npz):
identical separations, resolved flags, peak / valley frequencies (bin picks) and minimum resolved
separations; dB fields within 1e-8 dB (the fp64 transforms' 1e-10 relative error through 20 log10)."""
import numpy as np
import pytest

import paper_2108_03948_b200 as sk
from paper_2108_03948_b200.workloads import SCAN_CASES

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(SCAN_CASES))
def test_scan_matches_reference(golden, name):
    g = golden("scan")
    got = sk.resolvability_scan(**SCAN_CASES[name])
    assert np.array_equal(got["separations_hz"], g[f"{name}_sep"])
    for route in ("fft", "czt"):
        a, b = got[route], g[f"{name}_{route}"]
        assert np.array_equal(a[:, 0], b[:, 0]), route                   # resolved
        assert np.array_equal(a[:, [2, 4, 6]], b[:, [2, 4, 6]]), route   # peak / valley frequencies
        fin = np.isfinite(b[:, [1, 3, 5, 7]])
        assert np.array_equal(fin, np.isfinite(a[:, [1, 3, 5, 7]]))
        assert np.max(np.abs(a[:, [1, 3, 5, 7]][fin] - b[:, [1, 3, 5, 7]][fin]), initial=0.0) <= 1e-8, route
    assert got["min_resolved_fft_hz"] == g[f"{name}_minfft"] or (np.isnan(got["min_resolved_fft_hz"]) and
                                                                 np.isnan(g[f"{name}_minfft"]))
    assert got["min_resolved_czt_hz"] == g[f"{name}_minczt"] or (np.isnan(got["min_resolved_czt_hz"]) and
                                                                 np.isnan(g[f"{name}_minczt"]))
