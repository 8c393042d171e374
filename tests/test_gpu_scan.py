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


# The picks that differ from the reference's, enumerated (case, route, separation index, column):
# every one is a valley of a symmetric pair — the mirror bin about the centre or a bin at the fp64 noise
# floor — decided by the last bits of the transform (tools/scan_ties.py lists them). Any other
# difference, or one of these disappearing, fails.
KNOWN_TIES = {("pow2", "fft", 26, 6), ("pow2", "czt", 23, 6), ("pow2", "czt", 33, 6)}


def test_scan_ties_are_exactly_the_enumerated_ones(golden):
    g = golden("scan")
    found = set()
    for name in SCAN_CASES:
        got = sk.resolvability_scan(**SCAN_CASES[name])
        for route in ("fft", "czt"):
            a, b = got[route], g[f"{name}_{route}"]
            for col in (2, 4, 6):
                found |= {(name, route, int(i), col) for i in np.nonzero(a[:, col] != b[:, col])[0]}
    assert found == KNOWN_TIES


@pytest.mark.parametrize("name", list(SCAN_CASES))
def test_scan_matches_reference(golden, name):
    g = golden("scan")
    got = sk.resolvability_scan(**SCAN_CASES[name])
    assert np.array_equal(got["separations_hz"], g[f"{name}_sep"])
    for route in ("fft", "czt"):
        a, b = got[route], g[f"{name}_{route}"]
        assert np.array_equal(a[:, 0], b[:, 0]), route                   # resolved
        # Peak / valley picks. Two ill-conditioned cases are decided by rounding, not by the algorithm
        # (the reference's radix-2 FFT vs our radix-16 Stockham differ in the last bits):
        #  * a symmetric tone pair centred ON a bin has mirror bins of equal magnitude: a differing
        #    pick must be the mirror image about the centre, with the same dB value;
        #  * a valley at an exact zero of the spectrum sits at the fp64 noise floor (> 200 dB below the
        #    peaks), where the minimum among several ~1e-16 bins is noise: both picks must be there.
        centre = SCAN_CASES[name].get("center_hz") or 0.5 * (SCAN_CASES[name].get("f1_hz", 100.0) +
                                                             SCAN_CASES[name].get("f2_hz", 1000.0))
        floor = np.minimum(b[:, 3], b[:, 5]) - 200.0
        noise = (a[:, 7] < floor) & (b[:, 7] < floor)
        for col in (2, 4, 6):
            diff = a[:, col] != b[:, col]
            mirror = np.abs(a[:, col] + b[:, col] - 2 * centre) <= 1e-9 * centre
            ok = ~diff | mirror | (noise if col == 6 else False)
            assert np.all(ok), (route, col, a[~ok, col], b[~ok, col])
        for col in (3, 5):   # peak dB
            assert np.max(np.abs(a[:, col] - b[:, col])) <= 1e-8, (route, col)
        q = ~noise   # valley dB and dip dB above the noise floor
        assert np.max(np.abs(a[q, 7] - b[q, 7]), initial=0.0) <= 1e-8, route
        fin = q & np.isfinite(b[:, 1])
        assert np.array_equal(np.isfinite(a[q, 1]), np.isfinite(b[q, 1]))
        assert np.max(np.abs(a[fin, 1] - b[fin, 1]), initial=0.0) <= 1e-8, route
        assert np.all((a[noise, 1] > 150) & (b[noise, 1] > 150))
    assert got["min_resolved_fft_hz"] == g[f"{name}_minfft"] or (np.isnan(got["min_resolved_fft_hz"]) and
                                                                 np.isnan(g[f"{name}_minfft"]))
    assert got["min_resolved_czt_hz"] == g[f"{name}_minczt"] or (np.isnan(got["min_resolved_czt_hz"]) and
                                                                 np.isnan(g[f"{name}_minczt"]))


def test_curve_csv(tmp_path):
    """sk_resolvability_write_csv (serialize.cpp:39-45, 141-154): the header, two rows per separation,
    %.17g fields — checked against Python's printf formatting of the same curve values."""
    p = tmp_path / "curve.csv"
    got = sk.resolvability_scan(csv_path=str(p), **SCAN_CASES["default"])
    lines = p.read_text().splitlines()
    assert lines[0] == ("separation_hz,method,resolved,dip_db,f_peak_a_hz,peak_a_db,f_peak_b_hz,peak_b_db,"
                        "f_valley_hz,valley_db")
    assert len(lines) == 1 + 2 * got["separations_hz"].size
    for i, sep in enumerate(got["separations_hz"]):
        for j, route in enumerate(("fft", "czt")):
            m = got[route][i]
            want = ",".join(["%.17g" % sep, route, "%d" % int(m[0])] + ["%.17g" % v for v in m[1:]])
            assert lines[1 + 2 * i + j] == want


def test_curve_files_match_reference_layout(golden, tmp_path):
    """sk_resolvability_write_json / _csv against the reference's own files for the default sweep:
    identical text once the numbers are masked (layout, key order, booleans, integers, nulls), and the
    numbers equal to the reference's within the route's tolerance (separations exact)."""
    import json
    import re
    g = golden("scan")
    pj, pc = tmp_path / "c.json", tmp_path / "c.csv"
    sk.resolvability_scan(csv_path=str(pc), json_path=str(pj), **SCAN_CASES["default"])
    num = re.compile(r"-?\d+(\.\d+)?(e[+-]\d+)?")
    ours, ref = pj.read_text(), bytes(g["default_json"]).decode()
    assert num.sub("#", ours) == num.sub("#", ref)
    a, b = json.loads(ours), json.loads(ref)
    assert a["separations_hz"] == b["separations_hz"] and a["config"] == b["config"]
    assert a["min_resolved_fft_hz"] == b["min_resolved_fft_hz"] and a["min_resolved_czt_hz"] == b["min_resolved_czt_hz"]
    for route in ("fft", "czt"):
        for x, y in zip(a[route], b[route]):
            assert x["resolved"] == y["resolved"]
            for k in ("peak_a_db", "peak_b_db"):
                assert abs(x[k] - y[k]) <= 1e-8
    assert num.sub("#", pc.read_text()) == num.sub("#", bytes(g["default_csv"]).decode())
