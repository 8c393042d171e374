"""Host side of the resolvability sweep (analysis.cpp:30-195, resolution.cpp:18-47): validation order
and messages of sk_resolvability_scan (raised before any device work) and the valley test
sk_dip_metric_compute, restated from the reference, on spectra with known answers."""
import numpy as np
import pytest

import paper_2108_03948_b200 as sk


@pytest.mark.parametrize("kw,msg", [
    (dict(sample_rate_hz=0.0), "sample rate must be positive"),
    (dict(n=1), "record too short"),
    (dict(f2_hz=5000.0), "band must satisfy"),
    (dict(m=1), "need at least 2 band bins"),
    (dict(sep_step_hz=0.0), "bad separation sweep"),
    (dict(sep_stop_hz=5000.0), "tone pair leaves the band"),
    (dict(n=4096), "coarser than the unpadded spacing"),
])
def test_scan_validation(kw, msg):
    with pytest.raises(sk.SkError, match=msg) as e:
        sk.resolvability_scan(**kw)
    assert e.value.status == 1


def test_dip_metric_known_answers():
    f = np.arange(16.0)
    mag = np.array([0, 1, 2, 5, 2, 1, 0.5, 1, 3, 6, 3, 1, 0, 0, 0, 0], float)
    m = sk.dip_metric(mag.astype(complex), 0.0, 1.0, 3.0, 9.0)
    assert m[0] == 1 and m[2] == 3.0 and m[4] == 9.0 and m[6] == 6.0
    assert abs(m[1] - 20 * np.log10(5 / 0.5)) < 1e-12 and abs(m[7] - 20 * np.log10(0.5)) < 1e-12
    # merged tones: adjacent peaks, no valley
    m = sk.dip_metric(np.array([0, 1, 4, 5, 1, 0], complex), 0.0, 1.0, 1.9, 4.1)
    assert m[0] == 0 and m[2] == m[4] == m[6] == 3.0
    # flat: no local maxima, the default (all-zero) metric
    assert sk.dip_metric(np.ones(8, complex), 0.0, 1.0, 1.0, 5.0) == (0.0,) * 8
    with pytest.raises(sk.SkError) as e:
        sk.dip_metric(np.ones(8, complex), 0.0, 1.0, 2.0, 3.0)
    assert e.value.status == 5 and "fewer than 3 bins" in e.value.message
    with pytest.raises(sk.SkError, match="fall off the axis"):
        sk.dip_metric(np.ones(8, complex), 0.0, 1.0, 2.0, 9.0)
    with pytest.raises(sk.SkError, match="f_a < f_b"):
        sk.dip_metric(np.ones(8, complex), 0.0, 1.0, 3.0, 2.0)
