"""List the resolvability-scan peak / valley picks that differ from the reference's golden curves
(tests/golden/scan.npz): (case, route, separation index, column, ours, reference). These are the
rounding-decided ties tests/test_gpu_scan.py enumerates."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2108_03948_b200 as sk  # noqa: E402
from paper_2108_03948_b200.workloads import SCAN_CASES  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "scan.npz"))
out = []
for name in SCAN_CASES:
    got = sk.resolvability_scan(**SCAN_CASES[name])
    for route in ("fft", "czt"):
        a, b = got[route], g[f"{name}_{route}"]
        for col in (2, 4, 6):
            for i in np.nonzero(a[:, col] != b[:, col])[0]:
                out.append([name, route, int(i), col, float(a[i, col]), float(b[i, col])])
print(json.dumps(out))
