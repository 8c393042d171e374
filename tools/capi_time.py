import time, ctypes as C, numpy as np, sys
sys.path.insert(0, '.')
import paper_2108_03948_b200 as sk
from paper_2108_03948_b200 import workloads as W
r1, s1 = W.cfg1_pair()
sk.fft_spectrum(s1, W.FS, 4096)
L = sk.lib()
t = sk.Trace(s1, W.FS)
for name, fn in [("Trace()", lambda: sk.Trace(s1, W.FS)),
                 ("sk_fft_spectrum", None),
                 ("full fft_spectrum", lambda: sk.fft_spectrum(s1, W.FS, 4096)),
                 ("sk_czt_spectrum", None)]:
    if name == "sk_fft_spectrum":
        def fn():
            h = C.c_void_p()
            L.sk_fft_spectrum(t.handle, 4096, C.byref(h))
            L.sk_spectrum_free(h)
    if name == "sk_czt_spectrum":
        def fn():
            h = C.c_void_p()
            L.sk_czt_spectrum(t.handle, 0.1e12, 3e12, 2048, C.byref(h))
            L.sk_spectrum_free(h)
    fn()
    t0 = time.perf_counter()
    for _ in range(50):
        fn()
    print(f"{name}: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us")
