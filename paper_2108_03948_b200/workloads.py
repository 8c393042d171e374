"""Seeded synthetic THz-TDS inputs for the BASELINE.json configs (host-side input preparation).

The reference evaluates on no public dataset and its experimental traces are not distributed
(SURVEY §8d), so these generators stand in. They restate the reference's pulse model
(gen_thz_pulse, signals.cpp:46-88: first derivative of a Gaussian, -A sqrt(e) u exp(-u^2/2),
u = (t - t_c)/sigma, peak |A| at u = -/+1) and add seeded white Gaussian noise
(add_noise, signals.cpp:90-99). std::normal_distribution is implementation defined, so the noise
comes from numpy's PCG64 instead; parity never depends on it because the GPU and the CPU oracle
always consume the same host-generated buffers. Inputs are generated once in fp64
and rounded to fp32 for fp32 mode. None of this is timed.
"""
from __future__ import annotations

import numpy as np

FS = 20e12            # Ts = 0.05 ps
SIGMA = 0.3e-12       # pulse width (Gaussian sigma)
T_REF = 10e-12        # reference pulse centre
NOISE = 1e-3
SEED = 2108039480     # SURVEY §8d parameter seed


def thz_pulse(n, fs=FS, center=T_REF, sigma=SIGMA, amplitude=1.0):
    """gen_thz_pulse (gaussian_derivative) for one or many centres/amplitudes (broadcast)."""
    t = np.arange(n, dtype=np.float64) / fs
    center = np.asarray(center, dtype=np.float64)
    amplitude = np.asarray(amplitude, dtype=np.float64)
    if center.ndim or amplitude.ndim:
        center, amplitude = center[..., None], amplitude[..., None]
    u = (t - center) / sigma
    return -(amplitude * np.exp(0.5)) * u * np.exp(-0.5 * u * u)


def cfg1_pair(n=1024, seed=SEED):
    """configs[0]: one reference/sample pair, fp64. Sample = 0.6 x pulse delayed 2 ps plus a 0.15 echo
    read as +8 ps from the reference pulse."""
    rng = np.random.default_rng(seed)
    ref = thz_pulse(n) + NOISE * rng.standard_normal(n)
    sample = (thz_pulse(n, center=T_REF + 2e-12, amplitude=0.6)
              + thz_pulse(n, center=T_REF + 8e-12, amplitude=0.15)
              + NOISE * rng.standard_normal(n))
    return ref, sample


def sample_traces(count, n, seed=SEED + 1):
    """cfg2/cfg5 sample traces: a_i pulse(10 ps + d_i) + 0.25 a_i pulse(10 ps + d_i + 6 ps) + noise,
    d_i ~ U(1, 4) ps, a_i ~ U(0.3, 0.9) (keeps cfg1's 0.15/0.6 echo ratio and 6 ps spacing)."""
    rng = np.random.default_rng(seed)
    d = rng.uniform(1e-12, 4e-12, count)
    a = rng.uniform(0.3, 0.9, count)
    x = np.empty((count, n))
    step = 4096
    for s in range(0, count, step):
        e = min(count, s + step)
        x[s:e] = (thz_pulse(n, center=T_REF + d[s:e], amplitude=a[s:e])
                  + thz_pulse(n, center=T_REF + d[s:e] + 6e-12, amplitude=0.25 * a[s:e]))
    x += NOISE * rng.standard_normal((count, n))
    return x


def reference_traces(count, n, seed=SEED + 2):
    rng = np.random.default_rng(seed)
    return thz_pulse(n)[None, :] + NOISE * rng.standard_normal((count, n))


def cfg2_batch(pairs=4096, n=1024, seed=SEED):
    """configs[1]: `pairs` reference/sample pairs -> 2*pairs traces (refs first, then samples)."""
    return np.concatenate([reference_traces(pairs, n, seed + 2), sample_traces(pairs, n, seed + 1)])


def cfg2_czt_params(m=2048, fs=FS, f1=0.1e12, f2=3.0e12):
    """A = exp(j 2pi f1/fs), W = exp(-j 2pi ((f2-f1)/(M-1))/fs) — the (M-1) step of the config text,
    passed explicitly through sk_czt."""
    a = np.exp(2j * np.pi * f1 / fs)
    w = np.exp(-2j * np.pi * ((f2 - f1) / (m - 1)) / fs)
    return complex(a), complex(w)


def lorentz_lines(x, fs=FS, lines=(0.557e12, 1.097e12), fwhm=20e9, alpha=0.5, pad=4):
    """Imprint absorption lines on the sample spectrum: X(f) * exp(-alpha * sum_l L_l(|f|)) on a
    `pad`-times zero-padded grid, back to time and truncated (cfg3)."""
    n = x.shape[-1]
    L = pad * n
    X = np.fft.rfft(x, L, axis=-1)
    f = np.fft.rfftfreq(L, 1.0 / fs)
    g = 0.5 * fwhm
    att = np.zeros_like(f)
    for f0 in lines:
        att += g * g / ((f - f0) ** 2 + g * g)
    return np.fft.irfft(X * np.exp(-alpha * att), L, axis=-1)[..., :n]


def cfg3_batch(count=4096, n=4096, seed=SEED + 3):
    return lorentz_lines(sample_traces(count, n, seed))


def thickness_map(h=256, w=256, seed=SEED + 4, lo=0.0, hi=3e-12):
    """Smooth seeded 'Perlin-like' map: normalised sum of 8 sinusoids with u_i, v_i in [0.5, 4]."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    s = np.zeros((h, w))
    for _ in range(8):
        c = rng.uniform(0.5, 1.0)
        u, v = rng.uniform(0.5, 4.0, 2)
        ph = rng.uniform(0, 2 * np.pi)
        s += c * np.sin(2 * np.pi * (u * xx / w + v * yy / h) + ph)
    s = (s - s.min()) / (s.max() - s.min())
    return lo + (hi - lo) * s


def cfg4_cube(h=256, w=256, n=2048, seed=SEED + 5, dtype=np.float32):
    """configs[3]: pixel = a(x,y) pulse(10 ps + tau(x,y)) + noise, fp32, plus the shared reference."""
    tau = thickness_map(h, w, seed).ravel()
    amp = thickness_map(h, w, seed + 1, 0.4, 0.9).ravel()
    rng = np.random.default_rng(seed + 2)
    cube = np.empty((h * w, n), dtype=dtype)
    step = 4096
    for s in range(0, h * w, step):
        e = min(h * w, s + step)
        blk = thz_pulse(n, center=T_REF + tau[s:e], amplitude=amp[s:e]) + NOISE * rng.standard_normal((e - s, n))
        cube[s:e] = blk.astype(dtype)
    ref = thz_pulse(n) + NOISE * np.random.default_rng(seed + 3).standard_normal(n)
    return cube, ref


# resolvability sweeps used for parity against the reference's own curves (tests/golden/scan.npz) and
# in bench.py: the reference defaults (chirp route, fft_len 1138), a power-of-two
# padded route (fft_len 512), and a THz-scale sweep (fft_len 14124, multi-pass Bluestein)
SCAN_CASES = {
    "default": {},
    "pow2": dict(f1_hz=0.0, f2_hz=4000.0, m=256, center_hz=2000.0, sep_start_hz=20.0, sep_stop_hz=400.0,
                 sep_step_hz=10.0),
    "thz": dict(sample_rate_hz=20e12, n=1024, f1_hz=0.1e12, f2_hz=3.0e12, m=2048, center_hz=1.0e12,
                sep_start_hz=5e9, sep_stop_hz=200e9, sep_step_hz=5e9),
}
