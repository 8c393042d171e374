"""GPU memory-safety checks (compute-sanitizer cannot attach on the GPU pool): every batched entry
point runs on strided input rows whose gaps hold poison values and writes into strided output
rows whose gaps hold a canary. The result must equal the contiguous run bit for bit (any read of a
gap would change it) and every canary must survive (any stray write would overwrite one)."""
import numpy as np
import pytest

import paper_2108_03948_b200 as sk
from paper_2108_03948_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CANARY = 7.25 - 3.5j
POISON = 1e30


def _strided_in(x, pad=5):
    """rows of x inside a wider buffer whose gaps are poison"""
    b, n = x.shape
    buf = torch.full((b, n + pad), POISON, dtype=x.dtype, device=x.device)
    buf[:, 2:2 + n] = x
    return buf[:, 2:2 + n]


def _strided_out(b, n, dtype, pad=7, off=3):
    buf = torch.full((b, n + pad), CANARY if dtype.is_complex else CANARY.real, dtype=dtype, device="cuda")
    return buf, buf[:, off:off + n], off, n


def _canaries_ok(buf, off, n):
    host = buf.cpu().numpy()
    want = CANARY if np.iscomplexobj(host) else CANARY.real
    mask = np.ones(host.shape, bool)
    mask[:, off:off + n] = False
    return bool(np.all(host[mask] == want))


def _same(a, b):
    return np.array_equal(a.cpu().numpy(), b.cpu().numpy())


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n,L,layout", [(1000, 4096, sk.SKG_FULL), (1024, 4096, sk.SKG_HALF), (3000, 16384, sk.SKG_FULL),
                                        (20000, 65536, sk.SKG_HALF), (700, 1000, sk.SKG_FULL)])
def test_fft_spectrum_guards(prec, n, L, layout):
    x = torch.from_numpy(W.sample_traces(37, n)).cuda()
    x = x if prec == "f64" else x.float()
    ref = sk.fft_spectrum_batch(x, L, layout)
    buf, out, off, nb = _strided_out(37, ref.shape[1], ref.dtype)
    sk.fft_spectrum_batch(_strided_in(x), L, layout, out=out)
    torch.cuda.synchronize()
    assert _same(out, ref) and _canaries_ok(buf, off, nb)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n,m", [(1024, 2048), (1000, 1000), (1024, 333), (4096, 4096), (16384, 16384), (77, 5)])
def test_czt_guards(prec, n, m):
    x = torch.from_numpy(W.sample_traces(29, n)).cuda()
    x = x if prec == "f64" else x.float()
    a, w = W.cfg2_czt_params(m)
    p = sk.CztPlanGPU(n, a, w, m, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
    ref = p.execute(x)
    buf, out, off, nb = _strided_out(29, m, ref.dtype)
    p.execute(_strided_in(x), out=out)
    torch.cuda.synchronize()
    assert _same(out, ref) and _canaries_ok(buf, off, nb)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("kw", [{"decimation": 8, "num_taps": 65}, {"decimation": 5}, {"decimation": 3},
                                {"decimation": 6}, {"decimation": 16}, {"decimation": 4, "circular": 0,
                                                                        "trim_transient": 1}])
def test_zoom_guards(prec, kw):
    x = torch.from_numpy(W.cfg3_batch(23, 4096)).cuda()
    x = x if prec == "f64" else x.float()
    p = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, sk.SKG_F64 if prec == "f64" else sk.SKG_F32, **kw)
    ref = p.execute(x)
    buf, out, off, nb = _strided_out(23, p.bins, ref.dtype)
    p.execute(_strided_in(x, pad=6), out=out)
    torch.cuda.synchronize()
    assert _same(out, ref) and _canaries_ok(buf, off, nb)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_transfer_guards(prec):
    ref_t, smp = W.cfg1_pair()
    x = torch.from_numpy(np.stack([smp] * 19)).cuda()
    x = x if prec == "f64" else x.float()
    tp = sk.TransferPlanGPU(ref_t, 4096, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
    m0, p0 = tp.execute(x)
    rdt = m0.dtype
    bm, mag, off, nb = _strided_out(19, tp.bins, rdt)
    bp, ph, _, _ = _strided_out(19, tp.bins, rdt)
    tp.execute(_strided_in(x), mag=mag, phase=ph)
    torch.cuda.synchronize()
    assert _same(mag, m0) and _same(ph, p0)
    assert _canaries_ok(bm, off, nb) and _canaries_ok(bp, off, nb)


def _sizes(seed, count, lo, hi):
    rng = np.random.default_rng(seed)
    return [int(v) for v in rng.integers(lo, hi, size=count)]


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("case", range(12))
def test_czt_random_sizes_guarded(prec, case):
    """Seeded random (N, M) from 1 to ~20000 (every kernel class: resident-table, per-trace,
    multi-pass, segmented): parity vs the oracle on 2 rows and canaries around strided outputs."""
    import oracle as O
    from helpers import TOL_F32, TOL_F64, rel_l2_rows, rel_max_rows
    rng = np.random.default_rng(1000 + case)
    n = int(rng.integers(1, 20000)) if case % 3 else int(rng.integers(1, 300))
    m = int(rng.integers(1, 20000)) if case % 2 else int(rng.integers(1, 300))
    xs = W.sample_traces(3, n)
    a, w = complex(np.exp(2j * np.pi * rng.uniform(0, 0.5))), complex(np.exp(-2j * np.pi * rng.uniform(1e-5, 1e-3)))
    x = torch.from_numpy(xs).cuda()
    x = x if prec == "f64" else x.float()
    p = sk.CztPlanGPU(n, a, w, m, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
    buf, out, off, nb = _strided_out(3, m, torch.complex128 if prec == "f64" else torch.complex64)
    p.execute(_strided_in(x), out=out)
    torch.cuda.synchronize()
    assert _canaries_ok(buf, off, nb)
    want = O.CztPlan(n, a, w, m).batch_real(xs[:2].astype(np.float32).astype(np.float64) if prec == "f32" else xs[:2])
    got = out[:2].cpu().numpy()
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64, (n, m)
    else:
        assert rel_l2_rows(got, want) <= TOL_F32, (n, m)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("case", range(10))
def test_fft_spectrum_random_sizes_guarded(prec, case):
    """Seeded random trace lengths and transform lengths (powers of two up to 2^18 and arbitrary
    lengths through the chirp route), full and half layouts, vs the oracle, canaries intact."""
    import oracle as O
    from helpers import TOL_F32, TOL_F64, rel_l2_rows, rel_max_rows
    rng = np.random.default_rng(2000 + case)
    n = int(rng.integers(1, 40000))
    L = 1 << int(rng.integers(max(0, int(np.ceil(np.log2(n)))), 19)) if case % 2 == 0 else int(rng.integers(n, n + 5000))
    layout = sk.SKG_HALF if (case % 4 == 0 and L & (L - 1) == 0) else sk.SKG_FULL
    xs = W.sample_traces(3, n)
    x = torch.from_numpy(xs).cuda()
    x = x if prec == "f64" else x.float()
    nbins = L if layout == sk.SKG_FULL else L // 2 + 1
    buf, out, off, nb = _strided_out(3, nbins, torch.complex128 if prec == "f64" else torch.complex64)
    sk.fft_spectrum_batch(_strided_in(x), L, layout, out=out)
    torch.cuda.synchronize()
    assert _canaries_ok(buf, off, nb)
    src = xs[:2].astype(np.float32).astype(np.float64) if prec == "f32" else xs[:2]
    want = O.fft_spectrum_batch(src, L)[:, :nbins]
    got = out[:2].cpu().numpy()
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64, (n, L)
    else:
        assert rel_l2_rows(got, want) <= TOL_F32, (n, L)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n,L", [(1024, 4096), (3000, 16384), (16384, 65536), (700, 1000)])
def test_band_db_guards(prec, n, L):
    """skg_fft_spectrum_band_batch (fused band + dB store, and the chirp / multi-pass fallback through
    skg_band_db_batch) on poisoned strided input rows into canaried strided bins and dB rows."""
    import ctypes as C
    x = torch.from_numpy(W.sample_traces(23, n)).cuda()
    x = x if prec == "f64" else x.float()
    ref_bins, ref_db, _, _ = sk.fft_spectrum_band_batch(x, W.FS, 0.1e12, 3.0e12, L)
    k_lo, cnt, _ = sk.band_bins(L, 0.0, W.FS / L, 0.1e12, 3.0e12)
    bbuf, bins, boff, _ = _strided_out(23, cnt, ref_bins.dtype)
    dbuf, db, doff, _ = _strided_out(23, cnt, ref_db.dtype)
    xs = _strided_in(x)
    P = sk.SKG_F64 if prec == "f64" else sk.SKG_F32
    rc = sk.lib().skg_fft_spectrum_band_batch(n, L, P, k_lo, cnt, C.c_void_p(xs.data_ptr()), xs.stride(0), 23,
                                              C.c_void_p(bins.data_ptr()), bins.stride(0),
                                              C.c_void_p(db.data_ptr()), db.stride(0), sk._stream())
    assert rc == 0
    torch.cuda.synchronize()
    assert _same(bins, ref_bins) and _same(db, ref_db)
    assert _canaries_ok(bbuf, boff, cnt) and _canaries_ok(dbuf, doff, cnt)
