"""GPU parity for lengths beyond one CTA's shared memory: the four-step multi-pass path
(complex FFT up to 2^20, cfg5's long zero-padded spectra and CZTs up to L = 2^19)."""
import numpy as np
import pytest

import oracle as O
import paper_2108_03948_b200 as sk
from helpers import TOL_F32, TOL_F64, rel_l2_rows, rel_max_rows
from paper_2108_03948_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda"


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("lg", [14, 15, 16, 17, 18, 20])
def test_c2c_large(prec, lg):
    if prec == "f32" and lg == 14:
        pytest.skip("single-CTA size for fp32")
    n = 1 << lg
    b = 3 if lg < 18 else 1
    rng = np.random.default_rng(lg)
    x = rng.uniform(-1, 1, (b, n)) + 1j * rng.uniform(-1, 1, (b, n))
    dt = torch.complex128 if prec == "f64" else torch.complex64
    xd = torch.from_numpy(x).to(dt).to(DEV)
    xin = xd.cpu().numpy().astype(np.complex128)
    want = np.stack([O.fft(r) for r in xin])
    got = sk.fft_batch(xd).cpu().numpy()
    back = sk.fft_batch(torch.from_numpy(got).to(DEV), inverse=True).cpu().numpy()
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64
        assert rel_max_rows(back, xin) <= TOL_F64
    else:
        assert rel_l2_rows(got, want) <= TOL_F32
        assert rel_l2_rows(back, xin) <= TOL_F32
    if lg == 16:   # the C ABI one-shot path uses the same engine (sk_fft in place)
        g = sk.fft(xin[0]) if prec == "f64" else None
        if g is not None:
            assert rel_max_rows([g], want[:1]) <= TOL_F64


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n", [16384, 65536])
def test_cfg5_long_spectra(prec, n):
    L = 4 * n
    x = W.sample_traces(2, n)
    dt = torch.float64 if prec == "f64" else torch.float32
    xd = torch.from_numpy(x).to(dt).to(DEV)
    xin = xd.cpu().double().numpy()
    want = O.fft_spectrum_batch(xin, L)
    got = sk.fft_spectrum_batch(xd, L).cpu().numpy()
    half = sk.fft_spectrum_batch(xd, L, layout=sk.SKG_HALF).cpu().numpy()
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64
    else:
        assert rel_l2_rows(got, want) <= TOL_F32
    np.testing.assert_array_equal(half, got[:, : L // 2 + 1])


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n,m", [(4096, 16384), (16384, 4096), (16384, 16384), (3000, 12000), (65536, 16384)])
def test_cfg5_long_czt(prec, n, m):
    x = W.sample_traces(2, n)
    a, w = W.cfg2_czt_params(m)
    dt = torch.float64 if prec == "f64" else torch.float32
    xd = torch.from_numpy(x).to(dt).to(DEV)
    xin = xd.cpu().double().numpy()
    plan = sk.CztPlanGPU(n, a, w, m, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
    got = plan.execute(xd).cpu().numpy()
    want = O.CztPlan(n, a, w, m).batch_real(xin)
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64
    else:
        assert rel_l2_rows(got, want) <= TOL_F32


def test_largest_czt_row_fp64():
    """cfg5's largest row: N=65536, M=4N, L=2^19 (one trace; the oracle takes ~0.5 s)."""
    n, m = 65536, 262144
    x = W.sample_traces(1, n)
    a, w = W.cfg2_czt_params(m)
    got = sk.CztPlanGPU(n, a, w, m).execute(torch.from_numpy(x).to(DEV)).cpu().numpy()
    assert rel_max_rows(got, O.CztPlan(n, a, w, m).batch_real(x)) <= TOL_F64


def test_chunking_many_traces():
    """More traces than one L2-resident chunk: results must not depend on the chunk boundaries."""
    n, L = 16384, 65536
    x = W.sample_traces(200, n)
    xd = torch.from_numpy(x).to(DEV)
    got = sk.fft_spectrum_batch(xd, L).cpu().numpy()
    for i in (0, 95, 96, 97, 199):
        assert rel_max_rows(got[i:i + 1], O.fft_spectrum_batch(x[i:i + 1], L)) <= TOL_F64


@pytest.mark.parametrize("path", ["cluster", "four-step"])
@pytest.mark.parametrize("prec,L", [("f64", 32768), ("f64", 65536), ("f32", 65536), ("f32", 131072)])
def test_long_fft_batches(prec, L, path, monkeypatch):
    """both long-transform paths — the 8-CTA cluster FFT (kernels_cluster.cu, opt-in SKG_CLUSTER=1)
    and the four-step passes: more traces than resident CTAs (persistent loops), a length that is no
    multiple of 8 (partial residue classes), strided rows, half layout, an in-place complex round trip."""
    monkeypatch.setenv("SKG_CLUSTER", "1" if path == "cluster" else "0")
    n = L // 4 - 3
    b = 40
    x = W.sample_traces(b, n)
    dt = torch.float64 if prec == "f64" else torch.float32
    xs = torch.zeros((b, n + 5), dtype=dt, device=DEV)
    xs[:, :n] = torch.from_numpy(x).to(dt)
    xin = xs[:, :n].cpu().double().numpy()
    want = O.fft_spectrum_batch(xin, L)
    got = sk.fft_spectrum_batch(xs[:, :n], L).cpu().numpy()
    half = sk.fft_spectrum_batch(xs[:, :n], L, layout=sk.SKG_HALF).cpu().numpy()
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64
    else:
        assert rel_l2_rows(got, want) <= TOL_F32
    np.testing.assert_array_equal(half, got[:, : L // 2 + 1])
    c = torch.from_numpy(got[:4]).to(DEV)
    ref_back = np.stack([O.ifft(r.astype(np.complex128)) for r in got[:4]])
    sk.fft_batch(c, inverse=True, out=c)   # in place
    cb = c.cpu().numpy()
    if prec == "f64":
        assert rel_max_rows(cb, ref_back) <= TOL_F64
    else:
        assert rel_l2_rows(cb, ref_back) <= TOL_F32


@pytest.mark.parametrize("real_path", ["1", "0"])
@pytest.mark.parametrize("prec,L", [("f64", 32768), ("f64", 65536), ("f64", 262144), ("f32", 65536), ("f32", 131072),
                                    ("f32", 262144), ("f32", 1048576)])
def test_real_fourstep_paths(prec, L, real_path, monkeypatch):
    """fft_spectrum beyond one CTA: the Hermitian-half four-step (kernels_4step_real.cuh: paired real
    columns, work rows k1 <= R/2, mirrored conjugate store) and the complex four-step it replaces
    (SKG_4STEP_REAL=0) against the oracle — every zero-padding class of the column pass (N = L/4, L/2,
    L, and ragged lengths between), odd N, both layouts, more units than resident CTAs."""
    monkeypatch.setenv("SKG_CLUSTER", "0")
    monkeypatch.setenv("SKG_4STEP_REAL", real_path)
    dt = torch.float64 if prec == "f64" else torch.float32
    for n, b in ((L // 4, 9), (L // 4 - 3, 2), (L // 2 + 1, 2), (L, 2), (L - 1, 1), (7, 1)):
        if L > 262144:
            b = 1
        x = W.sample_traces(b, n) if n >= 64 else np.arange(1.0, n + 1.0)[None, :] * np.ones((b, 1))
        xd = torch.from_numpy(x).to(dt).to(DEV)
        xin = xd.cpu().double().numpy()
        want = O.fft_spectrum_batch(xin, L)
        got = sk.fft_spectrum_batch(xd, L).cpu().numpy()
        half = sk.fft_spectrum_batch(xd, L, layout=sk.SKG_HALF).cpu().numpy()
        if prec == "f64":
            assert rel_max_rows(got, want) <= TOL_F64, (n, b)
        else:
            assert rel_l2_rows(got, want) <= TOL_F32, (n, b)
        np.testing.assert_array_equal(half, got[:, : L // 2 + 1])


@pytest.mark.parametrize("variant", ["default", "short-lookahead", "small-grid"])
@pytest.mark.parametrize("prec,L,b", [("f32", 65536, 330), ("f64", 65536, 200), ("f32", 262144, 64), ("f64", 262144, 64)])
def test_real_fourstep_fused_ring(prec, L, b, variant, monkeypatch):
    """The one-launch Hermitian four-step (k4_rfused: column and row units interleaved in one persistent
    cooperative grid, work rows in an L2-resident ring reused every `slots` traces, release/acquire
    counters between the passes) gives the two-launch path's bits for every trace, and the oracle's
    spectrum on the first / middle / last traces — with the default look-ahead, with a look-ahead so short
    that row units block on their column units and rows are staged late, and with a small grid."""
    monkeypatch.setenv("SKG_CLUSTER", "0")
    monkeypatch.setenv("SKG_4STEP_REAL", "1")
    if variant == "short-lookahead":
        monkeypatch.setenv("SKG_4STEP_DELTA_X10", "1")
    dt = torch.float64 if prec == "f64" else torch.float32
    n = L // 4 - 3
    x = W.sample_traces(b, n)
    xd = torch.from_numpy(x).to(dt).to(DEV)
    xin = xd.cpu().double().numpy()
    monkeypatch.setenv("SKG_4STEP_FUSED", "0")
    two = sk.fft_spectrum_batch(xd, L)
    two_half = sk.fft_spectrum_batch(xd, L, layout=sk.SKG_HALF)
    monkeypatch.setenv("SKG_4STEP_FUSED", "1")
    with sk.grid_cap(61 if variant == "small-grid" else 0):
        n0 = sk.launch_count()
        one = sk.fft_spectrum_batch(xd, L)
        assert sk.launch_count() - n0 == 1, "the fused path did not run"
        one_half = sk.fft_spectrum_batch(xd, L, layout=sk.SKG_HALF)
        torch.cuda.synchronize()
    assert torch.equal(one, two)
    assert torch.equal(one_half, two_half)
    # strided output rows with a canary in the gaps, strided (odd: unaligned pairs) input rows with poison
    canary = complex(7.5, -3.25)
    buf = torch.full((b, L + 5), canary, dtype=one.dtype, device=DEV)
    xs = torch.full((b, n + 3), float("nan"), dtype=dt, device=DEV)
    xs[:, :n] = xd
    sk.fft_spectrum_batch(xs[:, :n], L, out=buf[:, :L])
    torch.cuda.synchronize()
    assert torch.equal(buf[:, :L], two) and bool((buf[:, L:] == canary).all())
    got = one.cpu().numpy()
    for i in (0, b // 2, b - 1):
        want = O.fft_spectrum_batch(xin[i:i + 1], L)
        if prec == "f64":
            assert rel_max_rows(got[i:i + 1], want) <= TOL_F64
        else:
            assert rel_l2_rows(got[i:i + 1], want) <= TOL_F32


@pytest.mark.parametrize("variant", ["default", "short-lookahead", "small-grid"])
@pytest.mark.parametrize("prec,n,m,b", [("f64", 3000, 12000, 200), ("f64", 16384, 16384, 100), ("f32", 16384, 16384, 200),
                                        ("f32", 30000, 30000, 80), ("f32", 65536, 16384, 64), ("f64", 16384, 65536, 120),
                                        ("f32", 65536, 262144, 48), ("f32", 200000, 20000, 16), ("f64", 300000, 100000, 10)])
def test_czt_fourstep_fused_ring(prec, n, m, b, variant, monkeypatch):
    """The one-launch multi-pass CZT (k4_czt_fused: forward column, Bluestein-middle row and inverse column
    units interleaved in one persistent cooperative grid, work rows in an L2-resident ring) gives the
    three-launch path's bits for every trace and the oracle's bins on the first / middle / last traces, for
    square and 1:2 factorisations, with the default look-ahead, one so short that units block on their
    producers, and a small grid."""
    if variant == "short-lookahead":
        monkeypatch.setenv("SKG_4STEP_DELTA_X10", "1")
    dt = torch.float64 if prec == "f64" else torch.float32
    x = W.sample_traces(b, n)
    a, w = W.cfg2_czt_params(m)
    xd = torch.from_numpy(x).to(dt).to(DEV)
    xin = xd.cpu().double().numpy()
    plan = sk.CztPlanGPU(n, a, w, m, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
    monkeypatch.setenv("SKG_4STEP_FUSED", "0")
    three = plan.execute(xd)   # (also builds the plan's device tables)
    n0 = sk.launch_count()
    three = plan.execute(xd)
    n3 = sk.launch_count() - n0   # three launches per output segment
    monkeypatch.setenv("SKG_4STEP_FUSED", "1")
    with sk.grid_cap(61 if variant == "small-grid" else 0):
        n0 = sk.launch_count()
        one = plan.execute(xd)
        assert 3 * (sk.launch_count() - n0) == n3, "the fused path did not run"
        torch.cuda.synchronize()
    assert torch.equal(one, three)
    canary = complex(7.5, -3.25)
    buf = torch.full((b, m + 3), canary, dtype=one.dtype, device=DEV)
    xs = torch.full((b, n + 3), float("nan"), dtype=dt, device=DEV)
    xs[:, :n] = xd
    plan.execute(xs[:, :n], out=buf[:, :m])
    torch.cuda.synchronize()
    assert torch.equal(buf[:, :m], three) and bool((buf[:, m:] == canary).all())
    got = one.cpu().numpy()
    oplan = O.CztPlan(n, a, w, m)
    for i in (0, b // 2, b - 1):
        want = oplan.batch_real(xin[i:i + 1])
        if prec == "f64":
            assert rel_max_rows(got[i:i + 1], want) <= TOL_F64
        else:
            assert rel_l2_rows(got[i:i + 1], want) <= TOL_F32


def test_fused_paths_stress():
    """tools/fused_stress.py: 450 (grid size, look-ahead, shape, precision) variants of the one-launch
    four-step spectrum and CZT, each bit-identical to the multi-launch path; a dependency cycle or a lost
    release would show as the timeout."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "fused_stress.py")], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "all ok: 450" in r.stdout
