"""GPU parity: fused Zoom FFT (zoom_fft, zoomfft.cpp:183-239) via sk_zoom_* and skg_zoom_*."""
import numpy as np
import pytest

import oracle as O
import paper_2108_03948_b200 as sk
from helpers import TOL_F32, TOL_F64, rel_l2_rows, rel_max, rel_max_rows
from paper_2108_03948_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda"


def _dev(x, prec):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.float64 if prec == "f64" else torch.float32).to(DEV)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n_fft", [0, 2048])
def test_golden_cfg3(golden, prec, n_fft):
    """configs[2]: N=4096, [0.4, 1.2] THz, D=8, 65 taps (64 is rejected by the reference, §9 D1);
    n_fft 512 (reference sizing) and 2048 (the config text, §9 D2)."""
    g = golden("zoom")
    key = "cfg3_Z2048" if n_fft else "cfg3_Z512"
    plan = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, sk.SKG_F64 if prec == "f64" else sk.SKG_F32,
                          n_fft=n_fft, decimation=8, num_taps=65)
    assert plan.n_fft == (n_fft or 512) and plan.bins == g[key].shape[1]
    f0 = float(g["cfg3_f0_2048" if n_fft else "cfg3_f0_512"])
    assert abs(plan.f_start_hz - f0) < 1e-3
    xd = _dev(g["cfg3_x"], prec)
    got = plan.execute(xd).cpu().numpy()
    if prec == "f64":
        assert rel_max_rows(got, g[key]) <= TOL_F64
    else:
        want = [O.ZoomPlan(4096, 0.4e12, 1.2e12, W.FS, decimation=8, num_taps=65,
                           **({"n_fft": n_fft} if n_fft else {}))(r)[0] for r in xd.cpu().double().numpy()]
        assert rel_l2_rows(got, want) <= TOL_F32


def test_golden_500_sample_plans_through_c_abi(golden):
    g = golden("zoom")
    p500 = g["p500"]
    s = sk.ZoomPlan(500, 0.5e12, 2.0e12, 10e12).spectrum(p500)
    assert rel_max(s.bins, g["p500_default"][0]) <= TOL_F64
    assert abs(s.f_start_hz - float(g["p500_default_f0"])) < 1e-3
    lt = sk.ZoomPlan(500, 0.5e12, 2.0e12, 10e12, decimation=4, circular=0, trim_transient=1).spectrum(p500)
    assert rel_max(lt.bins, g["p500_lin_trim"][0]) <= TOL_F64
    d2 = sk.ZoomPlan(500, 0.5e12, 2.0e12, 10e12, decimation=2).spectrum(p500)
    assert rel_max(d2.bins, g["p500_d2"][0]) <= TOL_F64


def test_zoom_accessors_and_115_bins():   # test_capi.cpp:333-363
    p = sk.ZoomPlan(500, 0.5e12, 2.0e12, 10e12)
    s = p.spectrum(W.thz_pulse(500, fs=10e12))
    assert s.bins.size == 115 and s.f_start_hz >= 0.5e12 and s.frequency(114) <= 2.0e12
    assert abs(s.f_step_hz - p.f_step_hz) < 1e-6
    with pytest.raises(sk.SkError):
        p.spectrum(W.thz_pulse(400, fs=10e12))
    with pytest.raises(sk.SkError):
        p.spectrum(W.thz_pulse(500, fs=10e12), fs=9e12)


def test_degenerate_zoom_equals_sliced_fft():   # test_zoomfft.cpp:89-108
    x = np.random.default_rng(17).uniform(-1, 1, 256)
    z = sk.ZoomPlan(256, 32.0, 96.0, 256.0, decimation=1).spectrum(x, 256.0)
    full = sk.slice_band(sk.fft_spectrum(x, 256.0, 256), 32.0, 96.0)
    assert z.bins.size == full.bins.size and abs(z.f_start_hz - full.f_start_hz) < 1e-9
    assert np.max(np.abs(z.bins - full.bins)) < 1e-10 * np.max(np.abs(full.bins))


def test_zoom_tracks_fft_and_rejects_off_band():   # acceptance.cpp:207-259 (crit7)
    main = W.thz_pulse(500, fs=10e12)
    trace = main + W.thz_pulse(500, fs=10e12, center=30e-12, amplitude=0.25)
    plan = sk.ZoomPlan(500, 0.5e12, 2.0e12, 10e12, decimation=2)
    zoom = plan.spectrum(trace)
    full = sk.fft_spectrum(trace, 10e12, 512)
    idx = np.rint(zoom.frequency(np.arange(zoom.bins.size)) / full.f_step_hz).astype(int)
    pk = 20 * np.log10(np.max(np.abs(zoom.bins)) / np.max(np.abs(full.bins[idx])))
    assert abs(pk) <= 0.5
    tone = np.array([O.cis_cycles(204.0 / 512.0, i).real for i in range(500)])
    leak = np.max(np.abs(plan.spectrum(tone).bins)) / np.max(np.abs(sk.fft_spectrum(tone, 10e12, 512).bins))
    assert 20 * np.log10(leak) <= -50


def test_even_tap_extension_vs_oracle():
    """The 64-tap design of the config text via the explicit-filter extension (§9 D1)."""
    T = 64
    fc = 0.4e12 / W.FS
    k = np.arange(T) - (T - 1) / 2
    h = 2 * fc * np.sinc(2 * fc * k) * (0.54 - 0.46 * np.cos(2 * np.pi * np.arange(T) / (T - 1)))
    h /= h.sum()
    x = W.cfg3_batch(4, 4096)
    plan = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, taps=h, decimation=8, num_taps=65)
    assert plan.num_taps == 64
    got = plan.execute(_dev(x, "f64")).cpu().numpy()
    ref = O.ZoomPlan(4096, 0.4e12, 1.2e12, W.FS, taps=h, decimation=8, num_taps=65)
    assert rel_max_rows(got, [ref(r)[0] for r in x]) <= TOL_F64


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n,D", [(1000, 4), (1000, 16), (1024, 4), (1024, 16), (3000, 4), (3000, 16), (4096, 4),
                                 (4096, 16), (16384, 4), (16384, 16), (65536, 4), (65536, 16)])
def test_cfg5_zoom_rows(prec, n, D):
    """configs[4] zoom rows: band [0.4, 1.2] THz (§9 D3), default 101 taps and cutoff."""
    x = W.sample_traces(4, n)
    plan = sk.ZoomPlanGPU(n, 0.4e12, 1.2e12, W.FS, sk.SKG_F64 if prec == "f64" else sk.SKG_F32, decimation=D)
    xd = _dev(x, prec)
    got = plan.execute(xd).cpu().numpy()
    ref = O.ZoomPlan(n, 0.4e12, 1.2e12, W.FS, decimation=D)
    want = [ref(r)[0] for r in xd.cpu().double().numpy()]
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64
    else:
        assert rel_l2_rows(got, want) <= TOL_F32


def test_linear_mode_and_centre_override():
    x = W.sample_traces(3, 2000)
    for kw in ({"circular": 0, "decimation": 5}, {"circular": 0, "trim_transient": 1, "decimation": 4},
               {"center_hz": 0.9e12, "decimation": 6}, {"cutoff_hz": 0.3e12, "num_taps": 33, "decimation": 8}):
        plan = sk.ZoomPlanGPU(2000, 0.4e12, 1.2e12, W.FS, **kw)
        got = plan.execute(_dev(x, "f64")).cpu().numpy()
        ref = O.ZoomPlan(2000, 0.4e12, 1.2e12, W.FS, **kw)
        assert rel_max_rows(got, [ref(r)[0] for r in x]) <= TOL_F64, kw


def test_natural_length_mode_chirp_route():   # test_zoomfft.cpp:110-126 (n_fft = 125, dft_any)
    p = sk.ZoomPlan(500, 0.5e12, 2.0e12, 10e12, decimation=4, pad_pow2=0)
    assert p.n_fft == 125 and abs(p.f_step_hz - 20e9) < 1e-3
    t = W.thz_pulse(500, fs=10e12)
    s = p.spectrum(t)
    assert s.bins.size == 75 and abs(s.f_start_hz - (1.25e12 - 37 * 20e9)) < 1.0 and s.source_n == 125
    want, f0, _ = O.ZoomPlan(500, 0.5e12, 2.0e12, 10e12, decimation=4, pad_pow2=0)(t)
    assert rel_max(s.bins, want) <= TOL_F64


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n,D", [(16384, 4), (65536, 4), (65536, 16)])
def test_cfg5_zoom_long_records_unfused(prec, n, D):
    """Records / short transforms beyond one CTA: chunked FIR -> (multi-pass) FFT -> band gather."""
    x = W.sample_traces(2, n)
    plan = sk.ZoomPlanGPU(n, 0.4e12, 1.2e12, W.FS, sk.SKG_F64 if prec == "f64" else sk.SKG_F32, decimation=D)
    xd = _dev(x, prec)
    got = plan.execute(xd).cpu().numpy()
    ref = O.ZoomPlan(n, 0.4e12, 1.2e12, W.FS, decimation=D)
    want = [ref(r)[0] for r in xd.cpu().double().numpy()]
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64
    else:
        assert rel_l2_rows(got, want) <= TOL_F32


def test_unfused_linear_trim_long():
    x = W.sample_traces(2, 40000)
    kw = {"circular": 0, "trim_transient": 1, "decimation": 4}
    got = sk.ZoomPlanGPU(40000, 0.4e12, 1.2e12, W.FS, **kw).execute(_dev(x, "f64")).cpu().numpy()
    ref = O.ZoomPlan(40000, 0.4e12, 1.2e12, W.FS, **kw)
    assert rel_max_rows(got, [ref(r)[0] for r in x]) <= TOL_F64


_ROUTE_SNIPPET = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2108_03948_b200 as sk
from paper_2108_03948_b200 import workloads as W
x = W.cfg3_batch(6, 4096)
outs = []
for prec in ("f64", "f32"):
    for kw in ({{"decimation": 8, "num_taps": 65}}, {{"decimation": 4, "circular": 0, "trim_transient": 1}},
               {{"decimation": 5}}, {{"decimation": 16}}, {{"decimation": 3}}):
        p = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, sk.SKG_F64 if prec == "f64" else sk.SKG_F32, **kw)
        xd = torch.from_numpy(x).to(torch.float64 if prec == "f64" else torch.float32).cuda()
        outs.append(p.execute(xd).cpu().numpy().astype(np.complex128))
np.savez({out!r}, *outs)
"""


@pytest.mark.parametrize("env", [{}, {"SKG_ZOOM_SPLIT": "1"}, {"SKG_ZOOM_NO_PFIR": "1"},
                                 {"SKG_ZOOM_NO_PFIR": "1", "SKG_ZOOM_NO_CFIR": "1"},
                                 {"SKG_ZOOM_PATH": "fused"}, {"SKG_ZOOM_PATH": "unfused"}],
                         ids=["default(pfir+fft one kernel where instantiated)", "split-pfir", "split-cfir", "split-wfir",
                              "fused", "unfused"])
def test_zoom_routes_match_oracle(env, tmp_path):
    """Every zoom route (phase-lane FIR, constant-bank FIR, warp-window FIR, fused single kernel,
    unfused FIR + FFT + gather) on linear/circular, power-of-two and odd decimations, against the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "routes.npz")
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, "-c", _ROUTE_SNIPPET.format(root=root, out=out)], check=True, env=e, timeout=600)
    got = np.load(out)
    x = W.cfg3_batch(6, 4096)
    i = 0
    for prec in ("f64", "f32"):
        for kw in ({"decimation": 8, "num_taps": 65}, {"decimation": 4, "circular": 0, "trim_transient": 1},
                   {"decimation": 5}, {"decimation": 16}, {"decimation": 3}):
            ref = O.ZoomPlan(4096, 0.4e12, 1.2e12, W.FS, **kw)
            want = np.array([ref(r)[0] for r in x])
            g = got[f"arr_{i}"]
            i += 1
            if prec == "f64":
                assert rel_max_rows(g, want) <= TOL_F64, (env, kw)
            else:
                assert rel_l2_rows(g, want) <= TOL_F32, (env, kw)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("D", list(range(2, 18)))
def test_zoom_decimation_sweep(prec, D):
    """Every decimation 2..17 (power-of-two, odd, composite: each FIR route and its window sizing)
    with the reference's default 101-tap filter, circular, vs the oracle."""
    x = W.cfg3_batch(5, 4096)
    try:
        ref = O.ZoomPlan(4096, 0.4e12, 1.2e12, W.FS, decimation=D)
    except O.OracleError:
        pytest.skip("the reference rejects this decimation for the band")
    p = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, sk.SKG_F64 if prec == "f64" else sk.SKG_F32, decimation=D)
    got = p.execute(_dev(x, prec)).cpu().numpy()
    want = np.array([ref(r)[0] for r in x])
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64
    else:
        assert rel_l2_rows(got, want) <= TOL_F32


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("D", [4, 16])
@pytest.mark.parametrize("n", [1000, 1024, 3000, 4096, 16384, 2000, 517])
def test_raw_window_fir_route(prec, D, n, monkeypatch):
    """configs[4] zoom geometry (101 taps, D in {4, 16}, circular): the whole-output FIR over a raw
    shared-memory window (kernels_zoom_rfir.cu) against the oracle on every row of a ragged batch — items
    whose windows start before the record, end past its usable length, a ragged last item, the circular
    wrap terms — and against the phase-lane / constant-bank routes it replaces (SKG_ZOOM_NO_RFIR=1),
    including strided rows and a circular=0 plan of the same geometry."""
    P = sk.SKG_F64 if prec == "f64" else sk.SKG_F32
    b = 77
    x = W.sample_traces(b, n)
    xd = _dev(x, prec)
    xin = xd.cpu().double().numpy()
    for circ in (1, 0):
        plan = sk.ZoomPlanGPU(n, 0.4e12, 1.2e12, W.FS, P, decimation=D, circular=circ)
        ref = O.ZoomPlan(n, 0.4e12, 1.2e12, W.FS, decimation=D, circular=circ)
        want = [ref(r)[0] for r in xin]
        got = plan.execute(xd).cpu().numpy()
        monkeypatch.setenv("SKG_ZOOM_NO_RFIR", "1")
        old = plan.execute(xd).cpu().numpy()
        monkeypatch.delenv("SKG_ZOOM_NO_RFIR")
        xs = torch.zeros((b, n + 12), dtype=xd.dtype, device=DEV)   # strided rows, 16-byte aligned
        xs[:, :n] = xd
        got_s = plan.execute(xs[:, :n]).cpu().numpy()
        xu = torch.zeros((b, n + 13), dtype=xd.dtype, device=DEV)   # odd stride: the element-copy fill
        xu[:, :n] = xd
        np.testing.assert_array_equal(plan.execute(xu[:, :n]).cpu().numpy(), got)
        if prec == "f64":
            assert rel_max_rows(got, want) <= TOL_F64, (n, D, circ)
            assert rel_max_rows(old, want) <= TOL_F64
        else:
            assert rel_l2_rows(got, want) <= TOL_F32, (n, D, circ)
            assert rel_l2_rows(old, want) <= TOL_F32
        np.testing.assert_array_equal(got_s, got)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n", [4096, 4000, 2048])
def test_raw_window_fir_fft_fused(prec, n, monkeypatch):
    """configs[2] as written (D = 8, 65 taps, n_fft 2048): raw-window FIR + 2048-point transform + band in one
    launch (k_zoom_rfir_fft) against the oracle on every row of a batch larger than the grid's first wave is
    not needed here (persistent loop: 700 records on <= 592 CTAs), against the two-launch route, with
    unaligned strided rows, and with output rows whose gaps hold a canary."""
    P = sk.SKG_F64 if prec == "f64" else sk.SKG_F32
    b = 700
    x = W.cfg3_batch(b, 4096)[:, :n] if n <= 4096 else W.sample_traces(b, n)
    xd = _dev(x, prec)
    xin = xd.cpu().double().numpy()
    plan = sk.ZoomPlanGPU(n, 0.4e12, 1.2e12, W.FS, P, n_fft=2048, decimation=8, num_taps=65)
    ref = O.ZoomPlan(n, 0.4e12, 1.2e12, W.FS, decimation=8, num_taps=65, n_fft=2048)
    n0 = sk.launch_count()
    got_t = plan.execute(xd)
    assert sk.launch_count() - n0 == 1, "the one-launch route did not run"
    got = got_t.cpu().numpy()
    rows = [0, 1, 147, 148, 349, 591, 592, 699]
    want = [ref(xin[i])[0] for i in rows]
    if prec == "f64":
        assert rel_max_rows(got[rows], want) <= TOL_F64
    else:
        assert rel_l2_rows(got[rows], want) <= TOL_F32
    monkeypatch.setenv("SKG_ZOOM_NO_RFIR_FFT", "1")
    two = plan.execute(xd).cpu().numpy()
    monkeypatch.delenv("SKG_ZOOM_NO_RFIR_FFT")
    if prec == "f64":
        assert rel_max_rows(got, two) <= TOL_F64
    else:
        assert rel_l2_rows(got, two) <= TOL_F32
    xu = torch.full((b, n + 13), float("nan"), dtype=xd.dtype, device=DEV)
    xu[:, :n] = xd
    canary = complex(7.5, -3.25)
    buf = torch.full((b, plan.bins + 3), canary, dtype=got_t.dtype, device=DEV)
    plan.execute(xu[:, :n], out=buf[:, : plan.bins])
    torch.cuda.synchronize()
    assert torch.equal(buf[:, : plan.bins], got_t) and bool((buf[:, plan.bins:] == canary).all())
