"""GPU parity: fused Bluestein CZT (CztPlan::execute, czt.cpp:116-130) via sk_czt and the batched
skg_czt_* extension, against reference golden vectors and the pinned CPU oracle."""
import numpy as np
import pytest

import oracle as O
import paper_2108_03948_b200 as sk
from helpers import TOL_F32, TOL_F64, rel_l2_rows, rel_max, rel_max_rows
from paper_2108_03948_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda"


def test_golden_czt_through_sk_czt(golden):
    g = golden("czt")
    a, w = complex(g["cfg2_a"]), complex(g["cfg2_w"])
    for r, want in zip(g["cfg2_x"], g["cfg2_X"]):
        assert rel_max(sk.czt(r, a, w, 2048), want) <= TOL_F64
    for i, (n, m, ar, ai, wr, wi) in enumerate(g["rand_params"]):
        got = sk.czt(g[f"r{i}_x"], complex(ar, ai), complex(wr, wi), int(m))
        assert rel_max(got, g[f"r{i}_X"]) <= TOL_F64, (n, m)
    got = sk.czt(g["spiral_x"], complex(g["spiral_a"]), complex(g["spiral_w"]), 24)   # off-circle
    assert rel_max(got, g["spiral_X"]) <= TOL_F64


def test_czt_matches_direct_route():   # test_capi.cpp:90-119
    n, m = 32, 24
    a, w = sk.czt_params_for_band(100.0, 900.0, 8000.0, m)
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    fast, direct = sk.czt(x, a, w, m), sk.czt_direct(x, a, w, m)
    assert rel_max(fast, direct) <= 1e-9
    assert rel_max(direct, O.czt_direct(x, a, w, m)) <= 1e-12


def test_full_circle_equals_dft():   # acceptance.cpp:96-112
    rng = np.random.default_rng(202)
    for n in (7, 16, 100, 128, 500, 1024):
        x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        w = O.cis_cycles(-1.0 / n, 1.0)
        assert rel_max(sk.czt(x, 1.0, w, n), O.dft_naive(x)) <= 1e-9


def test_czt_spectrum_axis_and_impulse():   # test_czt.cpp:123-139
    x = np.zeros(128)
    x[3] = 1.0
    s = sk.czt_spectrum(x, 8000.0, 100.0, 1000.0, 128)
    assert s.bins.size == 128 and s.f_start_hz == 100.0 and abs(s.f_step_hz - 7.03125) < 1e-12
    assert s.source_n == 128
    np.testing.assert_allclose(np.abs(s.bins), 1.0, atol=1e-9)
    with pytest.raises(sk.SkError):
        sk.czt_spectrum(x, 8000.0, 100.0, 5000.0, 128)
    with pytest.raises(sk.SkError):
        sk.czt_spectrum(x, 8000.0, 1000.0, 100.0, 128)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_cfg2_batch(prec):
    """configs[1] shape: N=1024 real traces, M=2048, L=4096, (M-1) W step."""
    x = W.cfg2_batch(48, 1024)
    a, w = W.cfg2_czt_params(2048)
    dt = torch.float64 if prec == "f64" else torch.float32
    xd = torch.from_numpy(x).to(dt).to(DEV)
    xin = xd.cpu().double().numpy()
    plan = sk.CztPlanGPU(1024, a, w, 2048, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
    assert plan.conv_size == 4096
    got = plan.execute(xd).cpu().numpy()
    want = O.CztPlan(1024, a, w, 2048).batch_real(xin)
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64
    else:
        assert rel_l2_rows(got, want) <= TOL_F32


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n,m", [(1, 1), (1, 5), (5, 1), (2, 2), (16, 16), (100, 25), (1000, 250), (1000, 1000),
                                 (1000, 4000), (1024, 256), (3000, 750), (3000, 3000), (4096, 1024),
                                 (4096, 4096), (2000, 6000)])
def test_sweep_vs_oracle(prec, n, m):
    L = O.next_pow2(n + m - 1)
    if L > (8192 if prec == "f64" else 16384):
        pytest.skip("multi-pass length")
    x = W.sample_traces(5, n) if n >= 1000 else np.random.default_rng(n * 7 + m).uniform(-1, 1, (5, n))
    a, w = W.cfg2_czt_params(max(m, 2))
    dt = torch.float64 if prec == "f64" else torch.float32
    xd = torch.from_numpy(x).to(dt).to(DEV)
    xin = xd.cpu().double().numpy()
    got = sk.CztPlanGPU(n, a, w, m, sk.SKG_F64 if prec == "f64" else sk.SKG_F32).execute(xd).cpu().numpy()
    want = O.CztPlan(n, a, w, m).batch_real(xin)
    if prec == "f64":
        assert rel_max_rows(got, want) <= TOL_F64
    else:
        assert rel_l2_rows(got, want) <= TOL_F32


def test_complex_input_and_ragged_batches():
    rng = np.random.default_rng(8)
    n, m = 300, 77
    a, w = 1.001 * np.exp(0.3j), 0.9999 * np.exp(-0.011j)   # mild spiral: |a^-n|, |w^(k^2/2)| stay O(1)
    plan = sk.CztPlanGPU(n, a, w, m)
    ref = O.CztPlan(n, a, w, m)
    for b in (1, 3, 17, 129):
        x = rng.uniform(-1, 1, (b, n)) + 1j * rng.uniform(-1, 1, (b, n))
        got = plan.execute(torch.from_numpy(x).to(DEV)).cpu().numpy()
        assert rel_max_rows(got, [ref.execute(r) for r in x]) <= TOL_F64


def test_plan_errors():
    for args in ((0, 1.0, 1.0, 4), (4, 0.0, 1.0, 4), (4, 1.0, 0.0, 4), (4, 1.0, 1.0, 0)):
        with pytest.raises(sk.SkError) as e:
            sk.CztPlanGPU(*args)
        assert e.value.status == sk.SK_ERR_INVALID_ARGUMENT
