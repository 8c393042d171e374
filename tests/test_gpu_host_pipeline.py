"""GPU parity of the host-buffer batched entry points (skg_*_host): host rows in, host rows out
through the library's chunked H2D / kernel / D2H pipeline — the batched counterpart of the
reference's host-buffer one-shot calls (sk_czt, capi.cpp:197-205; sk_fft_spectrum; sk_zoom_spectrum).
Each must equal the device-resident call bit for bit (same kernels on the same rows), whatever the
chunking, for pinned and pageable buffers, and match the oracle within the north_star tolerance."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2108_03948_b200 as sk
from helpers import TOL_F32, TOL_F64, rel_l2_rows, rel_max_rows
from paper_2108_03948_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda"
THREADS = os.cpu_count() or 4


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("chunk", [0, 1, 128, 5000])
def test_czt_host_equals_device(prec, pinned, chunk):
    x = W.cfg2_batch(500, 1024).astype(np.float64 if prec == "f64" else np.float32)   # 1000 traces
    a, w = W.cfg2_czt_params(2048)
    plan = sk.CztPlanGPU(1024, a, w, 2048, sk.SKG_F64 if prec == "f64" else sk.SKG_F32)
    xh = torch.from_numpy(x).pin_memory() if pinned else x
    got = plan.execute_host(xh, chunk=chunk)
    dev = plan.execute(torch.from_numpy(x).to(DEV)).cpu().numpy()
    assert np.array_equal(got, dev)
    if chunk == 0:
        want = O.CztPlan(1024, a, w, 2048).batch_real(x.astype(np.float64), threads=THREADS)
        if prec == "f64":
            assert rel_max_rows(got, want) <= TOL_F64
        else:
            assert rel_l2_rows(got, want) <= TOL_F32


def test_strided_host_rows_and_canaries():
    x = W.sample_traces(77, 1000)
    big = np.full((77, 1100), np.nan)
    big[:, :1000] = x
    a, w = W.cfg2_czt_params(250)
    plan = sk.CztPlanGPU(1000, a, w, 250)
    out_big = np.full((77, 300), 7.0 + 7.0j)
    plan.execute_host(big[:, :1000], out=out_big[:, :250], chunk=10)
    assert np.all(out_big[:, 250:] == 7.0 + 7.0j)   # gaps between output rows untouched
    want = plan.execute(torch.from_numpy(x).to(DEV)).cpu().numpy()
    assert np.array_equal(out_big[:, :250], want)


@pytest.mark.parametrize("layout", [sk.SKG_FULL, sk.SKG_HALF])
def test_fft_spectrum_host(layout):
    x = W.sample_traces(300, 1024)
    got = sk.fft_spectrum_host(x, 4096, layout=layout, chunk=64)
    dev = sk.fft_spectrum_batch(torch.from_numpy(x).to(DEV), 4096, layout=layout).cpu().numpy()
    assert np.array_equal(got, dev)
    want = O.fft_spectrum_batch(x, 4096, threads=THREADS)
    if layout == sk.SKG_HALF:
        want = want[:, :2049]
    assert rel_max_rows(got, want) <= TOL_F64


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_zoom_and_transfer_host(prec):
    dt = np.float64 if prec == "f64" else np.float32
    p = sk.SKG_F64 if prec == "f64" else sk.SKG_F32
    z = W.cfg3_batch(200, 4096).astype(dt)
    zp = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, p, decimation=8, num_taps=65)
    assert np.array_equal(zp.execute_host(z, chunk=33), zp.execute(torch.from_numpy(z).to(DEV)).cpu().numpy())
    cube, ref = W.cfg4_cube(10, 30, 2048, dtype=dt)
    tp = sk.TransferPlanGPU(ref, 8192, p)
    mag, ph = tp.execute_host(torch.from_numpy(cube).pin_memory(), chunk=70)
    md, pd = tp.execute(torch.from_numpy(cube).to(DEV))
    assert np.array_equal(mag.numpy() if hasattr(mag, "numpy") else mag, md.cpu().numpy())
    assert np.array_equal(ph if isinstance(ph, np.ndarray) else ph.numpy(), pd.cpu().numpy())


def test_host_argument_errors():
    a, w = W.cfg2_czt_params(64)
    plan = sk.CztPlanGPU(100, a, w, 64)
    with pytest.raises(TypeError):
        plan.execute_host(np.zeros((3, 100), np.float32))          # fp32 rows on an fp64 plan
    with pytest.raises(ValueError):
        plan.execute_host(np.zeros((3, 99)))                        # wrong row length
    with pytest.raises(ValueError):
        plan.execute_host(torch.zeros((3, 100), dtype=torch.float64, device=DEV))
    with pytest.raises(ValueError):
        plan.execute_host(np.zeros((3, 100)), out=np.zeros((2, 64), np.complex128))
    xd = torch.zeros((3, 100), dtype=torch.float32, device=DEV)
    with pytest.raises(TypeError):
        plan.execute(xd)                                            # device path checks too
    with pytest.raises(ValueError):
        plan.execute(torch.zeros((3, 100), dtype=torch.float64, device=DEV),
                     out=torch.empty((3, 10), dtype=torch.complex128, device=DEV))
    with pytest.raises(TypeError):
        plan.execute(torch.zeros((3, 100), dtype=torch.float64, device=DEV),
                     out=torch.empty((3, 64), dtype=torch.complex64, device=DEV))


def test_c_abi_rejects_short_strides():
    import ctypes as C
    a, w = W.cfg2_czt_params(64)
    plan = sk.CztPlanGPU(100, a, w, 64)
    xd = torch.zeros((3, 100), dtype=torch.float64, device=DEV)
    od = torch.empty((3, 64), dtype=torch.complex128, device=DEV)
    st = sk.lib().skg_czt_execute(plan._h, C.c_void_p(xd.data_ptr()), 0, 50, 3, C.c_void_p(od.data_ptr()), 64, None)
    assert st == sk.SK_ERR_INVALID_ARGUMENT and "stride" in sk.last_error()
    st = sk.lib().skg_czt_execute(plan._h, C.c_void_p(xd.data_ptr()), 0, 100, 3, C.c_void_p(od.data_ptr()), 32, None)
    assert st == sk.SK_ERR_INVALID_ARGUMENT
    st = sk.lib().skg_fft_spectrum_batch(100, 256, 7, 0, C.c_void_p(xd.data_ptr()), 100, 3,
                                         C.c_void_p(od.data_ptr()), 256, None)
    assert st == sk.SK_ERR_INVALID_ARGUMENT and "precision" in sk.last_error()
