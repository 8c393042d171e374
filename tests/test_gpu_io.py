"""GPU path of the batched file boundary: skg_traces_read_csv (parallel parse ->
pinned staging -> one H2D copy) and skg_spectra_write_csv (one D2H copy -> parallel reference-format
writers). Parity: the batched ingest equals the drop-in sk_trace_read_csv file by file (bit-exact,
itself pinned to the reference by tests/test_csv_io.py), the batched writer's files are
byte-identical to sk_spectrum_write_csv of the same bins, and errors are the lowest-index failing
file's status and message."""
import numpy as np
import pytest

import paper_2108_03948_b200 as sk
from paper_2108_03948_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _write_traces(tmp_path, x, fs=W.FS, t0_step=1e-12):
    paths = []
    for i, r in enumerate(x):
        p = str(tmp_path / f"trace_{i:04d}.csv")
        sk.trace_write_csv(r, fs, t0_step * i, p)
        paths.append(p)
    return paths


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_ingest_matches_dropin(tmp_path, dtype):
    x = W.sample_traces(37, 1024)
    paths = _write_traces(tmp_path, x)
    dt = getattr(torch, dtype)
    got, fs, t0 = sk.traces_read_csv(paths, 1024, dtype=dt, threads=4)
    for i, p in enumerate(paths):
        want, f, t = sk.trace_read_csv(p)
        assert f == fs[i] and t == t0[i]
        assert np.array_equal(got[i].cpu().numpy(), want.astype(dtype))


def test_ingest_errors(tmp_path):
    x = W.sample_traces(12, 256)
    paths = _write_traces(tmp_path, x)
    with open(paths[9], "a") as f:
        f.write("oops\n")
    with open(paths[5], "w") as f:
        f.write("0,1\n1,2\n")   # wrong length
    with pytest.raises(sk.SkError) as e:
        sk.traces_read_csv(paths, 256)
    assert e.value.status == 4 and e.value.message == f"{paths[5]}: expected 256 samples, got 2"
    paths[5] = str(tmp_path / "nope.csv")
    with pytest.raises(sk.SkError) as e:
        sk.traces_read_csv(paths, 256)
    assert e.value.status == 2 and "cannot open trace file" in e.value.message


def test_pipeline_files_to_files(tmp_path):
    """CSV traces -> batched ingest -> fused band FFT -> batched writer, against the single-trace
    drop-in chain (sk_trace_read_csv, sk_fft_spectrum, sk_spectrum_slice_band, sk_spectrum_write_csv):
    byte-identical output files."""
    x = W.sample_traces(16, 1024)
    # one time axis for the batch: the parsed rate is 1 / median step of the %.17g-printed times, so
    # files with different t0 can differ in the last bit of fs (and of the frequency column)
    paths = _write_traces(tmp_path, x, t0_step=0.0)
    dev, fs, _ = sk.traces_read_csv(paths, 1024)
    assert np.all(fs == fs[0])
    bins, _, f0, df = sk.fft_spectrum_band_batch(dev, fs[0], 0.1e12, 3.0e12, 4096, db=False)
    outs = [str(tmp_path / f"spec_{i:04d}.csv") for i in range(16)]
    sk.spectra_write_csv(outs, bins, f0, df, threads=3)
    for i, p in enumerate(paths):
        s, f, _ = sk.trace_read_csv(p)
        band = sk.slice_band(sk.fft_spectrum(s, f, 4096), 0.1e12, 3.0e12)
        ref_out = str(tmp_path / f"ref_{i:04d}.csv")
        sk.spectrum_write_csv(band.bins, band.f_start_hz, band.f_step_hz, ref_out)
        assert open(outs[i], "rb").read() == open(ref_out, "rb").read()


def test_writer_fp32_promotes(tmp_path):
    b = (torch.randn(3, 50, dtype=torch.complex64, device="cuda"))
    outs = [str(tmp_path / f"w{i}.csv") for i in range(3)]
    sk.spectra_write_csv(outs, b, [0.0, 1.0, 2.0], 0.5)
    h = b.cpu().numpy().astype(np.complex128)
    for i in range(3):
        ref_out = str(tmp_path / f"r{i}.csv")
        sk.spectrum_write_csv(h[i], float(i), 0.5, ref_out)
        assert open(outs[i], "rb").read() == open(ref_out, "rb").read()
