"""Trace ingest and spectrum serialisation through the drop-in C ABI, against
fixtures produced by the REFERENCE ITSELF (tests/golden/csv.npz, tests/golden/make_golden.py:
sk_trace_read_csv on each case file, sk_trace_write_csv / sk_spectrum_write_csv bytes). Host-only:
no GPU needed. Parity bar: identical status code and message, bit-identical samples / fs / t0,
byte-identical files (signals.cpp:100-189, spectra.cpp:63-78)."""
import os

import numpy as np
import pytest

import paper_2108_03948_b200 as sk

CASES = ["crlf_blank_ws", "header_notrail", "jitter_ok", "malformed", "three_cols", "bad_number", "nonuniform",
         "decreasing", "one_sample", "header_only", "empty", "nan_sample", "plus_sign", "two_headers"]


@pytest.mark.parametrize("name", CASES)
def test_trace_read_matches_reference(golden, tmp_path, name):
    g = golden("csv")
    path = tmp_path / f"{name}.csv"
    path.write_bytes(bytes(g[f"in_{name}"]))
    rc = int(g[f"rc_{name}"])
    if rc == 0:
        x, fs, t0 = sk.trace_read_csv(str(path))
        assert np.array_equal(x, g[f"x_{name}"]) and fs == g[f"fs_{name}"] and t0 == g[f"t0_{name}"]
    else:
        with pytest.raises(sk.SkError) as e:
            sk.trace_read_csv(str(path))
        assert e.value.status == rc
        assert str(e.value.message) == str(g[f"msg_{name}"]).replace("<PATH>", str(path))


def test_missing_file(golden, tmp_path):
    g = golden("csv")
    with pytest.raises(sk.SkError) as e:
        sk.trace_read_csv(str(tmp_path / "missing.csv"))
    assert e.value.status == int(g["rc_missing"])
    assert e.value.message == str(g["msg_missing"]).replace("<DIR>", str(tmp_path))


def test_writers_byte_identical(golden, tmp_path):
    g = golden("csv")
    p = tmp_path / "t.csv"
    sk.trace_write_csv(g["w_trace_x"], 20e12, 1.25e-12, str(p))
    assert p.read_bytes() == bytes(g["w_trace"])
    x, fs, t0 = sk.trace_read_csv(str(p))   # round trip through our parser = the reference's
    assert np.array_equal(x, g["rt_x"]) and fs == g["rt_fs"] and t0 == g["rt_t0"]
    q = tmp_path / "s.csv"
    sk.spectrum_write_csv(g["w_spec_X"], float(g["w_spec_f0"]), float(g["w_spec_df"]), str(q))
    assert q.read_bytes() == bytes(g["w_spec"])
    o = tmp_path / "o.csv"
    sk.spectrum_write_csv(g["w_odd_X"], -5.0, 1.0 / 3.0, str(o))
    assert o.read_bytes() == bytes(g["w_odd"])


def test_writer_formatting_random(tmp_path):
    """%.17g via to_chars == printf's %.17g on adversarial doubles (subnormals, huge, negative zero,
    exact powers, shortest-repr traps)."""
    rng = np.random.default_rng(5)
    v = np.concatenate([rng.standard_normal(200) * 10.0 ** rng.integers(-320, 300, 200),
                        [5e-324, -5e-324, 1.7976931348623157e308, -0.0, 0.0, 1.0, 0.1, 1e21, 1e-7, 123456789012345680.0]])
    v = v[np.isfinite(v)]
    bins = v[: v.size // 2 * 2].reshape(-1, 2) @ np.array([1, 1j])
    p = tmp_path / "r.csv"
    sk.spectrum_write_csv(bins, 0.0, 1.0, str(p))
    rows = p.read_text().splitlines()[1:]
    for k, (row, b) in enumerate(zip(rows, bins)):
        f, re, im, _ = row.split(",")
        assert (f, re, im) == ("%.17g" % float(k), "%.17g" % b.real, "%.17g" % b.imag)


def test_invalid_trace_write(tmp_path):
    with pytest.raises(sk.SkError) as e:
        sk.trace_write_csv(np.array([1.0, 2.0]), 1.0, 0.0, str(tmp_path / "no" / "dir.csv"))
    assert e.value.status == 2 and "cannot open trace file for writing" in e.value.message


SPEC_CASES = ["three_fields", "five_fields", "nonuniform", "decreasing", "single", "header_only", "crlf_ws",
              "jitter", "written"]


@pytest.mark.parametrize("name", SPEC_CASES)
def test_spectrum_read_matches_reference(golden, tmp_path, name):
    """sk_spectrum_read_csv (spectra.cpp:94-156) against the reference on the same file bytes."""
    g = golden("csv")
    path = tmp_path / f"sp_{name}.csv"
    path.write_bytes(bytes(g[f"sin_{name}"]))
    rc = int(g[f"src_{name}"])
    if rc == 0:
        s = sk.spectrum_read_csv(str(path))
        assert np.array_equal(s.bins, g[f"sX_{name}"])
        assert s.f_start_hz == g[f"sf0_{name}"] and s.f_step_hz == g[f"sdf_{name}"]
        assert s.source_n == int(g[f"sn_{name}"])
    else:
        with pytest.raises(sk.SkError) as e:
            sk.spectrum_read_csv(str(path))
        assert e.value.status == rc
        assert e.value.message == str(g[f"smsg_{name}"]).replace("<PATH>", str(path))


def test_sizing_helpers():
    """resolution.cpp:18-63 (the reference's sizing arithmetic, restated) incl. its errors."""
    assert sk.record_len_for_step(10e12, 20e9) == 500 and sk.record_len_for_step(10e12, 6e9) == 1667
    assert sk.fft_resolution(20e12, 4096) == 20e12 / 4096
    assert sk.zeros_for_resolution(20e12, 1024, 2.9e12 / 2048) == 14125 - 1024   # ceil(14124.1)
    assert sk.zeros_for_resolution(8000.0, 128, 62.5) == 0
    assert sk.czt_len_for_matched_resolution(0.5e12, 2.0e12, 10e12, 1667) == 250
    with pytest.raises(sk.SkError, match="coarser than the unpadded spacing"):
        sk.zeros_for_resolution(8000.0, 128, 100.0)
    with pytest.raises(sk.SkError, match="band edge exceeds"):
        sk.czt_len_for_matched_resolution(0.0, 6e12, 10e12, 100)
    with pytest.raises(sk.SkError, match="positive and finite"):
        sk.fft_resolution(0.0, 10)


def test_spectrum_json_byte_identical(golden, tmp_path):
    """sk_spectrum_write_json (spectra.cpp:161-183) against the reference's files: the band spectrum,
    adversarial values (subnormal, huge, negative zero, non-terminating), 1500 random bit patterns."""
    g = golden("csv")
    for name, bins, f0, df in (("j_spec", g["w_spec_X"], float(g["w_spec_f0"]), float(g["w_spec_df"])),
                               ("j_odd", g["w_odd_X"], -5.0, 1.0 / 3.0),
                               ("j_rand", g["j_rand_X"], 0.0, 4882812500.0)):
        p = tmp_path / f"{name}.json"
        sk.spectrum_write_json(bins, f0, df, str(p))
        assert p.read_bytes() == bytes(g[name]), name


def test_spectrum_json_differential_vs_reference(tmp_path):
    """Number formatting against the compiled reference on 200k random doubles (bit patterns over the
    whole range, powers of two and their neighbours); runs where oracle/_ref is built."""
    import ctypes as C

    import oracle as O
    R = O.ref()
    if R is None:
        pytest.skip("oracle/_ref not built here")
    R.sk_spectrum_create.argtypes = [O.dp, O.dp, C.c_size_t, C.c_double, C.c_double, C.POINTER(C.c_void_p)]
    R.sk_spectrum_write_json.argtypes = [C.c_void_p, C.c_char_p]
    R.sk_spectrum_free.argtypes = [C.c_void_p]
    rng = np.random.default_rng(2024)
    bits = rng.integers(0, 2**63, 150000, dtype=np.uint64) | (rng.integers(0, 2, 150000, dtype=np.uint64) << np.uint64(63))
    v = bits.view(np.float64)
    p2 = np.ldexp(1.0, rng.integers(-1074, 1023, 20000))
    v = np.concatenate([v[np.isfinite(v)], p2, np.nextafter(p2, np.inf), np.nextafter(p2, 0)])
    v = v[: v.size // 2 * 2]
    bins = v[0::2] + 1j * v[1::2]
    re, im = np.ascontiguousarray(bins.real), np.ascontiguousarray(bins.imag)
    h = C.c_void_p()
    assert R.sk_spectrum_create(O._p(re), O._p(im), re.size, 1.5, 0.1, C.byref(h)) == 0
    ref = tmp_path / "ref.json"
    assert R.sk_spectrum_write_json(h, str(ref).encode()) == 0
    R.sk_spectrum_free(h)
    ours = tmp_path / "ours.json"
    sk.spectrum_write_json(bins, 1.5, 0.1, str(ours))
    assert ours.read_bytes() == ref.read_bytes()
