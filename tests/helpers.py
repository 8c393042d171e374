"""Shared tolerances (BASELINE.json north_star) and metrics for the parity tests."""
import numpy as np

TOL_F64 = 1e-10   # fp64 mode: max|d| / max|X_ref|
TOL_F32 = 1e-5    # fp32 mode: relative L2


def rel_max(got, want):
    """acceptance.cpp:54-60: max_k |got - want| / max_k |want|."""
    got = np.asarray(got)
    want = np.asarray(want)
    den = np.max(np.abs(want))
    num = np.max(np.abs(got - want))
    return num / den if den > 0 else num


def rel_max_rows(got, want):
    return max(rel_max(g, w) for g, w in zip(got, want))


def rel_l2(got, want):
    got = np.asarray(got, np.complex128)
    want = np.asarray(want, np.complex128)
    return np.linalg.norm(got - want) / np.linalg.norm(want)


def rel_l2_rows(got, want):
    return max(rel_l2(g, w) for g, w in zip(got, want))
