"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/ots.h declares; the facade validates
shapes / arguments with the reference's exception classes before touching
the device; no CPU fallback exists."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ots.h")).read()
    return sorted(set(re.findall(r"\b(ots_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_all_declared_symbols():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_native.EXPORTED_SYMBOLS) <= set(syms)


def test_version_callable_without_gpu():
    assert _native.lib().ots_version() == 1


def test_api_surface_names():
    for name in ["two_stage_qr", "householder_qr", "modified_lu", "block_householder_qr",
                 "reorthogonalized_two_stage", "TwoStageResult", "BlockQRResult",
                 "ReflectorDiagnostics", "MLUResult", "GenHouseholder", "QRPair", "EPS",
                 "OrthoError", "DimensionError", "OrthonormalityError", "IntraFailure",
                 "ParameterError", "NormBoundError", "SingularTError", "NotPositiveDefinite"]:
        assert hasattr(P, name), name
    assert issubclass(P.OrthonormalityError, P.OrthoError)
    assert P.IntraFailure("x", block=3).block == 3


def test_validation_before_device():
    # shape errors are raised by host validation (same order as twostage.py:73-80)
    with pytest.raises(P.DimensionError):
        P.two_stage_qr(np.ones((5, 3, 1)), np.ones((5, 2)))
    with pytest.raises(P.DimensionError):
        P.two_stage_qr(np.eye(6, 3), np.ones((7, 2)))
    with pytest.raises(P.DimensionError):
        P.two_stage_qr(np.eye(5, 3), np.ones((5, 3)))
    with pytest.raises(P.DimensionError):
        P.householder_qr(np.ones((2, 3)))
    with pytest.raises(P.ParameterError):
        P.block_householder_qr([])


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.NativeUnavailable):
        P.two_stage_qr(np.eye(10, 3), np.ones((10, 2)))
    with pytest.raises(P.NativeUnavailable):
        P.householder_qr(np.ones((10, 2)))
    ip = P.InnerProduct.weighted(np.arange(1.0, 11.0))
    with pytest.raises(P.NativeUnavailable):
        P.b_householder_qr(np.ones((10, 2)), P.initial_b_basis(ip, 2), ip)
    with pytest.raises(P.NativeUnavailable):
        P.b_build_reflector(P.initial_b_basis(ip, 2), P.initial_b_basis(ip, 2), ip)
    with pytest.raises(P.NativeUnavailable):
        P.b_block_householder_qr([np.ones((10, 2))], ip)


def test_drop_in_surface():
    """every name of the reference's path surface."""
    for name in ("two_stage_qr", "build_reflector", "apply_reflector", "reflector_diagnostics", "modified_lu",
                 "b_two_stage_qr", "b_build_reflector", "b_apply_reflector", "b_householder_qr",
                 "b_block_householder_qr", "InnerProduct", "initial_b_basis", "BGenHouseholder",
                 "block_householder_qr", "reorthogonalized_two_stage", "householder_qr", "TwoStageResult",
                 "BlockQRResult", "GenHouseholder", "ReflectorDiagnostics"):
        assert callable(getattr(P, name)), name


def test_b_path_validation_on_host():
    """Shape / basis checks of the B-path primitives run before any device work
    (oblique.py:125-151, 170-238 error behaviour)."""
    from paper_2602_14449_b200.oblique import _is_canonical_basis
    d = np.arange(1.0, 13.0)
    ip = P.InnerProduct.weighted(d)
    u = P.initial_b_basis(ip, 4)
    assert _is_canonical_basis(u, ip.diag, 4)
    assert not _is_canonical_basis(2.0 * u, ip.diag, 4)
    with pytest.raises(P.DimensionError):
        P.b_householder_qr(np.ones((11, 2)), u, ip)          # row mismatch
    with pytest.raises(P.DimensionError):
        P.b_householder_qr(np.ones((12, 5)), u, ip)          # u_init too narrow
    with pytest.raises(P.DimensionError):
        P.b_build_reflector(u[:, :3], u, ip)                  # v / u0 shapes differ
    with pytest.raises(P.DimensionError):
        P.b_build_reflector(np.zeros((12, 0)), np.zeros((12, 0)), ip)
    with pytest.raises(P.ParameterError):
        P.b_block_householder_qr([], ip)
    with pytest.raises(P.DimensionError):
        P.b_block_householder_qr([np.ones((12, 8)), np.ones((12, 8))], ip)   # sum k_i > n
    q = P.b_householder_qr(np.zeros((12, 0)), u, ip)
    assert q.q.shape == (12, 0) and q.r.shape == (0, 0)
