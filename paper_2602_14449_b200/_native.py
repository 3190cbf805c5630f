"""ctypes binding of the C-ABI in include/ots.h (libots.so, built in-tree by
`make` / __graft_entry__.build()).  No CPU fallback: if the library or a CUDA
device is missing every call raises NativeUnavailable."""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OTS_LIB") or os.path.join(_HERE, "libots.so")

CHOICES = {"mlu": 0, "qr": 1, "polar": 2, "explicit": 3}
INTRA = {"householder": 0, "cholshift": 1}

_CODE_TO_EXC = {
    -1: E.DimensionError, -2: E.NotHermitian, -3: E.NotPositiveDefinite,
    -4: E.ConvergenceError, -5: E.SingularError, -6: E.NormBoundError,
    -7: E.SingularTError, -8: E.OrthonormalityError, -9: E.IntraFailure,
    -10: E.BreakdownError, -12: E.ParameterError, -20: ValueError,
}

_lib = None
_lock = threading.Lock()
_ctx = {}

_vp, _i64, _int, _dbl = C.c_void_p, C.c_int64, C.c_int, C.c_double


def lib():
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise E.NativeUnavailable(
                        f"{LIB_PATH} not built; run `make` (or __graft_entry__.build())")
                L = C.CDLL(LIB_PATH)
                L.ots_ctx_create.argtypes = [_int, C.POINTER(_vp)]
                L.ots_ctx_destroy.argtypes = [_vp]
                L.ots_last_error.argtypes = [_vp]
                L.ots_last_error.restype = C.c_char_p
                L.ots_sm_count.argtypes = [_vp]
                L.ots_last_fast.argtypes = [_vp]
                L.ots_version.restype = _int
                L.ots_set_profiling.argtypes = [_vp, _int]
                L.ots_last_launch_count.argtypes = [_vp]
                L.ots_fp64_peak.argtypes = [_vp, C.POINTER(_dbl)]
                L.ots_last_profile.argtypes = [_vp, C.c_char_p, _int, C.POINTER(C.c_float), _int]
                L.ots_two_stage_f64.argtypes = [
                    _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _int, _int, _vp, _i64,
                    _dbl, _int, _vp, _i64, _vp, _i64, _vp, _i64, C.POINTER(_dbl), _vp]
                L.ots_b_two_stage_diag_f64.argtypes = [
                    _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _int, _vp, _i64, _dbl,
                    _vp, _i64, _vp, _i64, _vp, _i64, C.POINTER(_dbl), _vp]
                L.ots_dense_cholesky_f64.argtypes = [_vp, _i64, _vp, _i64, _vp, _i64, _vp]
                L.ots_dense_trsm_lt_f64.argtypes = [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp]
                L.ots_dense_trmm_lt_f64.argtypes = [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp]
                L.ots_b_two_stage_dense_f64.argtypes = [
                    _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int, _vp, _i64, _dbl,
                    _vp, _i64, _vp, _i64, _vp, _i64, C.POINTER(_dbl), _vp]
                L.ots_build_reflector_f64.argtypes = [
                    _vp, _i64, _i64, _vp, _i64, _int, _vp, _i64, _dbl, _int, C.POINTER(_vp),
                    C.POINTER(_dbl), _vp]
                L.ots_reflector_destroy.argtypes = [_vp]
                L.ots_apply_reflector_f64.argtypes = [_vp, _vp, _i64, _vp, _i64, _vp, _i64, _int, _vp]
                L.ots_reflector_diagnostics_f64.argtypes = [_vp, _vp, C.POINTER(_dbl), _vp]
                L.ots_reflector_tsolve_f64.argtypes = [_vp, _vp, _i64, _vp, _i64, _int, _vp]
                L.ots_reflector_get_f64.argtypes = [_vp, _vp, _int, _vp, _i64, _vp]
                L.ots_householder_qr_f64.argtypes = [
                    _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int, _vp]
                L.ots_two_stage_c128.argtypes = L.ots_two_stage_f64.argtypes
                L.ots_householder_qr_c128.argtypes = L.ots_householder_qr_f64.argtypes
                L.ots_b_two_stage_diag_c128.argtypes = L.ots_b_two_stage_diag_f64.argtypes
                L.ots_stability_f64.argtypes = [
                    _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int,
                    _vp, _i64, C.POINTER(_dbl), _vp]
                L.ots_stability_c128.argtypes = L.ots_stability_f64.argtypes
                L.ots_orthonormality_defect_f64.argtypes = [_vp, _i64, _i64, _vp, _i64, C.POINTER(_dbl), _vp]
                L.ots_orthonormality_defect_c128.argtypes = L.ots_orthonormality_defect_f64.argtypes
                L.ots_shifted_cholesky_qr_ex_f64.argtypes = [
                    _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int, _vp]
                L.ots_shifted_cholesky_qr_ex_c128.argtypes = L.ots_shifted_cholesky_qr_ex_f64.argtypes
                L.ots_gram_f64.argtypes = [_vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp]
                L.ots_gram_c128.argtypes = L.ots_gram_f64.argtypes
                L.ots_update_f64.argtypes = [_vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64,
                                             _vp]
                L.ots_update_c128.argtypes = L.ots_update_f64.argtypes
                L.ots_gram_extremes_f64.argtypes = L.ots_orthonormality_defect_f64.argtypes
                L.ots_gram_extremes_c128.argtypes = L.ots_orthonormality_defect_f64.argtypes
                L.ots_qr_signs_f64.argtypes = [_vp, _i64, _vp, _i64, _vp, _vp]
                L.ots_qr_signs_c128.argtypes = L.ots_qr_signs_f64.argtypes
                L.ots_build_reflector_c128.argtypes = L.ots_build_reflector_f64.argtypes
                L.ots_zreflector_destroy.argtypes = [_vp]
                L.ots_apply_reflector_c128.argtypes = L.ots_apply_reflector_f64.argtypes
                L.ots_reflector_diagnostics_c128.argtypes = L.ots_reflector_diagnostics_f64.argtypes
                L.ots_reflector_tsolve_c128.argtypes = L.ots_reflector_tsolve_f64.argtypes
                L.ots_reflector_get_c128.argtypes = L.ots_reflector_get_f64.argtypes
                L.ots_two_stage_gram_f64.argtypes = [
                    _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _int, _int, _vp, _i64,
                    _dbl, _int, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, C.POINTER(_dbl), _vp]
                L.ots_debug_counters.argtypes = [C.POINTER(C.c_ulonglong), _int]
                L.ots_modified_lu_f64.argtypes = [_vp, _i64, _vp, _i64, _vp, _vp, _vp]
                L.ots_shifted_cholesky_qr_f64.argtypes = [
                    _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp]
                L.ots_dist_begin.argtypes = [
                    _vp, _i64, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int, _vp,
                    _i64, _dbl, _vp]
                L.ots_dist_sizes.argtypes = [_vp, C.POINTER(_i64)]
                L.ots_dist_gram.argtypes = [_vp, _vp]
                L.ots_dist_top_rows.argtypes = [_vp, _vp]
                L.ots_dist_seed.argtypes = [_vp, _vp, _vp]
                L.ots_dist_seed_early.argtypes = [_vp, _vp]
                L.ots_dist_factor.argtypes = [_vp, _vp]
                L.ots_dist_tree.argtypes = [_vp, _vp, _int, _int]
                L.ots_dist_qform.argtypes = [_vp, _vp, _vp]
                L.ots_dist_finish.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _i64, C.POINTER(_dbl)]
                # complex variants share their real twins' signatures (set above)
                L.ots_shifted_cholesky_qr_c128.argtypes = L.ots_shifted_cholesky_qr_f64.argtypes
                L.ots_modified_lu_c128.argtypes = L.ots_modified_lu_f64.argtypes
                for fn in EXPORTED_SYMBOLS:
                    if fn.startswith("ots_") and getattr(L, fn).argtypes is None and fn not in _NO_ARGS:
                        raise E.NativeUnavailable(f"{fn}: argtypes not declared")
                _lib = L
    return _lib


_NO_ARGS = {"ots_version"}

EXPORTED_SYMBOLS = [
    "ots_ctx_create", "ots_ctx_destroy", "ots_last_error", "ots_sm_count", "ots_last_fast", "ots_version",
    "ots_two_stage_f64", "ots_householder_qr_f64", "ots_modified_lu_f64",
    "ots_two_stage_c128", "ots_householder_qr_c128", "ots_b_two_stage_diag_c128", "ots_stability_f64",
    "ots_shifted_cholesky_qr_c128", "ots_modified_lu_c128",
    "ots_shifted_cholesky_qr_f64", "ots_b_two_stage_diag_f64",
    "ots_build_reflector_f64", "ots_reflector_destroy", "ots_apply_reflector_f64",
    "ots_reflector_diagnostics_f64", "ots_reflector_tsolve_f64", "ots_reflector_get_f64",
    "ots_set_profiling", "ots_last_profile", "ots_last_launch_count", "ots_fp64_peak",
    "ots_debug_counters",
    "ots_dist_begin", "ots_dist_sizes", "ots_dist_gram", "ots_dist_seed", "ots_dist_seed_early", "ots_dist_top_rows", "ots_dist_factor",
    "ots_dist_tree", "ots_dist_qform", "ots_dist_finish",
    "ots_stability_c128", "ots_orthonormality_defect_f64", "ots_orthonormality_defect_c128",
    "ots_shifted_cholesky_qr_ex_f64", "ots_shifted_cholesky_qr_ex_c128",
    "ots_gram_f64", "ots_gram_c128", "ots_update_f64", "ots_update_c128",
    "ots_gram_extremes_f64", "ots_gram_extremes_c128", "ots_qr_signs_f64", "ots_qr_signs_c128",
    "ots_build_reflector_c128", "ots_zreflector_destroy", "ots_apply_reflector_c128",
    "ots_reflector_diagnostics_c128", "ots_reflector_tsolve_c128", "ots_reflector_get_c128",
    "ots_two_stage_gram_f64",
    "ots_dense_cholesky_f64", "ots_dense_trsm_lt_f64", "ots_dense_trmm_lt_f64", "ots_b_two_stage_dense_f64",
]


def context(device):
    """C context of (device, calling thread), created lazily.  ots.h: one
    context per (device, host thread) -- ctypes releases the GIL during a
    call, so two threads must never share a context's workspace.  Contexts of
    threads that have exited are destroyed when a new one is created."""
    key = (int(device), threading.get_ident())
    h = _ctx.get(key)
    if h is None:
        L = lib()
        with _lock:
            alive = {t.ident for t in threading.enumerate()}
            for dead in [kk for kk in _ctx if kk[1] not in alive]:
                L.ots_ctx_destroy(_ctx.pop(dead))
        h = _vp()
        rc = L.ots_ctx_create(int(device), C.byref(h))
        if rc != 0:
            msg = L.ots_last_error(h).decode() if h.value else "ots_ctx_create failed"
            raise E.NativeUnavailable(f"CUDA context on device {device}: {msg}")
        with _lock:
            _ctx[key] = h
    return h


def new_context(device):
    """A fresh, uncached C context (e.g. one per simulated rank)."""
    L = lib()
    h = _vp()
    rc = L.ots_ctx_create(int(device), C.byref(h))
    if rc != 0:
        raise E.NativeUnavailable(f"CUDA context on device {device}")
    return h


def check(rc, ctx, block=None):
    if rc == 0:
        return
    msg = lib().ots_last_error(ctx).decode()
    exc = _CODE_TO_EXC.get(rc)
    if exc is E.IntraFailure:
        raise E.IntraFailure(msg, block)
    if exc is None:
        if rc == -31:
            raise NotImplementedError(msg)
        raise RuntimeError(f"libots error {rc}: {msg}")
    raise exc(msg)


def last_fast(ctx):
    """1 when the last two_stage call on ctx took the direct-Q pipeline
    (csrc/fastpath.cu), 0 when it took the materialised-X pipeline."""
    return int(lib().ots_last_fast(ctx))


def profile(ctx):
    """[(phase, ms)] of the last call (when profiling is enabled)."""
    L = lib()
    buf = C.create_string_buffer(4096)
    ms = (C.c_float * 64)()
    n = L.ots_last_profile(ctx, buf, 4096, ms, 64)
    names = buf.value.decode().split("\n")
    return [(names[i], float(ms[i])) for i in range(n)]
