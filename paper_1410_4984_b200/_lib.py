"""ctypes binding of include/sgpx.h (libsgpx.so, built in-tree for sm_100a).

Loading fails loudly when the shared library is missing: there is no
Python / CPU fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG_DIR)
# SGPX_LIB: alternative in-tree build (A/B timing experiments)
LIB_PATH = os.path.join(PKG_DIR, os.environ.get("SGPX_LIB", "libsgpx.so"))
HEADER_PATH = os.path.join(ROOT, "include", "sgpx.h")

SGPX_OK, SGPX_INVALID_ARGUMENT, SGPX_NUMERIC, SGPX_CUDA, SGPX_NCCL, SGPX_INTERNAL, SGPX_IO = range(7)
SGPX_PREC_AUTO, SGPX_PREC_FAST, SGPX_PREC_PRECISE, SGPX_PREC_DIRECT, SGPX_PREC_SYRK = 0, 2, 3, 4, 5
PRECISION_NAMES = {SGPX_PREC_AUTO: "auto", SGPX_PREC_FAST: "fast", SGPX_PREC_PRECISE: "precise",
                   SGPX_PREC_DIRECT: "direct", SGPX_PREC_SYRK: "syrk"}


class cmat(C.Structure):
    _fields_ = [("data", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64)]


mmat = cmat  # same layout, mutable data


class kernel_spec(C.Structure):
    _fields_ = [("variance", C.c_double), ("lengthscales", C.c_void_p), ("q", C.c_int64)]


class tile_config(C.Structure):
    _fields_ = [("block_span", C.c_int64), ("thread_span", C.c_int64)]


class stats_adjoints(C.Structure):
    _fields_ = [("d_phi", C.c_double), ("d_psi_y", cmat), ("d_phi_big", cmat)]


class sufficient_stats(C.Structure):
    _fields_ = [("phi", C.c_double), ("psi_y", mmat), ("phi_big", mmat), ("yy", C.c_double), ("n_count", C.c_int64)]


class stats_grads(C.Structure):
    _fields_ = [("d_mu", mmat), ("d_s", mmat), ("d_z", mmat), ("d_variance", C.c_double),
                ("d_lengthscales", C.c_void_p)]


class bound_breakdown(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("total", "log_det_term", "data_fit_term", "quadratic_term",
                                          "trace_phi_term", "trace_kmm_term", "kl_term")]


class engine_config(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_global", C.c_int64), ("row_begin", C.c_int64), ("n_local", C.c_int64),
                ("q", C.c_int64), ("d", C.c_int64), ("m", C.c_int64), ("jitter_factor", C.c_double),
                ("precision", C.c_int)]


class eval_result(C.Structure):
    _fields_ = [("bound", bound_breakdown), ("phi", C.c_double), ("yy", C.c_double), ("n_count", C.c_int64),
                ("psi_y", C.c_void_p), ("phi_big", C.c_void_p), ("has_grads", C.c_int), ("d_z", C.c_void_p),
                ("d_lengthscales", C.c_void_p), ("d_variance", C.c_double), ("d_beta", C.c_double),
                ("jitter_factor_used", C.c_double), ("stats_pass_s", C.c_double), ("coordinator_s", C.c_double),
                ("grad_pass_s", C.c_double), ("wall_s", C.c_double), ("fwd_kernel_s", C.c_double),
                ("bwd_kernel_s", C.c_double), ("fwd_grid", C.c_int), ("bwd_grid", C.c_int),
                ("precision_used", C.c_int), ("z_spread", C.c_double), ("psi2_fwd_kernel_s", C.c_double),
                ("psi2_bwd_kernel_s", C.c_double)]


class lbfgs_options(C.Structure):
    _fields_ = [("memory", C.c_int), ("c1", C.c_double), ("c2", C.c_double), ("g_tol", C.c_double),
                ("f_tol", C.c_double), ("max_iters", C.c_int), ("max_evals", C.c_int), ("max_line_search", C.c_int)]


FIT_STATUS = {-1: "running", 0: "gradient_converged", 1: "value_converged", 2: "max_iterations",
              3: "max_evaluations", 4: "line_search_failed"}

# name -> (restype, argtypes)
SIGNATURES = {
    "sgpx_last_error": (C.c_char_p, []),
    "sgpx_abi_version": (C.c_int, []),
    "sgpx_device_count": (C.c_int, []),
    "sgpx_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "sgpx_ctx_destroy": (C.c_int, [C.c_void_p]),
    "sgpx_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sgpx_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "sgpx_ctx_launch_count": (C.c_int64, [C.c_void_p]),
    "sgpx_ctx_set_precision": (C.c_int, [C.c_void_p, C.c_int]),
    "sgpx_ctx_last_precision": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "sgpx_sweep_stats": (C.c_int, [C.c_void_p, C.c_int, cmat, cmat, cmat, cmat, C.POINTER(kernel_spec),
                                   C.POINTER(tile_config), C.POINTER(stats_adjoints), C.POINTER(sufficient_stats),
                                   C.POINTER(stats_grads)]),
    "sgpx_psi1_expected": (C.c_int, [C.c_void_p, cmat, cmat, cmat, C.POINTER(kernel_spec), mmat]),
    "sgpx_psi0_expected": (C.c_int, [cmat, cmat, C.POINTER(kernel_spec), C.POINTER(C.c_double)]),
    "sgpx_packed_stats_count": (C.c_int64, [C.c_int64, C.c_int64]),
    "sgpx_packed_grads_count": (C.c_int64, [C.c_int64, C.c_int64]),
    "sgpx_coordinate_host": (C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, cmat,
                                       C.POINTER(kernel_spec), C.c_double, C.c_double, C.POINTER(bound_breakdown),
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sgpx_finish_host": (C.c_int, [C.c_int64, C.c_int64, C.c_void_p, cmat, C.POINTER(kernel_spec), C.c_void_p,
                                   C.c_double, C.c_void_p, C.POINTER(C.c_double), C.c_void_p]),
    "sgpx_engine_create": (C.c_int, [C.c_void_p, C.POINTER(engine_config), C.POINTER(C.c_void_p)]),
    "sgpx_engine_destroy": (C.c_int, [C.c_void_p]),
    "sgpx_engine_set_data": (C.c_int, [C.c_void_p, cmat, cmat, cmat, C.c_int]),
    "sgpx_engine_broadcast": (C.c_int, [C.c_void_p, C.POINTER(kernel_spec), C.c_double, cmat, cmat, cmat, C.c_int]),
    "sgpx_engine_evaluate": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(eval_result)]),
    "sgpx_engine_stats_pass": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "sgpx_engine_coordinate": (C.c_int, [C.c_void_p, C.c_int]),
    "sgpx_engine_grad_pass": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "sgpx_engine_finish": (C.c_int, [C.c_void_p, C.POINTER(eval_result)]),
    "sgpx_engine_local_grads_device": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "sgpx_engine_copy_local_grads": (C.c_int, [C.c_void_p, mmat, mmat]),
    "sgpx_engine_set_local_grads_out": (C.c_int, [C.c_void_p, mmat, mmat]),
    "sgpx_engine_predict": (C.c_int, [C.c_void_p, cmat, C.c_int, mmat, mmat, C.POINTER(C.c_double)]),
    "sgpx_multi_create": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(engine_config), C.POINTER(C.c_void_p)]),
    "sgpx_multi_destroy": (C.c_int, [C.c_void_p]),
    "sgpx_multi_workers": (C.c_int, [C.c_void_p]),
    "sgpx_multi_set_data": (C.c_int, [C.c_void_p, cmat, cmat, cmat]),
    "sgpx_multi_broadcast": (C.c_int, [C.c_void_p, C.POINTER(kernel_spec), C.c_double, cmat, cmat, cmat]),
    "sgpx_multi_evaluate": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(eval_result), mmat, mmat]),
    "sgpx_lbfgs_default_options": (None, [C.POINTER(lbfgs_options)]),
    "sgpx_fit_create": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(kernel_spec), C.c_double, cmat, cmat, cmat,
                                  C.POINTER(lbfgs_options), C.POINTER(C.c_void_p)]),
    "sgpx_fit_step": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    "sgpx_fit_state": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int),
                                 C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sgpx_fit_message": (C.c_char_p, [C.c_void_p]),
    "sgpx_fit_last_error": (C.c_char_p, []),
    "sgpx_fit_params": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_double), mmat, mmat,
                                  mmat]),
    "sgpx_fit_destroy": (C.c_int, [C.c_void_p]),
    "sgpx_rng_normal_matrix": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int64, C.c_int64, mmat, C.c_int]),
    "sgpx_rng_choose_rows": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.c_void_p]),
    "sgpx_io_matrix_shape": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "sgpx_io_read_matrix": (C.c_int, [C.c_char_p, mmat]),
    "sgpx_io_write_matrix": (C.c_int, [C.c_char_p, cmat]),
    "sgpx_io_load_matrix_device": (C.c_int, [C.c_void_p, C.c_char_p, mmat]),
}

_lib = None


def load():
    """Load libsgpx.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (or python "
                          f"paper_1410_4984_b200/build.py); the B200 engine has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class SgpxError(RuntimeError):
    code = SGPX_INTERNAL


class SgpxInvalidArgument(SgpxError, ValueError):
    """std::invalid_argument of the reference (common.hpp:24-26)."""
    code = SGPX_INVALID_ARGUMENT


class SgpxNumericError(SgpxError, ArithmeticError):
    """sgp::NumericError (common.hpp:20-22)."""
    code = SGPX_NUMERIC


class SgpxCudaError(SgpxError):
    code = SGPX_CUDA


class SgpxNcclError(SgpxError):
    code = SGPX_NCCL


class SgpxIoError(SgpxError, OSError):
    """std::runtime_error of the reference's io.hpp."""
    code = SGPX_IO


_ERRORS = {SGPX_INVALID_ARGUMENT: SgpxInvalidArgument, SGPX_NUMERIC: SgpxNumericError, SGPX_CUDA: SgpxCudaError,
           SGPX_IO: SgpxIoError, SGPX_NCCL: SgpxNcclError}


def check(rc: int):
    if rc == SGPX_OK:
        return
    msg = load().sgpx_last_error().decode(errors="replace")
    raise _ERRORS.get(rc, SgpxError)(msg)
