"""ctypes binding of the C ABI declared in include/kronprec_b200.h.

The shared library is built in-tree by ``paper_2311_15393_b200.build`` and
loaded from ``paper_2311_15393_b200/_lib``. There is no fallback: if the
library is missing every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libkronprec_b200.so")

KP_OK = 0
KP_ERR_INVALID_ARGUMENT = 1
KP_ERR_RUNTIME = 2
KP_ERR_NO_ROOT = 3
KP_ERR_CUDA = 4
KP_ERR_UNSUPPORTED = 5

KP_ACCUM_REFERENCE = 0
KP_ACCUM_TENSOR = 1

KP_FP16_PRODUCTS_AUTO = 0
KP_FP16_PRODUCTS_CUDA_CORES = 1
KP_FP16_PRODUCTS_TENSOR = 2

KP_OP_AUTO = 0
KP_OP_DENSE = 1
KP_OP_BANDED = 2


class kp_format(C.Structure):
    _fields_ = [("significand_bits", C.c_int), ("max_exponent", C.c_int),
                ("subnormals_enabled", C.c_int)]


class kp_solver_options(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("max_iterations", C.c_int),
                ("rel_residual_tol", C.c_double), ("x_true", C.c_void_p),
                ("track_search_direction_orthogonality", C.c_int),
                ("record_iterates", C.c_int), ("device_pointers", C.c_int)]


class kp_history(C.Structure):
    _fields_ = [("capacity", C.c_int), ("relative_error", C.c_void_p),
                ("residual_norm", C.c_void_p), ("work_units", C.c_void_p),
                ("residual_cosines", C.c_void_p), ("iterates", C.c_void_p),
                ("rows", C.c_int), ("n_cosines", C.c_int), ("iterations_used", C.c_int),
                ("converged", C.c_int), ("msolve_count", C.c_int),
                ("abort_reason", C.c_char * 192)]


class kp_param_choice(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("method", C.c_int), ("omega", C.c_double),
                ("eta", C.c_double), ("noise_norm", C.c_double),
                ("objective_value", C.c_double), ("bracket_lo", C.c_double),
                ("bracket_hi", C.c_double), ("flat_objective", C.c_int),
                ("grid_index", C.c_int)]


# every symbol the public header declares (checked by tests/test_abi.py)
EXPORTS = [
    "kp_last_error", "kp_init", "kp_synchronize", "kp_device_alloc", "kp_device_free",
    "kp_memcpy_h2d", "kp_memcpy_d2h", "kp_profile_enable", "kp_profile_read",
    "kp_profile_reset", "kp_launch_count", "kp_drive_stats", "kp_operator_create", "kp_operator_destroy",
    "kp_operator_info", "kp_kronsum_apply", "kp_kronsum_apply_transpose", "kp_normal_matvec",
    "kp_precond_build", "kp_precond_build_from_svd", "kp_precond_with_lambda",
    "kp_precond_destroy", "kp_precond_solve", "kp_precond_export", "kp_precond_info",
    "kp_cgls", "kp_pcg", "kp_fpcg", "kp_spectral_create", "kp_spectral_destroy",
    "kp_spectral_export", "kp_gcv_objective", "kp_discrepancy_gap", "kp_gcv_grid", "kp_gcv",
    "kp_discrepancy", "kp_operator_set_mode", "kp_operator_get_mode", "kp_event_record", "kp_event_elapsed", "kp_host_alloc", "kp_host_free",
    "kp_spectral_create_x", "kp_spectral_export_xhat", "kp_opt_objective", "kp_wgcv_objective",
    "kp_lambda_opt", "kp_wgcv", "kp_filtered_solution", "kp_round_array", "kp_lp_matmul",
    "kp_lp_matmul_ex", "kp_set_fp16_products", "kp_get_fp16_products", "kp_psf_to_kronsum",
    "kp_nearest_kron", "kp_pcg_batch", "kp_fpcg_batch", "kp_svd", "kp_set_svd_backend",
    "kp_get_svd_backend", "kp_discrepancy_batch", "kp_generate_test_problems", "kp_rng_raw",
    "kp_round_value", "kp_round_call_count", "kp_discrepancy_batch_ex",
]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with paper_2311_15393_b200.build "
                "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, D, I, V = C.c_void_p, C.c_double, C.c_int, C.c_void_p
        sig = {
            "kp_last_error": ([], C.c_char_p),
            "kp_init": ([I], I), "kp_synchronize": ([], I),
            "kp_device_alloc": ([C.c_size_t, C.POINTER(C.c_void_p)], I),
            "kp_device_free": ([P], I),
            "kp_memcpy_h2d": ([P, P, C.c_size_t], I), "kp_memcpy_d2h": ([P, P, C.c_size_t], I),
            "kp_profile_enable": ([I], I),
            "kp_profile_read": ([I, C.POINTER(D), C.POINTER(C.c_longlong)], I),
            "kp_profile_reset": ([], I), "kp_launch_count": ([], C.c_longlong),
            "kp_drive_stats": ([C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)], I),
            "kp_operator_create": ([I, I, P, P, C.POINTER(V)], I),
            "kp_operator_destroy": ([P], I),
            "kp_operator_info": ([P, C.POINTER(I), C.POINTER(I)], I),
            "kp_kronsum_apply": ([P, P, P], I), "kp_kronsum_apply_transpose": ([P, P, P], I),
            "kp_normal_matvec": ([P, D, P, P], I),
            "kp_precond_build": ([P, P, I, D, kp_format, I, C.POINTER(V)], I),
            "kp_precond_build_from_svd": ([I, P, P, P, P, P, P, D, kp_format, I, C.POINTER(V)], I),
            "kp_precond_with_lambda": ([P, D, C.POINTER(V)], I),
            "kp_precond_destroy": ([P], I), "kp_precond_solve": ([P, P, P], I),
            "kp_precond_export": ([P, I, P], I),
            "kp_precond_info": ([P, C.POINTER(I), C.POINTER(D), C.POINTER(kp_format),
                                 C.POINTER(I)], I),
            "kp_cgls": ([P, P, C.POINTER(kp_solver_options), P, C.POINTER(kp_history)], I),
            "kp_pcg": ([P, P, P, C.POINTER(kp_solver_options), P, C.POINTER(kp_history)], I),
            "kp_fpcg": ([P, P, P, C.POINTER(kp_solver_options), P, C.POINTER(kp_history)], I),
            "kp_svd": ([P, I, I, P, P, P], I), "kp_set_svd_backend": ([I], I),
            "kp_get_svd_backend": ([C.POINTER(I)], I),
            "kp_discrepancy_batch": ([P, I, P, P, D, P, P], I),
            "kp_discrepancy_batch_ex": ([P, I, P, P, D, P, P, I], I),
            "kp_generate_test_problems": ([P, I, P, I, P, P, P, P, P, P, I], I),
            "kp_rng_raw": ([P, I, C.c_long, P], I),
            "kp_pcg_batch": ([P, P, I, P, P, C.POINTER(kp_solver_options), P, C.POINTER(kp_history)], I),
            "kp_fpcg_batch": ([P, P, I, P, P, C.POINTER(kp_solver_options), P, C.POINTER(kp_history)], I),
            "kp_spectral_create": ([P, P, C.POINTER(V)], I),
            "kp_spectral_destroy": ([P], I), "kp_spectral_export": ([P, P, P], I),
            "kp_gcv_objective": ([P, D, C.POINTER(D)], I),
            "kp_discrepancy_gap": ([P, D, D, C.POINTER(D)], I),
            "kp_gcv_grid": ([P, P, I, P, C.POINTER(kp_param_choice)], I),
            "kp_gcv": ([P, C.POINTER(kp_param_choice)], I),
            "kp_spectral_create_x": ([P, P, P, C.POINTER(V)], I),
            "kp_spectral_export_xhat": ([P, P], I),
            "kp_opt_objective": ([P, D, C.POINTER(D)], I),
            "kp_wgcv_objective": ([P, D, D, C.POINTER(D)], I),
            "kp_lambda_opt": ([P, C.POINTER(kp_param_choice)], I),
            "kp_wgcv": ([P, D, C.POINTER(kp_param_choice)], I),
            "kp_filtered_solution": ([P, P, D, P], I),
            "kp_round_array": ([P, C.c_long, kp_format, P], I),
            "kp_round_value": ([D, kp_format, C.POINTER(D)], I),
            "kp_round_call_count": ([C.POINTER(C.c_ulonglong)], I),
            "kp_lp_matmul": ([I, I, I, P, P, kp_format, P], I),
            "kp_lp_matmul_ex": ([I, I, I, P, P, kp_format, I, P], I),
            "kp_discrepancy": ([P, D, D, C.POINTER(kp_param_choice)], I),
            "kp_event_record": ([I], I),
            "kp_operator_set_mode": ([P, I], I),
            "kp_operator_get_mode": ([P, C.POINTER(I), C.POINTER(I), C.POINTER(I)], I),
            "kp_event_elapsed": ([I, I, C.POINTER(C.c_float)], I),
            "kp_host_alloc": ([C.c_size_t, C.POINTER(C.c_void_p)], I),
            "kp_host_free": ([P], I),
            "kp_set_fp16_products": ([I], I),
            "kp_psf_to_kronsum": ([P, I, I, I, I, D, I, I, P, P, C.POINTER(I)], I),
            "kp_nearest_kron": ([P, I, I, I, I, I, P, P], I),
            "kp_get_fp16_products": ([I, C.POINTER(I)], I),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        # host-side problem generation (csrc/problem.cpp)
        U64, L64 = C.c_uint64, C.c_long
        gen = {
            "kpg_last_error": ([], C.c_char_p),
            "kpg_rng_normals": ([U64, L64, P], None),
            "kpg_rng_uniforms": ([U64, L64, D, D, P], None),
            "kpg_make_psf": ([I, I, D, D, I, I, I, D, U64, P], I),
            "kpg_psf_aniso_gaussian": ([I, D, D, D, P], I),
            "kpg_psf_gauss_motion": ([I, D, I, D, P], I),
            "kpg_default_test_image": ([I, P], I),
            "kpg_blob_image": ([I, U64, I, P], I),
            "kpg_psf_to_kronsum": ([P, I, I, I, I, D, I, I, P, P, C.POINTER(I), P], I),
            "kpg_nearest_kron": ([P, I, I, I, I, I, P, P], I),
            "kpg_kronsum_apply_host": ([I, I, P, P, P, P], I),
            "kpg_add_noise": ([L64, P, D, U64, P, P], I),
            "kpg_svd": ([P, I, I, P, P, P], I),
            "kpg_set_blas_threads": ([I], None),
        }
        for name, (args, res) in gen.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


class NoRootError(RuntimeError):
    """kronprec::NoRootError (regparam.hpp:51-53)."""


class CudaError(RuntimeError):
    """CUDA failure on the B200 path (there is no CPU fallback)."""


class UnsupportedError(NotImplementedError):
    """Option combination not implemented on the device path."""


def check(status: int) -> None:
    if status == KP_OK:
        return
    msg = lib().kp_last_error().decode()
    if status == KP_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == KP_ERR_NO_ROOT:
        raise NoRootError(msg)
    if status == KP_ERR_CUDA:
        raise CudaError(msg)
    if status == KP_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise RuntimeError(msg)


def ptr(a: np.ndarray | None) -> int | None:
    if a is None:
        return None
    assert a.flags["F_CONTIGUOUS"] or a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def f64(a, copy: bool = False) -> np.ndarray:
    """Column-major float64 view/copy (Eigen's storage order)."""
    return np.array(a, dtype=np.float64, order="F", copy=copy or None)
