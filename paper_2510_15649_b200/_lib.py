"""ctypes binding of libladlasso_b200.so (the C ABI in include/ladlasso_b200.h).

There is no fallback: if the library is missing or fails to load, every entry
point raises.  The CUDA kernels are the only implementation of the solver.
"""

from __future__ import annotations

import ctypes as C
import os

from . import _build

SYMBOLS = (
    "lad_version",
    "lad_last_error",
    "lad_kernel_launches",
    "lad_copy_h2d",
    "lad_default_params",
    "lad_set_kernel_policy",
    "lad_set_axis_parallel",
    "lad_locus_solve_f64",
    "lad_locus_solve_host_f64",
    "lad_ccd_descend_f64",
    "lad_brute_solve_f64",
    "lad_fp64_peak_tflops",
    "lad_objective_f64",
    "lad_generate_f64",
    "lad_subsets_f64",
    "lad_locus_solve_f32",
    "lad_locus_solve_host_f32",
    "lad_ccd_descend_f32",
    "lad_fp32_peak_tflops",
    "lad_axiswise_minimum_f64",
    "lad_lp_solve_f64",
    "lad_locus_solve_bracketed_f64",
    "lad_locus_solve_bracketed_host_f64",
    "lad_genspec_generate_f64",
)

LAD_OK = 0
LAD_E_INVALID = -1
LAD_E_TOO_LARGE = -2
LAD_E_CUDA = -3
LAD_E_UNSUPPORTED = -4
STATUS_SCRATCH = 3  # per-problem: the evaluator's curve-point list outgrew prm.seen_capacity

KERNEL_AUTO = 0
KERNEL_THREAD = 1
KERNEL_WARP = 2


def set_kernel_policy(policy: int) -> None:
    """Choose the locus kernel mapping (auto / thread-per-problem / warp-per-problem)."""
    rc = load().lad_set_kernel_policy(policy)
    if rc != LAD_OK:
        raise ValueError(last_error())


def set_axis_parallel(enable) -> None:
    """Axis-parallel mode of the warp kernel (bit-identical results): False/0 off,
    True/1 for batches smaller than the resident warps (default), 2 for every batch."""
    load().lad_set_axis_parallel(int(enable))


class LocusParams(C.Structure):
    _fields_ = [
        ("outer_axis", C.c_int32),
        ("outer_search", C.c_int32),
        ("outer_tolerance", C.c_double),
        ("outer_probes", C.c_int32),
        ("outer_max_iterations", C.c_int32),
        ("has_bracket", C.c_int32),
        ("bracket_lo", C.c_double),
        ("bracket_hi", C.c_double),
        ("inner_sweep_tol", C.c_double),
        ("inner_max_sweeps", C.c_int32),
        ("lambda_floor", C.c_double),
        ("seen_capacity", C.c_int32),
    ]


class LocusOut(C.Structure):
    _fields_ = [
        ("beta", C.c_void_p),
        ("objective", C.c_void_p),
        ("iterations", C.c_void_p),
        ("objective_evals", C.c_void_p),
        ("converged", C.c_void_p),
        ("status", C.c_void_p),
        ("descents", C.c_void_p),
        ("steps", C.c_void_p),
    ]


_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = False):
    """Load the shared library (optionally building it first)."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    if not os.path.exists(path):
        if not build_if_missing:
            raise RuntimeError(
                f"{path} is missing: build it with `python -m paper_2510_15649_b200._build` "
                "(there is no CPU fallback)")
        _build.build()
    L = C.CDLL(path)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    L.lad_version.restype = C.c_int
    L.lad_last_error.restype = C.c_char_p
    L.lad_default_params.argtypes = [C.POINTER(LocusParams)]
    L.lad_default_params.restype = None
    L.lad_set_kernel_policy.argtypes = [i32]
    L.lad_set_axis_parallel.argtypes = [i32]
    L.lad_locus_solve_f64.argtypes = [vp, vp, vp, vp, i64, i64, i32, i32, C.POINTER(LocusParams), C.POINTER(LocusOut),
                                      vp]
    L.lad_locus_solve_host_f64.argtypes = [vp, vp, vp, vp, i64, i64, i32, i32, C.POINTER(LocusParams),
                                           C.POINTER(LocusOut), vp]
    L.lad_locus_solve_bracketed_f64.argtypes = [vp, vp, vp, vp, i64, i64, i32, i32, vp, C.POINTER(LocusParams),
                                                C.POINTER(LocusOut), vp]
    L.lad_locus_solve_bracketed_host_f64.argtypes = L.lad_locus_solve_bracketed_f64.argtypes
    L.lad_genspec_generate_f64.argtypes = [i64, i32, i32, i32, vp, dbl, dbl, dbl, vp, vp, vp, vp, vp]
    L.lad_fp64_peak_tflops.argtypes = [C.POINTER(C.c_double), vp]
    L.lad_fp32_peak_tflops.argtypes = [C.POINTER(C.c_double), vp]
    L.lad_locus_solve_f32.argtypes = L.lad_locus_solve_f64.argtypes
    L.lad_locus_solve_host_f32.argtypes = L.lad_locus_solve_host_f64.argtypes
    L.lad_ccd_descend_f64.argtypes = [vp, vp, vp, i64, i32, i32, vp, vp, dbl, i32, dbl, C.POINTER(LocusOut), vp]
    L.lad_ccd_descend_f32.argtypes = L.lad_ccd_descend_f64.argtypes
    L.lad_brute_solve_f64.argtypes = [vp, vp, vp, i64, i32, i32, i32, i64, dbl, vp, vp, vp, vp]
    L.lad_objective_f64.argtypes = [vp, vp, vp, i64, i32, i32, vp, dbl, vp, vp]
    L.lad_axiswise_minimum_f64.argtypes = [vp, vp, vp, i64, i32, i32, vp, vp, dbl, dbl, vp, vp]
    L.lad_lp_solve_f64.argtypes = [vp, vp, vp, i64, i32, i32, i32, i32, dbl, dbl, vp, vp, vp, vp, vp, vp, vp, vp,
                                   i32, vp]
    L.lad_generate_f64.argtypes = [i32, C.c_uint64, i64, i64, i32, i32, vp, vp, vp, vp, vp]
    L.lad_subsets_f64.argtypes = [vp, vp, i32, i32, i32, i64, i64, vp, vp, vp]
    L.lad_copy_h2d.argtypes = [vp, vp, C.c_size_t, vp]
    L.lad_kernel_launches.restype = C.c_longlong
    for name in SYMBOLS:
        if name not in ("lad_version", "lad_last_error", "lad_kernel_launches", "lad_default_params"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def kernel_launches() -> int:
    """Kernels launched by the library so far (the bench's gpu_launches evidence)."""
    return int(load().lad_kernel_launches())


def last_error() -> str:
    return load().lad_last_error().decode(errors="replace")
