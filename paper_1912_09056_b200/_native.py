"""ctypes binding of libcamg.so (include/camg.h).

The library is REQUIRED: importing a compute path without it raises
`NativeError` -- there is no CPU fallback of the solve path.  Status codes
are mapped onto the reference exception classes (errors.py:4-25).
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import (
    ConfigError,
    DimensionError,
    NativeError,
    SetupError,
    SingularMatrixError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
# CAMG_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("CAMG_LIB") or os.path.join(_HERE, "libcamg.so")

i64 = C.c_int64
i32 = C.c_int32
f64 = C.c_double
vp = C.c_void_p
P64 = C.POINTER(C.c_int64)


class SmootherCfg(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("alpha", f64), ("outer_sweeps", C.c_int), ("a_hat_mode", C.c_int),
        ("pred_kind", C.c_int), ("pred_sweeps", C.c_int), ("pred_damping", f64),
        ("corr_kind", C.c_int), ("corr_sweeps", C.c_int), ("corr_damping", f64),
        ("node_block", C.c_int),
    ]


# camg_apply_fn: int (*)(void* user, const double* x, double* y, void* stream)
APPLY_FN = C.CFUNCTYPE(C.c_int, vp, vp, vp, vp)


class LevelInfo(C.Structure):
    """camg_level_info: formats and execution paths of one level's smoother."""
    _fields_ = [
        ("n_u", i64), ("n_lam", i64), ("nnz", i64),
        ("sell_block", C.c_int), ("sell_masked", C.c_int), ("sell_lanes", C.c_int),
        ("sell_rows", i64), ("sell_slices", i64),
        ("overlap", C.c_int), ("overlap_indep_slices", i64), ("overlap_dep_slices", i64),
        ("pred_path", C.c_int), ("pred_colors", C.c_int), ("corr_path", C.c_int), ("corr_colors", C.c_int),
        ("transfer_block_rows", C.c_int), ("restrict_block_rows", C.c_int), ("watchdog", C.c_int),
        ("sell_shared_values", C.c_int), ("sell_value_groups", i64), ("sell_value_groups_full", i64),
    ]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["pred_path"] = PATHS[d["pred_path"]]
        d["corr_path"] = PATHS[d["corr_path"]]
        return d


# CAMG_PATH_* (include/camg.h)
PATHS = ("none", "fused", "dense_lu", "colour_csr", "colour_sell", "cta", "cluster", "inner_amg", "lex_trsv", "lam_fused", "dense_inv", "lam_engine")


_SIGS = {
    "camg_last_error": (C.c_char_p, []),
    "camg_version": (C.c_int, []),
    "camg_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "camg_launch_count": (i64, []),
    "camg_csr_from_host": (C.c_int, [i64, i64, i64, vp, vp, vp, C.POINTER(vp)]),
    "camg_csr_from_device": (C.c_int, [i64, i64, i64, vp, vp, vp, C.POINTER(vp)]),
    "camg_csr_alloc": (C.c_int, [i64, i64, i64, C.POINTER(vp)]),
    "camg_csr_destroy": (C.c_int, [vp]),
    "camg_csr_shape": (C.c_int, [vp, P64, P64, P64]),
    "camg_csr_to_host": (C.c_int, [vp, vp, vp, vp]),
    "camg_csr_saddle_merge": (C.c_int, [vp, vp, vp, vp, C.POINTER(vp)]),
    "camg_spmv": (C.c_int, [vp, f64, vp, f64, vp, vp]),
    "camg_transpose": (C.c_int, [vp, C.POINTER(vp)]),
    "camg_spgemm": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "camg_galerkin": (C.c_int, [vp, vp, vp, C.POINTER(vp)]),
    "camg_diagonal": (C.c_int, [vp, C.c_int, vp]),
    "camg_ilu0_factor": (C.c_int, [i64, vp, vp, vp]),
    "camg_csr_axpby": (C.c_int, [f64, vp, f64, vp, C.POINTER(vp)]),
    "camg_csr_scale_rows": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "camg_power_step": (C.c_int, [vp, vp, vp, vp, vp]),
    "camg_vec_scale_div": (C.c_int, [i64, vp, f64, vp, vp]),
    "camg_smooth_prolongator": (C.c_int, [vp, vp, vp, f64, C.POINTER(vp)]),
    "camg_lambda_max": (C.c_int, [vp, vp, C.c_int, C.POINTER(f64)]),
    "camg_schur": (C.c_int, [vp, vp, vp, vp, f64, C.POINTER(vp)]),
    "camg_node_graph": (C.c_int, [vp, vp, i64, vp, f64, C.POINTER(vp), P64]),
    "camg_pattern_to_host": (C.c_int, [vp, vp, vp]),
    "camg_free_host": (None, [vp]),
    "camg_aggregate_greedy": (C.c_int, [i64, vp, vp, i64, vp, P64, vp, P64]),
    "camg_aggregate_lagrange": (C.c_int, [vp, i64, vp, vp, vp, vp, vp, vp, i64, vp, P64, vp, P64]),
    "camg_tentative_csr": (C.c_int, [i64, i64, i64, vp, vp, i64, vp, i64, vp, vp, i64, C.POINTER(vp)]),
    "camg_assemble_stencil": (C.c_int, [C.c_int, vp, C.c_int, C.c_int, i64, i64, vp, vp, i64]),
    "camg_stencil_block_counts": (C.c_int, [C.c_int, vp, C.c_int, C.c_int, vp, P64]),
    "camg_level_create": (C.c_int, [vp, vp, vp, vp, C.POINTER(SmootherCfg), C.c_int, C.c_int, C.POINTER(vp)]),
    "camg_level_create_shared": (C.c_int, [vp, vp, vp, vp, vp, C.POINTER(SmootherCfg), C.c_int, C.c_int,
                                           C.POINTER(vp)]),
    "camg_level_destroy": (C.c_int, [vp]),
    "camg_csr_attach_blocks": (C.c_int, [vp, C.c_int, i64]),
    "camg_csr_attach_rect_blocks": (C.c_int, [vp, C.c_int, C.c_int, i64, i64]),
    "camg_csr_stream_bytes": (C.c_int, [vp, C.POINTER(f64)]),
    "camg_csr_value_groups": (C.c_int, [vp, C.POINTER(i64), C.POINTER(i64)]),
    "camg_csr_slot_stats": (C.c_int, [vp, vp]),
    "camg_csr_uniform_slices": (C.c_int, [vp, vp]),
    "camg_level_block_transfer": (C.c_int, [vp, C.c_int, C.c_int, i64]),
    "camg_level_fine_pass": (C.c_int, [vp, C.c_int, vp, vp, vp, C.POINTER(f64), C.POINTER(f64)]),
    "camg_level_schur": (C.c_int, [vp, C.POINTER(vp)]),
    "camg_level_operator": (C.c_int, [vp, C.POINTER(vp)]),
    "camg_level_set_corrector_lu": (C.c_int, [vp, i64, vp, vp]),
    "camg_level_set_k_lu": (C.c_int, [vp, i64, vp, vp]),
    "camg_level_set_schur": (C.c_int, [vp, vp]),
    "camg_point_create": (C.c_int, [vp, C.c_int, C.c_int, f64, C.POINTER(vp)]),
    "camg_point_set_lu": (C.c_int, [vp, i64, vp, vp]),
    "camg_point_smooth": (C.c_int, [vp, vp, vp, vp, vp]),
    "camg_point_destroy": (C.c_int, [vp]),
    "camg_level_set_transfer": (C.c_int, [vp, vp, vp]),
    "camg_level_sweep": (C.c_int, [vp, vp, vp, vp, vp]),
    "camg_hierarchy_create": (C.c_int, [C.POINTER(vp), C.c_int, C.c_int, C.POINTER(vp)]),
    "camg_hierarchy_set_coarse_lu": (C.c_int, [vp, i64, vp, vp]),
    "camg_hierarchy_set_coarse_inverse": (C.c_int, [vp, i64, vp]),
    "camg_hierarchy_coarse_solve": (C.c_int, [vp, vp, vp, vp]),
    "camg_hierarchy_coarse_factor": (C.c_int, [vp, C.c_int]),
    "camg_hierarchy_destroy": (C.c_int, [vp]),
    "camg_vcycle": (C.c_int, [vp, vp, vp, vp]),
    "camg_hierarchy_use_graph": (C.c_int, [vp, C.c_int]),
    "camg_scalar_hierarchy_create": (C.c_int, [C.c_int, vp, vp, vp, C.c_int, C.c_int, f64, C.POINTER(vp)]),
    "camg_scalar_hierarchy_set_coarse_lu": (C.c_int, [vp, i64, vp, vp]),
    "camg_scalar_hierarchy_apply": (C.c_int, [vp, vp, vp, vp]),
    "camg_scalar_hierarchy_destroy": (C.c_int, [vp]),
    "camg_level_set_predictor_solver": (C.c_int, [vp, vp]),
    "camg_hierarchy_vcycle_bytes": (C.c_int, [vp, C.POINTER(f64), C.POINTER(f64)]),
    "camg_gmres": (C.c_int, [vp, vp, vp, vp, f64, C.c_int, C.c_int, C.POINTER(C.c_int), vp,
                             C.POINTER(C.c_int), vp]),
    "camg_gmres_ex": (C.c_int, [i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, f64, C.c_int, C.c_int,
                                C.POINTER(C.c_int), vp, C.POINTER(C.c_int), vp]),
    "camg_gmres_release": (C.c_int, []),
    "camg_gmres_workspace_create": (C.c_int, [i64, C.c_int, C.c_int, C.POINTER(vp)]),
    "camg_gmres_workspace_destroy": (C.c_int, [vp]),
    "camg_vcycle_workspace_create": (C.c_int, [vp, C.POINTER(vp)]),
    "camg_vcycle_workspace_destroy": (C.c_int, [vp]),
    "camg_vcycle_ws": (C.c_int, [vp, vp, vp, vp, vp]),
    "camg_hierarchy_kernels_per_cycle": (C.c_int, [vp, P64]),
    "camg_level_get_info": (C.c_int, [vp, C.POINTER(LevelInfo)]),
    "camg_qr_batch": (C.c_int, [C.c_char_p, i64, C.c_int, C.c_int, vp, i64, vp, vp, vp, vp, C.c_int, P64]),
    "camg_tentative": (C.c_int, [C.c_char_p, i64, C.c_int, vp, vp, vp, i64, i64, f64, C.c_int, C.POINTER(vp), vp, vp,
                                 P64]),
    "camg_tentative_device": (C.c_int, [i64, C.c_int, vp, vp, vp, i64, i64, f64, C.POINTER(vp), vp, vp,
                                        C.POINTER(i64)]),
    "camg_dot": (C.c_int, [i64, vp, vp, C.POINTER(f64), vp]),
    "camg_axpy": (C.c_int, [i64, f64, vp, vp, vp]),
}

_lib = None


def lib():
    """Load libcamg.so once; raise NativeError when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(make -C paper_1912_09056_b200/csrc); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


_CODES = {
    1: DimensionError,
    2: SingularMatrixError,
    3: ConfigError,
    4: SetupError,
    5: NativeError,
    6: NativeError,
    7: ValueError,
}


def check(status: int):
    if status != 0:
        msg = lib().camg_last_error().decode(errors="replace")
        raise _CODES.get(status, NativeError)(msg)


def call(name, *args):
    check(getattr(lib(), name)(*args))


def exported_symbols():
    return list(_SIGS)


def require_device():
    """Raise unless a CUDA device is visible to the library."""
    n = C.c_int(0)
    check(lib().camg_device_count(C.byref(n)))
    if n.value < 1:
        raise NativeError("no CUDA device visible: the contactamg-b200 solve path runs only on the GPU")


def launch_count() -> int:
    return int(lib().camg_launch_count())


def synchronize():
    """Wait for all device work (setup phase timing)."""
    import torch

    if torch.cuda.is_available():
        torch.cuda.synchronize()
