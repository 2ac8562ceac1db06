"""ctypes binding of libvreg_b200.so (include/vreg_cuda.h, include/vreg_b200.h).

The product path: every call goes to the sm_100a kernels through the C ABI.
There is no CPU fallback -- importing this module without the built library
raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# VREG_LIB_PATH: an alternative in-tree build of the same library (A/B measurements)
LIB_PATH = os.environ.get("VREG_LIB_PATH") or os.path.join(PKG, "libvreg_b200.so")


class VregGrid(C.Structure):
    """vreg_grid (include/vreg_cuda.h; grid.hpp:13-17)."""
    _fields_ = [("n1", C.c_int), ("n2", C.c_int), ("n3", C.c_int), ("nt", C.c_int)]


VP = C.c_void_p
I = C.c_int
D = C.c_double
GP = C.POINTER(VregGrid)

_SIGS = {
    "vreg_last_error": (C.c_char_p, []),
    "vreg_status_exit_code": (I, [I]),
    "vreg_ctx_create": (I, [I, C.POINTER(VP)]),
    "vreg_nccl_unique_id": (I, [VP]),
    "vreg_ctx_create_dist": (I, [I, I, I, VP, C.POINTER(VP)]),
    "vreg_ctx_destroy": (I, [VP]),
    "vreg_ctx_rank": (I, [VP, C.POINTER(I), C.POINTER(I)]),
    "vreg_ctx_set_stream": (I, [VP, VP]),
    "vreg_ctx_get_stream": (I, [VP, C.POINTER(VP)]),
    "vreg_ctx_set_deterministic": (I, [VP, I]),
    "vreg_ctx_set_reg_order": (I, [VP, I]),
    "vreg_ctx_reserve": (I, [VP, C.c_size_t]),
    "vreg_halo_chunks": (I, [I, I, I, C.POINTER(I), C.POINTER(I), C.POINTER(C.c_longlong),
                             C.POINTER(C.c_longlong)]),
    "vreg_two_level_begin": (I, [VP, C.POINTER(VregGrid), VP, C.c_double, VP, VP]),
    "vreg_two_level_end": (I, [VP, C.POINTER(VregGrid), VP, VP]),
    "vreg_volume_save": (I, [C.c_char_p, I, I, I, I, I, VP]),
    "vreg_volume_header": (I, [C.c_char_p, C.POINTER(I)]),
    "vreg_volume_load": (I, [C.c_char_p, VP, C.c_size_t]),
    "vreg_ctx_stream": (VP, [VP]),
    "vreg_ctx_synchronize": (I, [VP]),
    "vreg_slab": (I, [VP, GP, C.POINTER(I), C.POINTER(I)]),
    "vreg_ctx_enable_timers": (I, [VP, I]),
    "vreg_ctx_timers": (I, [VP, C.POINTER(D)]),
    "vreg_ctx_comm": (I, [VP, C.POINTER(C.c_uint64)]),
    "vreg_ctx_kernel_stats": (I, [VP, I, C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(D)]),
    "vreg_ctx_reset_kernel_stats": (I, [VP]),
    "vreg_ctx_launches": (I, [VP, C.POINTER(C.c_uint64)]),
    "vreg_ctx_tile_stats": (I, [VP, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "vreg_alloc": (I, [VP, C.c_size_t, C.POINTER(VP)]),
    "vreg_free": (I, [VP, VP]),
    "vreg_memcpy_d2d": (I, [VP, VP, VP, C.c_size_t]),
    "vreg_memcpy_h2d": (I, [VP, VP, VP, C.c_size_t]),
    "vreg_memcpy_d2h": (I, [VP, VP, VP, C.c_size_t]),
    "vreg_fill": (I, [VP, GP, I, VP, D]),
    "vreg_copy": (I, [VP, GP, I, VP, VP]),
    "vreg_axpy": (I, [VP, GP, I, D, VP, VP]),
    "vreg_scale": (I, [VP, GP, I, VP, D]),
    "vreg_aypx": (I, [VP, GP, I, D, VP, VP]),
    "vreg_sub": (I, [VP, GP, I, VP, VP, VP]),
    "vreg_hadamard": (I, [VP, GP, VP, VP, VP]),
    "vreg_pointwise_dot": (I, [VP, GP, VP, VP, VP]),
    "vreg_axpy_scaled_vector": (I, [VP, GP, D, VP, VP, VP]),
    "vreg_inner": (I, [VP, GP, I, VP, VP, C.POINTER(D)]),
    "vreg_max_abs": (I, [VP, GP, I, VP, C.POINTER(D)]),
    "vreg_fd_grad": (I, [VP, GP, VP, VP]),
    "vreg_fd_div": (I, [VP, GP, VP, VP]),
    "vreg_characteristics": (I, [VP, GP, VP, I, VP, C.POINTER(I)]),
    "vreg_interp": (I, [VP, GP, VP, VP, I, I, VP]),
    "vreg_scatter": (I, [VP, GP, VP, VP, I, I, VP]),
    "vreg_interp_points": (I, [VP, GP, VP, VP, C.c_int64, I, VP]),
    "vreg_scatter_points": (I, [VP, GP, VP, VP, C.c_int64, I, VP]),
    "vreg_solve_state": (I, [VP, GP, VP, I, I, VP]),
    "vreg_inc_state": (I, [VP, GP, VP, I, I, VP, VP, VP, VP]),
    "vreg_transpose_assemble": (I, [VP, GP, VP, I, I, VP, VP, VP]),
    "vreg_gn_matvec": (I, [VP, GP, VP, I, I, VP, D, VP, VP]),
    "vreg_adjoint_source_factor": (I, [VP, GP, VP, VP, I, I, VP]),
    "vreg_adjoint_sweep": (I, [VP, GP, VP, I, I, VP, VP]),
    "vreg_integrate_lambda_grad_m": (I, [VP, GP, VP, VP, VP]),
    "vreg_regop": (I, [VP, GP, VP, D, I, VP]),
    "vreg_inv_regop": (I, [VP, GP, VP, D, VP]),
    "vreg_seminorm": (I, [VP, GP, VP, C.POINTER(D)]),
    "vreg_leray": (I, [VP, GP, VP, VP]),
    "vreg_restrict": (I, [VP, GP, I, VP, VP]),
    "vreg_prolong": (I, [VP, GP, I, VP, VP]),
    "vreg_high_pass": (I, [VP, GP, I, VP, VP]),
    "vreg_h0_matvec": (I, [VP, GP, VP, VP, D, VP]),
    "vreg_fft_forward": (I, [VP, GP, VP, VP]),
    "vreg_syn_template": (I, [VP, GP, VP]),
    "vreg_syn_velocity": (I, [VP, GP, VP]),
    "vreg_from_global": (I, [VP, GP, I, VP, VP]),
    "vreg_to_global": (I, [VP, GP, I, VP, VP]),
}

# solver-level C ABI (include/vreg_b200.h); bound when present
_SOLVER_SIGS: dict = {}

_lib = None


class VregError(RuntimeError):
    """Raised for a non-zero status; `kind` mirrors the reference exception
    type (proj/include/vreg/types.hpp:19-41)."""
    KINDS = {2: "parameter_error", 3: "numerical_error", 4: "io_error", 5: "input_error",
             6: "dimension_error", 7: "config_error", 8: "cuda_error"}

    def __init__(self, status: int, msg: str):
        self.status = status
        self.kind = self.KINDS.get(status, "error")
        super().__init__(f"{self.kind}: {msg}")


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA library must be built "
                "(python -m paper_2008_12820_b200.build); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in list(_SIGS.items()) + list(_SOLVER_SIGS.items()):
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS) + list(_SOLVER_SIGS)


def check(status: int):
    if status != 0:
        raise VregError(status, lib().vreg_last_error().decode())
