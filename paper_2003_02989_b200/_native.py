"""ctypes binding of libqfb200.so (the C ABI in include/qfb200.h).

The product path has exactly one backend: this library.  If it cannot be
loaded on a machine with a GPU the import of any compute function raises --
there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqfb200.so")

EXPORTS = (
    "qf_last_error", "qf_version", "qf_device_sm_count", "qf_build_ops", "qf_run_passes",
    "qf_adjoint_passes", "qf_reduce_slots", "qf_pauli_expect", "qf_pauli_apply", "qf_sample",
    "qf_jit_compile", "qf_jit_free", "qf_jit_load", "qf_jit_function", "qf_jit_unload", "qf_jit_run",
    "qf_reduce_slots_scaled", "qf_frame_walk", "qf_jit_occupancy", "qf_frame_walk_ckpt", "qf_block_grads",
    "qf_sample_multi", "qf_reduce_slots_offset", "qf_permute_bits", "qf_dense4_tc_prepare", "qf_dense4_tc",
    "qf_tc_build", "qf_jit_global", "qf_jit_cm_stage",
)

_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64


class QfProgram(C.Structure):
    _fields_ = [
        ("passes", _p), ("stages", _p), ("ops", _p), ("term_mask", _p), ("term_idx", _p),
        ("term_w", _p), ("grp", _p), ("genmats", _p),
        ("n_passes", _i32), ("n_slots", _i32), ("n_mat", _i32), ("n_ang", _i32), ("n_coef", _i32),
        ("L", _i32), ("R", _i32), ("coef_row_stride", _i32), ("host_passes", _p),
    ]


class QfBuildRecipe(C.Structure):
    _fields_ = [
        ("n_gen", _i32), ("gen_sym", _p), ("gen_coeff", _p), ("gen_const", _p), ("gen_dim", _p),
        ("gen_eval", _p), ("gen_evec", _p),
        ("n_fixed", _i32), ("fixed", _p), ("fixed_rows", _i32),
        ("n_dense", _i32), ("dense_mat", _p), ("dense_dim", _p), ("dense_fbeg", _p), ("factor", _p),
        ("n_terms", _i32), ("term_src", _p), ("term_beta", _p), ("term_const", _p),
        ("const_rows", _i32), ("n_const", _i32), ("max_dim", _i32),
    ]


class QfFrame(C.Structure):
    _fields_ = [("x", C.c_uint32), ("z", C.c_uint32), ("m", C.c_double)]


class NativeError(RuntimeError):
    pass


_lib = None


def load(build_if_missing: bool = True):
    """Load (building in-tree first if needed) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        from .build import build

        build()
    lib = C.CDLL(LIB_PATH)
    lib.qf_last_error.restype = C.c_char_p
    lib.qf_version.restype = C.c_int
    lib.qf_device_sm_count.argtypes = [C.c_int]
    lib.qf_build_ops.argtypes = [C.POINTER(QfBuildRecipe), _p, _i64, C.c_int, _p, C.c_int, _p, C.c_int, _p]
    lib.qf_run_passes.argtypes = [C.POINTER(QfProgram), C.c_int, C.c_int, _p, C.c_int, C.c_int, _p, _p, _p, _p,
                                  C.c_int, _p]
    lib.qf_adjoint_passes.argtypes = [C.POINTER(QfProgram), C.c_int, C.c_int, _p, _p, C.c_int, C.c_int, _p, _p,
                                      _p, _p, C.c_int, _p]
    lib.qf_reduce_slots.argtypes = [_p, C.c_int, C.c_int, C.c_int, _p, _p, C.c_int, _p, C.c_int, _p]
    lib.qf_reduce_slots_scaled.argtypes = [_p, C.c_int, C.c_int, C.c_int, _p, _p, C.c_int, _p, C.c_int, _p, _p]
    lib.qf_frame_walk.argtypes = [_p, C.c_int, C.c_int, C.c_int, _p, C.c_int, _p, C.c_int, _p, C.c_int, _p, _p,
                                  _p]
    lib.qf_frame_walk_ckpt.argtypes = [_p, C.c_int, C.c_int, C.c_int, _p, C.c_int, _p, C.c_int, _p, C.c_int, _p,
                                       _p, _p, C.c_int, C.c_int, _p]
    lib.qf_block_grads.argtypes = [_p, C.c_int, _p, C.c_int, _p, _p, C.c_int, _p, C.c_int, _p, C.c_int, _p]
    lib.qf_pauli_expect.argtypes = [_p, C.c_int, C.c_int, C.c_int, _p, _p, _p, _p, _i64, _p, _p]
    lib.qf_pauli_apply.argtypes = [_p, _p, C.c_int, C.c_int, C.c_int, _p, _p, _p, _p, _i64, _p]
    lib.qf_sample.argtypes = [_p, C.c_int, C.c_int, C.c_int, _p, _p, _p, _p, _p]
    lib.qf_permute_bits.argtypes = [_p, _p, C.c_int, C.c_int, _p, _p]
    lib.qf_dense4_tc_prepare.argtypes = [_p, _p]
    lib.qf_dense4_tc.argtypes = [_p, _p, C.c_int, C.c_int, _p, _p]
    lib.qf_tc_build.argtypes = [_p, C.c_int, C.c_int, _p, _p, C.c_int, _p, _p]
    lib.qf_sample_multi.argtypes = [_p, C.c_int, C.c_int, C.c_int, C.c_int, _p, _p, _p, _p, _p]
    lib.qf_reduce_slots_offset.argtypes = [_p, C.c_int, C.c_int, C.c_int, _p, _p, C.c_int, _p, C.c_int, _p, _p,
                                           _p]
    lib.qf_jit_compile.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p), C.c_int, C.POINTER(C.c_void_p),
                                   C.POINTER(C.c_size_t)]
    lib.qf_jit_free.argtypes = [_p]
    lib.qf_jit_load.argtypes = [_p, C.POINTER(C.c_void_p)]
    lib.qf_jit_function.argtypes = [_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
    lib.qf_jit_unload.argtypes = [_p]
    lib.qf_jit_occupancy.argtypes = [_p, C.c_int, C.c_int, C.POINTER(C.c_int)]
    lib.qf_jit_run.argtypes = [_p, _p, _p, _p, C.c_int, _p, _p, C.c_size_t]
    lib.qf_jit_global.argtypes = [_p, C.c_char_p, C.POINTER(_p), C.POINTER(C.c_size_t)]
    lib.qf_jit_cm_stage.argtypes = [_p, C.c_int, C.c_int, _p, C.c_int, _p, _p, C.c_size_t, _p]
    for name in EXPORTS:
        getattr(lib, name).restype = C.c_int if name != "qf_last_error" else C.c_char_p
    lib.qf_jit_free.restype = None
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.qf_last_error().decode(errors="replace") if _lib is not None else "?"
        if rc == 3:
            raise MemoryError(msg)
        if rc == 2:
            raise ValueError(msg)
        raise NativeError(f"libqfb200 error {rc}: {msg}")
