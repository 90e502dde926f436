"""ctypes binding of libcurvkit_b200.so (the C-ABI in include/curvkit_b200.h).

There is no fallback: if the shared library is missing or fails to load,
importing the package's compute entry points raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libcurvkit_b200.so")

i32, i64, u64 = C.c_int32, C.c_int64, C.c_uint64
dptr = C.POINTER(C.c_double)
fptr = C.POINTER(C.c_float)
vptr = C.c_void_p


class Model(C.Structure):
    _fields_ = [("num_layers", i32), ("layer_widths", C.POINTER(i64)), ("hidden_activation", i32),
                ("output_mode", i32)]


class CurvatureConfig(C.Structure):
    _fields_ = [("batch_size_h", i64), ("batch_size_g", i64), ("parallelism", i64), ("memory_cap", i64)]


# name -> argtypes (all return int status unless listed in _RESTYPES)
_MP = C.POINTER(Model)
_CP = C.POINTER(CurvatureConfig)
SIGNATURES = {
    "curvkit_last_error": [],
    "curvkit_version": [],
    "curvkit_launch_count": [],
    "curvkit_profile_begin": [],
    "curvkit_profile_end": [C.c_char_p, i64],
    "curvkit_param_count": [_MP, C.POINTER(i64)],
    "curvkit_assemble_jacobian": [_MP, dptr, dptr, dptr, i64, i32, dptr],
    "curvkit_grad_batch": [_MP, dptr, dptr, dptr, i64, i32, dptr],
    "curvkit_hvp": [_MP, dptr, dptr, dptr, i64, dptr, i64, i32, dptr],
    "curvkit_hvp_operator_apply": [_MP, dptr, dptr, dptr, i64, i64, dptr, i64, i32, dptr],
    "curvkit_assemble_hessian": [_MP, dptr, dptr, dptr, i64, _CP, i32, i32, dptr, dptr],
    "curvkit_assemble_opg": [_MP, dptr, dptr, dptr, i64, _CP, i32, dptr],
    "curvkit_assemble_hessian_f32": [_MP, dptr, dptr, dptr, i64, _CP, i32, fptr],
    "curvkit_assemble_opg_f32": [_MP, dptr, dptr, dptr, i64, _CP, i32, fptr],
    "curvkit_opg_topk": [_MP, dptr, dptr, dptr, i64, i64, i64, i64, u64, i32, dptr, dptr],
    "curvkit_opg_topk_filtered": [_MP, dptr, dptr, dptr, i64, i64, i64, i64, i64, u64, i32, dptr, dptr],
    "curvkit_dev_assemble_hessian": [_MP, vptr, vptr, vptr, i64, i32, vptr, i64, vptr],
    "curvkit_dev_assemble_opg": [_MP, vptr, vptr, vptr, i64, i32, vptr, i64, vptr],
    "curvkit_dev_assemble_jacobian": [_MP, vptr, vptr, vptr, i64, i32, vptr, i64, vptr],
    "curvkit_shard_units": [_MP, i64, i64, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)],
    "curvkit_dev_assemble_band": [_MP, i32, vptr, vptr, vptr, i64, i32, i64, i64, vptr, i64, vptr],
    "curvkit_dev_band_scatter": [_MP, i32, i64, i64, vptr, i64, vptr, i64, vptr],
    "curvkit_dev_symmetrize_units": [_MP, i32, vptr, i64, vptr],
    "curvkit_dev_gather_bands": [_MP, i32, vptr, i64, vptr, i64, vptr, vptr],
    "curvkit_comm_init_host": [i32, i32, vptr, vptr, vptr, C.POINTER(vptr)],
    "curvkit_opg_topk_auto": [_MP, dptr, dptr, dptr, i64, i64, i64, C.c_double, i64, u64, i32, dptr, dptr],
    "curvkit_dev_opg_topk_auto": [_MP, vptr, vptr, vptr, i64, i64, i64, C.c_double, i64, u64, i32, vptr, vptr, vptr],
    "curvkit_dev_opg_topk_sharded_auto": [_MP, vptr, vptr, vptr, i64, i64, i64, C.c_double, i64, u64, i32, vptr, vptr,
                                          vptr, vptr],
    "curvkit_dev_gemm": [i64, i64, i64, vptr, i64, i32, vptr, i64, i32, vptr, i64, C.c_float, i32, vptr],
    "curvkit_dev_opg_topk": [_MP, vptr, vptr, vptr, i64, i64, i64, i64, u64, i32, vptr, vptr, vptr],
    "curvkit_dev_opg_topk_filtered": [_MP, vptr, vptr, vptr, i64, i64, i64, i64, i64, u64, i32, vptr, vptr, vptr],
    "curvkit_comm_unique_id": [C.POINTER(C.c_uint8)],
    "curvkit_comm_init": [C.POINTER(C.c_uint8), i32, i32, C.POINTER(vptr)],
    "curvkit_comm_destroy": [vptr],
    "curvkit_incr_opg_create": [i64, i64, C.POINTER(vptr)],
    "curvkit_incr_opg_push_block": [vptr, dptr, i64],
    "curvkit_incr_opg_dev_push_block": [vptr, vptr, i64, i64, vptr],
    "curvkit_incr_opg_counts": [vptr, C.POINTER(i64), C.POINTER(i64)],
    "curvkit_incr_opg_finalize": [vptr, i64, dptr, dptr],
    "curvkit_incr_opg_dev_finalize": [vptr, i64, vptr, vptr, vptr],
    "curvkit_incr_opg_destroy": [vptr],
    "curvkit_topk_shard_rows": [_MP, i64, i64, C.POINTER(i64), C.POINTER(i64)],
    "curvkit_dev_opg_topk_sharded": [_MP, vptr, vptr, vptr, i64, i64, i64, i64, u64, i32, vptr, vptr, vptr, vptr],
    "curvkit_dev_opg_topk_sharded_filtered": [_MP, vptr, vptr, vptr, i64, i64, i64, i64, i64, u64, i32, vptr, vptr, vptr,
                                              vptr],
    "curvkit_dev_jacobian_apply": [_MP, vptr, vptr, vptr, i64, i32, i64, i64, i32, vptr, i64, i64, vptr, i64, vptr],
    "curvkit_forward": [_MP, dptr, dptr, i64, i32, dptr],
    "curvkit_cost": [_MP, dptr, dptr, dptr, i64, i32, dptr],
    "curvkit_opg_topk_from_jacobian": [dptr, i64, i64, i64, i64, i64, u64, i32, dptr, dptr],
    "curvkit_dev_opg_topk_from_jacobian": [vptr, i64, i64, i64, i64, i64, i64, u64, i32, vptr, vptr, vptr],
    "curvkit_eig_validate": [i64, i64, dptr, dptr, i64, C.c_double],
    "curvkit_eig_materialize": [i64, i64, dptr, dptr, i32, C.c_double, i64, i32, dptr],
    "curvkit_eig_apply": [i64, i64, dptr, dptr, i32, C.c_double, i64, dptr, i64, i32, dptr, dptr],
    "curvkit_dev_eig_materialize": [i64, i64, vptr, i64, vptr, i32, C.c_double, i32, vptr, i64, vptr],
    "curvkit_dev_eig_apply": [i64, i64, vptr, i64, vptr, i32, C.c_double, i64, vptr, i64, vptr, i64, dptr, i32, vptr],
    "curvkit_dev_eig_apply_sharded": [i64, i64, vptr, i64, vptr, i32, C.c_double, i64, vptr, i64, vptr, i64, dptr, i32,
                                      vptr, vptr],
    "curvkit_hessian_topk_lanczos": [_MP, dptr, dptr, dptr, i64, i64, i64, i64, C.c_double, u64, i32, dptr, dptr, dptr,
                                     C.POINTER(i64)],
}
# host-transport callbacks of curvkit_comm_init_host
HOST_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, i64, i32, C.c_void_p)
HOST_GATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, i64, C.c_void_p, C.POINTER(i64), i32, C.c_void_p)

_RESTYPES = {"curvkit_last_error": C.c_char_p, "curvkit_version": C.c_char_p, "curvkit_launch_count": i64}

_lib = None


def load(path: str = SO_PATH) -> C.CDLL:
    """Load (once) and type the library.  Raises OSError if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise OSError(f"libcurvkit_b200.so not built at {path}; run `python -m paper_1905_05559_b200.build`")
        lib = C.CDLL(path)
        for name, args in SIGNATURES.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = _RESTYPES.get(name, C.c_int)
        _lib = lib
    return _lib


def check(rc: int):
    if rc != 0:
        from .errors import raise_for
        raise_for(rc, load().curvkit_last_error().decode())
