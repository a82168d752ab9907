"""ctypes binding of the C ABI in include/wadg_b200.h (libwadg_b200.so,
built in-tree by __graft_entry__.build()).

There is no fallback: if the library is missing every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

LIB_NAME = "libwadg_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

WADG_F64, WADG_F32 = 0, 1
WADG_STRONG, WADG_STRONG_WEAK = 0, 1
ELEMS_PER_BLOCK = 32
ABI_VERSION = 6

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32


class WadgProblem(ctypes.Structure):
    _fields_ = [
        ("dim", _i32), ("dtype", _i32), ("K", _i32), ("Kpad", _i32),
        ("Np", _i32), ("Nq", _i32), ("Nqu", _i32),
        ("Nf", _i32), ("Nfp", _i32), ("Nfq", _i32),
        ("n_orient", _i32), ("formulation", _i32),
        ("Vq", _vp), ("Dq", _vp), ("Pq", _vp), ("DTW", _vp), ("Vu", _vp), ("Pu", _vp),
        ("Vfi", _vp), ("Pf", _vp),
        ("fmask", _vp), ("ext_node", _vp), ("fperm", _vp),
        ("geo", _vp), ("fgeo", _vp), ("wu", _vp), ("wp", _vp), ("c2", ctypes.c_double),
        ("nbr", _vp), ("ncode", _vp),
        ("halo", _vp), ("n_halo", _i32),
        ("Ne", _i32), ("Ve", _vp), ("we", _vp), ("ewp", _vp), ("ewu", _vp), ("e_recip", _i32),
        ("order", _i32), ("fused_kind", _i32), ("opVA", _vp), ("opVB", _vp), ("opU1", _vp), ("opU2", _vp), ("liftT", _vp),
        ("geo_il", _vp), ("fgeo_il", _vp), ("wu_il", _vp), ("wp_il", _vp), ("wbar", _vp),
        ("minv_p", _vp), ("minv_u", _vp),
    ]


EXPORTS = {
    "wadg_abi_version": ([], ctypes.c_int),
    "wadg_last_error": ([], ctypes.c_char_p),
    "wadg_volume": ([ctypes.POINTER(WadgProblem), _vp, _vp, _vp], ctypes.c_int),
    "wadg_surface": ([ctypes.POINTER(WadgProblem), _vp, _vp, ctypes.c_double, ctypes.c_double,
                      ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp], ctypes.c_int),
    "wadg_mass_inverse": ([ctypes.POINTER(WadgProblem), _vp, _vp, _vp], ctypes.c_int),
    "wadg_update_lsrk": ([ctypes.POINTER(WadgProblem), _vp, _vp, _vp, ctypes.c_double,
                          ctypes.c_double, ctypes.c_double, _vp], ctypes.c_int),
    "wadg_stage": ([ctypes.POINTER(WadgProblem), _vp, _vp, _vp, ctypes.c_double, ctypes.c_double,
                    ctypes.c_double, ctypes.c_double, ctypes.c_double, _vp], ctypes.c_int),
    "wadg_lsrk_axpy": ([ctypes.c_int, ctypes.c_int64, _vp, _vp, _vp, ctypes.c_double,
                        ctypes.c_double, ctypes.c_double, _vp], ctypes.c_int),
    "wadg_energy": ([ctypes.POINTER(WadgProblem), _vp, _vp, _vp, _vp], ctypes.c_int),
    "wadg_fused_config": ([ctypes.c_int, ctypes.c_int, ctypes.POINTER(_i32),
                           ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "wadg_fused_config_form": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_i32),
                                ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "wadg_debug_set_fused_variant": ([ctypes.c_int], ctypes.c_int),
    "wadg_stage_fused": ([ctypes.POINTER(WadgProblem), _vp, _vp, _vp, ctypes.c_double, ctypes.c_double,
                          ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                          _vp], ctypes.c_int),
    "wadg_stage_fused_rows": ([ctypes.POINTER(WadgProblem), _vp, _vp, _vp, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, _vp], ctypes.c_int),
    "wadg_debug_set_phase_clock_buffer": ([_vp], ctypes.c_int),
    "wadg_microbench_fma": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp], ctypes.c_int),
    "wadg_debug_umma_test": ([_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp], ctypes.c_int),
    "wadg_pack_halo": ([ctypes.POINTER(WadgProblem), _vp, _vp, _vp, _i32, _vp, _vp], ctypes.c_int),
    "wadg_rows_to_fields": ([ctypes.POINTER(WadgProblem), _vp, _i32, _i32, _vp, _vp], ctypes.c_int),
    "wadg_fields_to_rows": ([ctypes.POINTER(WadgProblem), _vp, _i32, _i32, _vp, _vp], ctypes.c_int),
    "wadg_debug_umma_rate": ([_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp], ctypes.c_int),
}

_lib = None


class NativeError(RuntimeError):
    pass


def load():
    """Load the in-tree shared library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("WADG_LIB", LIB_PATH)    # experiments: alternative in-tree build
    if not os.path.exists(path):
        raise NativeError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (args, res) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.wadg_abi_version() != ABI_VERSION:
        raise NativeError("ABI version mismatch between libwadg_b200.so and _native.py")
    _lib = lib
    return lib


def call(name, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise NativeError(f"{name} failed ({rc}): {lib.wadg_last_error().decode()}")


def fused_config(dtype_code, order, formulation=WADG_STRONG_WEAK):
    """Layout of the fused stage for (dtype, order, formulation) as a dict, or
    None when there is no fused stage for it (see include/wadg_b200.h)."""
    lib = load()
    info = (_i32 * 8)()
    smem = ctypes.c_int64()
    if lib.wadg_fused_config_form(dtype_code, order, formulation, info, ctypes.byref(smem)) != 0:
        return None
    keys = ("kind", "kb", "qc", "nch", "npp", "qcs", "njs", "nfq8")
    out = dict(zip(keys, list(info)))
    out["smem"] = smem.value
    return out
