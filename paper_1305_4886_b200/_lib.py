"""ctypes binding of libbgp.so (include/bgp.h).

The library is the only compute path: if it is missing or cannot be loaded,
every device operation raises `BackendUnavailable` -- there is no CPU
fallback.  Build it with `make` (or `__graft_entry__.build()`).
"""

import ctypes
import os

from .errors import BackendUnavailable

_HERE = os.path.dirname(os.path.abspath(__file__))
# BGP_LIB_PATH (diagnostics): load an alternative build of the library
LIB_PATH = os.environ.get("BGP_LIB_PATH") or os.path.join(_HERE, "libbgp.so")

BGP_OK = 0
BGP_E_CUDA = -1
BGP_E_ARG = -2
BGP_E_UNSUPPORTED = -3

BGP_TRI, BGP_RECT, BGP_VEC = 0, 1, 2
KIND_CODE = {"triangular": BGP_TRI, "rectangular": BGP_RECT, "vector": BGP_VEC}

GEN_ZERO, GEN_DELTA, GEN_LINEAR_INDEX, GEN_MATERN, GEN_SQEXP, GEN_WHITE, GEN_PRODUCT = range(7)
PART_COV, PART_CROSS, PART_PRED, PART_PREDVAR = range(4)


class Generator(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int), ("part", ctypes.c_int),
                ("nugget", ctypes.c_int), ("nparams", ctypes.c_int),
                ("params", ctypes.c_double * 8), ("nu", ctypes.c_double),
                ("nu2", ctypes.c_double), ("span", ctypes.c_double)]


_c_dp = ctypes.c_void_p           # device pointers travel as integers
_i64 = ctypes.c_int64
_int = ctypes.c_int

# name -> (restype, argtypes); mirrors include/bgp.h
SIGNATURES = {
    "bgp_init": (_int, [_int, ctypes.POINTER(ctypes.c_void_p)]),
    "bgp_finalize": (_int, [ctypes.c_void_p]),
    "bgp_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
    "bgp_version": (ctypes.c_char_p, []),
    "bgp_launch_count": (_i64, [ctypes.c_void_p]),
    "bgp_construct": (_int, [ctypes.c_void_p, _int, ctypes.POINTER(Generator), _c_dp, _i64,
                             _c_dp, _i64, _int, _int, _c_dp, _c_dp]),
    "bgp_potrf": (_int, [ctypes.c_void_p, _c_dp, _i64, _int, ctypes.POINTER(_i64), _c_dp]),
    "bgp_trsv": (_int, [ctypes.c_void_p, _c_dp, _i64, _int, _c_dp, _int,
                        ctypes.POINTER(_i64), _c_dp]),
    "bgp_trsm_rect": (_int, [ctypes.c_void_p, _c_dp, _i64, _int, _c_dp, _i64, _int,
                             ctypes.POINTER(_i64), _c_dp]),
    "bgp_xprod_mat_vec": (_int, [ctypes.c_void_p, _c_dp, _i64, _i64, _int, _c_dp, _c_dp, _c_dp]),
    "bgp_xprod_self_diag": (_int, [ctypes.c_void_p, _c_dp, _i64, _i64, _int, _c_dp, _c_dp]),
    "bgp_xprod_self": (_int, [ctypes.c_void_p, _c_dp, _i64, _i64, _int, _c_dp, _c_dp]),
    "bgp_trmm_rect": (_int, [ctypes.c_void_p, _c_dp, _i64, _int, _c_dp, _i64, _c_dp, _c_dp]),
    "bgp_rnorm": (_int, [ctypes.c_void_p, _i64, _i64, _i64, _i64, ctypes.c_uint64, ctypes.c_uint64,
                         ctypes.c_uint64, _int, _c_dp, _c_dp]),
    "bgp_tri_mv": (_int, [ctypes.c_void_p, _c_dp, _i64, _int, _c_dp, _c_dp, _int, _c_dp]),
    "bgp_logdet": (_int, [ctypes.c_void_p, _c_dp, _i64, _int, ctypes.POINTER(ctypes.c_double),
                          ctypes.POINTER(_i64), _c_dp]),
    "bgp_sumsq": (_int, [ctypes.c_void_p, _c_dp, _i64, ctypes.POINTER(ctypes.c_double), _c_dp]),
    "bgp_pack": (_int, [ctypes.c_void_p, _int, _c_dp, _i64, _i64, _i64, _int, _c_dp, _c_dp]),
    "bgp_unpack": (_int, [ctypes.c_void_p, _int, _c_dp, _i64, _i64, _int, _c_dp, _i64, _c_dp]),
    "bgp_tri_diagonal": (_int, [ctypes.c_void_p, _c_dp, _i64, _int, _c_dp, _c_dp]),
    "bgp_sub": (_int, [ctypes.c_void_p, _c_dp, _c_dp, _c_dp, _i64, _c_dp]),
    "bgp_tile_potrf": (_int, [ctypes.c_void_p, _c_dp, _int, _i64, ctypes.POINTER(_i64), _c_dp]),
    "bgp_tile_potrf_inv": (_int, [ctypes.c_void_p, _c_dp, _int, _c_dp, ctypes.POINTER(_i64), _c_dp]),
    "bgp_info_reset": (_int, [ctypes.c_void_p, _c_dp]),
    "bgp_info_read": (_int, [ctypes.c_void_p, ctypes.POINTER(_i64), _c_dp]),
    "bgp_tile_potrf_async": (_int, [ctypes.c_void_p, _c_dp, _int, _i64, _c_dp, _c_dp]),
    "bgp_panel_trsm_inv": (_int, [ctypes.c_void_p, _c_dp, _c_dp, _i64, _int, _c_dp]),
    "bgp_ipc_alloc": (_int, [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p]),
    "bgp_ipc_open": (_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "bgp_ipc_close": (_int, [ctypes.c_void_p, _c_dp]),
    "bgp_ipc_free": (_int, [ctypes.c_void_p, _c_dp]),
    "bgp_panel_trsm_push": (_int, [ctypes.c_void_p, _c_dp, _c_dp, _i64, _int, ctypes.POINTER(ctypes.c_void_p),
                                   _int, _i64, _i64, _c_dp]),
    "bgp_panel_trsm": (_int, [ctypes.c_void_p, _c_dp, _c_dp, _i64, _int, _c_dp]),
    "bgp_tile_update": (_int, [ctypes.c_void_p, _c_dp, _c_dp, _c_dp, _c_dp, _i64, _int, _c_dp]),
    "bgp_potrf_async": (_int, [ctypes.c_void_p, _c_dp, _i64, _int, _c_dp]),
    "bgp_trsv_async": (_int, [ctypes.c_void_p, _c_dp, _i64, _int, _c_dp, _int, _c_dp]),
    "bgp_logdet_async": (_int, [ctypes.c_void_p, _c_dp, _i64, _int, _c_dp, _c_dp]),
    "bgp_sumsq_async": (_int, [ctypes.c_void_p, _c_dp, _i64, _c_dp, _c_dp]),
    "bgp_info_copy": (_int, [ctypes.c_void_p, _c_dp, _c_dp]),
    "bgp_dist_begin": (_int, [ctypes.c_void_p, _int, _int, _c_dp]),
    "bgp_dist_step": (_int, [ctypes.c_void_p, _int, _c_dp, _i64, _c_dp, _i64, _c_dp, _i64, _i64, _c_dp, _i64,
                             _i64, _i64, _int, ctypes.POINTER(ctypes.c_void_p), _int, _i64, _i64, _int, _c_dp]),
    "bgp_construct_tiles": (_int, [ctypes.c_void_p, ctypes.POINTER(Generator), _c_dp, _i64, _int, _int,
                                   _c_dp, _i64, _c_dp, _c_dp]),
    "bgp_tile_trsv": (_int, [ctypes.c_void_p, _c_dp, _int, _i64, _i64, _c_dp, _int,
                             ctypes.POINTER(_i64), _c_dp]),
    "bgp_tile_gemv": (_int, [ctypes.c_void_p, _c_dp, _c_dp, _i64, _int, _c_dp, _c_dp, _int, _c_dp]),
    "bgp_tile_logdet": (_int, [ctypes.c_void_p, _c_dp, _c_dp, _i64, _int, _i64,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64), _c_dp]),
    "bgp_set_profiling": (_int, [ctypes.c_void_p, _int]),
    "bgp_set_tail": (_int, [ctypes.c_void_p, _int]),
    "bgp_set_grid_cap": (_int, [ctypes.c_void_p, _int]),
    "bgp_profile_read": (_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]),
    "bgp_profile_steps": (_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), _int]),
}

_LIB = None


def load(path=LIB_PATH):
    """Load libbgp.so and attach prototypes; raises BackendUnavailable."""
    global _LIB
    if _LIB is not None and path == LIB_PATH:
        return _LIB
    if not os.path.exists(path):
        raise BackendUnavailable(
            f"libbgp.so not built ({path}); run `make` -- there is no CPU fallback")
    try:
        lib = ctypes.CDLL(path)
    except OSError as exc:
        raise BackendUnavailable(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _LIB = lib
    return lib
