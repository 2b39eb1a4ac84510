"""ctypes loader for libskel.so (include/skel.h).  No fallback: a missing library raises."""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libskel.so")

c_i64 = ctypes.c_int64
c_dp = ctypes.c_void_p
c_int = ctypes.c_int

SK_OK, SK_E_ARG, SK_E_RANK, SK_E_CUDA, SK_E_NCCL, SK_E_NOMEM, SK_E_STATE = range(7)
STATUS_NAMES = {0: "SK_OK", 1: "SK_E_ARG", 2: "SK_E_RANK", 3: "SK_E_CUDA", 4: "SK_E_NCCL",
                5: "SK_E_NOMEM", 6: "SK_E_STATE"}

# name -> argtypes (restype sk_status = int unless noted)
_SIGS = {
    "sk_create": [ctypes.POINTER(c_dp), c_int, c_dp],
    "sk_set_stream": [c_dp, c_dp],
    "sk_set_sketch_tuning": [c_dp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_i64],
    "sk_sketch_dual": [c_dp, c_dp, c_int, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, ctypes.c_uint64, ctypes.c_uint64,
                       c_dp, c_i64, c_dp, c_i64],
    "sk_id_estimate_cols": [c_dp, c_dp, c_i64, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64, ctypes.POINTER(c_i64)],
    "sk_id_estimate_rows": [c_dp, c_dp, c_i64, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64, ctypes.POINTER(c_i64)],
    "sk_nccl_unique_id": [c_dp],
    "sk_create_dist": [ctypes.POINTER(c_dp), c_int, c_dp, c_dp, c_int, c_int, c_i64, c_i64, c_i64],
    "sk_set_dist_exchange": [c_dp, ctypes.c_int32],
    "sk_dist_info": [c_dp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(c_i64),
                     ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)],
    "sk_sketch": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_int, ctypes.c_int32, ctypes.c_uint64, c_dp, c_i64],
    "sk_sketch_cols": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_int, ctypes.c_int32, ctypes.c_uint64, c_dp, c_i64],
    "sk_sketch_power": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_int, ctypes.c_int32, ctypes.c_uint64,
                        ctypes.c_int32, c_dp, c_i64],
    "sk_sketch_power_ortho": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_int, ctypes.c_int32, ctypes.c_uint64,
                              ctypes.c_int32, c_dp, c_i64, ctypes.POINTER(c_i64)],
    "sk_select_cols": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_dp, c_dp, c_i64, c_dp, c_i64, c_dp,
                       ctypes.POINTER(c_i64)],
    "sk_select_cols_cpqr": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_dp, c_dp, c_i64, ctypes.POINTER(c_i64)],
    "sk_select_cols_deim": [c_dp, c_dp, c_i64, c_i64, c_i64, c_dp, c_i64, c_i64, c_i64, c_dp, ctypes.POINTER(c_i64)],
    "sk_gather_cols": [c_dp, c_dp, c_i64, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64],
    "sk_gather_cols_shard": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64],
    "sk_residual_cols": [c_dp, c_dp, c_i64, c_i64, c_i64, c_dp, c_i64, c_i64, ctypes.POINTER(ctypes.c_double)],
    "sk_select_rows": [c_dp, c_dp, c_i64, c_i64, c_i64, c_dp, c_dp, c_i64, c_dp, c_i64, c_dp,
                       ctypes.POINTER(c_i64)],
    "sk_id_coeffs": [c_dp, c_dp, c_i64, c_i64, c_i64, c_dp, c_dp, c_i64, ctypes.POINTER(ctypes.c_double)],
    "sk_residual": [c_dp, c_dp, c_i64, c_i64, c_i64, c_dp, c_dp, c_i64, c_int, c_dp, c_i64,
                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)],
    "sk_lupp_dist_begin": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_dp, c_dp, c_i64, c_dp, c_i64, c_dp],
    "sk_lupp_dist_step": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_dp, ctypes.c_int32, c_dp, c_dp, c_i64, c_dp,
                          c_i64, c_dp],
    "sk_lupp_dist_info": [c_dp, c_dp, ctypes.POINTER(c_i64)],
    "sk_lupp_dist_begin_p2p": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_dp, c_dp, c_i64, c_dp, c_i64, c_dp, c_dp,
                               c_dp, ctypes.c_int32, ctypes.c_int32],
    "sk_lupp_dist_step_p2p": [c_dp, c_dp, c_i64, c_i64, c_i64, c_i64, c_dp, ctypes.c_int32, ctypes.c_int32,
                              c_dp, c_dp, c_i64, c_dp, c_i64, c_dp],
    "sk_ipc_alloc": [c_dp, ctypes.c_size_t, ctypes.POINTER(c_dp)],
    "sk_ipc_free": [c_dp, c_dp],
    "sk_ipc_export": [c_dp, c_dp, c_dp],
    "sk_ipc_import": [c_dp, c_dp, ctypes.POINTER(c_dp)],
    "sk_ipc_close": [c_dp, c_dp],
    "sk_rand_lupp": [c_dp, c_dp, c_int, c_i64, c_i64, c_i64, c_i64, c_int, ctypes.c_int32, ctypes.c_uint64,
                     c_i64, c_dp, c_dp, ctypes.POINTER(c_i64)],
}
_VOID = {"sk_destroy": [c_dp]}
_OTHER = {
    "sk_last_error": ([c_dp], ctypes.c_char_p),
    "sk_version": ([], ctypes.c_char_p),
    "sk_workspace_bytes": ([c_dp], c_i64),
    "sk_launch_count": ([c_dp], c_i64),
    "sk_lupp_dist_state_bytes": ([c_i64, c_i64], ctypes.c_size_t),
    "sk_lupp_dist_mailbox_bytes": ([c_i64, ctypes.c_int32], ctypes.c_size_t),
}

# every symbol include/skel.h declares
EXPORTS = sorted(list(_SIGS) + list(_VOID) + list(_OTHER))

_lib = None


def load(path=LIB_PATH):
    """Load libskel.so and attach prototypes.  Raises OSError if the library is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"{path} not found: build it with `python -m paper_2104_05877_b200.build` "
                      "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = c_int
    for name, args in _VOID.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = None
    for name, (args, res) in _OTHER.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib
