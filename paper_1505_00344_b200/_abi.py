"""ctypes declarations of include/fireflies.h (argument marshalling only).

The product path is libfireflies.so; if it cannot be loaded this module raises -- there is no
CPU or Python fallback for any step of the hot path.
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfireflies.so")

FF_OK, FF_ERR_INVALID_ARG, FF_ERR_PARSE, FF_ERR_UNKNOWN_SYMBOL, FF_ERR_RANGE, FF_ERR_COMPILE, FF_ERR_CUDA, \
    FF_ERR_OOM, FF_ERR_STATE = range(9)
STATUS_NAMES = ["FF_OK", "FF_ERR_INVALID_ARG", "FF_ERR_PARSE", "FF_ERR_UNKNOWN_SYMBOL", "FF_ERR_RANGE",
                "FF_ERR_COMPILE", "FF_ERR_CUDA", "FF_ERR_OOM", "FF_ERR_STATE"]
FF_TILE = 512
FF_MAX_DIM = 64
FF_MAX_PARAMS = 128
FF_MAX_GROUPS = 16
FF_MAX_PEERS = 8

# Every symbol include/fireflies.h declares (checked by tests/test_abi.py).
EXPORTS = ["ff_last_error", "ff_abi_version", "ff_build_info", "ff_emit_source", "ff_compile_cubin", "ff_create", "ff_destroy",
           "ff_set_stream", "ff_set_shard", "ff_shard_range", "ff_bind_state", "ff_group_slots", "ff_init_group", "ff_group_info",
           "ff_set_param", "ff_get_param", "ff_sweep_param", "ff_project", "ff_step", "ff_set_reset",
           "ff_read_epochs", "ff_read_lifted", "ff_set_launch",
           "ff_read_state", "ff_write_state", "ff_read_image", "ff_render", "ff_project_colour", "ff_launch_count", "ff_sync",
           "ff_set_exchange", "ff_set_exchange_multicast", "ff_set_exchange_push", "ff_set_grid_limit", "ff_write_state_async", "ff_read_image_async"]


class FFError(RuntimeError):
    def __init__(self, status, message):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {message}")


class ff_system(C.Structure):
    _fields_ = [("dim", C.c_int), ("var_names", C.POINTER(C.c_char_p)), ("rhs", C.POINTER(C.c_char_p)),
                ("n_params", C.c_int), ("param_names", C.POINTER(C.c_char_p)),
                ("param_default", C.POINTER(C.c_float)), ("param_min", C.POINTER(C.c_float)),
                ("param_max", C.POINTER(C.c_float))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(the CUDA path has no fallback)")
        L = C.CDLL(LIB_PATH)
        P, i64, u64, f32, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_float, C.c_int
        sysp = C.POINTER(ff_system)
        sig = {
            "ff_last_error": ([], C.c_char_p),
            "ff_abi_version": ([], C.c_int),
            "ff_build_info": ([P, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
            "ff_emit_source": ([sysp, i32, P, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
            "ff_compile_cubin": ([sysp, i32, P, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
            "ff_create": ([sysp, i32, C.POINTER(P)], C.c_int),
            "ff_destroy": ([P], C.c_int),
            "ff_set_stream": ([P, P], C.c_int),
            "ff_set_shard": ([P, i32, i32], C.c_int),
            "ff_shard_range": ([i64, i32, i32, C.POINTER(i64), C.POINTER(i64)], C.c_int),
            "ff_bind_state": ([P, P, i64, i64], C.c_int),
            "ff_group_slots": ([P, i64, C.POINTER(i64)], C.c_int),
            "ff_init_group": ([P, P, P, i64, i32, i32, u64, C.POINTER(i32)], C.c_int),
            "ff_group_info": ([P, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)], C.c_int),
            "ff_set_param": ([P, C.c_char_p, f32], C.c_int),
            "ff_get_param": ([P, C.c_char_p, C.POINTER(f32)], C.c_int),
            "ff_sweep_param": ([P, i32, C.c_char_p, f32, f32, i32, u64], C.c_int),
            "ff_project": ([P, P, i32, P, i32, i32, i32, P], C.c_int),
            "ff_step": ([P, i64, f32], C.c_int),
            "ff_set_reset": ([P, i32, P, P, f32], C.c_int),
            "ff_read_epochs": ([P, i32, i64, i64, P], C.c_int),
            "ff_read_lifted": ([P, i32, i64, i64, P], C.c_int),
            "ff_set_launch": ([P, i32, i32], C.c_int),
            "ff_read_state": ([P, i32, i64, i64, P], C.c_int),
            "ff_write_state": ([P, i32, i64, i64, P], C.c_int),
            "ff_read_image": ([P, P], C.c_int),
            "ff_render": ([P, P, f32, f32, P], C.c_int),
            "ff_project_colour": ([P, P, P, P], C.c_int),
            "ff_launch_count": ([P, C.POINTER(i64)], C.c_int),
            "ff_sync": ([P], C.c_int),
            "ff_set_exchange": ([P, i32, i32, P, P, C.c_double], C.c_int),
            "ff_set_exchange_multicast": ([P, P], C.c_int),
            "ff_set_exchange_push": ([P, i32, P], C.c_int),
            "ff_set_grid_limit": ([P, i32], C.c_int),
            "ff_write_state_async": ([P, i32, i64, i64, P], C.c_int),
            "ff_read_image_async": ([P, P], C.c_int),
        }
        assert set(sig) == set(EXPORTS)
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def check(status):
    if status != FF_OK:
        raise FFError(status, lib().ff_last_error().decode(errors="replace"))
    return status


def make_system(var_names, rhs, params):
    """Build an ff_system from names, rhs strings and [(name, default, min, max)] (None = unbounded).

    Returns (struct, keepalive) -- keep the second element alive while the struct is in use."""
    dim = len(var_names)
    assert len(rhs) == dim
    vn = (C.c_char_p * dim)(*[v.encode() for v in var_names])
    rh = (C.c_char_p * dim)(*[r.encode() for r in rhs])
    n = len(params)
    pn = (C.c_char_p * max(n, 1))(*[p[0].encode() for p in params])
    pd = (C.c_float * max(n, 1))(*[p[1] for p in params])
    inf = float("inf")
    pmin = (C.c_float * max(n, 1))(*[(-inf if p[2] is None else p[2]) if len(p) > 2 else -inf for p in params])
    pmax = (C.c_float * max(n, 1))(*[(inf if p[3] is None else p[3]) if len(p) > 3 else inf for p in params])
    s = ff_system(dim, vn, rh, n, pn, pd, pmin, pmax)
    return s, (vn, rh, pn, pd, pmin, pmax)
