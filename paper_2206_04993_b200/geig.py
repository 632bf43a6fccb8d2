"""Thin ctypes binding of include/geig.h (argument marshalling only).

Every function has the C name and forwards to libgeig.so; torch tensors are
accepted for device / host buffers and passed as raw pointers after shape,
dtype, device and contiguity checks.  There is no Python or CPU fallback:
if the shared library is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgeig.so")

GEIG_OK, GEIG_ERR_ARG, GEIG_ERR_CUDA, GEIG_ERR_UNSUPPORTED, GEIG_ERR_STATE = range(5)
GEIG_DENSE, GEIG_CCA = 0, 1
GEIG_MATH_F32, GEIG_MATH_BF16, GEIG_MATH_TF32, GEIG_MATH_3XTF32, GEIG_MATH_BF16X2 = 0, 1, 2, 3, 4
GEIG_DATA_F32, GEIG_DATA_BF16 = 0, 1
GEIG_OPT_FUSED_M_TILES, GEIG_OPT_STAGED_PRODUCTS, GEIG_OPT_SMALL_STEP, GEIG_OPT_FUSED_PAIRS, GEIG_OPT_GRAM_TC, \
    GEIG_OPT_SMALL_CLUSTER = 1, 2, 3, 4, 5, 6

MATH_NAMES = {"f32": GEIG_MATH_F32, "bf16": GEIG_MATH_BF16, "tf32": GEIG_MATH_TF32,
              "3xtf32": GEIG_MATH_3XTF32, "bf16x2": GEIG_MATH_BF16X2}


class GeigError(RuntimeError):
    pass


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: the sm_100a CUDA library has not been built "
                      "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                      "there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)
_vp, _i64, _i32, _f32, _f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float, ctypes.c_double
_SIGS = {
    "geig_create": [ctypes.POINTER(_vp), ctypes.c_int, _i64, _i64, _i32, ctypes.c_int, ctypes.c_int,
                    _f64, _i64, ctypes.c_int],
    "geig_destroy": [_vp],
    "geig_set_stream": [_vp, _vp],
    "geig_sync": [_vp],
    "geig_init_state": [_vp, _vp],
    "geig_set_state": [_vp, _vp, _vp],
    "geig_get": [_vp, _vp, _vp],
    "geig_products_cca": [_vp, _vp, _vp, _i64, _f32, _vp, _vp],
    "geig_products_dense": [_vp, _vp, _vp, _i64, _i64, _vp, _vp],
    "geig_update": [_vp, _vp, _vp, _f64, _f64],
    "geig_products_cca_tables": [_vp, _vp, _vp, _i64, _f32, _vp, _vp, _vp],
    "geig_update_tables": [_vp, _vp, _vp, _vp, _f64, _f64],
    "geig_step_cca": [_vp, _vp, _vp, _i64, _f64, _f64],
    "geig_step_dense": [_vp, _vp, _vp, _f64, _f64],
    "geig_run_dense": [_vp, _vp, _vp, _i64, _f64, _f64],
    "geig_run_cca": [_vp, _vp, _vp, _i64, _i64, _f64, _f64],
    "geig_set_smooth": [_vp, _f64],
    "geig_smooth_state": [_vp, _vp, _vp],
    "geig_set_adam": [_vp, _f64, _f64, _f64],
    "geig_step_cca_host": [_vp, _vp, _vp, _i64, _f64, _f64, _vp, ctypes.POINTER(_i64),
                           ctypes.POINTER(_i64)],
    "geig_get_gram": [_vp, _vp, _vp, _vp],
    "geig_run_cca_host": [_vp, _vp, _vp, _i64, _i64, _f64, _f64, _vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
    "geig_update_phase_ns": [_vp, ctypes.POINTER(_i64)],
    "geig_set_option": [_vp, ctypes.c_int, _i64],
    "geig_set_partition": [_vp, ctypes.c_int, ctypes.c_int],
    "geig_shadow_buffer": [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_i64)],
    "geig_products_cca_owned": [_vp, _vp, _vp, _i64, _f32, _vp],
    "geig_update_owned": [_vp, _vp, _f64, _f64],
    "geig_peer_buffers": [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_i64), ctypes.POINTER(_vp), ctypes.POINTER(_i64)],
    "geig_set_peers": [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp)],
    "geig_step_cca_peer": [_vp, _vp, _vp, _i64, _f32, _f64, _f64],
    "geig_products_cca_peer": [_vp, _vp, _vp, _i64, _f32],
    "geig_update_peer": [_vp, _f64, _f64],
    "geig_ipc_handle": [_vp, _vp],
    "geig_ipc_open": [_vp, ctypes.POINTER(_vp)],
    "geig_ipc_close": [_vp],
}
for _name, _args in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = ctypes.c_int
_lib.geig_table_floats.argtypes = [_vp]
_lib.geig_table_floats.restype = _i64
_lib.geig_owned_chunk_floats.argtypes = [_vp]
_lib.geig_owned_chunk_floats.restype = _i64
_lib.geig_launch_count.argtypes = [_vp]
_lib.geig_launch_count.restype = _i64
_lib.geig_last_error.restype = ctypes.c_char_p
_lib.geig_version.restype = ctypes.c_char_p

EXPORTED = ["geig_create", "geig_destroy", "geig_set_stream", "geig_sync", "geig_init_state",
            "geig_set_state", "geig_get", "geig_products_cca", "geig_products_dense", "geig_update",
            "geig_step_cca", "geig_step_dense", "geig_run_dense", "geig_run_cca", "geig_step_cca_host", "geig_run_cca_host", "geig_get_gram",
            "geig_set_smooth", "geig_smooth_state", "geig_set_adam",
            "geig_launch_count", "geig_last_error", "geig_version", "geig_update_phase_ns",
            "geig_table_floats", "geig_products_cca_tables", "geig_update_tables", "geig_set_option",
            "geig_set_partition", "geig_owned_chunk_floats", "geig_shadow_buffer", "geig_products_cca_owned",
            "geig_update_owned", "geig_peer_buffers", "geig_set_peers", "geig_step_cca_peer", "geig_products_cca_peer", "geig_update_peer", "geig_ipc_handle",
            "geig_ipc_open", "geig_ipc_close"]


def _check(st: int):
    if st != GEIG_OK:
        raise GeigError(f"geig status {st}: {_lib.geig_last_error().decode()}")


def _ptr(t, dtype=None, device=True, numel=None):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"expected dtype {dtype}, got {t.dtype}")
    if device and not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not device and t.is_cuda:
        raise ValueError("expected a host tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"expected {numel} elements, got {t.numel()}")
    return ctypes.c_void_p(t.data_ptr())


def geig_version() -> str:
    return _lib.geig_version().decode()


def geig_last_error() -> str:
    return _lib.geig_last_error().decode()


def geig_create(problem: int, dx: int, dy: int, k: int, math: int, data_dtype: int, rho: float,
                max_rows: int = 0, device: int = 0):
    h = ctypes.c_void_p()
    _check(_lib.geig_create(ctypes.byref(h), problem, dx, dy, k, math, data_dtype, rho, max_rows, device))
    return h


def geig_destroy(h):
    _check(_lib.geig_destroy(h))


def geig_set_stream(h, stream: int | None):
    _check(_lib.geig_set_stream(h, ctypes.c_void_p(stream or 0)))


def geig_sync(h):
    _check(_lib.geig_sync(h))


def geig_init_state(h, G):
    _check(_lib.geig_init_state(h, _ptr(G, torch.float32)))


def geig_set_state(h, V, AUX=None):
    _check(_lib.geig_set_state(h, _ptr(V, torch.float32), _ptr(AUX, torch.float32)))


def geig_get(h, V=None, AUX=None):
    _check(_lib.geig_get(h, _ptr(V, torch.float32), _ptr(AUX, torch.float32)))


def geig_products_cca(h, X, Y, b: int, scale: float, AV, BV):
    _check(_lib.geig_products_cca(h, _ptr(X), _ptr(Y), b, scale, _ptr(AV, torch.float32),
                                  _ptr(BV, torch.float32)))


def geig_products_dense(h, A, B, r0: int, r1: int, AV, BV):
    _check(_lib.geig_products_dense(h, _ptr(A), _ptr(B), r0, r1, _ptr(AV, torch.float32),
                                    _ptr(BV, torch.float32)))


def geig_update(h, AV, BV, eta: float, gamma: float):
    _check(_lib.geig_update(h, _ptr(AV, torch.float32), _ptr(BV, torch.float32), eta, gamma))


def geig_table_floats(h) -> int:
    return int(_lib.geig_table_floats(h))


def geig_products_cca_tables(h, X, Y, b: int, scale: float, AV, BV, T):
    _check(_lib.geig_products_cca_tables(h, _ptr(X), _ptr(Y), b, scale, _ptr(AV, torch.float32),
                                         _ptr(BV, torch.float32), _ptr(T, torch.float32)))


def geig_update_tables(h, AV, BV, T, eta: float, gamma: float):
    _check(_lib.geig_update_tables(h, _ptr(AV, torch.float32), _ptr(BV, torch.float32), _ptr(T, torch.float32),
                                   eta, gamma))


def geig_step_cca(h, X, Y, b: int, eta: float, gamma: float):
    _check(_lib.geig_step_cca(h, _ptr(X), _ptr(Y), b, eta, gamma))


def geig_set_smooth(h, nu: float):
    _check(_lib.geig_set_smooth(h, nu))


def geig_smooth_state(h, z_in=None, z_out=None):
    _check(_lib.geig_smooth_state(h, _ptr(z_in, torch.float32), _ptr(z_out, torch.float32)))


def geig_set_adam(h, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8):
    _check(_lib.geig_set_adam(h, b1, b2, eps))


def cca_batches(Xs, Ys):
    """Marshal the minibatch lists of geig_run_cca once (device tensors):
    returns (n, X pointer array, Y pointer array)."""
    if len(Xs) != len(Ys):
        raise ValueError("Xs and Ys must have the same length")
    n = len(Xs)
    xa = (ctypes.c_void_p * max(n, 1))(*[_ptr(x).value for x in Xs])
    ya = (ctypes.c_void_p * max(n, 1))(*[_ptr(y).value for y in Ys])
    return n, xa, ya


def geig_run_cca(h, Xs, Ys, b: int, eta: float, gamma: float, batches=None):
    """nsteps = len(Xs) steps, step i on (Xs[i], Ys[i]) (device tensors);
    `batches` = a cca_batches(Xs, Ys) result to skip the marshalling."""
    n, xa, ya = batches if batches is not None else cca_batches(Xs, Ys)
    _check(_lib.geig_run_cca(h, ctypes.cast(xa, ctypes.c_void_p), ctypes.cast(ya, ctypes.c_void_p), b, n, eta,
                             gamma))


def geig_step_dense(h, A, B, eta: float, gamma: float):
    _check(_lib.geig_step_dense(h, _ptr(A), _ptr(B), eta, gamma))


def geig_run_dense(h, A, B, nsteps: int, eta: float, gamma: float):
    _check(_lib.geig_run_dense(h, _ptr(A), _ptr(B), nsteps, eta, gamma))


def geig_step_cca_host(h, X_host, Y_host, b: int, eta: float, gamma: float, ga_host=None):
    h2d, d2h = _i64(0), _i64(0)
    _check(_lib.geig_step_cca_host(h, _ptr(X_host, device=False), _ptr(Y_host, device=False), b, eta,
                                   gamma, _ptr(ga_host, torch.float32, device=False),
                                   ctypes.byref(h2d), ctypes.byref(d2h)))
    return h2d.value, d2h.value


def geig_run_cca_host(h, Xs_host, Ys_host, b: int, eta: float, gamma: float, ga_host=None):
    """T steps from pinned host batches (lists of tensors); returns (h2d, d2h) bytes."""
    n = len(Xs_host)
    if len(Ys_host) != n:
        raise ValueError("Xs_host and Ys_host differ in length")
    xs = (_vp * n)(*[_ptr(x, device=False) for x in Xs_host])
    ys = (_vp * n)(*[_ptr(y, device=False) for y in Ys_host])
    h2d, d2h = _i64(0), _i64(0)
    _check(_lib.geig_run_cca_host(h, xs, ys, b, n, eta, gamma, _ptr(ga_host, torch.float32, device=False),
                                  ctypes.byref(h2d), ctypes.byref(d2h)))
    return h2d.value, d2h.value


def geig_get_gram(h, GA=None, GB=None, GC=None):
    _check(_lib.geig_get_gram(h, _ptr(GA, torch.float32), _ptr(GB, torch.float32), _ptr(GC, torch.float32)))


def geig_set_option(h, option: int, value: int):
    _check(_lib.geig_set_option(h, option, value))


def geig_set_partition(h, world: int, rank: int):
    _check(_lib.geig_set_partition(h, world, rank))


def geig_owned_chunk_floats(h) -> int:
    return int(_lib.geig_owned_chunk_floats(h))


def geig_shadow_buffer(h):
    """(device pointer, bytes per rank) of the gathered bf16 shadow."""
    p, n = _vp(), _i64(0)
    _check(_lib.geig_shadow_buffer(h, ctypes.byref(p), ctypes.byref(n)))
    return p.value, n.value


def geig_products_cca_owned(h, X, Y, b: int, scale: float, buf):
    _check(_lib.geig_products_cca_owned(h, _ptr(X), _ptr(Y), b, scale, _ptr(buf, torch.float32)))


def geig_update_owned(h, chunk, eta: float, gamma: float):
    _check(_lib.geig_update_owned(h, _ptr(chunk, torch.float32), eta, gamma))


def geig_peer_buffers(h):
    """(recv_ptr, recv_bytes, flags_ptr, flags_bytes) of this rank (device)."""
    r, f = _vp(), _vp()
    rb, fb = _i64(), _i64()
    _check(_lib.geig_peer_buffers(h, ctypes.byref(r), ctypes.byref(rb), ctypes.byref(f), ctypes.byref(fb)))
    return r.value, rb.value, f.value, fb.value


def geig_set_peers(h, recv_ptrs, shadow_ptrs, flag_ptrs):
    """Arrays of `world` device pointers (ints), entry `rank` = own buffers."""
    n = len(recv_ptrs)
    arr = lambda xs: (_vp * n)(*[_vp(int(x)) for x in xs])
    _check(_lib.geig_set_peers(h, arr(recv_ptrs), arr(shadow_ptrs), arr(flag_ptrs)))


def geig_step_cca_peer(h, X, Y, b: int, scale: float, eta: float, gamma: float):
    _check(_lib.geig_step_cca_peer(h, _ptr(X), _ptr(Y), b, scale, eta, gamma))


def geig_products_cca_peer(h, X, Y, b: int, scale: float):
    _check(_lib.geig_products_cca_peer(h, _ptr(X), _ptr(Y), b, scale))


def geig_update_peer(h, eta: float, gamma: float):
    _check(_lib.geig_update_peer(h, eta, gamma))


def geig_ipc_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(_lib.geig_ipc_handle(_vp(int(ptr)), buf))
    return buf.raw


def geig_ipc_open(handle: bytes) -> int:
    out = _vp()
    _check(_lib.geig_ipc_open(ctypes.create_string_buffer(bytes(handle), 64), ctypes.byref(out)))
    return out.value


def geig_ipc_close(ptr: int):
    _check(_lib.geig_ipc_close(_vp(int(ptr))))


def geig_update_phase_ns(h):
    out = (_i64 * 5)()
    _check(_lib.geig_update_phase_ns(h, out))
    return list(out)


def geig_launch_count(h) -> int:
    return int(_lib.geig_launch_count(h))


class Solver:
    """Convenience owner of a geig_solver handle (marshalling only)."""

    def __init__(self, problem, dx, dy, k, math="f32", data_dtype=GEIG_DATA_F32, rho=0.0,
                 max_rows=0, device=0, stream=None):
        self.problem, self.dx, self.dy, self.k = problem, dx, dy, k
        self.d = dx + dy
        self.device = device
        self.math = MATH_NAMES[math] if isinstance(math, str) else math
        self.h = geig_create(problem, dx, dy, k, self.math, data_dtype, rho, max_rows, device)
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        geig_set_stream(self.h, stream)

    def close(self):
        if self.h is not None:
            geig_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init_state(self, G):
        geig_init_state(self.h, G)

    def set_state(self, V, AUX=None):
        geig_set_state(self.h, V, AUX)

    def state(self):
        V = torch.empty(self.k, self.d, device=f"cuda:{self.device}")
        AUX = torch.empty_like(V)
        geig_get(self.h, V, AUX)
        geig_sync(self.h)
        return V, AUX

    def gram(self):
        t = [torch.empty(self.k, self.k, device=f"cuda:{self.device}") for _ in range(3)]
        geig_get_gram(self.h, *t)
        geig_sync(self.h)
        return t

    def launches(self):
        return geig_launch_count(self.h)


class _DevArray:
    """__cuda_array_interface__ wrapper (zero-copy torch view of a device
    buffer the library owns)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


def shadow_tensor(h, world: int, k: int, W: int, device: int = 0):
    """The gathered bf16 shadow of a partitioned solver as a torch int16 view
    [world, 2, k, W] (the bytes the all-gather moves; bf16 hi | lo planes)."""
    ptr, nbytes = geig_shadow_buffer(h)
    if nbytes != 2 * k * W * 2:
        raise GeigError(f"shadow block is {nbytes} bytes, expected {2 * k * W * 2}")
    return torch.as_tensor(_DevArray(ptr, (world, 2, k, W), "<i2"), device=f"cuda:{device}")
