"""ctypes binding of oracle/kernels.c -- TEST INFRASTRUCTURE ONLY.

Builds oracle/_build/liboracle.so with the committed Makefile when missing
(gcc is present both here and on the GPU box).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_d = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64 = ctypes.c_int64


def build() -> str:
    src = os.path.join(_HERE, "kernels.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.or_affine_rows.argtypes = [_d, _d, _d, _i64, _i64, _i64, _d]
        L.or_relu.argtypes = [_d, _i64, _d]
        L.or_output_delta.argtypes = [_d, _i64p, _d, _i64, _i64, _d]
        L.or_weight_grad.argtypes = [_d, _d, _i64, _i64, _i64, _d]
        L.or_bias_grad.argtypes = [_d, _i64, _i64, _d]
        L.or_hidden_delta.argtypes = [_d, _d, _d, _i64, _i64, _i64, _d]
        L.or_rmsprop_flat.argtypes = [_d, _d, _d, _d, _i64, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double, _d, _d, _d]
        L.or_pcg64_random.argtypes = [_u64p]
        L.or_pcg64_random.restype = ctypes.c_double
        L.or_pcg64_integers.argtypes = [_u64p, ctypes.c_uint64, _i64, _i64p]
        L.or_pcg64_integers.restype = ctypes.c_int
        L.or_select_action.argtypes = [_u64p, _d, _i64, ctypes.c_double]
        L.or_select_action.restype = ctypes.c_int64
        L.or_set_threads.argtypes = [ctypes.c_int]
        L.or_get_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t=_d):
    return a.ctypes.data_as(t)


# --- the reference kernel module contract -------------------

BACKEND_NAME = "oracle-c"


def affine_rows(w, b, x):
    w, b, x = _f64(w), _f64(b), _f64(x)
    n, d = x.shape
    o = w.shape[0]
    out = np.empty((n, o), dtype=np.float64)
    lib().or_affine_rows(_p(w), _p(b), _p(x), n, o, d, _p(out))
    return out


def relu(x):
    x = _f64(x)
    out = np.empty_like(x)
    lib().or_relu(_p(x), x.size, _p(out))
    return out


def output_delta(q, actions, targets):
    q = _f64(q)
    a = np.ascontiguousarray(actions, dtype=np.int64)
    t = _f64(targets)
    n, o = q.shape
    out = np.empty_like(q)
    lib().or_output_delta(_p(q), _p(a, _i64p), _p(t), n, o, _p(out))
    return out


def weight_grad(delta, acts):
    delta, acts = _f64(delta), _f64(acts)
    n, o = delta.shape
    d = acts.shape[1]
    out = np.empty((o, d), dtype=np.float64)
    lib().or_weight_grad(_p(delta), _p(acts), n, o, d, _p(out))
    return out


def bias_grad(delta):
    delta = _f64(delta)
    n, o = delta.shape
    out = np.empty(o, dtype=np.float64)
    lib().or_bias_grad(_p(delta), n, o, _p(out))
    return out


def hidden_delta(delta, w, pre):
    delta, w, pre = _f64(delta), _f64(w), _f64(pre)
    n, o = delta.shape
    d = w.shape[1]
    out = np.empty((n, d), dtype=np.float64)
    lib().or_hidden_delta(_p(delta), _p(w), _p(pre), n, o, d, _p(out))
    return out


def rmsprop_flat(p, g, m, v, lr, rho, kappa):
    p, g, m, v = _f64(p), _f64(g), _f64(m), _f64(v)
    p2, m2, v2 = np.empty_like(p), np.empty_like(p), np.empty_like(p)
    lib().or_rmsprop_flat(_p(p), _p(g), _p(m), _p(v), p.size, lr, rho, kappa,
                          _p(p2), _p(m2), _p(v2))
    return p2, m2, v2


# --- PCG64 restatement ---------------------------------------------------------

def pcg_state_from_generator(rng: np.random.Generator) -> np.ndarray:
    """numpy Generator(PCG64) state -> u64[6] (state hi/lo, inc hi/lo, has32, u32)."""
    st = rng.bit_generator.state
    if st["bit_generator"] != "PCG64":
        raise ValueError("only PCG64 generators are supported")
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m, st["has_uint32"], st["uinteger"]],
                    dtype=np.uint64)


def pcg_state_to_generator(state: np.ndarray, rng: np.random.Generator) -> None:
    s = [int(v) for v in state]
    rng.bit_generator.state = {
        "bit_generator": "PCG64",
        "state": {"state": (s[0] << 64) | s[1], "inc": (s[2] << 64) | s[3]},
        "has_uint32": s[4],
        "uinteger": s[5],
    }


def pcg64_integers(state: np.ndarray, n: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.int64)
    rc = lib().or_pcg64_integers(_p(state, _u64p), n, count, _p(out, _i64p))
    if rc != 0:
        raise ValueError("n out of the 32-bit Lemire range")
    return out


def pcg64_random(state: np.ndarray) -> float:
    return lib().or_pcg64_random(_p(state, _u64p))


def select_action(state: np.ndarray, q_row, eps: float) -> int:
    q = _f64(q_row)
    return int(lib().or_select_action(_p(state, _u64p), _p(q), q.size, eps))
