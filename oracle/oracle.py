"""ctypes wrapper of the CPU ORACLE (oracle/liboracle.so).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module; the product never does.  See
oracle.h for what the oracle restates and how it is pinned.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2509_08383_b200 import _abi  # struct layouts of include/pam_c_api.h (types only)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_P = C.c_void_p
_I64 = C.c_int64
_PRM = C.POINTER(_abi.pam_cutmax_params)
_SIG = {
    "orc_ipow": (C.c_double, [C.c_double, C.c_int]),
    "orc_invsqrt_newton": (C.c_double, [C.c_double, C.c_int]),
    "orc_goldschmidt_inv": (C.c_double, [C.c_double, C.c_int]),
    "orc_invsqrt_cfg": (C.c_int, [C.c_double, C.POINTER(_abi.pam_approx_config), C.POINTER(C.c_double)]),
    "orc_inv_cfg": (C.c_int, [C.c_double, C.POINTER(_abi.pam_approx_config), C.POINTER(C.c_double)]),
    "orc_exp": (C.c_double, [C.c_double]),
    "orc_philox": (None, [_P, _P, _P]),
    "orc_log": (C.c_double, [C.c_double]),
    "orc_uniform": (C.c_double, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]),
    "orc_beta_icdf": (C.c_double, [C.c_double, C.c_double]),
    "orc_gumbel": (C.c_double, [C.c_double]),
    "orc_nucleus_alpha": (C.c_double, [C.c_double, C.c_double]),
    "orc_cutmax": (C.c_int, [_P, _I64, _PRM, _P, _P, _P, _P]),
    "orc_cutmax_f32": (C.c_int, [_P, _I64, _PRM, _P, _P, _P]),
    "orc_cutmax_batch": (C.c_int64, [_P, _I64, _I64, _I64, _PRM, _P, _I64, _P, _P, C.c_int]),
    "orc_cutmax_batch_f32": (C.c_int64, [_P, _I64, _I64, _I64, _PRM, _P, _I64, _P, _P, C.c_int]),
    "orc_cutmax_step": (C.c_int, [_P, _I64, C.c_int, C.c_double, C.c_double, _P, _P, _P, _P, _P]),
    "orc_fixed_point_target": (C.c_int, [_I64, C.c_int, C.c_double, _P, _P]),
    "orc_contraction_factor": (C.c_int, [_I64, C.c_int, C.c_double, _P]),
    "orc_convergence_trace": (C.c_int, [_P, _I64, _PRM, _P]),
    "orc_cutmax_jvp": (C.c_int, [_P, _P, _I64, _PRM, _P, _P]),
    "orc_tie_warning": (C.c_int, [_P, _I64]),
    "orc_nucleus_inside": (C.c_int, [_P, _I64, C.c_double, _I64]),
    "orc_sample": (C.c_int, [_P, _I64, C.POINTER(_abi.pam_sampler_cfg), _PRM, C.c_uint64, C.c_int, _P, _P, _P]),
    "orc_sample_batch": (C.c_int64, [_P, _I64, _I64, _I64, C.POINTER(_abi.pam_sampler_cfg), _PRM, C.c_int, _P, _P,
                                     _P, C.c_int]),
}

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        lib = C.CDLL(LIB_PATH)
        for k, (r, a) in _SIG.items():
            f = getattr(lib, k)
            f.restype = r
            f.argtypes = a
        _lib = lib
    return _lib


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def cutmax(x, prm: _abi.pam_cutmax_params):
    """-> (status, z, argmax, stats[T,2])"""
    lib = load()
    x = _f64(x)
    n = x.shape[-1]
    z = np.empty(n)
    am = C.c_int32(-1)
    stats = np.zeros((prm.T, 2))
    st = lib.orc_cutmax(x.ctypes.data, n, C.byref(prm), z.ctypes.data, C.byref(am), stats.ctypes.data, None)
    return st, z, am.value, stats


def cutmax_batch(X, prm, nthreads: int = 0):
    """-> (z, argmax, status)"""
    lib = load()
    X = np.asarray(X)
    if X.dtype == np.float32:
        X = np.ascontiguousarray(X)
        fn = lib.orc_cutmax_batch_f32
    else:
        X = _f64(X)
        fn = lib.orc_cutmax_batch
    B, n = X.shape
    z = np.empty_like(X)
    am = np.empty(B, dtype=np.int32)
    st = np.empty(B, dtype=np.int32)
    fn(X.ctypes.data, n, B, n, C.byref(prm), z.ctypes.data, n, am.ctypes.data, st.ctypes.data, nthreads)
    return z, am, st


def sample_batch(X, cfg: _abi.pam_sampler_cfg, prm, gumbel: bool = False, nthreads: int = 0):
    """-> (token, inside, status)"""
    lib = load()
    X = _f64(X)
    B, n = X.shape
    tok = np.empty(B, dtype=np.int32)
    ins = np.empty(B, dtype=np.uint8)
    st = np.empty(B, dtype=np.int32)
    lib.orc_sample_batch(X.ctypes.data, n, B, n, C.byref(cfg), C.byref(prm), int(gumbel), tok.ctypes.data,
                         ins.ctypes.data, st.ctypes.data, nthreads)
    return tok, ins, st


def nucleus_inside(x, p: float, tok: int) -> bool:
    x = _f64(x)
    return bool(load().orc_nucleus_inside(x.ctypes.data, x.shape[0], p, tok))


def cutmax_step(y, p: int, c: float, eps_var: float = 1e-24):
    """-> (status, next, residuals, mu, s2, dispersion)"""
    lib = load()
    y = _f64(y)
    n = y.shape[0]
    nx, r = np.empty(n), np.empty(n)
    mu, s2, d = C.c_double(), C.c_double(), C.c_double()
    st = lib.orc_cutmax_step(y.ctypes.data, n, p, c, eps_var, nx.ctypes.data, r.ctypes.data, C.byref(mu),
                             C.byref(s2), C.byref(d))
    return st, nx, r, mu.value, s2.value, d.value


def fixed_point_target(n: int, p: int, c: float):
    """-> (status, vector, s_star)"""
    out = np.empty(n)
    s = C.c_double()
    st = load().orc_fixed_point_target(n, p, c, out.ctypes.data, C.byref(s))
    return st, out, s.value


def contraction_factor(n: int, p: int, c: float):
    k = C.c_double()
    st = load().orc_contraction_factor(n, p, c, C.byref(k))
    return st, k.value


def convergence_trace(x, prm):
    x = _f64(x)
    out = np.zeros((prm.T, 4))
    st = load().orc_convergence_trace(x.ctypes.data, x.shape[0], C.byref(prm), out.ctypes.data)
    return st, out


def cutmax_jvp(x, v, prm):
    """-> (status, z, dz): forward-mode JVP of cutmax at x in direction v."""
    x = _f64(x)
    v = _f64(v)
    z = np.empty_like(x)
    dz = np.empty_like(x)
    st = load().orc_cutmax_jvp(x.ctypes.data, v.ctypes.data, x.shape[0], C.byref(prm), z.ctypes.data, dz.ctypes.data)
    return st, z, dz


def tie_warning(x) -> int:
    x = _f64(x)
    return load().orc_tie_warning(x.ctypes.data, x.shape[0])


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    load().orc_philox(c.ctypes.data, k.ctypes.data, o.ctypes.data)
    return [int(v) for v in o]


def scalar(name: str, *args):
    return getattr(load(), "orc_" + name)(*args)


def approx_cfg(x: float, cfg: _abi.pam_approx_config, inv: bool):
    out = C.c_double()
    fn = load().orc_inv_cfg if inv else load().orc_invsqrt_cfg
    st = fn(x, C.byref(cfg), C.byref(out))
    return st, out.value
