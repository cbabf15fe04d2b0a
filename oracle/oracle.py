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


class _abi:
    """ctypes restatement of the struct layouts in include/pam_c_api.h.

    Defined here, not imported from the product package, so loading the oracle
    never maps libpam.so (bench.py --impl reference must not touch the product).
    tests/test_abi.py checks these layouts against the product's _abi.py."""

    PAM_MAX_T = 16
    PAM_MODE_EXACT, PAM_MODE_POLY = 0, 1
    PAM_RESCALE_AUTO, PAM_RESCALE_STATIC, PAM_RESCALE_NONE = 0, 1, 2
    PAM_ROW_FLAG_TIE = 0x100

    class pam_approx_config(C.Structure):
        _fields_ = [("iterations", C.c_int32), ("alpha_bits", C.c_int32), ("rescale", C.c_int32),
                    ("scale_log2", C.c_int32), ("lo", C.c_double), ("hi", C.c_double)]

    class pam_cutmax_params(C.Structure):
        pass

    class pam_sampler_cfg(C.Structure):
        _fields_ = [("p", C.c_double), ("q", C.c_double), ("alpha", C.c_double), ("seed", C.c_uint64),
                    ("draw", C.c_uint64)]


_abi.pam_cutmax_params._fields_ = [
    ("T", C.c_int32), ("flags", C.c_int32), ("invsqrt_mode", C.c_int32), ("inv_mode", C.c_int32),
    ("p", C.c_int32 * _abi.PAM_MAX_T), ("c", C.c_double * _abi.PAM_MAX_T), ("eps_var", C.c_double),
    ("eps_stop", C.c_double), ("invsqrt", _abi.pam_approx_config * _abi.PAM_MAX_T),
    ("inv", _abi.pam_approx_config)]


def default_params(T: int = 4, p: int = 3, c: float = 5.0, eps_stop: float = 0.0) -> "_abi.pam_cutmax_params":
    """CutMaxParams defaults: p, c broadcast over T,
    eps_var = 1e-24, exact 1/sqrt and 1/S, invsqrt preset alpha=7 (5 Newton
    iterations, Table 3), Goldschmidt d=5, AUTO rescale.  Same
    values as the product's pam_default_params (checked by tests/test_abi.py)."""
    r = _abi.pam_cutmax_params()
    r.T = int(T)
    r.eps_var = 1e-24
    r.eps_stop = float(eps_stop)
    r.invsqrt_mode = _abi.PAM_MODE_EXACT
    r.inv_mode = _abi.PAM_MODE_EXACT
    for t in range(_abi.PAM_MAX_T):
        r.p[t] = int(p)
        r.c[t] = float(c)
        a = r.invsqrt[t]
        a.iterations, a.alpha_bits, a.rescale, a.lo, a.hi = 5, 7, _abi.PAM_RESCALE_AUTO, 0.25, 1.0
    r.inv.iterations, r.inv.alpha_bits, r.inv.rescale, r.inv.lo, r.inv.hi = 5, 7, _abi.PAM_RESCALE_AUTO, 0.5, 1.0
    return r


def _as(struct_type, v):
    """Accept the product's ctypes structs too (same layout, different class):
    tests lower parameters with the product's front end and hand them here."""
    if v is None or isinstance(v, struct_type):
        return v
    return struct_type.from_buffer_copy(bytes(memoryview(v)))


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
    "orc_exp_t": (C.c_double, [C.c_double]),
    "orc_log_t": (C.c_double, [C.c_double]),
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
    "orc_nucleus_set_batch": (C.c_int64, [_P, _I64, _I64, _I64, C.c_double, _P, _P, _P, _P]),
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
    st = lib.orc_cutmax(x.ctypes.data, n, C.byref(_as(_abi.pam_cutmax_params, prm)), z.ctypes.data, C.byref(am), stats.ctypes.data, None)
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
    fn(X.ctypes.data, n, B, n, C.byref(_as(_abi.pam_cutmax_params, prm)), z.ctypes.data, n, am.ctypes.data, st.ctypes.data, nthreads)
    return z, am, st


def sample_batch(X, cfg: _abi.pam_sampler_cfg, prm, gumbel: bool = False, nthreads: int = 0):
    """-> (token, inside, status)"""
    lib = load()
    X = _f64(X)
    B, n = X.shape
    tok = np.empty(B, dtype=np.int32)
    ins = np.empty(B, dtype=np.uint8)
    st = np.empty(B, dtype=np.int32)
    lib.orc_sample_batch(X.ctypes.data, n, B, n, C.byref(_as(_abi.pam_sampler_cfg, cfg)), C.byref(_as(_abi.pam_cutmax_params, prm)), int(gumbel), tok.ctypes.data,
                         ins.ctypes.data, st.ctypes.data, nthreads)
    return tok, ins, st


def nucleus_inside(x, p: float, tok: int) -> bool:
    x = _f64(x)
    return bool(load().orc_nucleus_inside(x.ctypes.data, x.shape[0], p, tok))


def nucleus_set_batch(X, p: float):
    """Top-p nucleus of every row -> (cutoff, size, mass, status)."""
    lib = load()
    X = _f64(X)
    if X.ndim == 1:
        X = X[None, :]
    B, n = X.shape
    cut, mass = np.empty(B), np.empty(B)
    size, st = np.empty(B, dtype=np.int32), np.empty(B, dtype=np.int32)
    lib.orc_nucleus_set_batch(X.ctypes.data, n, B, n, float(p), cut.ctypes.data, size.ctypes.data, mass.ctypes.data,
                              st.ctypes.data)
    return cut, size, mass, st


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
    st = load().orc_convergence_trace(x.ctypes.data, x.shape[0], C.byref(_as(_abi.pam_cutmax_params, prm)), out.ctypes.data)
    return st, out


def cutmax_jvp(x, v, prm):
    """-> (status, z, dz): forward-mode JVP of cutmax at x in direction v."""
    x = _f64(x)
    v = _f64(v)
    z = np.empty_like(x)
    dz = np.empty_like(x)
    st = load().orc_cutmax_jvp(x.ctypes.data, v.ctypes.data, x.shape[0], C.byref(_as(_abi.pam_cutmax_params, prm)), z.ctypes.data, dz.ctypes.data)
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
    st = fn(x, C.byref(_as(_abi.pam_approx_config, cfg)), C.byref(out))
    return st, out.value
