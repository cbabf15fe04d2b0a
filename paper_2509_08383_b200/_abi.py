"""ctypes mirror of include/pam_c_api.h and the loader for libpam.so.

The shared library is the product: sm_100a CUDA kernels behind a C ABI.  It is
built in-tree (``make -C paper_2509_08383_b200/csrc``, or ``__graft_entry__.build()``)
and loading fails loudly when it is missing — there is no Python fallback.
"""
from __future__ import annotations

import ctypes as C
import os

PAM_MAX_T = 16

PAM_OK = 0
PAM_ERR_INVALID_PARAMS = 1
PAM_ERR_DEGENERATE_INPUT = 2
PAM_ERR_RANGE = 3
PAM_ERR_DOMAIN = 4
PAM_ERR_NON_FINITE = 5
PAM_ERR_CUDA = 6
PAM_ERR_BAD_ARGUMENT = 7
PAM_ERR_UNSUPPORTED = 8
PAM_ERR_FORMAT = 9
PAM_ERR_SINGULAR = 10
PAM_ROW_FLAG_TIE = 0x100

PAM_RESCALE_AUTO, PAM_RESCALE_STATIC, PAM_RESCALE_NONE = 0, 1, 2
PAM_MODE_EXACT, PAM_MODE_POLY = 0, 1
PAM_F_UNCHECKED, PAM_F_GUARANTEE, PAM_F_NO_NORMALIZE = 0x1, 0x2, 0x4


class pam_approx_config(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("alpha_bits", C.c_int32),
        ("rescale", C.c_int32),
        ("scale_log2", C.c_int32),
        ("lo", C.c_double),
        ("hi", C.c_double),
    ]


class pam_cutmax_params(C.Structure):
    _fields_ = [
        ("T", C.c_int32),
        ("flags", C.c_int32),
        ("invsqrt_mode", C.c_int32),
        ("inv_mode", C.c_int32),
        ("p", C.c_int32 * PAM_MAX_T),
        ("c", C.c_double * PAM_MAX_T),
        ("eps_var", C.c_double),
        ("eps_stop", C.c_double),
        ("invsqrt", pam_approx_config * PAM_MAX_T),
        ("inv", pam_approx_config),
    ]


class pam_sampler_cfg(C.Structure):
    _fields_ = [
        ("p", C.c_double),
        ("q", C.c_double),
        ("alpha", C.c_double),
        ("seed", C.c_uint64),
        ("draw", C.c_uint64),
    ]


class pam_launch_info(C.Structure):
    _fields_ = [(k, C.c_int32) for k in
                ("threads", "elems_per_thread", "cluster", "clusters", "ctas", "smem_bytes", "tma", "kernel_id",
                 "groups")]


class pam_ingest_info(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("count", "n", "err_offset", "bad_vector")]


_P = C.c_void_p
_I64 = C.c_int64

# name -> (restype, argtypes); every function declared in include/pam_c_api.h
SIGNATURES = {
    "pam_abi_version": (C.c_int, []),
    "pam_status_string": (C.c_char_p, [C.c_int]),
    "pam_default_params": (None, [C.POINTER(pam_cutmax_params), C.c_int32, C.c_int32, C.c_double]),
    "pam_validate_cutmax_params": (C.c_int, [C.POINTER(pam_cutmax_params), _I64]),
    "pam_goldschmidt_inv": (C.c_int, [C.c_double, C.POINTER(pam_approx_config), C.POINTER(C.c_double)]),
    "pam_goldschmidt_invsqrt": (C.c_int, [C.c_double, C.POINTER(pam_approx_config), C.POINTER(C.c_double)]),
    "pam_nucleus_alpha": (C.c_int, [C.c_double, C.c_double, C.POINTER(C.c_double)]),
    "pam_beta_inverse_cdf": (C.c_double, [C.c_double, C.c_double]),
    "pam_gumbel_from_uniform": (C.c_int, [C.c_double, C.POINTER(C.c_double)]),
    "pam_uniform": (C.c_double, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]),
    "pam_cutmax_batch_f64": (C.c_int, [_P, _I64, _I64, _I64, C.POINTER(pam_cutmax_params), _P, _I64, _P, _P, _P, _P]),
    "pam_cutmax_batch_f32": (C.c_int, [_P, _I64, _I64, _I64, C.POINTER(pam_cutmax_params), _P, _I64, _P, _P, _P, _P]),
    "pam_cutmax_batch_host_f64": (C.c_int, [_P, _I64, _I64, C.POINTER(pam_cutmax_params), _P, _P, _P]),
    "pam_cutmax_batch_host_f32": (C.c_int, [_P, _I64, _I64, C.POINTER(pam_cutmax_params), _P, _P, _P]),
    "pam_nucleus_sample_batch_f64": (C.c_int, [_P, _I64, _I64, _I64, C.POINTER(pam_sampler_cfg),
                                               C.POINTER(pam_cutmax_params), _P, _P, _P, _I64, _P, _P]),
    "pam_gumbel_sample_batch_f64": (C.c_int, [_P, _I64, _I64, _I64, C.POINTER(pam_sampler_cfg),
                                              C.POINTER(pam_cutmax_params), _P, _P, _P, _I64, _P, _P]),
    "pam_nucleus_set_batch_f64": (C.c_int, [_P, _I64, _I64, _I64, C.c_double, _P, _P, _P, _P, _P]),
    "pam_query_launch": (C.c_int, [C.c_int, _I64, _I64, C.POINTER(pam_cutmax_params), C.POINTER(pam_launch_info)]),
    "pam_kernel_launch_count": (C.c_int64, []),
    "pam_last_cuda_error": (C.c_char_p, []),
    "pam_set_trace_buffer": (None, [_P, _I64]),
    "pam_set_geometry_override": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "pam_set_lean_p3": (C.c_int, [C.c_int]),
    "pam_set_host_chunk_bytes": (C.c_int, [_I64]),
    "pam_convergence_trace_batch_f64": (C.c_int, [_P, _I64, _I64, _I64, C.POINTER(pam_cutmax_params), _P, _P, _P]),
    "pam_cutmax_jvp_batch_f64": (C.c_int, [_P, _P, _I64, _I64, _I64, C.POINTER(pam_cutmax_params), _P, _P, _I64,
                                           _P, _P]),
    "pam_lgt1_probe": (C.c_int, [C.c_char_p, C.POINTER(pam_ingest_info)]),
    "pam_lgt1_read": (C.c_int, [C.c_char_p, _P, _I64, C.POINTER(pam_ingest_info)]),
    "pam_lgt1_write": (C.c_int, [C.c_char_p, _P, _I64, _I64]),
    "pam_jsonl_probe": (C.c_int, [C.c_char_p, C.POINTER(pam_ingest_info)]),
    "pam_jsonl_read": (C.c_int, [C.c_char_p, _P, _I64, C.POINTER(pam_ingest_info)]),
}

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PAM_LIB_PATH") or os.path.join(PKG_DIR, "libpam.so")  # override: dev trace build

_lib = None


def load() -> C.CDLL:
    """Load libpam.so (built in-tree).  Raises if it is missing — no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2509_08383_b200/csrc -j)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
