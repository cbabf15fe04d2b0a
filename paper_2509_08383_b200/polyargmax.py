"""Python host mirror of the reference's `polyargmax` interface for the CutMax
decoding core (SPEC.md modules `core`, `polyapprox` scalars, `sampling`).

Same operation names, argument meaning and error behaviour as the SPEC:

    cutmax(x, params)                      SPEC.md:60-69   -> ScoreVector
    cutmaxStep(y, p, c)                    SPEC.md:71-79   -> (next, ResidualStats)
    goldschmidtInv(x, cfg)
    goldschmidtInvSqrt(x, cfg)
    gumbelFromUniform(u)
    gumbelMaxSample(x, params, seed)
    betaInverseCdf(u, alpha)
    nucleusAlpha(p, q)
    nucleusOneShotSample(x, cfg, params)

plus batched forms over host arrays (numpy) and device tensors (torch, CUDA).
Every vector operation runs in libpam.so's sm_100a kernels; nothing here
computes on the CPU except argument marshalling.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

import numpy as np

from . import _abi
import warnings

from .errors import DomainError, InvalidParamsError, TieWarning, raise_for_status

_lib = _abi.load()

# ---------------------------------------------------------------- types ----


@dataclass
class ApproxConfig:
    """ApproxConfig.  rescale: 'auto' | 'static' | 'none'."""

    iterations: int = 5
    lo: float = 0.25
    hi: float = 1.0
    alphaBits: int = 7
    rescale: str = "auto"
    scaleLog2: int = 0

    @staticmethod
    def invsqrtPreset(alphaBits: int = 7) -> "ApproxConfig":
        """Table 3: invsqrt iterations 5/6/7/8 for alpha 7/9/11/13."""
        it = 5 if alphaBits <= 7 else 6 if alphaBits <= 9 else 7 if alphaBits <= 11 else 8
        return ApproxConfig(iterations=it, lo=0.25, hi=1.0, alphaBits=alphaBits)

    @staticmethod
    def invPreset(alphaBits: int = 7) -> "ApproxConfig":
        d = 0
        while (1 << (d + 1)) < alphaBits + 1:
            d += 1
        return ApproxConfig(iterations=max(d, 2), lo=0.5, hi=1.0, alphaBits=alphaBits)

    def lower(self) -> _abi.pam_approx_config:
        r = _abi.pam_approx_config()
        r.iterations = int(self.iterations)
        r.alpha_bits = int(self.alphaBits)
        r.rescale = {"auto": _abi.PAM_RESCALE_AUTO, "static": _abi.PAM_RESCALE_STATIC,
                     "none": _abi.PAM_RESCALE_NONE}[self.rescale]
        r.scale_log2 = int(self.scaleLog2)
        r.lo = float(self.lo)
        r.hi = float(self.hi)
        return r


def _sched(v, T, name):
    if isinstance(v, (int, float, np.integer, np.floating)):
        return [v] * T
    v = list(v)
    if len(v) == 1:
        return v * T
    if len(v) != T:
        raise InvalidParamsError(f"{name} schedule must have length 1 or T (SPEC.md:124)")
    return v


@dataclass
class CutMaxParams:
    """CutMaxParams: p odd >= 3, c > 0, T >= 1; scalars broadcast."""

    p: Union[int, Sequence[int]] = 3
    c: Union[float, Sequence[float]] = 5.0
    T: int = 4
    checked: bool = True
    guarantee: bool = False
    normalize: bool = True
    epsVar: float = 1e-24
    epsStop: float = 0.0
    invsqrtMode: str = "exact"  # 'exact' | 'poly'
    invMode: str = "exact"
    invsqrt: Union[ApproxConfig, Sequence[ApproxConfig]] = field(default_factory=ApproxConfig.invsqrtPreset)
    inv: ApproxConfig = field(default_factory=ApproxConfig.invPreset)

    def lower(self) -> _abi.pam_cutmax_params:
        T = int(self.T)
        if T < 1 or T > _abi.PAM_MAX_T:
            raise InvalidParamsError("T must be in [1, 16] (SPEC.md:67: T=0 is invalid)")
        r = _abi.pam_cutmax_params()
        _lib.pam_default_params(C.byref(r), T, 3, 5.0)
        r.flags = ((0 if self.checked else _abi.PAM_F_UNCHECKED) | (_abi.PAM_F_GUARANTEE if self.guarantee else 0)
                   | (0 if self.normalize else _abi.PAM_F_NO_NORMALIZE))
        r.eps_var = float(self.epsVar)
        r.eps_stop = float(self.epsStop)
        r.invsqrt_mode = {"exact": _abi.PAM_MODE_EXACT, "poly": _abi.PAM_MODE_POLY}[self.invsqrtMode]
        r.inv_mode = {"exact": _abi.PAM_MODE_EXACT, "poly": _abi.PAM_MODE_POLY}[self.invMode]
        ps = _sched(self.p, T, "p")
        cs = _sched(self.c, T, "c")
        inv = [self.invsqrt] if isinstance(self.invsqrt, ApproxConfig) else list(self.invsqrt)
        inv = _sched(inv, T, "invsqrt") if len(inv) != 1 else inv * T
        for t in range(T):
            r.p[t] = int(ps[t])
            r.c[t] = float(cs[t])
            r.invsqrt[t] = inv[t].lower()
        r.inv = self.inv.lower()
        return r


@dataclass
class ScoreVector:
    """ScoreVector plus the argmax computed by the kernel and the
    TieWarning flag."""

    values: np.ndarray
    normalized: bool
    argmax: int
    tieWarning: bool = False


@dataclass
class ResidualStats:
    """ResidualStats."""

    mu: float
    s2: float
    residuals: np.ndarray
    dispersion: float


@dataclass
class SamplerConfig:
    """SamplerConfig; alpha <= 0 derives ln(1-q)/ln(p)."""

    p: float = 0.9
    q: Optional[float] = None
    alpha: float = 0.0
    seed: int = 0
    draw: int = 0

    def lower(self) -> _abi.pam_sampler_cfg:
        r = _abi.pam_sampler_cfg()
        r.p = float(self.p)
        r.q = float(self.p if self.q is None else self.q)
        r.alpha = float(self.alpha)
        r.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        r.draw = int(self.draw) & 0xFFFFFFFFFFFFFFFF
        return r


@dataclass
class SampleOutcome:
    """SampleOutcome."""

    onehot: np.ndarray
    tokenIndex: int
    insideNucleus: bool


# ---------------------------------------------------------------- scalars --


def goldschmidtInv(x: float, cfg: Optional[ApproxConfig] = None) -> float:
    cfg = cfg or ApproxConfig(iterations=5, lo=1e-300, hi=2.0, rescale="none")
    out = C.c_double()
    c = cfg.lower()
    raise_for_status(_lib.pam_goldschmidt_inv(float(x), C.byref(c), C.byref(out)), what="goldschmidtInv")
    return out.value


def goldschmidtInvSqrt(x: float, cfg: Optional[ApproxConfig] = None) -> float:
    cfg = cfg or ApproxConfig(iterations=5, lo=1e-300, hi=2.0, rescale="none")
    out = C.c_double()
    c = cfg.lower()
    raise_for_status(_lib.pam_goldschmidt_invsqrt(float(x), C.byref(c), C.byref(out)), what="goldschmidtInvSqrt")
    return out.value


def nucleusAlpha(p: float, q: Optional[float] = None) -> float:
    out = C.c_double()
    raise_for_status(_lib.pam_nucleus_alpha(float(p), float(p if q is None else q), C.byref(out)),
                     what="nucleusAlpha")
    return out.value


def betaInverseCdf(u: float, alpha: float) -> float:
    if not (0.0 <= u <= 1.0) or not (alpha > 0.0):
        raise DomainError("betaInverseCdf needs u in [0,1] and alpha > 0")
    return _lib.pam_beta_inverse_cdf(float(u), float(alpha))


def gumbelFromUniform(u: float) -> float:
    out = C.c_double()
    raise_for_status(_lib.pam_gumbel_from_uniform(float(u), C.byref(out)), what="gumbelFromUniform")
    return out.value


def uniform(seed: int, row: int, draw: int, index: int) -> float:
    """The pinned Philox4x32-10 uniform for (seed, row, draw, element index)."""
    m = 0xFFFFFFFFFFFFFFFF
    return _lib.pam_uniform(seed & m, row & m, draw & m, index & m)


# ----------------------------------------------------- host-array batch API


def _as_rows(x, dtype):
    a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
    if a.ndim == 1:
        a = a[None, :]
    if a.ndim != 2:
        raise InvalidParamsError("expected a vector or a (B, n) matrix")
    return a


def cutmax_batch(X, params: Optional[CutMaxParams] = None, raise_on_error: bool = True):
    """Batched CutMax over host rows (float64 or float32): returns (Z, argmax, status).

    Host -> device copies, the fused kernel and device -> host copies all happen
    inside the library call (pam_cutmax_batch_host_*)."""
    params = params or CutMaxParams()
    dtype = np.float32 if np.asarray(X).dtype == np.float32 else np.float64
    a = _as_rows(X, dtype)
    B, n = a.shape
    z = np.empty_like(a)
    am = np.empty(B, dtype=np.int32)
    st = np.empty(B, dtype=np.int32)
    prm = params.lower()
    fn = _lib.pam_cutmax_batch_host_f32 if dtype == np.float32 else _lib.pam_cutmax_batch_host_f64
    rc = fn(a.ctypes.data, B, n, C.byref(prm), z.ctypes.data, am.ctypes.data, st.ctypes.data)
    raise_for_status(rc, what="cutmax_batch")
    if raise_on_error:
        bad = np.nonzero(st & 0xFF)[0]
        if len(bad):
            raise_for_status(int(st[bad[0]]), row=int(bad[0]))
    return z, am, st


def cutmax(x, params: Optional[CutMaxParams] = None) -> ScoreVector:
    """cutmax(x, params) -> ScoreVector."""
    params = params or CutMaxParams()
    z, am, st = cutmax_batch(np.asarray(x, dtype=np.float64)[None, :], params)
    tie = bool(int(st[0]) & _abi.PAM_ROW_FLAG_TIE)
    if tie:
        warnings.warn("cutmax: top-2 gap of the input < 1e-9 (SPEC.md:122)", TieWarning, stacklevel=2)
    return ScoreVector(values=z[0], normalized=params.normalize, argmax=int(am[0]), tieWarning=tie)


# --------------------------------------------------------- device API ------


def _torch():
    import torch  # plumbing only: device memory and streams

    return torch


def _stream_ptr(stream, device):
    """The launch stream: the caller's (it must belong to `device`) or the
    current stream of `device` (not of the current device)."""
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream(device)
    elif stream.device != device:
        raise InvalidParamsError(f"stream is on {stream.device}, tensors on {device}")
    return C.c_void_p(stream.cuda_stream)


def _check_out(t, name, device, dtype, shape, contiguous=False):
    """Caller-supplied output buffers: same device, dtype and shape as the call
    writes, unit stride along rows (and fully contiguous where the kernel
    indexes it flat), so the kernel can never write out of bounds."""
    if t.device != device:
        raise InvalidParamsError(f"{name} is on {t.device}, x on {device}")
    if t.dtype != dtype:
        raise InvalidParamsError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise InvalidParamsError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if t.dim() > 0 and t.stride(-1) != 1:
        raise InvalidParamsError(f"{name} must have unit stride along its last dimension")
    if contiguous and not t.is_contiguous():
        raise InvalidParamsError(f"{name} must be contiguous")
    return t


def cutmax_batch_device(x, params: Optional[CutMaxParams] = None, z=None, argmax=None, status=None,
                        stats=None, stream=None):
    """Batched CutMax on a CUDA tensor (B, n) float64/float32, stream-ordered.

    Returns (z, argmax, status) device tensors.  ``stats`` (optional float64
    tensor (B, T, 2)) receives {mu_t, s2_t}.  Raises only for invalid params or
    launch failures; data-dependent failures land in ``status``."""
    torch = _torch()
    params = params or CutMaxParams()
    if x.dim() != 2 or not x.is_cuda:
        raise InvalidParamsError("x must be a 2-D CUDA tensor")
    if x.dtype not in (torch.float64, torch.float32):
        raise InvalidParamsError("dtype must be float64 or float32")
    B, n = x.shape
    ld = x.stride(0)
    if x.stride(1) != 1:
        raise InvalidParamsError("rows must be contiguous")
    dev = x.device
    if z is None:
        z = torch.empty((B, n), dtype=x.dtype, device=dev)
    _check_out(z, "z", dev, x.dtype, (B, n))
    if argmax is None:
        argmax = torch.empty(B, dtype=torch.int32, device=dev)
    _check_out(argmax, "argmax", dev, torch.int32, (B,))
    if status is None:
        status = torch.empty(B, dtype=torch.int32, device=dev)
    _check_out(status, "status", dev, torch.int32, (B,))
    if stats is not None:
        _check_out(stats, "stats", dev, torch.float64, (B, int(params.T), 2), contiguous=True)
    prm = params.lower()
    fn = _lib.pam_cutmax_batch_f64 if x.dtype == torch.float64 else _lib.pam_cutmax_batch_f32
    with torch.cuda.device(dev):  # the C ABI launches on the current device
        rc = fn(x.data_ptr(), ld, B, n, C.byref(prm), z.data_ptr(), z.stride(0), argmax.data_ptr(),
                status.data_ptr(), stats.data_ptr() if stats is not None else None, _stream_ptr(stream, dev))
    raise_for_status(rc, what="cutmax_batch_device")
    return z, argmax, status


def _sample_device(fn_name, x, cfg: SamplerConfig, params: CutMaxParams, onehot=None, stream=None):
    torch = _torch()
    if x.dim() != 2 or not x.is_cuda or x.dtype != torch.float64:
        raise InvalidParamsError("x must be a 2-D float64 CUDA tensor")
    if x.stride(1) != 1:
        raise InvalidParamsError("rows must be contiguous")
    B, n = x.shape
    dev = x.device
    token = torch.empty(B, dtype=torch.int32, device=dev)
    inside = torch.empty(B, dtype=torch.uint8, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    if onehot is not None:
        _check_out(onehot, "onehot", dev, torch.float64, (B, n))
    c = cfg.lower()
    prm = params.lower()
    with torch.cuda.device(dev):
        rc = getattr(_lib, fn_name)(x.data_ptr(), x.stride(0), B, n, C.byref(c), C.byref(prm), token.data_ptr(),
                                    inside.data_ptr(), onehot.data_ptr() if onehot is not None else None,
                                    onehot.stride(0) if onehot is not None else 0, status.data_ptr(),
                                    _stream_ptr(stream, dev))
    raise_for_status(rc, what=fn_name)
    return token, inside, status


def nucleus_sample_batch_device(x, cfg: SamplerConfig, params: Optional[CutMaxParams] = None, onehot=None,
                                stream=None):
    """Fused Beta-cut nucleus sampling (Alg. 3) over CUDA rows; returns (token, inside, status)."""
    return _sample_device("pam_nucleus_sample_batch_f64", x, cfg, params or CutMaxParams(), onehot, stream)


def gumbel_sample_batch_device(x, cfg: SamplerConfig, params: Optional[CutMaxParams] = None, onehot=None,
                               stream=None):
    """Fused Gumbel-max sampling (Lemma 1) over CUDA rows; inside[] against nucleus mass cfg.p."""
    return _sample_device("pam_gumbel_sample_batch_f64", x, cfg, params or CutMaxParams(), onehot, stream)


def _one_row_sample(fn, x, cfg, params, row_index):
    torch = _torch()
    xv = torch.as_tensor(np.asarray(x, dtype=np.float64), device="cuda")[None, :]
    oh = torch.empty_like(xv)
    c2 = SamplerConfig(p=cfg.p, q=cfg.q, alpha=cfg.alpha, seed=(cfg.seed ^ row_index), draw=cfg.draw)
    tok, ins, st = fn(xv, c2, params, onehot=oh)
    s = int(st.item())
    raise_for_status(s, row=0)
    return SampleOutcome(onehot=oh[0].cpu().numpy(), tokenIndex=int(tok.item()), insideNucleus=bool(ins.item()))


def nucleusOneShotSample(x, cfg: SamplerConfig, params: Optional[CutMaxParams] = None,
                         row_index: int = 0) -> SampleOutcome:
    """nucleusOneShotSample: noise keyed by cfg.seed ^ row_index."""
    return _one_row_sample(nucleus_sample_batch_device, x, cfg, params or CutMaxParams(), row_index)


def gumbelMaxSample(x, params: Optional[CutMaxParams] = None, seed: int = 0, nucleus_p: float = 0.9) -> SampleOutcome:
    """gumbelMaxSample."""
    return _one_row_sample(gumbel_sample_batch_device, x, SamplerConfig(p=nucleus_p, seed=seed),
                           params or CutMaxParams(), 0)


# ---- the top-p nucleus itself (csrc/nucleus_set.cu) ----------------------
def nucleus_set_batch_device(x, p: float, stream=None):
    """Top-p nucleus of softmax(x_r) for CUDA rows (ties included): returns
    (cutoff [B] float64, size [B] int32, mass [B] float64, status [B] int32);
    entry k of row r is inside <=> x[r, k] >= cutoff[r].  Cluster histogram scan
    over fixed-point masses, so the result does not depend on the summation order."""
    torch = _torch()
    if x.dim() != 2 or not x.is_cuda or x.dtype != torch.float64:
        raise InvalidParamsError("x must be a 2-D float64 CUDA tensor")
    if x.stride(1) != 1:
        raise InvalidParamsError("rows must be contiguous")
    B, n = x.shape
    cutoff = torch.empty(B, dtype=torch.float64, device=x.device)
    mass = torch.empty(B, dtype=torch.float64, device=x.device)
    size = torch.empty(B, dtype=torch.int32, device=x.device)
    status = torch.empty(B, dtype=torch.int32, device=x.device)
    with torch.cuda.device(x.device):
        rc = _lib.pam_nucleus_set_batch_f64(x.data_ptr(), x.stride(0), B, n, float(p), cutoff.data_ptr(),
                                            size.data_ptr(), mass.data_ptr(), status.data_ptr(),
                                            _stream_ptr(stream, x.device))
    raise_for_status(rc, what="nucleus_set_batch_device")
    return cutoff, size, mass, status


def nucleusSet(x, p: float):
    """The top-p nucleus of one logit vector: dict(cutoff, size, mass)."""
    torch = _torch()
    xv = torch.as_tensor(np.asarray(x, dtype=np.float64), device="cuda")[None, :]
    cut, size, mass, st = nucleus_set_batch_device(xv, p)
    raise_for_status(int(st.item()), row=0)
    return dict(cutoff=float(cut.item()), size=int(size.item()), mass=float(mass.item()))


# ---- analysis (csrc/analysis_kernel.cuh) ---------------------------------
def convergence_trace_batch_device(x, params: Optional[CutMaxParams] = None, stream=None):
    """convergenceTrace for CUDA rows: returns (out [B, T, 4] = {mu, s2, U,
    fraction below mean} per iteration, status [B])."""
    torch = _torch()
    if x.dim() != 2 or not x.is_cuda or x.dtype != torch.float64:
        raise InvalidParamsError("x must be a 2-D float64 CUDA tensor")
    params = params or CutMaxParams()
    if x.stride(1) != 1:
        raise InvalidParamsError("rows must be contiguous")
    B, n = x.shape
    out = torch.zeros((B, params.T, 4), dtype=torch.float64, device=x.device)
    status = torch.empty(B, dtype=torch.int32, device=x.device)
    prm = params.lower()
    with torch.cuda.device(x.device):
        rc = _lib.pam_convergence_trace_batch_f64(x.data_ptr(), x.stride(0), B, n, C.byref(prm), out.data_ptr(),
                                                  status.data_ptr(), _stream_ptr(stream, x.device))
    raise_for_status(rc, what="convergence_trace_batch_device")
    return out, status


def convergenceTrace(x, params: Optional[CutMaxParams] = None):
    """convergenceTrace on the GPU: one dict per iteration with
    mu, s2, dispersion (non-top U) and fractionBelowMean."""
    torch = _torch()
    xv = torch.as_tensor(np.asarray(x, dtype=np.float64), device="cuda")[None, :]
    out, st = convergence_trace_batch_device(xv, params)
    raise_for_status(int(st.item()))
    o = out[0].cpu().numpy()
    return [dict(mu=float(r[0]), s2=float(r[1]), dispersion=float(r[2]), fractionBelowMean=float(r[3])) for r in o]


def cutmax_jvp_batch_device(x, v, params: Optional[CutMaxParams] = None, want_z: bool = False, stream=None):
    """Forward-mode JVP of CutMax for CUDA rows x in directions v (same shape):
    returns (z or None, dz, status)."""
    torch = _torch()
    if x.shape != v.shape or x.dim() != 2 or not (x.is_cuda and v.is_cuda) or x.dtype != torch.float64 \
            or v.dtype != torch.float64:
        raise InvalidParamsError("x, v must be 2-D float64 CUDA tensors of one shape")
    x = x.contiguous()
    v = v.contiguous()
    params = params or CutMaxParams()
    B, n = x.shape
    dz = torch.empty_like(x)
    z = torch.empty_like(x) if want_z else None
    status = torch.empty(B, dtype=torch.int32, device=x.device)
    prm = params.lower()
    if v.device != x.device:
        raise InvalidParamsError("x and v must be on one device")
    with torch.cuda.device(x.device):
        rc = _lib.pam_cutmax_jvp_batch_f64(x.data_ptr(), v.data_ptr(), n, B, n, C.byref(prm),
                                           z.data_ptr() if z is not None else None, dz.data_ptr(), n,
                                           status.data_ptr(), _stream_ptr(stream, x.device))
    raise_for_status(rc, what="cutmax_jvp_batch_device")
    return z, dz, status


def _check_rows(status):
    st = status.cpu().numpy() & 0xFF
    bad = np.nonzero(st)[0]
    if bad.size:
        raise_for_status(int(st[bad[0]]), row=int(bad[0]))


def cutmaxJvp(x, v, params: Optional[CutMaxParams] = None) -> np.ndarray:
    """cutmaxJvp: d cutmax(x)/dx . v on the GPU (forward mode)."""
    torch = _torch()
    xv = torch.as_tensor(np.asarray(x, dtype=np.float64), device="cuda")[None, :]
    vv = torch.as_tensor(np.asarray(v, dtype=np.float64), device="cuda")[None, :]
    _, dz, st = cutmax_jvp_batch_device(xv, vv, params)
    _check_rows(st)
    return dz[0].cpu().numpy()


def cutmaxJacobian(x, params: Optional[CutMaxParams] = None) -> np.ndarray:
    """cutmaxJacobian: J[i, j] = dZ_i/dx_j from n JVPs with the
    basis directions, one batched launch."""
    torch = _torch()
    xh = np.asarray(x, dtype=np.float64)
    n = xh.shape[0]
    X = torch.as_tensor(xh, device="cuda")[None, :].repeat(n, 1)
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    _, dz, st = cutmax_jvp_batch_device(X, V, params)
    _check_rows(st)
    return dz.cpu().numpy().T.copy()


# ---- logit files (csrc/ingest.cpp) --------------------------------
def _read_file(path: str, pinned: bool):
    info = _abi.pam_ingest_info()
    bpath = os.fsencode(path)
    st = _lib.pam_lgt1_probe(bpath, C.byref(info))
    kind, dtype = "lgt1", np.float32
    if st == _abi.PAM_ERR_FORMAT and info.err_offset == 0:  # no LGT1 magic: JSON lines
        st = _lib.pam_jsonl_probe(bpath, C.byref(info))
        kind, dtype = "jsonl", np.float64
    raise_for_status(st, row=info.err_offset, what=f"ingest {path}")
    shape = (int(info.count), int(info.n))
    if pinned:
        torch = _torch()
        buf = torch.empty(shape, dtype=torch.float32 if dtype == np.float32 else torch.float64, pin_memory=True)
        ptr = buf.data_ptr()
    else:
        buf = np.empty(shape, dtype=dtype)
        ptr = buf.ctypes.data
    fn = _lib.pam_lgt1_read if kind == "lgt1" else _lib.pam_jsonl_read
    st = fn(bpath, ptr, shape[0] * shape[1], C.byref(info))
    raise_for_status(st, row=info.bad_vector if st == _abi.PAM_ERR_NON_FINITE else info.err_offset,
                     what=f"ingest {path}")
    return buf


def ingest(path: str) -> np.ndarray:
    """ingest: an LGT1 file (float32 [count, n]) or JSON lines
    (float64 [count, n]).  Raises FormatError (byte offset) / NonFiniteError (vector)."""
    return _read_file(path, pinned=False)


def ingest_pinned(path: str):
    """ingest straight into pinned host memory (a torch tensor) so the batch API
    can take it to the GPU with one async copy: ingest_pinned(p).cuda(non_blocking=True)."""
    return _read_file(path, pinned=True)


def write_lgt1(path: str, vectors) -> None:
    """LGT1 writer; ingest(write_lgt1(v)) == float32(v) bit-exact."""
    a = np.ascontiguousarray(np.asarray(vectors, dtype=np.float32))
    if a.ndim != 2:
        raise InvalidParamsError("write_lgt1 expects a 2-D array [count, n]")
    raise_for_status(_lib.pam_lgt1_write(os.fsencode(path), a.ctypes.data, a.shape[0], a.shape[1]))


def violationExperiment(prompts, cfg: SamplerConfig, draws: int, params: Optional[CutMaxParams] = None) -> dict:
    """violationExperiment (§4.3 / Fig. 4) on the GPU
    samplers.  For every prompt, `draws` independent samples (noise keyed by
    (seed ^ prompt) ^ draw-row) from the Beta-cut sampler and from Gumbel-max;
    a violation is a token outside the plaintext top-p nucleus.
    Returns per-method (mean, std) of the per-prompt violation fractions and
    the per-prompt arrays.  Deterministic under a fixed seed."""
    torch = _torch()
    if draws < 1:
        raise InvalidParamsError("draws must be >= 1")
    params = params or CutMaxParams()
    rates = {"betaCut": [], "gumbel": []}
    for i, x in enumerate(prompts):
        xv = torch.as_tensor(np.asarray(x, dtype=np.float64), device="cuda")
        X = xv[None, :].repeat(draws, 1)
        c = SamplerConfig(p=cfg.p, q=cfg.q, alpha=cfg.alpha, seed=cfg.seed ^ i, draw=cfg.draw)
        for name, fn in (("betaCut", nucleus_sample_batch_device), ("gumbel", gumbel_sample_batch_device)):
            _, inside, st = fn(X, c, params)
            st_h = st.cpu().numpy() & 0xFF  # the TieWarning bit is not an error
            if np.any(st_h != 0):
                raise_for_status(int(st_h[st_h != 0][0]), row=int(np.nonzero(st_h)[0][0]))
            rates[name].append(1.0 - float(inside.double().mean().item()))
    out = {}
    for name, r in rates.items():
        a = np.asarray(r)
        out[name + "Rate"] = (float(a.mean()), float(a.std()))
        out[name + "PerPrompt"] = a
    return out


def cutmaxStep(y, p: int, c: float, epsVar: float = 1e-24):
    """cutmaxStep: next_i = (1 + r_i/c)^p on the GPU (T=1,
    un-normalised), with mu/s2 from the kernel's stats output.  Residuals and
    the non-top dispersion are derived from those stats."""
    torch = _torch()
    yv = torch.as_tensor(np.asarray(y, dtype=np.float64), device="cuda")[None, :]
    prm = CutMaxParams(p=p, c=c, T=1, checked=False, normalize=False, epsVar=epsVar)
    stats = torch.empty((1, 1, 2), dtype=torch.float64, device="cuda")
    z, _, st = cutmax_batch_device(yv, prm, stats=stats)
    raise_for_status(int(st.item()))
    mu, s2 = (float(v) for v in stats[0, 0].cpu().numpy())
    yh = np.asarray(y, dtype=np.float64)
    r = (yh - mu) * (1.0 / np.sqrt(s2))
    top = int(np.argmax(yh))
    nt = np.delete(r, top)
    disp = float(((nt - nt.mean()) ** 2).sum())
    return z[0].cpu().numpy(), ResidualStats(mu=mu, s2=s2, residuals=r, dispersion=disp)


def launch_info(dtype_bytes: int, B: int, n: int, params: Optional[CutMaxParams] = None) -> dict:
    """Launch geometry the library picks for (dtype, B, n) (needs a GPU)."""
    info = _abi.pam_launch_info()
    prm = (params or CutMaxParams()).lower()
    raise_for_status(_lib.pam_query_launch(dtype_bytes, B, n, C.byref(prm), C.byref(info)))
    return {k: getattr(info, k) for k, _ in info._fields_}


def kernel_launch_count() -> int:
    return int(_lib.pam_kernel_launch_count())


class geometry_override:
    """Tuning / test hook: force the CutMax launch geometry for one dtype
    (dtype_bytes 8 or 4) to a compiled variant (threads x elems per thread) and
    a cluster size, for the duration of a ``with`` block (pam_set_geometry_override)."""

    def __init__(self, dtype_bytes: int, threads: int, elems: int, cluster: int, min_blocks: int = 0):
        self.args = (int(dtype_bytes), int(threads), int(elems), int(cluster), int(min_blocks))

    def __enter__(self):
        raise_for_status(_lib.pam_set_geometry_override(*self.args), what="geometry_override")
        return self

    def __exit__(self, *exc):
        _lib.pam_set_geometry_override(self.args[0], 0, 0, 0, 0)
        return False


class general_p3_kernel:
    """Test hook: inside the ``with`` block, p = 3 rows run on the general
    CutMax kernel instead of the lean p = 3 kernel (pam_set_lean_p3(0)); both
    must give bit-identical results."""

    def __enter__(self):
        _lib.pam_set_lean_p3(0)
        return self

    def __exit__(self, *exc):
        _lib.pam_set_lean_p3(1)
        return False
