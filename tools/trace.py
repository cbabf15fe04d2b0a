"""Per-phase timing of the CutMax kernel from the debug trace buffer (dev tool).
Needs the trace build:  make -C paper_2509_08383_b200/csrc trace  and
PAM_LIB_PATH=paper_2509_08383_b200/libpam_trace.so  (set below if present)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PAM_LIB_PATH", os.path.join(ROOT, "paper_2509_08383_b200", "libpam_trace.so"))
import numpy as np
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

CLK = 1.965e3  # cycles per us (SM clock under load)


def names(T):  # p = 3 analytic-normaliser flow (the headline kernel)
    nm = {2: "input pass + xchg (1st row)", 4: "input moments"}
    for t in range(T - 1):
        nm[13 + t] = f"control {t} (moments+chain, bcast)"
        nm[5 + 2 * t] = f"pass {t}" + (" (+3rd moment)" if t == T - 2 else "")
        nm[16 + t] = f"push {t} (bfly+barrier+send)"
        nm[6 + 2 * t] = f"wait {t} (warp 0: records)"
    nm.update({22: "control + normaliser", 23: "X(next) wait", 24: "fused last pass + swap",
               6 + 2 * (T - 1): "closing xchg", 21: "status"})
    return nm


def seq(T):
    s = [0, 2]
    for t in range(T - 1):
        s += [13 + t, 5 + 2 * t, 16 + t, 6 + 2 * t]
    s += [22, 23, 24, 6 + 2 * (T - 1), 21]
    return s


def run(B, n, dtype, cfg=None, T=4):
    """cfg: "NTGxExC[xMINB]" forces the geometry (pam_set_geometry_override)."""
    import contextlib
    ov = contextlib.nullcontext()
    if cfg:
        g = [int(v) for v in cfg.split("x")]
        ov = pam.geometry_override(8 if dtype == torch.float64 else 4, g[0], g[1], g[2], g[3] if len(g) > 3 else 0)
    with ov:
        _run(B, n, dtype, T)


def _run(B, n, dtype, T):
    x = W.torch_gaussian(B, n, seed=1, dtype=dtype)
    prm = pam.CutMaxParams(T=T)
    info = pam.launch_info(x.element_size(), B, n, prm)
    buf = torch.zeros(info["ctas"] * 8 * 32, dtype=torch.int64, device="cuda")
    lib = pam._abi.load()
    pam.cutmax_batch_device(x, prm); torch.cuda.synchronize()
    lib.pam_set_trace_buffer(buf.data_ptr(), buf.numel())
    pam.cutmax_batch_device(x, prm); torch.cuda.synchronize()
    lib.pam_set_trace_buffer(None, 0)
    tr = buf.view(info["ctas"], 8, 32).cpu().numpy().astype(np.float64)
    print(f"== B={B} n={n} {dtype} T={T} cfg={info['threads']}x{info['elems_per_thread']} C={info['cluster']} "
          f"ctas={info['ctas']}")
    rows = tr[:, 1:7, :]  # skip the first (cold) row and the last
    nm = names(T)
    s = seq(T)
    period = np.median(tr[:, 2:8, 0] - tr[:, 1:7, 0])
    for a, b in zip(s, s[1:]):
        v = np.median(rows[:, :, b] - rows[:, :, a])
        print(f"   {nm.get(b, b):28s} {v:8.0f} cyc  {v / CLK:6.2f} us  {100 * v / period:5.1f}%")
    for a, b, nm in ((0, 25, "DMA: hook ex0 done (half X(next))"), (0, 26, "DMA: hook ex1 done (all X(next))"),
                     (0, 23, "X(next) landed (last pass start)")):
        print(f"   {nm:28s} at {np.median(rows[:, :, b] - rows[:, :, a]):8.0f} cyc after row start")
    # exchange latency spread over CTAs (pass end -> records combined, thread 0)
    for t in range(T):
        a_, b_ = (16 + t, 6 + 2 * t) if t < T - 1 else (24, 6 + 2 * t)
        d = (rows[:, :, b_] - rows[:, :, a_]).ravel()
        print(f"   xchg {t} wait spread: min {np.min(d):6.0f} p10 {np.percentile(d, 10):6.0f} med {np.median(d):6.0f} "
              f"p90 {np.percentile(d, 90):6.0f} max {np.max(d):6.0f}")
    for k, nm in ((30, "warp 5"), (31, "warp 10"), (19, "warp 15")):
        d = (rows[:, :, k] - rows[:, :, 7]).ravel()  # vs warp 0's pass-1 end (event 7)
        print(f"   pass-1 end, {nm} - warp 0: med {np.median(d):6.0f} p10 {np.percentile(d, 10):6.0f} "
              f"p90 {np.percentile(d, 90):6.0f}")
    print(f"   {'-> next row start':28s} {np.median(tr[:, 2:8, 0] - tr[:, 1:7, 21]):8.0f} cyc")
    print(f"   {'row period':28s} {period:8.0f} cyc  {period / CLK:6.2f} us")


if __name__ == "__main__":
    if len(sys.argv) > 1:  # n B cfg...
        for c in sys.argv[3:] or [None]:
            run(int(sys.argv[2]), int(sys.argv[1]), torch.float64, c)
        sys.exit(0)
    run(4096, 151936, torch.float64)
    run(4096, 32768, torch.float64)
