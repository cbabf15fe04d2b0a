"""Per-phase timing of the CutMax kernel from the debug trace buffer (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

NAMES = {0: "row start", 1: "TMA wait done", 2: "LDS+sync+next TMA", 3: "input pass", 4: "xchg0",
         20: "core done (normaliser)", 21: "final pass (Z, stores)", 22: "argmax gather"}
for t in range(8):
    NAMES[5 + 2 * t] = f"iter{t} pass"; NAMES[6 + 2 * t] = f"iter{t} xchg"

def run(B, n, dtype, cfg=None):
    if cfg:
        os.environ["PAM_FORCE_CFG_F64" if dtype == torch.float64 else "PAM_FORCE_CFG_F32"] = cfg
    x = W.torch_gaussian(B, n, seed=1, dtype=dtype)
    prm = pam.CutMaxParams()
    info = pam.launch_info(x.element_size(), B, n, prm)
    buf = torch.zeros(info["ctas"] * 8 * 32, dtype=torch.int64, device="cuda")
    lib = pam._abi.load()
    pam.cutmax_batch_device(x, prm); torch.cuda.synchronize()
    lib.pam_set_trace_buffer(buf.data_ptr(), buf.numel())
    pam.cutmax_batch_device(x, prm); torch.cuda.synchronize()
    lib.pam_set_trace_buffer(None, 0)
    tr = buf.view(info["ctas"], 8, 32).cpu().numpy().astype(np.float64)
    ev = [0, 1, 2, 3, 4] + [k for t in range(4) for k in (5 + 2 * t, 6 + 2 * t)] + [20, 21, 22]
    print(f"== B={B} n={n} {dtype} cfg={info['threads']}x{info['elems_per_thread']} G={info['groups']} C={info['cluster']} ctas={info['ctas']}")
    rows = tr[:, 1:7, :]  # skip the first row (cold)
    d = {}
    for a, b in zip(ev, ev[1:]):
        dd = rows[:, :, b] - rows[:, :, a]
        d[(a, b)] = np.median(dd)
    nxt = tr[:, 2:8, 0] - tr[:, 1:7, 22]
    tot = np.median(tr[:, 2:8, 0] - tr[:, 1:7, 0])
    for (a, b), v in d.items():
        print(f"   {NAMES.get(b, b):28s} {v:8.0f} cyc  {v/1.965e3:7.2f} us  {100*v/tot:5.1f}%")
    print(f"   {'gap to next row':28s} {np.median(nxt):8.0f} cyc")
    for a, b, nm in ((3, 24, "xchg0: warp tree + push"), (24, 25, "xchg0: mbarrier wait"), (25, 26, "xchg0: slot reduce"),
                     (26, 4, "xchg0: return"), (4, 28, "  guard"), (28, 29, "  loop top/status"), (29, 30, "  invsqrt"), (30, 27, "  k, b"), (4, 27, "scalar math (iter0)")):
        print(f"   {nm:28s} {np.median(rows[:, :, b] - rows[:, :, a]):8.0f} cyc")
    sk = tr[:, 1:7, 24].reshape(-1, info['cluster'], 6) if False else None
    print(f"   {'row period':28s} {tot:8.0f} cyc  {tot/1.965e3:7.2f} us")
    os.environ.pop("PAM_FORCE_CFG_F64", None); os.environ.pop("PAM_FORCE_CFG_F32", None)

run(4096, 151936, torch.float64)
run(4096, 151936, torch.float64, "256,38,16,2")
run(4096, 32768, torch.float64, "256,38,4,2")
run(4096, 32768, torch.float64)
run(4096, 151936, torch.float32)
run(4096, 1024, torch.float64)
