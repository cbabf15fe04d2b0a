"""Absolute per-event timelines of both row groups of one CTA (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

def run(B, n, cfg, T=4):
    os.environ["PAM_FORCE_CFG_F64"] = cfg
    x = W.torch_gaussian(B, n, seed=1)
    prm = pam.CutMaxParams(T=T)
    info = pam.launch_info(8, B, n, prm)
    buf = torch.zeros(info["ctas"] * 8 * 32, dtype=torch.int64, device="cuda")
    lib = pam._abi.load()
    pam.cutmax_batch_device(x, prm); torch.cuda.synchronize()
    lib.pam_set_trace_buffer(buf.data_ptr(), buf.numel())
    pam.cutmax_batch_device(x, prm); torch.cuda.synchronize()
    lib.pam_set_trace_buffer(None, 0)
    tr = buf.view(info["ctas"], 8, 32).cpu().numpy()
    cta = 5
    t0 = tr[cta, 0, 0]
    G = info["groups"]
    print(f"== {cfg} B={B} n={n}: CTA {cta}, times relative to group-0 row-0 start (cycles)")
    ev = [0, 1, 2, 3, 4] + [k for t in range(T) for k in (5 + 2 * t, 6 + 2 * t)] + [20, 21]
    names = ["start", "tma", "lds", "in.pass", "x0"] + [f"p{t}|x{t+1}" if False else n for t in range(T) for n in (f"pass{t}", f"xchg{t+1}")] + ["core", "stores"]
    for rr in range(1, 3):
        for g in range(G):
            row = g * (8 // G) + rr
            vals = [tr[cta, row, e] - t0 for e in ev]
            print(f"  g{g} row{rr}: " + " ".join(f"{nm}={v}" for nm, v in zip(names, vals)))
    os.environ.pop("PAM_FORCE_CFG_F64")

run(4096, 151936, "256,38,16,2")
run(4096, 151936, "512,38,8,1")
