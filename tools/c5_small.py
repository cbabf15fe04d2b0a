"""Dev tool: C5 points at n = 1024 (and other short rows) through the product
path (warp-per-row kernel) vs the cluster kernel (forced geometry), fp64 and
fp32, with an L2 flush between timed launches for inputs that fit in L2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

PEAK = 6547.5
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(f, reps):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


prm = pam.CutMaxParams()
for dt in (torch.float64, torch.float32):
    esz = 8 if dt == torch.float64 else 4
    for n in [int(a) for a in (sys.argv[1:] or ["1024"])]:
        for B in (1, 16, 256, 4096):
            x = W.torch_gaussian(B, n, seed=1, dtype=dt)
            z = torch.empty_like(x)
            am = torch.empty(B, dtype=torch.int32, device="cuda")
            st = torch.empty_like(am)
            ms = t(lambda: pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st), 20)
            info = pam.launch_info(esz, B, n, prm)
            ok = bool(torch.equal(am.long(), x.argmax(dim=1)))
            gbs = B * (2 * n * esz + 4) / ms / 1e6
            print(f"{str(dt)[6:]:8s} B={B:5d} n={n:6d} kid={info['kernel_id']:5d} {ms*1e3:8.1f} us {B/ms/1e3:9.3f} Mrow/s {gbs:7.0f} GB/s {100*gbs/PEAK:5.1f}%  argmax ok={ok}")
