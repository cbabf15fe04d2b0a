"""Phase clocks of the nucleus-set kernel (dev tool): CTA 0's first row."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

lib = pam._abi.load()
lib.pam_dev_nucleus_set_clocks.argtypes = [C.c_void_p]
for B, n in ((128, 32768), (64, 151936)):
    x = torch.as_tensor(W.zipf_logits(B, n, seed=2), device="cuda")
    buf = torch.zeros(40, dtype=torch.int64, device="cuda")
    pam.nucleus_set_batch_device(x, 0.9)
    lib.pam_dev_nucleus_set_clocks(buf.data_ptr())
    pam.nucleus_set_batch_device(x, 0.9)
    torch.cuda.synchronize()
    lib.pam_dev_nucleus_set_clocks(None)
    t = buf.cpu().numpy()
    print(f"B={B} n={n}: load {t[1]-t[0]}, sync {t[2]-t[1]}, weights {t[3]-t[2]}, sync {t[4]-t[3]}")
    prev = t[4]
    for l in range(8):
        h, s, g, sc = t[5+4*l], t[6+4*l], t[7+4*l], t[8+4*l]
        print(f"  level {l}: hist {h-prev}, cluster sync {s-h}, gather {g-s}, scan {sc-g}")
        prev = sc
    print(f"  total {prev - t[0]}")
