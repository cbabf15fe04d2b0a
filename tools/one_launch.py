"""One (or a few) CutMax launches on synthetic N(0,3^2) rows (for ncu captures; dev tool).
usage: python tools/one_launch.py B n [launches] [T]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

B, n = int(sys.argv[1]), int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 else 2
T = int(sys.argv[4]) if len(sys.argv) > 4 else 4
x = W.torch_gaussian(B, n, seed=1)
prm = pam.CutMaxParams(T=T)
z = torch.empty_like(x)
for _ in range(k):
    pam.cutmax_batch_device(x, prm, z=z)
torch.cuda.synchronize()
print("ok", pam.launch_info(8, B, n, prm))
