"""A few sampler launches on C4-shaped rows (for ncu captures; dev tool). usage: one_sample.py B n [launches]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

B, n = int(sys.argv[1]), int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 else 2
x = torch.as_tensor(W.zipf_logits(B, n, seed=3), device="cuda")
for _ in range(k):
    pam.nucleus_sample_batch_device(x, pam.SamplerConfig(p=0.9, seed=1), pam.CutMaxParams())
torch.cuda.synchronize()
print("ok")
