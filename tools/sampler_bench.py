"""Sampler throughput at the C4 shape (dev tool): Beta-cut and Gumbel-max over
B x 32768 fp64 Zipf-shaped rows, CUDA events on device-resident inputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
x = torch.as_tensor(W.zipf_logits(B, 32768, seed=5), device="cuda")
cfg = pam.SamplerConfig(p=0.9, seed=7)
prm = pam.CutMaxParams()
for name, fn in (("beta-cut", pam.nucleus_sample_batch_device), ("gumbel", pam.gumbel_sample_batch_device)):
    for _ in range(2):
        fn(x, cfg, prm)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn(x, cfg, prm)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name}: B={B} n=32768 {ms:.3f} ms  {B / ms * 1e3:.3g} rows/s  {B * (8 * 32768 + 9) / ms / 1e6:.0f} GB/s")
