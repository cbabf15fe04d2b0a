"""Fig. 4 reproduction on the GPU samplers (§4.3):
S prompts x N draws, p = 0.9, peaked Zipf(1.1)-shaped synthetic logits (the
paper's Mistral-7B logits are not available).  Prints per-method mean +- std of
the per-prompt violation rates."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

S = int(sys.argv[1]) if len(sys.argv) > 1 else 100
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
n = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
prompts = W.zipf_logits(S, n, seed=11)
t0 = time.time()
out = pam.violationExperiment(prompts, pam.SamplerConfig(p=0.9, seed=2024), draws=N)
dt = time.time() - t0
print(f"S={S} prompts x N={N} draws, n={n}, p=0.9 ({S * N * 2 / dt:.3g} samples/s incl. host loop)")
for k in ("betaCut", "gumbel"):
    m, s = out[k + "Rate"]
    print(f"  {k:8s} violation rate {100 * m:6.2f}% +- {100 * s:5.2f}%")
