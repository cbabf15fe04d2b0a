"""Per-phase timing of the sampler kernel (trace build; dev tool)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PAM_LIB_PATH", os.path.join(ROOT, "paper_2509_08383_b200", "libpam_trace.so"))
import numpy as np, torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

B, n = 4096, 32768
x = torch.as_tensor(W.zipf_logits(B, n, seed=5), device="cuda")
cfg = pam.SamplerConfig(p=0.9, seed=7)
ctas = 148
buf = torch.zeros(ctas * 8 * 32, dtype=torch.int64, device="cuda")
lib = pam._abi.load()
pam.nucleus_sample_batch_device(x, cfg); torch.cuda.synchronize()
lib.pam_set_trace_buffer(buf.data_ptr(), buf.numel())
pam.nucleus_sample_batch_device(x, cfg); torch.cuda.synchronize()
lib.pam_set_trace_buffer(None, 0)
tr = buf.view(ctas, 8, 32).cpu().numpy().astype(np.float64)
rows = tr[:, 1:7, :]
names = {1: "sync + load issue + noise", 2: "load wait + x+G + max", 3: "cutmax (input + T iterations)",
         4: "token candidate + gather", 5: "nucleus pass + exchange"}
period = np.median(tr[:, 2:8, 0] - tr[:, 1:7, 0])
for a, b in ((0, 1), (1, 2), (2, 3), (3, 4), (4, 5)):
    v = np.median(rows[:, :, b] - rows[:, :, a])
    print(f"   {names[b]:32s} {v:8.0f} cyc  {100 * v / period:5.1f}%")
print(f"   row period {period:8.0f} cyc")
