"""Per-phase timing of the two-iterations-per-exchange kernel (dev tool).
Needs the trace build (make -C paper_2509_08383_b200/csrc trace)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PAM_LIB_PATH", os.path.join(ROOT, "paper_2509_08383_b200", "libpam_trace.so"))
import numpy as np
import torch
os.environ.setdefault("PAM_ENABLE_AHEAD", "1")
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

SEQ = [(0, "row start"), (1, "stage0 wait (warp0: records)"), (2, "stage0 chain"), (3, "bar1 (coef bcast)"),
       (4, "mid pass (warp 0)"), (5, "mid push (barrier+reduce+send)"), (14, "stage1 wait"), (15, "stage1 chain"),
       (16, "bar1"), (9, "X(next) wait"), (10, "last pass (warp 0)"), (11, "boundary push")]


def run(B, n, T=4):
    x = W.torch_gaussian(B, n, seed=1)
    prm = pam.CutMaxParams(T=T)
    info = pam.launch_info(8, B, n, prm)
    buf = torch.zeros(info["ctas"] * 8 * 32, dtype=torch.int64, device="cuda")
    lib = pam._abi.load()
    pam.cutmax_batch_device(x, prm)
    torch.cuda.synchronize()
    lib.pam_set_trace_buffer(buf.data_ptr(), buf.numel())
    pam.cutmax_batch_device(x, prm)
    torch.cuda.synchronize()
    lib.pam_set_trace_buffer(None, 0)
    tr = buf.view(info["ctas"], 8, 32).cpu().numpy().astype(np.float64)
    print(f"== B={B} n={n} T={T} cfg={info['threads']}x{info['elems_per_thread']} C={info['cluster']} "
          f"clusters={info['clusters']} kernel_id={info['kernel_id']}")
    rows = tr[:, 1:7, :]  # skip the first row (prologue)
    prev = None
    tot = 0.0
    for k, nm in SEQ:
        if prev is not None:
            d = np.median(rows[:, :, k] - rows[:, :, prev])
            tot += d
            print(f"  {nm:36s} {d:8.0f}")
        prev = k
    per_row = np.median(tr[:, 2:7, 0] - tr[:, 1:6, 0])
    print(f"  {'boundary push -> next row start':36s} {np.median(tr[:, 2:7, 0] - tr[:, 1:6, 11]):8.0f}")
    print(f"  row period (cycles)                  {per_row:8.0f}")
    # cross-CTA skew from %globaltimer (ns): per cluster, spread of the push times
    C = info["cluster"]
    g = tr.reshape(-1, C, 8, 32)[:, :, 1:7, :]
    for k_push, k_recv, nm in ((20, 21, "mid exchange"), (23, 22, "boundary exchange")):
        push = g[:, :, :-1, k_push] if k_push == 23 else g[:, :, :, k_push]
        recv = g[:, :, 1:, k_recv] if k_push == 23 else g[:, :, :, k_recv]
        spread = np.median(push.max(axis=1) - push.min(axis=1))
        transit = np.median(recv - push.max(axis=1, keepdims=True))
        print(f"  {nm}: push-time spread over CTAs {spread * 1.965:7.0f} cyc, last push -> records {transit * 1.965:7.0f} cyc")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] != "-":
        os.environ["PAM_DEBUG_FLAGS"] = sys.argv[1]
    if len(sys.argv) > 2:
        os.environ["PAM_FORCE_AHEAD"] = sys.argv[2]
        run(4096, 151936)
    else:
        run(4096, 151936)
        run(4096, 32768)
