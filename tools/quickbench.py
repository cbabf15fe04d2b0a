"""Quick device-side timing of the CutMax kernel (dev tool, not the bench contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

def run(B, n, dtype, reps=10, **kw):
    x = W.torch_gaussian(B, n, seed=1, dtype=dtype)
    z = torch.empty_like(x); am = torch.empty(B, dtype=torch.int32, device='cuda'); st = torch.empty_like(am)
    prm = pam.CutMaxParams(**kw)
    for _ in range(3): pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort(); ms = ts[len(ts)//2]
    esz = x.element_size()
    gbs = B * (2 * n * esz + 4) / ms / 1e6
    info = pam.launch_info(esz, B, n, prm)
    print(f"B={B:5d} n={n:6d} {str(dtype):14s} {ms:9.4f} ms  {B/ms*1e3/1e6:8.4f} Mrows/s  {gbs:8.1f} GB/s  {100*gbs/6540.2:5.1f}% "
          f"st_bad={int((st!=0).sum())} cfg={info['threads']}x{info['elems_per_thread']} C={info['cluster']} clusters={info['clusters']} smem={info['smem_bytes']}", flush=True)

if __name__ == "__main__":
    for dt in (torch.float64, torch.float32):
        for n in (1024, 32768, 151936):
            for B in (1, 16, 256, 4096):
                run(B, n, dt)
