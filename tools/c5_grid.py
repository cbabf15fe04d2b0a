"""Every BASELINE C5 point (B in {1,16,256,4096} x n in {1024,32768,151936}, fp64
and fp32) plus the C4 sampler shape, timed with CUDA events on device-resident
inputs (dev tool; SURVEY.md §8(d) asks for every C5 point).  Prints a markdown
table; the headline line is bench.py's."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

PEAK = 6547.5


def time_fn(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    prm = pam.CutMaxParams()
    print("| dtype | B | n | geometry | ms | rows/s | GB/s | % of HBM |")
    print("|---|---|---|---|---|---|---|---|")
    for dt in (torch.float64, torch.float32):
        esz = 8 if dt == torch.float64 else 4
        for n in (1024, 32768, 151936):
            for B in (1, 16, 256, 4096):
                x = W.torch_gaussian(B, n, seed=1, dtype=dt)
                z = torch.empty_like(x)
                am = torch.empty(B, dtype=torch.int32, device="cuda")
                st = torch.empty_like(am)
                reps = 50 if B * n < 1 << 24 else 10
                ms = time_fn(lambda: pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st), reps)
                info = pam.launch_info(esz, B, n, prm)
                geo = f"{info['threads']}x{info['elems_per_thread']} C={info['cluster']} cl={info['clusters']}"
                gbs = B * (2 * n * esz + 4) / ms / 1e6
                print(f"| {'fp64' if esz == 8 else 'fp32'} | {B} | {n} | {geo} | {ms:.4f} | {B / ms * 1e3:.3g} | "
                      f"{gbs:.0f} | {100 * gbs / PEAK:.1f}% |", flush=True)
    # C4: nucleus sampler, 128 x 32768 fp64 (and a large batch for throughput)
    print()
    print("| sampler | B | n | ms | rows/s | GB/s (8n+9 B/row) |")
    print("|---|---|---|---|---|---|")
    for B in (128, 4096):
        x = W.torch_gaussian(B, 32768, seed=2, dtype=torch.float64)
        for gumbel in (False, True):
            cfg = pam.SamplerConfig(p=0.9, q=0.9, seed=7)
            fn = (lambda: pam.gumbel_sample_batch_device(x, cfg, prm)) if gumbel else \
                (lambda: pam.nucleus_sample_batch_device(x, cfg, prm))
            ms = time_fn(fn, 10)
            gbs = B * (8 * 32768 + 9) / ms / 1e6
            print(f"| {'gumbel' if gumbel else 'beta-cut'} | {B} | 32768 | {ms:.4f} | {B / ms * 1e3:.3g} | {gbs:.0f} |",
                  flush=True)


main()
