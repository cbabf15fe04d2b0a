"""Every BASELINE C5 point (B in {1,16,256,4096} x n in {1024,32768,151936}, fp64
and fp32), C3 (64 x 151936 Zipf logits), polynomial-mode scalars, the Table-1
schedules (generic p) and the C4 sampler shape, timed with CUDA events on
device-resident inputs through the product path (dev tool).

Working sets that fit in the 126 MB L2 (2 * B * n * size < 256 MB) are timed one
launch at a time with a 256 MB L2 flush before each launch; larger ones
back-to-back.  Small-B rows are dominated by launch latency (~5-9 us per call,
reported as is).  Prints a markdown table."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

PEAK = 6547.5
try:
    import json
    PEAK = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass
_flush = None


def time_fn(fn, reps, flush):
    global _flush
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if not flush:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    if _flush is None:
        _flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tot = 0.0
    for _ in range(reps):
        _flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


def kernel_name(info):
    k = info["kernel_id"]
    if k >= 2000:
        return f"warp/row E={info['elems_per_thread']}"
    kind = "lean" if k >= 1000 else "general"
    return f"{kind} {info['threads']}x{info['elems_per_thread']} C={info['cluster']} cl={info['clusters']}"


def row(label, x, prm, esz, reps=None):
    B, n = x.shape
    z = torch.empty_like(x)
    am = torch.empty(B, dtype=torch.int32, device="cuda")
    st = torch.empty_like(am)
    flush = 2 * B * n * esz < (256 << 20)
    reps = reps or (30 if flush else 10)
    ms = time_fn(lambda: pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st), reps, flush)
    info = pam.launch_info(esz, B, n, prm)
    gbs = B * (2 * n * esz + 4) / ms / 1e6
    ok = int(((st & 0xFF) != 0).sum()) == 0
    print(f"| {label} | {B} | {n} | {kernel_name(info)} | {ms * 1e3:.1f} | {B / ms * 1e3:.3g} | {gbs:.0f} | "
          f"{100 * gbs / PEAK:.1f}% | {'flush' if flush else 'stream'} |{'' if ok else ' ROW ERRORS'}", flush=True)


def main():
    prm = pam.CutMaxParams()
    print("| case | B | n | kernel / geometry | us | rows/s | GB/s | % of HBM | L2 |")
    print("|---|---|---|---|---|---|---|---|---|")
    for dt in (torch.float64, torch.float32):
        esz = 8 if dt == torch.float64 else 4
        for n in (1024, 32768, 151936):
            for B in (1, 16, 256, 4096):
                row(f"C5 {'fp64' if esz == 8 else 'fp32'}", W.torch_gaussian(B, n, seed=1, dtype=dt), prm, esz)
    xz = torch.as_tensor(W.zipf_logits(64, 151936, seed=3), device="cuda")
    row("C3 fp64 Zipf T=4", xz, prm, 8)
    x = W.torch_gaussian(4096, 151936, seed=1)
    row("fp64 poly scalars", x, pam.CutMaxParams(invsqrtMode="poly", invMode="poly"), 8)
    row("fp64 Table 1 (4,13,15)", x, pam.CutMaxParams(T=4, p=13, c=15.0), 8)
    row("fp64 Table 1 (5,9,15)", x, pam.CutMaxParams(T=5, p=9, c=15.0), 8)
    row("fp64 HE schedule p=[16,4,4,6]", x, pam.CutMaxParams(T=4, p=[16, 4, 4, 6], c=[5.0, 3.0, 3.0, 3.0],
                                                                checked=False), 8)
    del x
    # C4: nucleus sampler, 128 x 32768 fp64 (and a large batch for throughput)
    print()
    print("| sampler | B | n | us | rows/s | GB/s (8n+9 B/row) | L2 |")
    print("|---|---|---|---|---|---|---|")
    for B in (128, 4096):
        x = torch.as_tensor(W.zipf_logits(B, 32768, seed=2), device="cuda")
        flush = B * 32768 * 8 < (256 << 20)
        for gumbel in (False, True):
            cfg = pam.SamplerConfig(p=0.9, q=0.9, seed=7)
            fn = (lambda: pam.gumbel_sample_batch_device(x, cfg, prm)) if gumbel else \
                (lambda: pam.nucleus_sample_batch_device(x, cfg, prm))
            ms = time_fn(fn, 10, flush)
            gbs = B * (8 * 32768 + 9) / ms / 1e6
            print(f"| {'gumbel' if gumbel else 'beta-cut'} | {B} | 32768 | {ms * 1e3:.1f} | {B / ms * 1e3:.3g} | "
                  f"{gbs:.0f} | {'flush' if flush else 'stream'} |", flush=True)
        ms = time_fn(lambda: pam.nucleus_set_batch_device(x, 0.9), 10, flush)
        print(f"| nucleus set (cutoff/size/mass) | {B} | 32768 | {ms * 1e3:.1f} | {B / ms * 1e3:.3g} | "
              f"{B * (8 * 32768 + 24) / ms / 1e6:.0f} | {'flush' if flush else 'stream'} |", flush=True)
    x = torch.as_tensor(W.zipf_logits(1024, 151936, seed=3), device="cuda")
    ms = time_fn(lambda: pam.nucleus_set_batch_device(x, 0.9), 5, False)
    print(f"| nucleus set (cutoff/size/mass) | 1024 | 151936 | {ms * 1e3:.1f} | {1024 / ms * 1e3:.3g} | "
          f"{1024 * (8 * 151936 + 24) / ms / 1e6:.0f} | stream |", flush=True)


main()
