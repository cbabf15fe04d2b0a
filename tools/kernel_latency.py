"""Kernel-only latency of the small-batch C5 points (dev tool): run under
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file out.csv python tools/kernel_latency.py
Each (dtype, n, B) point launches the product path 3 times with the L2 flushed in
between (cold input, as in decode); tools/kernel_latency.py --summarise out.csv prints the table."""
import csv, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

POINTS = [(dt, n, B) for dt in ("f64", "f32") for n in (1024, 32768, 151936) for B in (1, 16, 256)]


def run():
    import torch
    import paper_2509_08383_b200 as pam
    from paper_2509_08383_b200 import workloads as W
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    prm = pam.CutMaxParams()
    for dt, n, B in POINTS:
        x = W.torch_gaussian(B, n, seed=1, dtype=torch.float64 if dt == "f64" else torch.float32)
        z = torch.empty_like(x)
        am = torch.empty(B, dtype=torch.int32, device="cuda")
        st = torch.empty_like(am)
        for _ in range(3):
            flush.zero_()
            pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st)
        torch.cuda.synchronize()


def summarise(path):
    rows = [r for r in csv.reader(open(path, errors="ignore")) if len(r) > 5]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    iu = hdr.index("Metric Unit")
    ours = [(r[ik], float(r[iv].replace(",", "")) * (1e-3 if r[iu] == "ns" else 1.0)) for r in rows[1:]
            if "cutmax" in r[ik]]
    assert len(ours) == 3 * len(POINTS), (len(ours), len(POINTS))
    print("| dtype | n | B | kernel | kernel time, us (median of 3, L2 flushed) |")
    print("|---|---|---|---|---|")
    for i, (dt, n, B) in enumerate(POINTS):
        ks = sorted(v for _, v in ours[3 * i:3 * i + 3])
        name = ours[3 * i][0].split("(")[0].replace("void pam::", "")
        print(f"| {dt} | {n} | {B} | `{name}` | {ks[1]:.1f} |")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarise":
        summarise(sys.argv[2])
    else:
        run()
