"""Dev tool: time the p = 3 CutMax kernel at forced geometries on one (dtype, B, n)
and check each against the default geometry (argmax/status identical, Z within
1e-12 normwise).  usage: python tools/geo_ab.py [n] [B] NTGxExC[xMINB] ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

PEAK = 6547.5


def run(x, prm, reps=20):
    z = torch.empty_like(x)
    B = x.shape[0]
    am = torch.empty(B, dtype=torch.int32, device=x.device)
    st = torch.empty_like(am)
    f = lambda: pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, z, am, st


def main():
    n = int(sys.argv[1]); B = int(sys.argv[2])
    dt = torch.float32 if os.environ.get("GEO_F32") else torch.float64
    esz = 4 if dt == torch.float32 else 8
    prm = pam.CutMaxParams()
    x = W.torch_gaussian(B, n, seed=1, dtype=dt)
    ms, z0, a0, s0 = run(x, prm)
    info = pam.launch_info(esz, B, n, prm)
    gbs = B * (2 * n * esz + 4) / ms / 1e6
    print(f"default {info['threads']}x{info['elems_per_thread']} C={info['cluster']}: {ms:.4f} ms {gbs:.0f} GB/s {100*gbs/PEAK:.1f}%")
    for g in sys.argv[3:]:
        parts = [int(v) for v in g.split("x")]
        ntg, e, c = parts[:3]
        mb = parts[3] if len(parts) > 3 else 0
        try:
            with pam.geometry_override(esz, ntg, e, c, mb):
                ms, z, a, s = run(x, prm)
                info = pam.launch_info(esz, B, n, prm)
        except Exception as ex:  # noqa: BLE001
            print(g, "failed:", ex)
            continue
        err = ((z.double() - z0.double()).abs().amax(1) / z0.double().abs().amax(1)).max().item()
        same = bool(torch.equal(a, a0) and torch.equal(s, s0))
        gbs = B * (2 * n * esz + 4) / ms / 1e6
        print(f"{g}: clusters={info['clusters']} {ms:.4f} ms {gbs:.0f} GB/s {100*gbs/PEAK:.1f}%  argmax/status same={same} normwise-vs-default={err:.1e}")


if __name__ == "__main__":
    main()
