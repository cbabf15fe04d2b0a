"""Geometry sweep (dev tool): time every (NT, E, C) candidate for a shape via
the PAM_FORCE_CFG_* override and print rows/s and % of the HBM roofline."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W

VARS = {8: [(64,2,0),(128,4,0),(128,8,0),(256,8,0),(256,16,0),(512,16,0),(256,38,0),(512,24,0),(512,30,0),(512,34,0),
            (512,38,0),(256,38,2)],
        4: [(64,4,0),(128,8,0),(256,8,0),(256,16,0),(512,16,0),(256,40,0),(512,24,0),(512,40,0),(256,76,0),(256,76,2)]}

def bench(x, prm, reps=5):
    z = torch.empty_like(x); B = x.shape[0]
    am = torch.empty(B, dtype=torch.int32, device='cuda'); st = torch.empty_like(am)
    for _ in range(2): pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st)
    e1.record(); torch.cuda.synchronize()
    ok = bool(torch.equal(am.long(), x.argmax(dim=1))) and int((st != 0).sum()) == 0
    return e0.elapsed_time(e1) / reps, ok

def tsweep():
    for B, n, dt in [(4096, 151936, torch.float64), (4096, 32768, torch.float64)]:
        x = W.torch_gaussian(B, n, seed=1, dtype=dt)
        for dbg in ("0", "1"):
            os.environ["PAM_DEBUG_FLAGS"] = dbg
            for T in (1, 2, 3, 4, 6, 8):
                ms, ok = bench(x, pam.CutMaxParams(T=T))
                print(f"B={B} n={n} T={T} nostore={dbg}: {ms:8.4f} ms  ({ms/ (B/15) * 1e3:7.2f} us/row/cluster)", flush=True)
        os.environ.pop("PAM_DEBUG_FLAGS")

def main():
    if len(sys.argv) > 1 and sys.argv[1] == "tsweep":
        return tsweep()
    shapes = [(4096, 151936, torch.float64), (4096, 151936, torch.float32), (4096, 32768, torch.float64),
              (4096, 32768, torch.float32), (4096, 1024, torch.float64), (256, 151936, torch.float64),
              (64, 151936, torch.float64)]
    if len(sys.argv) > 1:
        sel = sys.argv[1]
        # "5" = first five shapes; "@0,2" = shapes 0 and 2
        shapes = [shapes[int(i)] for i in sel[1:].split(",")] if sel.startswith("@") else shapes[:int(sel)]
    prm = pam.CutMaxParams()
    for B, n, dt in shapes:
        x = W.torch_gaussian(B, n, seed=1, dtype=dt)
        esz = x.element_size(); vec = 16 // esz
        key = "PAM_FORCE_CFG_F64" if esz == 8 else "PAM_FORCE_CFG_F32"
        res = []
        for C in range(1, 17):
            L = ((n + C - 1) // C + vec - 1) // vec * vec
            for nt, e, mb in VARS[esz]:
                G = mb
                if nt * e < L or nt * e > 1.3 * L: continue
                os.environ[key] = f"{nt},{e},{C},{mb}"
                try:
                    ms, ok = bench(x, prm)
                    info = pam.launch_info(esz, B, n, prm)
                except Exception as ex:
                    print("fail", nt, e, C, ex); continue
                gbs = B * (2 * n * esz + 4) / ms / 1e6
                res.append((gbs, nt, e, C, G, ms, ok, info['clusters'], info['ctas']))
        os.environ.pop(key, None)
        res.sort(reverse=True)
        ms_auto, _ = bench(x, prm)
        ia = pam.launch_info(esz, B, n, prm)
        print(f"== B={B} n={n} {dt}  [auto: {ia['threads']}x{ia['elems_per_thread']} C={ia['cluster']} -> {B*(2*n*esz+4)/ms_auto/1e6/65.402:.1f}%]")
        for gbs, nt, e, C, G, ms, ok, ncl, ctas in res:
            print(f"   NTG={nt:4d} E={e:3d} C={C:2d} MINB={G}  {ms:8.4f} ms  {gbs:7.1f} GB/s  {100*gbs/6540.2:5.1f}%  clusters={ncl} ctas={ctas} ok={ok}", flush=True)

main()
