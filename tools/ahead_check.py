"""Dev check of the two-iterations-per-exchange kernel: parity vs the oracle on
the BASELINE shapes + edge rows, then device timing against the
one-exchange-per-iteration kernel (PAM_DISABLE_AHEAD)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
os.environ.setdefault("PAM_ENABLE_AHEAD", "1")
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W
from oracle import oracle as orc


def nw(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def check(name, x, **kw):
    prm = pam.CutMaxParams(**kw)
    xt = torch.as_tensor(x, device="cuda")
    t0 = time.time()
    z, am, st = pam.cutmax_batch_device(xt, prm)
    torch.cuda.synchronize()
    z, am, st = z.cpu().numpy(), am.cpu().numpy(), st.cpu().numpy()
    zr, amr, sr = orc.cutmax_batch(x, prm.lower())
    ok = sr == 0
    worst = max([nw(z[r], zr[r]) for r in np.nonzero(ok)[0]], default=0.0)
    print(f"{name:34s} status_eq={np.array_equal(st, sr)} argmax_eq={np.array_equal(am[ok], amr[ok])} "
          f"worst={worst:.2e} bad_status={int((sr != 0).sum())} {time.time()-t0:.2f}s", flush=True)
    return np.array_equal(st, sr) and np.array_equal(am[ok], amr[ok]) and worst <= 1e-12


def timeit(B, n, reps=10, **kw):
    x = W.torch_gaussian(B, n, seed=1)
    z = torch.empty_like(x)
    am = torch.empty(B, dtype=torch.int32, device="cuda")
    st = torch.empty_like(am)
    prm = pam.CutMaxParams(**kw)
    for _ in range(3):
        pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    gbs = B * (2 * n * 8 + 4) / ms / 1e6
    return ms, gbs, int((st != 0).sum())


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "all"
    if mode in ("all", "parity"):
        allok = True
        allok &= check("gauss 8x32768 T4", W.gaussian(8, 32768, 1), T=4)
        for T in (1, 2, 3, 5, 6):
            allok &= check(f"gauss 8x32768 T{T}", W.gaussian(8, 32768, 10 + T), T=T)
        allok &= check("zipf 8x151936 T4", W.zipf_logits(8, 151936, 2), T=4)
        allok &= check("gauss 8x151936 T4", W.gaussian(8, 151936, 3), T=4)
        x, _, _ = W.planted(32, 32768, 4)
        allok &= check("planted 32x32768 T3", x, T=3)
        allok &= check("planted 32x32768 T4", x, T=4)
        allok &= check("gauss 64x1024 T4", W.gaussian(64, 1024, 5), T=4)
        x = W.gaussian(700, 6000, 6)
        x[5] += 300.0
        x[6, :] = 2.5
        x[9, 3] = np.nan
        x[11, 0] = 40.0
        allok &= check("pipeline 700x6000 T4 (+edge rows)", x, T=4)
        allok &= check("pipeline 700x6000 T3", x, T=3)
        x = np.random.default_rng(7).standard_cauchy((16, 32768))
        allok &= check("cauchy 16x32768 T4", x, T=4)
        allok &= check("n=2 B=5", W.gaussian(5, 2, 8), T=4)
        allok &= check("n=4096 c=1.5 T4", W.gaussian(16, 4096, 9), T=4, c=1.5)
        print("PARITY", "OK" if allok else "FAIL", flush=True)
    if mode in ("all", "time"):
        for (B, n) in ((4096, 151936), (256, 151936), (4096, 32768), (256, 32768), (4096, 1024)):
            for dis in (False, True):
                if dis:
                    os.environ["PAM_DISABLE_AHEAD"] = "1"
                else:
                    os.environ.pop("PAM_DISABLE_AHEAD", None)
                ms, gbs, bad = timeit(B, n)
                print(f"B={B:5d} n={n:6d} {'old  ' if dis else 'ahead'} {ms:8.4f} ms {gbs:8.1f} GB/s "
                      f"{100 * gbs / 6547.5:5.1f}% bad={bad}", flush=True)
        os.environ.pop("PAM_DISABLE_AHEAD", None)
    if mode in ("all", "time", "flags"):
        os.environ["PAM_DEBUG_FLAGS"] = "1"
        ms, gbs, bad = timeit(4096, 151936)
        print(f"B= 4096 n=151936 ahead debug_flags=1 {ms:8.4f} ms {gbs:8.1f} GB/s {100 * gbs / 6547.5:5.1f}%")
        os.environ.pop("PAM_DEBUG_FLAGS", None)
    if mode in ("all", "lat", "skip"):
        os.environ["PAM_DEBUG_FLAGS"] = "2"
        for (B, n) in ((4096, 151936), (4096, 32768)):
            ms, gbs, bad = timeit(B, n)
            info = pam.launch_info(8, B, n, pam.CutMaxParams())
            print(f"skip passes B={B} n={n}: {ms * 1.965e6 / (B / info['clusters']):8.0f} cycles/row "
                  f"(clusters={info['clusters']}, C={info['cluster']})")
        os.environ.pop("PAM_DEBUG_FLAGS", None)
    if mode in ("all", "lat"):
        # exchange-latency probe: tiny slices (128 threads x 8 per CTA), C = 9 and 2
        for C in (9, 2):
            n = 1024 * C
            os.environ["PAM_FORCE_AHEAD"] = f"128,8,{C}"
            ms, gbs, bad = timeit(4096, n)
            info = pam.launch_info(8, 4096, n, pam.CutMaxParams())
            cyc = ms * 1.965e6 / (4096 / info["clusters"])
            print(f"lat probe ahead C={C} clusters={info['clusters']}: {cyc:8.0f} cycles/row (2 exchanges)")
            os.environ.pop("PAM_FORCE_AHEAD", None)
            os.environ["PAM_FORCE_CFG_F64"] = f"128,8,{C}"
            ms, gbs, bad = timeit(4096, n)
            info = pam.launch_info(8, 4096, n, pam.CutMaxParams())
            cyc = ms * 1.965e6 / (4096 / info["clusters"])
            print(f"lat probe old   C={C} clusters={info['clusters']}: {cyc:8.0f} cycles/row (4 exchanges)")
            os.environ.pop("PAM_FORCE_CFG_F64", None)
