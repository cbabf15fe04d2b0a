"""Adversarial parity fuzz (dev tool): heavy tails, outliers, near-degenerate and
constant rows, huge offsets, small c, against the oracle, for the rows kernel
and the two-iterations-per-exchange kernel.  usage: fuzz_adversarial.py [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_08383_b200 as pam
from oracle import oracle as orc


def rows(rng, B, n):
    kind = rng.integers(0, 9)
    if kind == 0:
        return rng.standard_cauchy((B, n)), "cauchy"
    if kind == 1:
        return rng.lognormal(0, 2.5, (B, n)) * rng.choice([-1, 1]), "lognormal"
    if kind == 2:
        x = rng.normal(0, 1e-3, (B, n)); x[:, rng.integers(0, n)] = 30.0; return x, "outlier"
    if kind == 3:
        x = np.full((B, n), 2.5); x[:, rng.integers(0, n)] += 1e-10; return x, "near-constant"
    if kind == 4:
        return rng.normal(1e9, 1e-2, (B, n)), "offset1e9"
    if kind == 5:
        return rng.standard_t(2, (B, n)), "t2"
    if kind == 6:
        x = rng.normal(0, 3, (B, n)); x[:, :: 7] = -40.0; return x, "bimodal-heavy"
    if kind == 7:
        return rng.uniform(-1, 1, (B, n)) ** 9, "peaked"
    return rng.normal(0, 3, (B, n)), "gauss"


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(7)
    fails = 0
    for it in range(iters):
        B = int(rng.integers(1, 12)); n = int(rng.choice([64, 1000, 4096, 20000, 65536]))
        T = int(rng.integers(1, 7)); c = float(rng.choice([0.7, 1.5, 5.0, 20.0]))
        x, kind = rows(rng, B, n)
        prm = pam.CutMaxParams(p=3, c=c, T=T)
        zr, amr, sr = orc.cutmax_batch(x, prm.lower())
        for k in ("product", "general"):  # the product path (lean / warp kernel where they apply) and the general kernel
            import contextlib
            with (pam.general_p3_kernel() if k == "general" else contextlib.nullcontext()):
                z, am, st = pam.cutmax_batch_device(torch.as_tensor(x, device="cuda"), prm)
                torch.cuda.synchronize()
            z, am, st = z.cpu().numpy(), am.cpu().numpy(), st.cpu().numpy()
            ok = sr == 0
            err = max([float(np.max(np.abs(z[r] - zr[r])) / np.max(np.abs(zr[r]))) for r in np.nonzero(ok)[0]], default=0.0)
            tol = 1e-12 * max(1.0, 3.0 ** T / 81.0)
            good = np.array_equal(st, sr) and np.array_equal(am[ok], amr[ok]) and err <= tol
            if not good:
                fails += 1
                print(f"FAIL it={it} kernel={k} kind={kind} B={B} n={n} T={T} c={c}: status_eq={np.array_equal(st, sr)} "
                      f"argmax_eq={np.array_equal(am[ok], amr[ok])} err={err:.2e} st={st.tolist()} sr={sr.tolist()}",
                      flush=True)
    print(f"done: {iters} cases x 2 kernels, {fails} failures")


if __name__ == "__main__":
    main()
