"""Small launches of every kernel family: the lean and general CutMax kernels at
cluster sizes 1, 2, 9 and 16, generic p, early stop, fp32, unaligned rows, the
TieWarning fallback, the samplers and the analysis kernels.  Outputs are
pre-filled with NaN and must come back fully written; argmax must equal the
argmax of x.  Meant for the checked build (compute-sanitizer is closed on the
GPU pool):  make -C paper_2509_08383_b200/csrc checked &&
PAM_LIB_PATH=paper_2509_08383_b200/libpam_checked.so python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W


def check_argmax(x, am, st):
    ok = (st & 0xFF) == 0
    assert torch.equal(am[ok].long(), x[ok].argmax(dim=1)), "argmax"


def main():
    torch.cuda.set_device(0)
    prm = pam.CutMaxParams()
    cases = [(151936, 12, (512, 34, 9)), (32768, 6, (512, 32, 2)), (9000, 5, (128, 8, 9)),
             (16000, 4, (128, 8, 16)), (1024, 40, (128, 8, 1))]
    for n, B, g in cases:
        x = W.torch_gaussian(B, n, seed=n)
        x[0, 3] = x[0, 7] = x[0].max() + 1.0  # duplicated max: TieWarning fallback
        for general in (False, True):
            z = torch.full_like(x, float("nan"))
            with pam.geometry_override(8, *g):
                if general:
                    with pam.general_p3_kernel():
                        z, am, st = pam.cutmax_batch_device(x, prm, z=z)
                else:
                    z, am, st = pam.cutmax_batch_device(x, prm, z=z)
            torch.cuda.synchronize()
            check_argmax(x, am, st)
            assert bool(torch.isfinite(z).all()), "unwritten Z"
            assert int(st[0]) & 0x100, "TieWarning"
        print(f"cutmax n={n} B={B} geometry={g}: ok", flush=True)
    x = W.torch_gaussian(6, 20000, seed=3)
    for p in (pam.CutMaxParams(p=5, c=12.0, T=3), pam.CutMaxParams(p=13, c=15.0, T=4, epsStop=1e-3),
              pam.CutMaxParams(T=1), pam.CutMaxParams(invsqrtMode="poly", invMode="poly")):
        z, am, st = pam.cutmax_batch_device(x, p)
        torch.cuda.synchronize()
        check_argmax(x, am, st)
    xf = x.float()
    z, am, st = pam.cutmax_batch_device(xf, prm)
    torch.cuda.synchronize()
    check_argmax(xf, am, st)
    xu = W.torch_gaussian(4, 20001, seed=5)  # odd n: unaligned rows, direct loads
    z, am, st = pam.cutmax_batch_device(xu, prm)
    torch.cuda.synchronize()
    check_argmax(xu, am, st)
    print("generic p / early stop / T=1 / poly / fp32 / unaligned: ok", flush=True)
    xs = torch.as_tensor(W.zipf_logits(4, 32768, seed=4), device="cuda")
    tok, ins, st = pam.nucleus_sample_batch_device(xs, pam.SamplerConfig(p=0.9, seed=1), prm)
    torch.cuda.synchronize()
    tok2, ins2, st2 = pam.nucleus_sample_batch_device(xs, pam.SamplerConfig(p=0.9, seed=1), prm)
    torch.cuda.synchronize()
    assert torch.equal(tok, tok2)
    print("sampler: ok", flush=True)
    xa = W.torch_gaussian(3, 4096, seed=6)
    pam.convergence_trace_batch_device(xa, prm)
    pam.cutmax_jvp_batch_device(xa, torch.ones_like(xa), prm)
    torch.cuda.synchronize()
    print("analysis: ok", flush=True)
    print("SANITIZE CASES DONE", flush=True)


if __name__ == "__main__":
    main()
