import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W
from oracle import oracle as orc
def normwise(a,b):
    a=np.asarray(a,np.float64); b=np.asarray(b,np.float64); return float(np.max(np.abs(a-b))/np.max(np.abs(b)))
for T in (2, 4):
    x = W.gaussian(700, 6000, seed=40 + T); x[5] += 300.0; x[6,:] = 2.5
    prm = pam.CutMaxParams(T=T)
    for dt in (np.float32, np.float64):
        xx = x.astype(dt)
        zr, ar, sr = orc.cutmax_batch(xx, prm.lower())
        z64, _, _ = orc.cutmax_batch(xx.astype(np.float64), prm.lower())
        key = "PAM_FORCE_CFG_F32" if dt == np.float32 else "PAM_FORCE_CFG_F64"
        os.environ[key] = "256,40,1" if dt == np.float32 else "256,24,1"
        for gen in (0, 1):
            if gen: os.environ["PAM_FORCE_GENERIC_P"] = "1"
            xt = torch.as_tensor(xx, device='cuda')
            z, am, st = pam.cutmax_batch_device(xt, prm); torch.cuda.synchronize()
            z = z.cpu().numpy(); am = am.cpu().numpy(); st = st.cpu().numpy()
            os.environ.pop("PAM_FORCE_GENERIC_P", None)
            ok = sr == 0
            e_or = {r: normwise(z[r], zr[r]) for r in np.nonzero(ok)[0]}
            e_ex = {r: normwise(z[r], z64[r]) for r in np.nonzero(ok)[0]}
            w1 = max(e_or, key=e_or.get); w2 = max(e_ex, key=e_ex.get)
            print(f"T={T} {dt.__name__} generic={gen}: vs oracle max {e_or[w1]:.3e} (row {w1}); vs f64 exact max {e_ex[w2]:.3e} (row {w2}); status eq {np.array_equal(st, sr)} argmax eq {np.array_equal(am[ok], ar[ok])}")
        os.environ.pop(key)
