"""fp32 accuracy probe (dev tool): per-iteration (mu, s2) of the GPU kernel vs the oracle."""
import os, sys, numpy as np, torch, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_08383_b200 as pam
from paper_2509_08383_b200 import workloads as W
from oracle import oracle as orc
T = 4
x = W.gaussian(700, 6000, seed=40 + T); x[5] += 300.0; x[6, :] = 2.5
x32 = x.astype(np.float32)
prm = pam.CutMaxParams(T=T)
os.environ["PAM_FORCE_CFG_F32"] = "256,40,1"
xt = torch.as_tensor(x32, device="cuda")
stt = torch.zeros((700, T, 2), dtype=torch.float64, device="cuda")
z, am, st = pam.cutmax_batch_device(xt, prm, stats=stt)
torch.cuda.synchronize()
z = z.cpu().numpy(); stt = stt.cpu().numpy()
lib = orc.load()
for row in (298, 331, 0, 1, 150):
    n = 6000
    zz = np.empty(n, np.float32); a = C.c_int32(-1); s = np.zeros((T, 2))
    lib.orc_cutmax_f32(x32[row].ctypes.data, n, C.byref(prm.lower()), zz.ctypes.data, C.byref(a), s.ctypes.data)
    zd, _, _ = orc.cutmax_batch(x32[row:row + 1].astype(np.float64), prm.lower())
    err = np.max(np.abs(z[row] - zd[0])) / np.max(zd[0])
    print(f"row {row}: gpu-vs-exact {err:.3e}  oracle32-vs-exact {np.max(np.abs(zz - zd[0])) / np.max(zd[0]):.3e}")
    for t in range(T):
        print(f"   t={t} gpu mu={stt[row,t,0]:.10f} s2={stt[row,t,1]:.10e} | orc mu={s[t,0]:.10f} s2={s[t,1]:.10e} | dmu={stt[row,t,0]-s[t,0]:.2e} ds2/s2={(stt[row,t,1]-s[t,1])/s[t,1]:.2e}")
    i = int(np.argmax(np.abs(z[row] - zd[0])))
    print(f"   worst elem {i}: gpu {z[row,i]:.9e} exact {zd[0,i]:.9e} oracle32 {zz[i]:.9e} x={x32[row,i]}")
