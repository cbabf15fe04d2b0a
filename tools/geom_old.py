"""Time cutmax_rows_kernel under forced geometries (dev tool).  usage: geom_old.py B n NTG,E,C [...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ahead_check import timeit
B, n = int(sys.argv[1]), int(sys.argv[2])
os.environ.pop("PAM_ENABLE_AHEAD", None)
for g in sys.argv[3:]:
    os.environ["PAM_FORCE_CFG_F64"] = g
    ms, gbs, bad = timeit(B, n)
    print(f"rows kernel {g:10s} B={B} n={n}: {ms:.4f} ms {100 * gbs / 6547.5:.1f}% bad={bad}", flush=True)
