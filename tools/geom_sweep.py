import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
from ahead_check import timeit
os.environ.setdefault("PAM_ENABLE_AHEAD", "1")
import paper_2509_08383_b200 as pam
for g in ["512,34,9", "512,32,10", "512,24,13", "256,16,16"]:
    os.environ["PAM_FORCE_AHEAD"] = g
    try:
        ms, gbs, bad = timeit(4096, 151936)
        info = pam.launch_info(8, 4096, 151936, pam.CutMaxParams())
        print(f"ahead {g}: {ms:.4f} ms {100*gbs/6547.5:.1f}% clusters={info['clusters']} C={info['cluster']} cfg={info['threads']}x{info['elems_per_thread']}", flush=True)
    except Exception as e:
        print(g, "ERR", e)
os.environ.pop("PAM_FORCE_AHEAD")
