"""Summarise ptxas -v logs: registers / spills per kernel instantiation."""
import glob, re, subprocess, sys
for f in sorted(glob.glob("build/obj/*.ptxas.log")):
    cur = None
    for l in open(f):
        m = re.search(r"Compiling entry function '(\w+)'", l)
        if m: cur = m.group(1); spill = 0; stack = 0
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", l)
        if m and cur: stack, spill = int(m.group(1)), int(m.group(2))
        m = re.search(r"Used (\d+) registers", l)
        if m and cur:
            name = subprocess.run(["cu++filt", cur], capture_output=True, text=True).stdout.strip()
            name = re.sub(r"void pam::|\(pam::\w+\)|\(int\)|\(bool\)", "", name)
            if "-a" in sys.argv or spill or stack:
                print(f"{name:55s} regs={m.group(1):>4s} stack={stack:4d} spill={spill}")
            cur = None
