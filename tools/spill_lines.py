"""Attribute local-memory spills (STL/LDL) of one kernel to source lines (dev tool).
usage: python tools/spill_lines.py build/obj/cutmax_variants.o <mangled-substring>"""
import re, subprocess, sys, tempfile, os, collections
obj, pat = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
out = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
on, cur, cnt = False, None, collections.Counter()
for l in out.split("\n"):
    if ".text." in l and l.rstrip().endswith(":"):
        on = pat in l
    if not on: continue
    m = re.search(r'//## File "(?:.*/)?([^/"]+)", line (\d+)', l)
    if m: cur = f"{m.group(1)}:{m.group(2)}"
    m = re.search(r"\b(STL|LDL)(\.\w+)*\b", l)
    if m: cnt[(cur, m.group(1))] += 1
for (loc, k), v in sorted(cnt.items(), key=lambda x: -x[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{k} {v:4d}  {loc}")
