"""Aggregate ncu per-instruction stall samples (source page, SASS) by CUDA
source line, using the cubin's line table (dev tool).
usage: python tools/ncu_lines.py <rep.ncu-rep> <object.o> <mangled-kernel-substring> [top]"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, pat = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
f = lambda x: float(x) if x not in ("", None) else 0.0
base = int(data[0][ix["Address"]], 16)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [x for x in os.listdir(d) if x.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
on, cur, line_of = False, None, {}
for l in dis.split("\n"):
    if ".text." in l and l.rstrip().endswith(":"):
        on = pat in l
    if not on:
        continue
    m = re.search(r'//## File "(?:.*/)?([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
    m = re.match(r"\s*/\*([0-9a-f]{4,6})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: collections.Counter())
tot = 0.0
for r in data:
    off = int(r[ix["Address"]], 16) - base
    a = f(r[ix["Warp Stall Sampling (All Samples)"]])
    tot += a
    ln = line_of.get(off, "?")
    agg[ln]["all"] += a
    for s in stalls:
        agg[ln][s] += f(r[ix[s]])
for ln, c in sorted(agg.items(), key=lambda x: -x[1]["all"])[:top]:
    t = sorted(((k, v) for k, v in c.items() if k != "all"), key=lambda x: -x[1])[:3]
    print(f"{100 * c['all'] / tot:6.2f}%  {ln:34s} " + " ".join(f"{k[6:]}={100 * v / tot:.1f}" for k, v in t))
