"""Stall samples of one kernel in an ncu report, attributed to CUDA source lines via the
cubin's line table (needs -lineinfo).  usage: ncu_lines.py REPORT OBJ.o MANGLED_FN SRC.cu [N]"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

rep, obj, fn, srcf = sys.argv[1:5]
n = int(sys.argv[5]) if len(sys.argv) > 5 else 30
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr, data = rows[1], rows[2:]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
lines = dis.split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":")][0]
cur, m = None, {}
for l in lines[start + 1:]:
    if l.startswith(".text.") or "\t.section" in l:
        break
    mm = re.search(r'File "([^"]+)", line (\d+)', l) if "//##" in l else None
    if mm:
        cur = (os.path.basename(mm.group(1)), int(mm.group(2)))
        continue
    mm = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if mm and cur:
        m[int(mm.group(1), 16)] = cur
i_s, i_a = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Address")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][i_a], 16)
tot, per = Counter(), {}
for r in data:
    ln = m.get(int(r[i_a], 16) - base)
    tot[ln] += float(r[i_s] or 0)
    pr = per.setdefault(ln, Counter())
    for i in stalls:
        try:
            pr[hdr[i][6:]] += float(r[i] or 0)
        except ValueError:
            pass
srcs = {}


def text(ln):
    if not ln:
        return ""
    f, k = ln
    if f not in srcs:
        path = os.path.join(os.path.dirname(os.path.abspath(srcf)), f)
        srcs[f] = open(path).read().split("\n") if os.path.exists(path) else []
    return srcs[f][k - 1].strip()[:70] if k <= len(srcs[f]) else ""
T = sum(tot.values())
print(f"total samples {T:.0f}")
for ln, v in tot.most_common(n):
    top = ",".join(f"{k}:{int(x)}" for k, x in per[ln].most_common(3))
    print(f"{ln[0][:10] if ln else '-'}:{ln[1] if ln else 0}\t{100*v/T:5.1f}%\t{top}\t{text(ln)}")
