"""Per-kernel table of an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file).
usage: python tools/launch_table.py launches.csv "command description" [bench.json]"""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iu = hdr.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    v = v / 1e6 if r[iu] == "ns" else (v / 1e3 if r[iu] == "us" else v)  # -> ms
    name = r[ik].split("(")[0]
    tot[name] += v
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"ncu --metrics gpu__time_duration.sum --clock-control none of: {sys.argv[2]} "
      "(cold-cache serialised launches: compare shares)")
print(f"{'kernel':44s} {'launches':>9s} {'total ms':>10s} {'ms/launch':>10s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:44s} {cnt[k]:9d} {tot[k]:10.3f} {tot[k] / cnt[k]:10.4f} {tot[k] / all_ms:6.3f}")
ops = {"K-A": "k_xfwd", "K-B": "k_yfwd", "K-C": "k_zconv", "K-D": "k_yinv", "K-E": "k_xinv"}
per = {}
for lab, pre in ops.items():
    ks = [k for k in tot if pre in k]
    if ks:
        per[lab] = sum(tot[k] for k in ks) / sum(cnt[k] for k in ks)
if len(per) == 5:
    step = sum(per.values())
    line = f"\nshare of the operator step (5 kernels): K-C {per['K-C']:.3f} / {step:.3f} = {per['K-C'] / step:.3f}"
    if len(sys.argv) > 3:
        b = json.load(open(sys.argv[3]))
        kk = b["kernels"]
        line += f" (bench CUDA events: {kk['K-C z-convolution']['ms'] / sum(v['ms'] for v in kk.values()):.3f})"
    print(line)
