"""Top stalled SASS instructions of an ncu report (source page, sass view), with the stall
reasons that dominate each.  usage: python tools/ncu_sass_hot.py report.ncu-rep [N]"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kf = os.environ.get("KREGEX")  # optional kernel filter (regex) for multi-kernel reports
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + (["-k", "regex:" + kf] if kf else [])
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = []
for r in rows[2:]:  # first kernel section only
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
ia, isrc, ism = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
tot = sum(float(r[ism] or 0) for r in data)
print(f"total samples {tot:.0f}, instructions {len(data)}")
agg = {}
for r in data:
    for i in stall_cols:
        agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
print("by reason:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][ism] or 0))[:n]:
    s = float(r[ism] or 0)
    reasons = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
    print(f"{idx:5d} {r[ia]} {s / tot:6.2%}  {r[isrc][:60]:60s} " + " ".join(f"{k}:{v / max(s, 1):.0%}" for v, k in reasons if v))

# samples per block of instructions (phase map), with the dominant stall per block
if len(sys.argv) > 3:
    b = int(sys.argv[3])
    for s0 in range(0, len(data), b):
        blk = data[s0:s0 + b]
        s = sum(float(r[ism] or 0) for r in blk)
        ops = {}
        for r in blk:
            op = r[isrc].split()[0] if r[isrc].split() else ""
            if op.startswith("@"):
                op = r[isrc].split()[1]
            ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + 1
        top = sorted(ops.items(), key=lambda x: -x[1])[:4]
        rs = sorted(((sum(float(r[i] or 0) for r in blk), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
        print(f"[{s0:5d},{s0 + b:5d}) {s / tot:6.1%}  {top}  " + " ".join(f"{k}:{v / max(s, 1):.0%}" for v, k in rs))
