"""Layered configurations with the physical three-layer table on the GPU: c3 operator leg,
s/position per scheme on c3capped and c3 (literal), and the c4 layered sweep (bench.py legs)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="op,c3capped,c3,c4")
ap.add_argument("--stations", default="0,31,63")
ap.add_argument("--freqs", default="4e5")
ap.add_argument("--c4runs", default="full:1,gauss_seidel:1")
ap.add_argument("--c4name", default="default")
ap.add_argument("--tol", type=float, default=None)
ap.add_argument("--out", default=None)
a = ap.parse_args()
w = a.what.split(",")
out = {}
if "op" in w:
    out["operator_c3"] = bench.layered_leg()
    print(json.dumps(out["operator_c3"]), flush=True)
if "c3capped" in w:
    out["dd_c3capped"] = bench.layered_dd_leg("c3capped")
    print(json.dumps(out["dd_c3capped"]), flush=True)
if "c3" in w:
    out["dd_c3"] = bench.layered_dd_leg("c3", runs=(("full", 1), ("gauss_seidel", 1), ("full", 0)), reps=0)
    print(json.dumps(out["dd_c3"]), flush=True)
if "c4" in w:
    variants = bench.C4_VARIANTS
    if a.c4name != "default":
        runs = tuple((r.split(":")[0], int(r.split(":")[1])) for r in a.c4runs.split(","))
        variants = ((a.c4name, a.tol if a.tol else 1e-6, runs),)
    st = tuple(range(64)) if a.stations == "all" else tuple(int(x) for x in a.stations.split(","))
    out["c4"] = bench.c4_layered_sweep(st,
                                       tuple(float(x) for x in a.freqs.split(",")), variants, verbose=True)
    print(json.dumps(out["c4"]), flush=True)
if a.out:
    json.dump(out, open(a.out, "w"))
