"""CLI for bench.c4_sweep: the c4 deviated-well logging sweep (s/position per DD scheme)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--stations", default="0,31,63")
ap.add_argument("--schemes", default="full,gauss_seidel")
ap.add_argument("--verbose", action="store_true")
a = ap.parse_args()
print(json.dumps(bench.c4_sweep(tuple(int(x) for x in a.stations.split(",")), tuple(a.schemes.split(",")),
                                verbose=a.verbose)))
