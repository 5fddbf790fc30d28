"""CLI for bench.moving_window: the paper's moving-window logging simulation (section 3.3,
SURVEY 8(f)-1); window 1 = 256x128x128 cells (hole along x), 2 sub-domains; window 2 = 256^3,
8 sub-domains (--window 2)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--stations", type=int, default=5)
ap.add_argument("--window", type=int, default=1)
ap.add_argument("--scheme", default="gauss_seidel")
ap.add_argument("--precond", type=int, default=0)
ap.add_argument("--tol", type=float, default=1e-3)
a = ap.parse_args()
kw = dict(n=(256, 256, 256), splits=(2, 2, 2)) if a.window == 2 else {}
print(json.dumps(bench.moving_window(a.stations, scheme=a.scheme, precond=a.precond, tol=a.tol, **kw)))
