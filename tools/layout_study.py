"""GPU re-run of the reference's layout / traversal study.

    python tools/layout_study.py [--sizes 64,65,128,129,256,257] [--repeats 20]

Prints the reference's report table (bench.bench_report) for every size x
layout x traversal, plus the soft-ordering notes, on the current GPU.
"""
import argparse
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2211_16718_b200 import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="64,65,128,129,256,257")
ap.add_argument("--repeats", type=int, default=20)
ap.add_argument("--tile", default="32,8")
a = ap.parse_args()
sizes = [int(s) for s in a.sizes.split(",")]
tile = tuple(int(s) for s in a.tile.split(","))
recs = bench.layout_sweep(sizes=sizes, repeats=a.repeats, traversals=bench.TRAVERSALS, tile=tile)
print(bench.bench_report(recs), end="")
for r in recs:
    if r.wasted_lanes:
        print(f"# {r.size_label} {bench._layout_name(r.layout)} {r.traversal}: "
              f"wasted {r.wasted_fraction:.1%} of lanes")
with warnings.catch_warnings(record=True):
    warnings.simplefilter("always")
    for note in bench.soft_ordering_checks(recs):
        print("# note:", note)
