"""est-eval on the BASELINE config matrices on the GPU (reference
cli.py:301-341): python tools/est_eval.py [config ...] > profiles/r1_est_eval.csv"""
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19004_b200 import matgen  # noqa: E402
from paper_2604_19004_b200.est_eval import est_eval  # noqa: E402

cfgs = sys.argv[1:] or ["er10k", "poisson64", "rect", "rmat16", "rmat18", "rmat20"]
w = None
for name in cfgs:
    a, b = matgen.make_config(name)
    for r in est_eval(a, b, op="ab", name=name):
        if w is None:
            w = csv.DictWriter(sys.stdout, fieldnames=list(r))
            w.writeheader()
        w.writerow(r)
        sys.stdout.flush()
