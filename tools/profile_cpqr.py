"""pivoted_qr_partial of a 610 x 10000 Gaussian (the C3 sketch shape), k = 600,
twice (for ncu: -k regex:cpqr --launch-skip 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1502_05366_b200 as R

eng = R.Engine(0)
a = np.random.default_rng(0).standard_normal((int(os.environ.get("M", 610)), int(os.environ.get("N", 10000))))
for _ in range(2):
    eng.pivoted_qr_partial(a, int(os.environ.get("K", 600)))
print("ok")
