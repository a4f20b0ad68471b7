"""Run the default FWHT pass plan a few times (profiling driver for ncu);
the config input is regenerated before every transform, so each one runs the
plan fwht_array picks for that input (the compact plan at n = 26..32)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1607_01039_b200 as bw  # noqa: E402
from paper_1607_01039_b200 import signals  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=28)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
spec = signals.config(4, a.n)
t = signals.make(spec)
for rep in range(a.reps):
    if rep:
        signals.generate(spec, t)
    bw.fwht_array(t)
torch.cuda.synchronize()
print("ok", a.n)
