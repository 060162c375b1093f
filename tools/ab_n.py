#!/usr/bin/env python
"""Leja it/s of the config-1 workload (phi_0..phi_3) at several grid sizes (A/B helper)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import sweep  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
out = []
for n in [int(x) for x in sys.argv[1].split(",")]:
    r = sweep.cfg_leja(s, n, (0, 1, 2, 3), n, reps=5)
    out.append((n, round(r["leja_it_per_s"]), round(sum(c["ms"] for c in r["calls"]), 3)))
print(os.environ.get("TAG", ""), out)
