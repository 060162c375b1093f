#!/usr/bin/env python
"""A/B of the EXPRB43 Allen-Cahn integrate metric (bench.py exprb43_steps), repeated."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2310_08344_b200 as lx  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
vals = []
for _ in range(3):
    r = bench.exprb43_steps(lx, torch, s, n=n)
    vals.append(round(r["value"], 1))
print(os.environ.get("TAG", ""), "exprb43 steps/s", vals, "iters/step", r["leja_iters_per_step"])
