#!/usr/bin/env python
"""One cfg5-style basis sweep (reading R27) on an N³ Laplacian, for ncu captures of the sweep kernels:
  python tools/sweep_once.py --N 256 --t 16 --nblocks 4 [--reps 1]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import eks_inputs as ei  # noqa: E402
import paper_1804_10629_b200 as eks  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=256)
ap.add_argument("--t", type=int, default=16)
ap.add_argument("--nblocks", type=int, default=4)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
A = ei.cfg5_operator(a.N)
S = eks.Solver(A)
X0 = ei.cfg5_start_block_torch(A.n, a.t, "cuda")
W = torch.empty_like(X0)
for _ in range(a.reps):
    rep = eks.eks_basis_sweep(S.ctx, a.t, a.nblocks, X0, W)
print({"n": A.n, "t": a.t, "nblocks": a.nblocks, "ms": rep["solve_seconds"] * 1e3, "launches": rep["gpu_launches"]})
S.close()
