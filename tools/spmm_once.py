#!/usr/bin/env python
"""The solve's SpMM-block step (eks_k_time_spmm variant 7) on the N³ Laplacian at one t, for ncu:
  python tools/spmm_once.py --N 384 --t 32 [--reps 1]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import eks_inputs as ei  # noqa: E402
import paper_1804_10629_b200 as eks  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=384)
ap.add_argument("--t", type=int, default=16)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
A = ei.cfg5_operator(a.N)
S = eks.Solver(A)
X = ei.uniform_pm1_torch(77, A.n * a.t, "cuda").view(A.n, a.t)
Y = torch.empty_like(X)
v = ei.uniform_pm1_torch(78, A.n, "cuda")
ms = eks.eks_k_time_spmm(S.ctx, a.t, X, Y, v, 7, a.reps)
print({"n": A.n, "t": a.t, "ms": ms, "gbs": (56.0 * A.n + 16.0 * A.n * a.t + 8.0 * A.n) / (ms * 1e-3) / 1e9})
S.close()
