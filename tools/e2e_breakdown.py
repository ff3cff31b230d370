"""Where the cfg5 end-to-end step goes: eks_setup_csr from pinned host CSR, eks_basis_sweep from / to pinned
host blocks, and the same sweep on device-resident blocks (wall clock, 3 repetitions each)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import eks_inputs as ei  # noqa: E402
import paper_1804_10629_b200 as eks  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 384
t, s_ = 16, 4
A = ei.cfg5_operator(N)
n = A.n


def pinned(a):
    tt = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
    tt.numpy()[...] = a
    return tt


hrp, hcol, hval = pinned(A.row_ptr), pinned(A.col), pinned(A.val)
S = eks.Solver(None)
X0 = ei.cfg5_start_block_torch(n, t, "cuda")
W = torch.empty_like(X0)
hX0 = X0.cpu().pin_memory()
hW = torch.empty_like(hX0).pin_memory()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S.setup(n, 0, n, hrp.numpy(), hcol.numpy(), hval.numpy())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    eks.eks_basis_sweep(S.ctx, t, 20 * s_, hX0.numpy(), hW.numpy())
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    eks.eks_basis_sweep(S.ctx, t, 20 * s_, X0, W)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    gb = (hrp.numel() * 8 + hcol.numel() * 4 + hval.numel() * 8) / 1e9
    print(f"rep {rep}: setup {t1 - t0:.3f} s ({gb:.2f} GB CSR), sweep host->host {t2 - t1:.3f} s "
          f"({hX0.numel() * 8 / 1e9:.2f} GB in, {hW.numel() * 8 / 1e9:.2f} GB out), sweep device {t3 - t2:.3f} s")
S.close()
