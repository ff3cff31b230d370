"""Host-side eks_setup_csr time on cfg2 (pinned host CSR), averaged over 5 calls."""
import sys
import time
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import eks_inputs as ei  # noqa: E402
import paper_1804_10629_b200 as eks  # noqa: E402

p = ei.cfg2()
A = p.A
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
rp, cl, vl = pin(A.row_ptr), pin(A.col), pin(A.val)
S = eks.Solver(None)
S.setup(A.n, 0, A.n, rp, cl, vl)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    S.setup(A.n, 0, A.n, rp, cl, vl)
torch.cuda.synchronize()
print(f"setup_csr: {1e3 * (time.perf_counter() - t0) / 5:.1f} ms per call (EKS_SPMM_PATH={os.environ.get('EKS_SPMM_PATH', '')})")
b = pin(p.b)
x = pin(np.zeros(A.n))
t0 = time.perf_counter()
for _ in range(3):
    x[:] = 0
    st, rep = eks.eks_solve_ex(S.ctx, "sre-cg", 3, 16, 1e-8, b, x)
print(f"solve (host b/x): {1e3 * (time.perf_counter() - t0) / 3:.1f} ms per call, outer {rep['outer_iters']}")
