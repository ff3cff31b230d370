import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import eks_inputs as ei, paper_1804_10629_b200 as eks
A = ei.cfg5_operator() if os.environ.get("OP") == "cfg5" else ei.cfg4().A
S = eks.Solver(A)
t = int(sys.argv[1]) if len(sys.argv) > 1 else 64
var = int(sys.argv[2]) if len(sys.argv) > 2 else 2
X = ei.uniform_pm1_torch(77, A.n * t, "cuda").view(A.n, t)
v = ei.uniform_pm1_torch(78, A.n, "cuda")
Y0 = torch.zeros_like(X)
eks.eks_k_time_spmm(S.ctx, t, X, Y0, v, 0, 1)  # plain CSR reference
Yfix = torch.empty_like(X)
for rep in range(4):
    fresh = rep % 2 == 1
    Y = torch.full_like(X, float("nan")) if fresh else Yfix.fill_(float("nan"))
    eks.eks_k_time_spmm(S.ctx, t, X, Y, v, var, 1)
    torch.cuda.synchronize()
    bad = (Y != Y0).any(dim=1).nonzero()
    nan = torch.isnan(Y).any(dim=1).sum().item()
    print(f"var {var} rep {rep} fresh={fresh} Y@{Y.data_ptr():#x} X@{X.data_ptr():#x}: bad {bad.numel()} nanrows {nan}",
          (bad[:2].flatten().tolist(), bad[-1:].flatten().tolist()) if bad.numel() else "", flush=True)
