#!/usr/bin/env python
"""Full-size solves of the BASELINE configs to tol (cfg3: MSDO-CG t=32 s=4; cfg4: SRE-CG t=64 s=2),
one JSON line per solve: outer iterations, status, device seconds, true residual, memory.

  python tools/full_solves.py --cfg cfg4 [--max-outer 3000] [--repeat 1] [--out gpurun_out/x.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import eks_inputs as ei  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg4")
    ap.add_argument("--N", type=int, default=0, help="grid size override (analog)")
    ap.add_argument("--max-outer", type=int, default=0)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--method", default="")
    ap.add_argument("--s", type=int, default=0)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch
    import paper_1804_10629_b200 as eks
    t0 = time.time()
    kw = {"N": args.N} if args.N else {}
    p = {"cfg2": ei.cfg2, "cfg3": ei.cfg3, "cfg4": ei.cfg4}[args.cfg](**kw)
    method = args.method or p.method
    s = args.s or p.s
    gen_s = time.time() - t0
    t1 = time.time()
    S = eks.Solver(p.A)
    setup_s = time.time() - t1
    b = torch.from_numpy(p.b).cuda()
    lines = []
    for rep_i in range(args.repeat):
        x = torch.zeros_like(b)
        st, rep = eks.eks_solve_ex(S.ctx, method, s, p.t, p.tol, b, x, max_outer=args.max_outer,
                                   profile=args.profile, raise_on=(5, 6, 1, 2, 3))
        free, total = torch.cuda.mem_get_info()
        line = {"cfg": p.name, "n": p.A.n, "nnz": p.A.nnz, "method": method, "s": s, "t": p.t, "tol": p.tol,
                "status": eks.STATUS.get(st, st), "outer_iters": rep["outer_iters"], "converged": rep["converged"],
                "solve_seconds": rep["solve_seconds"],
                "outer_it_per_s": rep["outer_iters"] / max(rep["solve_seconds"], 1e-9),
                "true_relres": rep["true_relres"], "rho_ratio": rep["rho"] / rep["rho0"],
                "max_outer_fit": rep["max_outer_fit"], "gpu_launches": rep["gpu_launches"],
                "model_bytes": rep["model_bytes"], "model_flops": rep["model_flops"],
                "hist_tail": [float(h) / rep["rho0"] for h in rep["hist"][-5:]] if rep["hist"] is not None else None,
                "hist_every_10": [float(h) / rep["rho0"] for h in rep["hist"][::10]] if rep["hist"] is not None else None,
                "device_free_gb": free / 1e9, "device_total_gb": total / 1e9, "gen_s": gen_s, "setup_s": setup_s,
                "err": eks.eks_error_string(S.ctx) if st else ""}
        if args.profile:
            pr = eks.eks_get_profile(S.ctx)
            line["profile_ms"] = pr["ms"]
            line["profile_launches"] = pr["launches"]
            line["profile_bytes"] = pr["bytes"]
            line["profile_flops"] = pr["flops"]
        print(json.dumps(line), flush=True)
        lines.append(line)
    if args.out:
        with open(args.out, "a") as f:
            for l in lines:
                f.write(json.dumps(l) + "\n")
    S.close()


if __name__ == "__main__":
    main()
