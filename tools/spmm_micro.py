"""SpMM-block micro-benchmark: device time of one Y = A·X launch (eks_k_time_spmm) on the
BASELINE operators, for the plain SpMM and the fused SpMM+Gram variants, as GB/s of the
algorithmic bytes B_spmm = 12·nnz + 4(n+1) + 16·n·t."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import eks_inputs as ei  # noqa: E402
import paper_1804_10629_b200 as eks  # noqa: E402


def ops(names):
    for nm in names:
        t0 = time.time()
        if nm == "cfg2":
            A = ei.cfg2().A
        elif nm == "cfg3":
            A = ei.cfg3().A
        elif nm == "cfg4":
            A = ei.cfg4().A
        elif nm == "cfg5":
            A = ei.cfg5_operator()
        else:
            raise SystemExit(nm)
        print(f"# {nm}: n={A.n} nnz={A.nnz} generated in {time.time() - t0:.1f}s", flush=True)
        yield nm, A


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="cfg2,cfg3")
    ap.add_argument("--ts", default="8,16,32,64")
    ap.add_argument("--variants", default="0,1,2,3")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6558.7) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6558.7
    torch.cuda.set_device(0)
    for nm, A in ops(a.ops.split(",")):
        s = eks.Solver(A)
        for t in [int(x) for x in a.ts.split(",")]:
            need = 2 * A.n * t * 8
            if need > 0.8 * torch.cuda.mem_get_info()[0]:
                print(f"{nm} t={t}: skipped (memory)")
                continue
            X = torch.rand(A.n, t, dtype=torch.float64, device="cuda") - 0.5
            Y = torch.empty_like(X)
            v = torch.rand(A.n, dtype=torch.float64, device="cuda")
            # algorithmic bytes: A in the representation the kernel streams (stencil operators on the
            # plane-marching path: 8·7 B of values per row; CSR otherwise) + X read + Y written + v read
            B = 8.0 * 7 * A.n + 16.0 * A.n * t + 8.0 * A.n
            Bcsr = 12.0 * A.nnz + 4.0 * (A.n + 1) + 16.0 * A.n * t
            res = {}
            for var in [int(x) for x in a.variants.split(",")]:
                ms = eks.eks_k_time_spmm(s.ctx, t, X, Y, v, var, a.reps)
                res[var] = (ms, B / (ms * 1e-3) / 1e9)
            print(f"{nm} t={t:2d} B_spmm={B / 1e6:9.1f} MB  " + "  ".join(
                f"v{k}: {ms * 1e3:8.1f} us {gbs:7.0f} GB/s ({gbs / peak:4.2f})" for k, (ms, gbs) in res.items()),
                flush=True)
            del X, Y, v
            torch.cuda.empty_cache()
        s.close()


if __name__ == "__main__":
    main()
