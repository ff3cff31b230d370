"""cfg1 (2D Poisson 64², launch-bound) and cfg2 solve time: plain (0), CUDA-graph replay with a host loop
test per outer iteration (1), and the device-resident loop (2: one graph launch for the steady solve)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import eks_inputs as ei  # noqa: E402
import paper_1804_10629_b200 as eks  # noqa: E402

for name, p in (("cfg1", ei.cfg1()), ("cfg2", ei.cfg2())):
    S = eks.Solver(p.A)
    b = torch.from_numpy(p.b).cuda()
    for g in (0, 1, 2, 0, 1, 2, 1, 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 5 if name == "cfg1" else 2
        for _ in range(reps):
            r = S.solve(b, p.method, p.s, p.t, p.tol, use_graph=g)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        print(f"{name} use_graph={g}: {1e3 * dt:.2f} ms per solve, {r['outer_iters']} outer, "
              f"{r['outer_iters'] / dt:.0f} outer it/s (device {r['outer_iters'] / r['solve_seconds']:.0f})")
    S.close()
