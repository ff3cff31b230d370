#!/usr/bin/env python
"""bench.py — outer iterations/s of the s-step enlarged CG hot path on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` (N>1 under
torchrun, one rank per GPU over NCCL).  A *step* is one full ``eks_solve`` of the
workload (every §8(a) row: split, s chained SpMMs per outer iteration, CGS2 +
A-CholQR, x/r update, loop control) with the inputs resident in HBM; ``value`` =
outer iterations of all timed steps ÷ device time (CUDA events on the solve
stream, max over ranks).  Rank 0 prints ONE JSON line.

``--impl reference`` times the CPU oracle (oracle/, plain C, single thread) on
the same workload instead: each step = a bounded sample of outer iterations.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import eks_inputs as ei  # noqa: E402

METRIC = "outer iterations/s and SpMM-block HBM GB/s vs peak, at 1/2/4/8 B200"
UNIT = "outer_iter/s"


def workload(name: str):
    """(Problem, description).  Default = configs[1] of BASELINE.json (cfg2, s-step SRE-CG)."""
    if name == "cfg2":
        return ei.cfg2(method="sre-cg")
    if name == "cfg2-sre-cg2":
        return ei.cfg2(method="sre-cg2")
    if name == "cfg1":
        return ei.cfg1()
    if name == "cfg3":
        return ei.cfg3()
    if name == "cfg4":
        return ei.cfg4()
    raise SystemExit(f"unknown workload {name}")


def spmm_block(eks, torch, peak_gbs, N=384, ts=(8, 16, 32), reps=10, solver=None, A=None):
    """The SpMM-block kernel of the solve (fused Y = A·X + Gram [XᵀY | Xᵀr], tail reduction)
    timed on the cfg5 operator (384³ 7-point Laplacian, BASELINE configs[4]) with CUDA events
    over `reps` back-to-back launches; GB/s of B_spmm = 12·nnz + 4(n+1) + 16·n·t."""
    A = ei.cfg5_operator(N) if A is None else A
    s = eks.Solver(A) if solver is None else solver
    out = {"workload": f"cfg5 operator {N}^3 7-point Laplacian, n={A.n}, nnz={A.nnz}; fused SpMM+Gram launch "
                       f"as in eks_solve; X uniform, L2 not flushed between the {reps} launches (inputs > L2)",
           "bytes_formula": "8*7*n (stencil values) + 16*n*t (X, Y) + 8*n (v); frac_csr_formula uses "
                            "12*nnz + 4*(n+1) + 16*n*t", "peak_gbs": peak_gbs, "t": {}}
    for t in ts:
        X = torch.rand(A.n, t, dtype=torch.float64, device="cuda") - 0.5
        Y = torch.empty_like(X)
        v = torch.rand(A.n, dtype=torch.float64, device="cuda")
        ms = eks.eks_k_time_spmm(s.ctx, t, X, Y, v, 2, reps)
        # algorithmic bytes of the launch: the 7 stencil values per row the plane-marching kernel
        # streams (no indices), X read, Y written, v read; B_csr = the north_star's CSR formula
        B = 8.0 * 7 * A.n + 16.0 * A.n * t + 8.0 * A.n
        Bcsr = 12.0 * A.nnz + 4.0 * (A.n + 1) + 16.0 * A.n * t
        gbs = B / (ms * 1e-3) / 1e9
        out["t"][str(t)] = {"us_per_launch": ms * 1e3, "gbs": gbs, "frac": gbs / peak_gbs,
                            "frac_of_8TBs": gbs / 8000.0, "bytes": B,
                            "frac_csr_formula": Bcsr / (ms * 1e-3) / 1e9 / peak_gbs}
        del X, Y, v
        torch.cuda.empty_cache()
    if solver is None:
        s.close()
    return out


def pin_one_core():
    """The oracle is single-threaded: pin it to one host core (the last one the process may use)."""
    try:
        cores = sorted(os.sched_getaffinity(0))
        os.sched_setaffinity(0, {cores[-1]})
        return cores[-1]
    except (AttributeError, OSError):
        return None


def cfg5_oracle_sample(t: int, s_: int, N: int = 384, planes: int = 2, iters: int = 2):
    """The oracle (as it stands, definition mode, one thread pinned to one core) on a bounded sample of
    the cfg5 workload: the first `iters` outer iterations (iters·s blocks, window 2t, reading R27) of
    the basis sweep on the first `planes` z-planes of the 384³ grid (a 384×384×planes Dirichlet
    Laplacian, n_s rows), scaled to the full grid by the row count (the sweep's work is linear in n at
    fixed t, s).  Returns (outer it/s at full size, seconds, n_s)."""
    import oracle
    oracle.build()
    A = ei.stencil_csr(N, N, planes, ndim=3)
    X0 = ei.cfg5_start_block(A.n, t)
    aff = None
    try:
        aff = os.sched_getaffinity(0)
    except AttributeError:
        pass
    pin_one_core()
    try:
        t0 = time.perf_counter()
        st, _ = oracle.basis_sweep(A, X0, iters * s_)
        dt = time.perf_counter() - t0
    finally:
        if aff:
            os.sched_setaffinity(0, aff)
    if st != 0:
        raise SystemExit(f"oracle basis sweep failed: {st}")
    n_full = N ** 3
    return iters / (dt * n_full / A.n), dt, A.n


def roofline_of(agg, c, peaks):
    """Roofline of kernel class c from the profile pass: algorithmic bytes (flops) per launch ÷ the
    launch's CUDA-event time on the solve stream."""
    if agg["ms"].get(c, 0) <= 0:
        return None
    n_l = max(1, agg["launches"][c])
    gbs = agg["bytes"][c] / (agg["ms"][c] * 1e-3) / 1e9
    tfl = agg["flops"][c] / (agg["ms"][c] * 1e-3) / 1e12
    intensity = agg["flops"][c] / max(agg["bytes"][c], 1.0)
    ridge = peaks["dmma_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    common = {"kernel": c, "launches": agg["launches"][c], "avg_launch_us": 1e3 * agg["ms"][c] / n_l,
              "bytes_per_launch": agg["bytes"][c] / n_l, "flops_per_launch": agg["flops"][c] / n_l,
              "intensity_flop_per_byte": intensity, "traffic": None}
    if intensity > ridge:
        return dict(common, bound="alu", achieved=tfl, peak=peaks["dmma_tflops"], unit="TFLOP/s",
                    frac=tfl / peaks["dmma_tflops"],
                    peak_source="measured fp64 DMMA (profiles/fp64_peaks_r01.json, tools/fp64_peaks.cu)")
    return dict(common, bound="hbm", achieved=gbs, peak=peaks["hbm_gbs"], unit="GB/s", frac=gbs / peaks["hbm_gbs"],
                peak_source=peaks["source"], frac_of_8TBs=gbs / 8000.0)


def attach_traffic(rf, name):
    """DRAM bytes per launch of the same kernel class from a committed ncu --set full capture."""
    tf = os.path.join(ROOT, "profiles", name)
    if rf is None or not os.path.exists(tf):
        return
    tr = json.load(open(tf)).get("classes", {})
    if tr.get(rf["kernel"]):
        rf["traffic"] = tr[rf["kernel"]]
        rf["traffic_source"] = f"profiles/{name} (ncu dram__bytes_read.sum + dram__bytes_write.sum per launch)"


def run_cfg5(args, eks, torch, dist, world, rank, local):
    """BASELINE configs[4] (the bench headline): basis-generation sweep only, 20 outer iterations of
    s blocks on the 384³ Laplacian from a seeded unit-norm random block (reading R27).  A step = one
    eks_basis_sweep call (20·s blocks: chained SpMM + CGS2 + A-CholQR, every §8(a) row except the
    x/r update, which cfg5 does not have); value = outer iterations/s."""
    N, t, s_ = args.cfg5_n, args.t or 16, args.s or 4
    t_gen = time.perf_counter()
    A = ei.cfg5_operator(N)
    gen_s = time.perf_counter() - t_gen
    n = A.n
    lo = (rank * (t // world)) * n // t
    hi = ((rank + 1) * (t // world)) * n // t
    slab = A.rows(lo, hi)
    uid = None
    if world > 1:
        obj = [eks.eks_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    solver = eks.Solver(None, rank=rank, nranks=world, device=local, nccl_id=uid)
    t_set = time.perf_counter()
    solver.setup(n, lo, hi, slab.row_ptr, slab.col, slab.val)
    setup_s = time.perf_counter() - t_set
    X0 = ei.cfg5_start_block_torch(n, t, "cuda")[lo:hi].contiguous()
    W = torch.empty_like(X0)
    nblocks = 20 * s_
    stream = torch.cuda.Stream()
    eks.eks_set_stream(solver.ctx, stream.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        eks.eks_basis_sweep(solver.ctx, t, nblocks, X0, W)
    torch.cuda.synchronize()
    barrier()
    # ---------------- timed region: K steps, CUDA events on the sweep's stream (inputs ≫ L2)
    clocks = ClockSampler(local)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    reps = []
    barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        evs[k][0].record(stream)
        reps.append(eks.eks_basis_sweep(solver.ctx, t, nblocks, X0, W))
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = 20 * args.steps / (ms * 1e-3)  # every rank builds its slab of the same 20 outer iterations
    launches = sum(r["gpu_launches"] for r in reps)
    # ---------------- per-kernel-class device time: one more sweep, CUDA events around every launch
    prof_rep = eks.eks_basis_sweep(solver.ctx, t, nblocks, X0, W, profile=True)
    agg = eks.eks_get_profile(solver.ctx)
    peaks = load_peaks()
    classes = [c for c in agg["ms"] if c != "comm" and agg["ms"][c] > 0]
    dom = max(classes, key=lambda c: agg["ms"][c])
    roofline = roofline_of(agg, dom, peaks)
    spmm_roof = roofline_of(agg, "spmm", peaks)
    for rf in (roofline, spmm_roof):
        attach_traffic(rf, f"ncu_traffic_cfg5_t{t}_r02.json")
    share = {c: agg["ms"][c] / max(1e-9, sum(agg["ms"].values())) for c in agg["ms"]}
    per_class = {c: roofline_of(agg, c, peaks) for c in classes}
    model_bytes = reps[0]["model_bytes"]

    # ---------------- e2e: the public C ABI with HOST buffers (pinned): eks_setup_csr of the host CSR
    # slab + eks_basis_sweep(host X0 → host W_last) per step, wall clock (max over ranks)
    e2e = None
    if not args.no_e2e:
        del W
        torch.cuda.empty_cache()

        def pinned(a):
            tt = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
            tt.numpy()[...] = a
            return tt
        hrp, hcol, hval = pinned(slab.row_ptr), pinned(slab.col), pinned(slab.val)
        hX0 = X0.cpu().pin_memory()
        hW = torch.empty_like(hX0).pin_memory()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            solver.setup(n, lo, hi, hrp.numpy(), hcol.numpy(), hval.numpy())
            eks.eks_set_stream(solver.ctx, stream.cuda_stream)
            eks.eks_basis_sweep(solver.ctx, t, nblocks, hX0.numpy(), hW.numpy())
        torch.cuda.synchronize()
        barrier()
        wall = time.perf_counter() - t0
        wt = torch.tensor([wall], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        wall = float(wt.item())
        h2d = hrp.numel() * 8 + hcol.numel() * 4 + hval.numel() * 8 + hX0.numel() * 8
        e2e = {"value": 20 * args.steps / wall, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(hW.numel() * 8),
               "note": "eks_setup_csr(pinned host CSR slab) + eks_basis_sweep(pinned host X0 -> pinned host W_last) "
                       "per step through the C ABI, wall clock; host-side setup (validation, stencil plan) included",
               "setup_s_first": setup_s}
        del hrp, hcol, hval, hX0, hW
    del X0
    torch.cuda.empty_cache()

    # ---------------- SpMM-block kernel at t = 8/16/32 on this operator (rank 0, N = 1)
    sblock = None
    if rank == 0 and world == 1 and not args.no_spmm_block:
        sblock = spmm_block(eks, torch, peaks["hbm_gbs"], solver=solver, A=A)
    solver.close()
    del A, slab

    # ---------------- CPU oracle baseline (rank 0, N = 1; bounded, scaled sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, dt, ns = cfg5_oracle_sample(t, s_, N, args.cpu_planes)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"oracle basis sweep (definition mode, 1 thread pinned to 1 of {os.cpu_count()} cores) of "
                         f"the first 2 outer iterations (2 x s={s_} blocks, t={t}) on the first {args.cpu_planes} "
                         f"z-planes of the {N}^3 grid (n={ns}), {dt:.1f} s, scaled by n_full/n_sample = {n / ns:.0f} "
                         f"to outer it/s at full size"}

    # ---------------- extra workloads (rank 0, N = 1): the cfg2 solve (BASELINE configs[1])
    extras = {}
    if rank == 0 and world == 1:
        for w in [x for x in args.extra.split(",") if x]:
            extras[w] = solve_summary(eks, torch, w, args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg5_config(N, n, t, s_, world),
            "roofline": roofline, "spmm_roofline": spmm_roof, "spmm_block": sblock,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "sweep": {"model_bytes_per_step": model_bytes * world,
                      "achieved_model_gbs": model_bytes * world / (ms * 1e-3 / args.steps) / 1e9,
                      "frac_of_hbm": model_bytes / (ms * 1e-3 / args.steps) / 1e9 / peaks["hbm_gbs"],
                      "breakdown": reps[0]["breakdown_block"]},
            "time_share": share, "per_class": per_class, "extras": extras,
            "host": {"operator_gen_s": gen_s, "setup_csr_s": setup_s},
        }
        print(json.dumps(line), flush=True)


def slab_nnz(n, N):
    return n + 6 * N * N * (N - 1)


def solve_summary(eks, torch, name, args, steps=3, warmup=2):
    """A full eks_solve of another BASELINE config (device inputs, graphs on for SRE-CG): outer it/s,
    outer iterations, convergence — reported beside the headline, not part of it.  cfg4 (a 30 s
    solve): one timed solve after a 3-iteration warm-up that allocates the workspace."""
    p = workload(name)
    S = eks.Solver(p.A)
    stream = torch.cuda.Stream()
    eks.eks_set_stream(S.ctx, stream.cuda_stream)
    b = torch.from_numpy(p.b).cuda()
    x = torch.zeros_like(b)
    long_solve = name in ("cfg3", "cfg4")
    if long_solve:
        steps, warmup = 1, 1
    for _ in range(warmup):
        x.zero_()
        eks.eks_solve_ex(S.ctx, p.method, p.s, p.t, p.tol, b, x, use_graph=True, max_outer=4 if long_solve else 0,
                         raise_on=(5, 6, 1, 2, 3))
    torch.cuda.synchronize()
    tot_ms, tot_it, last = 0.0, 0, None
    for _ in range(steps):
        x.zero_()
        a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        st, last = eks.eks_solve_ex(S.ctx, p.method, p.s, p.t, p.tol, b, x, use_graph=True)
        bb.record(stream)
        torch.cuda.synchronize()
        tot_ms += a.elapsed_time(bb)
        tot_it += last["outer_iters"]
    S.close()
    return {"workload": f"{p.name}: {p.note}; s-step {p.method}, s={p.s}, t={p.t}, tol={p.tol:g}",
            "outer_it_per_s": tot_it / (tot_ms * 1e-3), "outer_iters": last["outer_iters"],
            "converged": last["converged"], "true_relres": last["true_relres"], "status": int(st),
            "ms_per_solve": tot_ms / steps, "steps": steps, "warmup": warmup}


def load_peaks():
    peaks = {"hbm_gbs": 6558.7, "source": "fallback"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        peaks.update(hbm_gbs=d.get("hbm_gbs", peaks["hbm_gbs"]), source="MEASURED_PEAKS.json (measured copy)")
    f = os.path.join(ROOT, "profiles", "fp64_peaks_r01.json")
    peaks["dfma_tflops"] = 34.217  # measured, profiles/fp64_peaks_r01.json (tools/fp64_peaks.cu)
    peaks["dmma_tflops"] = 37.089
    if os.path.exists(f):
        for line in open(f):
            try:
                d = json.loads(line)
            except ValueError:
                continue
            for k in ("dfma_tflops", "dmma_tflops"):
                if k in d:
                    peaks[k] = d[k]
    return peaks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- reference arm (CPU oracle)
def oracle_sample(p, iters: int):
    """Time the oracle (as it stands) on the first `iters` outer iterations of the workload."""
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    if p.method.startswith("ca-"):
        r = oracle.solve_ca(p.A, p.b, p.method[3:], arnoldi=p.arnoldi, s=p.s, t=p.t, tol=0.0, kmax=iters + 1)
    else:
        L = oracle.ic0(p.A, p.precond, kind=getattr(p, "precond_kind", "ic0"))[1] if getattr(p, "precond", 0) else None
        r = oracle.solve(p.A, p.b, p.method, p.s, p.t, 0.0, kmax=iters + 1, ortho=getattr(p, "ortho", "acholqr"),
                         restructured=getattr(p, "restructured", False), L=L)
    dt = time.perf_counter() - t0
    return r["outer_iters"], dt


def problem_of(args):
    """The workload, with --method/--s/--arnoldi overrides (CA variants: §8(f) item 1)."""
    p = workload(args.workload)
    if args.method:
        p = dataclasses.replace(p, method=args.method)
    if args.s:
        p = dataclasses.replace(p, s=args.s)
    p.arnoldi = args.arnoldi if p.method.startswith("ca-") else 0
    p.ortho = args.ortho
    p.restructured = args.restructured
    p.precond = args.precond
    p.precond_kind = args.precond_kind
    return p


def cfg5_config(N, n, t, s_, world):
    return {"workload": f"cfg5 (BASELINE configs[4]): 3D 7-point Laplacian {N}^3 (n={n}, nnz={slab_nnz(n, N)}), "
                        f"basis-generation sweep only (reading R27): 20 outer iterations x s={s_} blocks, "
                        f"t={t}, window 2t, seeded unit-norm U[-1,1) start block",
            "n": n, "t": t, "s": s_, "outer_iters_per_step": 20,
            "parallelism": f"row-slabs x{world} (t/N domains per GPU)",
            "l2": "inputs > L2: every block is 8*n*t = %.2f GB, L2 = 126 MB; not flushed" % (8 * n * t / 1e9)}


def run_reference_cfg5(args):
    """Reference arm for the cfg5 headline: the oracle as it stands (one thread), each step one
    bounded sample (one outer iteration on the first --cpu-planes z-planes), scaled to full n."""
    N, t, s_ = args.cfg5_n, args.t or 16, args.s or 4
    for _ in range(args.warmup):  # warm-up: a one-iteration sample (the oracle has no state to warm)
        cfg5_oracle_sample(t, s_, N, args.cpu_planes, iters=1)
    tot_dt, ns = 0.0, 0
    for _ in range(args.steps):
        _, dt, ns = cfg5_oracle_sample(t, s_, N, args.cpu_planes)
        tot_dt += dt
    n = N ** 3
    value = 2 * args.steps / (tot_dt * n / ns)  # outer it/s at full size
    sample = (f"oracle basis sweep (definition mode, 1 thread pinned to 1 of {os.cpu_count()} cores) of the first 2 "
              f"outer iterations (2 x s={s_} blocks, t={t}) per step on the first {args.cpu_planes} z-planes of the "
              f"{N}^3 grid (n={ns}), scaled by n_full/n_sample = {n / ns:.0f}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_dt * (n / ns) / args.steps / 2 * 20,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg5_config(N, n, t, s_, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.workload == "cfg5":
        return run_reference_cfg5(args)
    p = problem_of(args)
    per_step = args.ref_iters
    for _ in range(args.warmup):
        oracle_sample(p, per_step)
    total_it, total_t = 0, 0.0
    for _ in range(args.steps):
        k, dt = oracle_sample(p, per_step)
        total_it += k
        total_t += dt
    value = total_it / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args, p, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"first {per_step} outer iteration(s) of {p.name} {p.method} per step "
                                   f"(definition mode, single thread, {os.cpu_count()} host cores present)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_of(args, p, N):
    kind = f"CA (Alg {p.arnoldi})" if p.method.startswith("ca-") else \
        ("restructured" if getattr(p, "restructured", False) else "s-step")
    if getattr(p, "ortho", "acholqr") != "acholqr":
        kind += f" + {p.ortho}"
    if getattr(p, "precond", 0):
        kind = f"split-preconditioned (block-Jacobi {p.precond_kind}, {p.precond} domains) " + kind
    return {"workload": f"{p.name}: {p.note}; {kind} {p.method}, s={p.s}, t={p.t}, tol={p.tol:g}",
            "n": p.A.n, "nnz": p.A.nnz, "method": p.method, "s": p.s, "t": p.t, "tol": p.tol,
            "parallelism": f"row-slabs x{N} (t/N domains per GPU)",
            "cuda_graphs": ("off" if getattr(args, "no_graph", False) or getattr(args, "impl", "eks") == "reference"
                            else "steady s-step SRE-CG outer iterations replayed as CUDA graphs (one rank)"),
            "l2": "flushed: 256 MiB buffer written between timed steps (outside the step events)"}


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="eks", choices=["eks", "reference"])
    ap.add_argument("--workload", default="cfg5", help="cfg5 (headline, BASELINE configs[4]) | cfg2 | cfg3 | cfg4 | ...")
    ap.add_argument("--ref-iters", type=int, default=1, help="oracle outer iterations per reference step")
    ap.add_argument("--cpu-iters", type=int, default=2, help="oracle outer iterations for cpu_baseline")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--max-outer", type=int, default=0, help="cap outer iterations per solve (profiling only)")
    ap.add_argument("--no-spmm-block", action="store_true", help="skip the large-operator SpMM-block measurement")
    ap.add_argument("--t", type=int, default=0, help="cfg5: block width t")
    ap.add_argument("--s", type=int, default=0, help="blocks per outer iteration s (cfg5, or override)")
    ap.add_argument("--method", default="", help="override the workload's method (e.g. ca-sre-cg)")
    ap.add_argument("--arnoldi", type=int, default=7, help="CA variants: Alg 5 or Alg 7")
    ap.add_argument("--ortho", default="acholqr", choices=["acholqr", "pre-cholqr"])
    ap.add_argument("--restructured", action="store_true", help="restructured Alg 2 / Alg 1 (SRE-CG / SRE-CG2)")
    ap.add_argument("--no-graph", action="store_true",
                    help="disable the CUDA-graph replay of steady s-step SRE-CG outer iterations (use_graph)")
    ap.add_argument("--precond", type=int, default=0,
                    help="split-preconditioned Alg 8-10 with block Jacobi of this many domains (64 in the paper)")
    ap.add_argument("--precond-kind", default="ic0", choices=["ic0", "chol"], help="IC(0) (Table 5) or Cholesky (Table 6)")
    ap.add_argument("--cfg5-n", type=int, default=384, help="cfg5 grid size (384 = BASELINE configs[4])")
    ap.add_argument("--cpu-planes", type=int, default=2, help="cfg5 cpu_baseline: z-planes of the oracle sample")
    ap.add_argument("--extra", default="cfg2,cfg4",
                    help="cfg5: comma-separated solve workloads reported beside the headline")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1804_10629_b200 as eks

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.workload == "cfg5":
        run_cfg5(args, eks, torch, dist, world, rank, local)
        if world > 1:
            dist.destroy_process_group()
        return

    p = problem_of(args)
    n, t = p.A.n, p.t
    if t % world:
        raise SystemExit("t must be divisible by the number of GPUs")
    lo = (rank * (t // world)) * n // t
    hi = ((rank + 1) * (t // world)) * n // t
    slab = p.A.rows(lo, hi)

    uid = None
    if world > 1:
        obj = [eks.eks_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    solver = eks.Solver(None, rank=rank, nranks=world, device=local, nccl_id=uid)
    solver.setup(n, lo, hi, slab.row_ptr, slab.col, slab.val)
    if p.precond:
        solver.setup_precond(p.precond, kind=p.precond_kind)
    stream = torch.cuda.Stream()
    eks.eks_set_stream(solver.ctx, stream.cuda_stream)

    b = torch.from_numpy(np.ascontiguousarray(p.b[lo:hi])).cuda()
    x = torch.zeros_like(b)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()

    def step(profile=False):
        with torch.cuda.stream(stream):
            x.zero_()
        st, rep = eks.eks_solve_ex(solver.ctx, p.method, p.s, p.t, p.tol, b, x, profile=profile,
                                   max_outer=args.max_outer, arnoldi=p.arnoldi, ortho=p.ortho,
                                   restructured=p.restructured, precond=bool(p.precond), use_graph=not args.no_graph)
        if st not in ((0, 8) if args.max_outer else (0,)):
            raise SystemExit(f"solve failed: {eks.STATUS.get(st)} {eks.eks_error_string(solver.ctx)}")
        return rep

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()

    # ---------------- timed region: K steps, CUDA events on the solve stream, L2 flushed between steps
    clocks = ClockSampler(local)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    reps = []
    barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        evs[k][0].record(stream)
        reps.append(step())
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = sum(a.elapsed_time(bb) for a, bb in evs)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    outer = sum(r["outer_iters"] for r in reps)
    value = outer / (ms * 1e-3)
    launches = sum(r["gpu_launches"] for r in reps)

    # ---------------- per-kernel-class device time (same K steps, events per launch on the solve stream)
    prof_reps, prof_ms = [], 0.0
    agg = None
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        prof_reps.append(step(profile=True))
        pr = eks.eks_get_profile(solver.ctx)
        if agg is None:
            agg = pr
        else:
            for key in ("ms", "launches", "bytes", "flops"):
                for c in agg[key]:
                    agg[key][c] += pr[key][c]
    torch.cuda.synchronize()
    peaks = load_peaks()
    classes = [c for c in agg["ms"] if c not in ("comm",)]
    dom = max(classes, key=lambda c: agg["ms"][c])

    def roof(c):
        if agg["ms"][c] <= 0:
            return None
        gbs = agg["bytes"][c] / (agg["ms"][c] * 1e-3) / 1e9
        tfl = agg["flops"][c] / (agg["ms"][c] * 1e-3) / 1e12
        intensity = agg["flops"][c] / max(agg["bytes"][c], 1.0)
        ridge = peaks["dfma_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
        if intensity > ridge:
            return {"kernel": c, "bound": "alu", "achieved": tfl, "peak": peaks["dfma_tflops"], "unit": "TFLOP/s",
                    "frac": tfl / peaks["dfma_tflops"], "traffic": None,
                    "peak_source": "measured DFMA (profiles/fp64_peaks_r01.json)",
                    "launches": agg["launches"][c], "avg_launch_us": 1e3 * agg["ms"][c] / max(1, agg["launches"][c])}
        return {"kernel": c, "bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": gbs / peaks["hbm_gbs"], "traffic": None, "peak_source": peaks["source"],
                "frac_of_8TBs": gbs / 8000.0, "launches": agg["launches"][c],
                "avg_launch_us": 1e3 * agg["ms"][c] / max(1, agg["launches"][c]),
                "bytes_per_launch": agg["bytes"][c] / max(1, agg["launches"][c])}

    roofline = roof(dom)
    spmm_roof = roof("spmm")
    # DRAM traffic per launch of the same kernel from the committed ncu --set full capture
    tf = os.path.join(ROOT, "profiles", "ncu_traffic_r01.json")
    if os.path.exists(tf) and args.workload == "cfg2":
        tr = json.load(open(tf)).get("classes", {})
        for rf in (roofline, spmm_roof):
            if rf is not None and tr.get(rf["kernel"]):
                rf["traffic"] = tr[rf["kernel"]]
                rf["traffic_source"] = "profiles/ncu_traffic_r01.json (ncu dram__bytes_read+write per launch)"
    share = {c: agg["ms"][c] / max(1e-9, sum(agg["ms"].values())) for c in agg["ms"]}

    # ---------------- e2e: C-ABI with pinned HOST buffers, setup + solve per step, wall clock
    e2e = None
    if not args.no_e2e:
        def pinned(a):
            tt = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            return tt.numpy()
        hrp, hcol, hval = pinned(slab.row_ptr), pinned(slab.col), pinned(slab.val)
        hb = pinned(p.b[lo:hi])
        hx = pinned(np.zeros(hi - lo))
        e2e_solver = eks.Solver(None, rank=rank, nranks=world, device=local, nccl_id=uid) if False else solver
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        e_outer = 0
        for k in range(args.steps):
            e2e_solver.setup(n, lo, hi, hrp, hcol, hval)
            if p.precond:
                e2e_solver.setup_precond(p.precond, kind=p.precond_kind)
            hx[:] = 0.0
            st, rep = eks.eks_solve_ex(e2e_solver.ctx, p.method, p.s, p.t, p.tol, hb, hx, arnoldi=p.arnoldi,
                                       ortho=p.ortho, restructured=p.restructured, precond=bool(p.precond),
                                       use_graph=not args.no_graph)
            e_outer += rep["outer_iters"]
        torch.cuda.synchronize()
        barrier()
        wall = time.perf_counter() - t0
        wt = torch.tensor([wall], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        wall = float(wt.item())
        h2d = hrp.nbytes + hcol.nbytes + hval.nbytes + hb.nbytes + hx.nbytes
        e2e = {"value": e_outer / wall, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(hx.nbytes),
               "note": "eks_setup_csr(host CSR) + eks_solve(host b, host x) per step, pinned host memory, wall clock"}

    # ---------------- CPU oracle baseline (rank 0, N=1 only; bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        k, dt = oracle_sample(p, args.cpu_iters)
        cpu = {"value": k / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"first {k} outer iterations of {p.name} {p.method} (definition mode, single thread, "
                         f"{os.cpu_count()} host cores present), {dt:.1f} s"}

    sblock = None
    if rank == 0 and world == 1 and not args.no_spmm_block:
        sblock = spmm_block(eks, torch, load_peaks()["hbm_gbs"])

    if rank == 0:
        r0 = reps[0]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(args, p, world),
            "roofline": roofline, "spmm_roofline": spmm_roof, "spmm_block": sblock,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "solve": {"outer_iters": r0["outer_iters"], "converged": r0["converged"],
                      "true_relres": r0["true_relres"], "rho_ratio": r0["rho"] / r0["rho0"],
                      "model_bytes_per_outer": r0["model_bytes"] / max(1, r0["outer_iters"]),
                      "achieved_model_gbs": r0["model_bytes"] / (ms * 1e-3 / args.steps) / 1e9},
            "time_share": share,
        }
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
