"""Multi-rank logic on CPUs (gloo, world_size 2 and 4): the row-slab partition of
§8(e), the halo plan that libeks.so builds on every rank (eks_plan_halo, the
same host code eks_setup_csr runs before its NCCL exchanges), the halo exchange
protocol (rank q sends rows need_p[q] to rank p), and the allreduce of per-rank
partial sums.  The distributed SpMM assembled from the plan must be BITWISE the
global SpMM (same fma order, reading R20); the distributed Gram must equal the
global one to rounding.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import eks_inputs as ei


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def slab(rank, world, n, t):
    """Rows of rank `rank`: the union of its t/world domains D_d = [⌊d n/t⌋, ⌊(d+1) n/t⌋) (reading R1)."""
    per = t // world
    return (rank * per) * n // t, ((rank + 1) * per) * n // t


def _matrix(kind):
    if kind == "bands2d":
        return ei.stencil_csr(24, 24, ndim=2, kappa=ei.bands_kappa(24, band=3))
    if kind == "aniso3d":
        return ei.stencil_csr(8, 8, 8, ndim=3, scale=(1.0, 1.0, 1e-2))
    # general sparse SPD: random symmetric pattern + dominant diagonal (non-banded ghost sets)
    n = 300
    rng = np.random.default_rng(7)
    D = np.zeros((n, n))
    for _ in range(900):
        i, j = rng.integers(0, n, 2)
        if i != j:
            D[i, j] = D[j, i] = -rng.random()
    D[np.arange(n), np.arange(n)] = np.abs(D).sum(1) + 1.0
    return ei.csr_from_dense(D)


def _worker(rank, world, port, kind, t, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1804_10629_b200 as eks
        A = _matrix(kind)
        n = A.n
        ranges = np.array([v for r in range(world) for v in slab(r, world, n, t)], np.int64)
        lo, hi = ranges[2 * rank], ranges[2 * rank + 1]
        S = A.rows(lo, hi)
        ext_col, need, geom = eks.eks_plan_halo(rank, world, ranges, S.row_ptr, S.col)
        # every rank learns every rank's needs (eks_setup_csr: ncclAllGather)
        need_t = torch.from_numpy(need.copy())
        all_need = [torch.zeros_like(need_t) for _ in range(world)]
        dist.all_gather(all_need, need_t)
        X = ei.uniform_pm1(11, n * t).reshape(n, t)  # same global block on every rank
        Xloc = X[lo:hi].copy()
        nloc = hi - lo
        next_ = geom["halo_before"] + nloc + geom["halo_after"]
        Xext = np.full((next_, t), np.nan)
        Xext[geom["halo_before"]:geom["halo_before"] + nloc] = Xloc
        # halo exchange: rank p sends to q the rows q asked from p; receives its own ghost ranges
        reqs = []
        for peer in range(world):
            if peer == rank:
                continue
            a, b = all_need[peer][rank].tolist()
            if b > a:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(Xloc[a - lo:b - lo])), dst=peer))
        off = 0
        recv_bufs = []
        for peer in range(world):
            if peer == rank:
                off += nloc
                continue
            a, b = need[peer].tolist()
            if b > a:
                buf = torch.empty((b - a, t), dtype=torch.float64)
                reqs.append(dist.irecv(buf, src=peer))
                recv_bufs.append((off, buf))
                off += b - a
        for r_ in reqs:
            r_.wait()
        for o, buf in recv_bufs:
            Xext[o:o + buf.shape[0]] = buf.numpy()
        assert off == next_
        # local SpMM on the extended layout vs the global SpMM: bitwise
        Aloc = ei.Csr(nloc, S.row_ptr, ext_col, S.val)
        Yloc = oracle.spmm(Aloc, Xext)[:nloc]  # the wrapper sizes Y like X; rows past nloc are unused
        Yglob = oracle.spmm(A, X)[lo:hi]
        bitwise = bool(np.array_equal(Yloc, Yglob))
        # interior rows only touch local columns
        ilo, ihi = geom["interior_lo"], geom["interior_hi"]
        interior_ok = True
        for i in range(ilo, ihi):
            cols = ext_col[S.row_ptr[i]:S.row_ptr[i + 1]]
            interior_ok &= bool(np.all((cols >= geom["halo_before"]) & (cols < geom["halo_before"] + nloc)))
        # Gram: per-rank partial XᵀY, allreduced (the stacked ncclAllReduce of §8(e))
        G = torch.from_numpy(Xloc.T @ Yloc)
        dist.all_reduce(G)
        Gref = X.T @ oracle.spmm(A, X)
        gram_err = float(np.abs(G.numpy() - Gref).max() / np.abs(Gref).max())
        # ghost-plane plan of the plane-marching SpMM (eks_plan_grid, what eks_setup_csr builds on every
        # rank): stencil operators with whole-plane slabs get one ghost plane per neighbour rank; the
        # SpMM from the slot values over [ghost plane | local planes | ghost plane] (absent neighbours:
        # value 0 on the row's own column, fma(0, x, y) = y) is bitwise the global one
        grid_ok = None
        if kind != "general":
            g, sv = eks.eks_plan_grid(lo, hi, S.row_ptr, S.col, S.val, geom["halo_before"], geom["halo_after"])
            plane = g["nx"] * g["ny"]
            grid_ok = g["w"] == (7 if kind == "aniso3d" else 5) and g["nz"] * plane == nloc
            grid_ok &= g["gb"] == (1 if rank > 0 else 0) and g["ga"] == (1 if rank < world - 1 else 0)
            grid_ok &= geom["halo_before"] == g["gb"] * plane and geom["halo_after"] == g["ga"] * plane
            offs = [-plane, -g["nx"], -1, 0, 1, g["nx"], plane] if g["w"] == 7 else [-g["nx"], -1, 0, 1, g["nx"]]
            rows = np.arange(nloc)
            cols = np.empty((nloc, g["w"]), np.int64)
            for k, o in enumerate(offs):
                c = geom["halo_before"] + rows + o
                inside = (c >= 0) & (c < next_) & (sv[:, k] != 0.0)
                cols[:, k] = np.where(inside, c, geom["halo_before"] + rows)
            Ag = ei.Csr(nloc, np.arange(0, nloc * g["w"] + 1, g["w"], dtype=np.int64),
                        cols.reshape(-1).astype(np.int32), np.ascontiguousarray(sv[:, :g["w"]]).reshape(-1))
            grid_ok &= bool(np.array_equal(oracle.spmm(Ag, Xext)[:nloc], Yglob))
        # max-over-ranks timing aggregation used by bench.py
        tt = torch.tensor([float(rank + 1)])
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        q.put((rank, bitwise, interior_ok, gram_err, float(tt.item()), int(nloc), geom, grid_ok))
    except Exception as e:  # report instead of leaving the parent waiting
        q.put((rank, f"error: {e!r}"))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,t", [(2, "bands2d", 4), (2, "aniso3d", 8), (4, "bands2d", 8),
                                          (4, "aniso3d", 4), (2, "general", 4), (4, "general", 8)])
def test_distributed_spmm_gram_protocol(world, kind, t):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, t, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    errors = [r for r in res if len(r) == 2]
    for p in procs:
        p.join(timeout=60)
        if errors and p.is_alive():
            p.kill()
    assert not errors, errors
    for p in procs:
        assert p.exitcode == 0
    res.sort()
    n = _matrix(kind).n
    assert sum(r[5] for r in res) == n
    for rank, bitwise, interior_ok, gram_err, tmax, nloc, geom, grid_ok in res:
        assert bitwise, (rank, kind)
        assert grid_ok is None if kind == "general" else grid_ok, (rank, kind)
        assert interior_ok
        assert gram_err <= 1e-13
        assert tmax == float(world)
        if kind == "bands2d":  # 24-wide grid, ≥ 6 grid rows per slab: the middle rows are interior
            assert geom["interior_hi"] - geom["interior_lo"] >= nloc - 2 * 24
    if kind == "bands2d":
        # first rank has no lower ghosts, last rank no upper ghosts
        assert res[0][6]["halo_before"] == 0 and res[-1][6]["halo_after"] == 0


def test_slabs_are_unions_of_domains():
    for n, t, world in [(262144, 16, 4), (16777216, 64, 8), (2097152, 32, 2), (4099, 8, 4)]:
        prev = 0
        for r in range(world):
            lo, hi = slab(r, world, n, t)
            assert lo == prev
            prev = hi
            for d in range(r * (t // world), (r + 1) * (t // world)):
                assert lo <= d * n // t and (d + 1) * n // t <= hi
        assert prev == n


def test_plan_halo_single_rank_is_identity():
    import paper_1804_10629_b200 as eks
    A = ei.poisson2d(10)
    ext, need, geom = eks.eks_plan_halo(0, 1, np.array([0, A.n]), A.row_ptr, A.col)
    assert np.array_equal(ext, A.col) and not need.any()
    assert geom == dict(halo_before=0, halo_after=0, interior_lo=0, interior_hi=A.n)


def _onesynch_worker(rank, world, port, t, q):
    """One block of one-synch CGS2 (DESIGN reading R36) on row slabs: rank-local partials, exactly two
    allreduces (C1, then the stacked [C2 | B1 | g1]), the local B/g correction — compared with the
    two-pass CGS2 + A-CholQR Gram of the whole block (R3/R4) computed on one process."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        A = ei.stencil_csr(20, 20, ndim=2, kappa=ei.bands_kappa(20, band=4, hi=1e2))
        n = A.n
        lo, hi = slab(rank, world, n, t)
        # a window Q of two A-orthonormal blocks (A-CholQR of a random n×2t block), Z, r, α of block 1
        V = ei.uniform_pm1(21, n * 2 * t).reshape(n, 2 * t)
        L = np.linalg.cholesky(V.T @ oracle.spmm(A, V))
        Q = np.linalg.solve(L, V.T).T
        AQ = oracle.spmm(A, Q)
        Z = ei.uniform_pm1(22, n * t).reshape(n, t)
        r = ei.uniform_pm1(23, n)
        alpha1 = Q[:, t:].T @ r  # α̃ of the window block built in this outer iteration (the older one: 0)
        ncoll = 0

        def allreduce(a):
            nonlocal ncoll
            ncoll += 1
            tt = torch.from_numpy(np.ascontiguousarray(a))
            dist.all_reduce(tt)
            return tt.numpy()
        sl = slice(lo, hi)
        C1 = allreduce(AQ[sl].T @ Z[sl])                       # synch 1
        Z1 = Z - Q @ C1                                         # (every rank: its rows; all rows kept here
        AZ1 = oracle.spmm(A, Z1)                                #  only to form A·Z1 without a halo exchange)
        stacked = np.concatenate([(AQ[sl].T @ Z1[sl]).ravel(), (Z1[sl].T @ AZ1[sl]).ravel(), Z1[sl].T @ r[sl]])
        red = allreduce(stacked)                                # synch 2: [C2 | B1 | g1]
        C2 = red[:2 * t * t].reshape(2 * t, t)
        B1 = red[2 * t * t:3 * t * t].reshape(t, t)
        g1 = red[3 * t * t:]
        B = B1 - C2.T @ C2
        g = g1 - C2[t:].T @ alpha1
        Z2 = Z1[sl] - Q[sl] @ C2
        AZ2 = AZ1[sl] - AQ[sl] @ C2
        # reference: two explicit CGS passes Qᵀ(A·Z) on one process, then the Gram of Z2
        Zr = Z - Q @ (Q.T @ oracle.spmm(A, Z))
        Zr = Zr - Q @ (Q.T @ oracle.spmm(A, Zr))
        AZr = oracle.spmm(A, Zr)
        Bref, gref = Zr.T @ AZr, Zr.T @ r
        errs = (float(np.abs(B - Bref).max() / np.abs(Bref).max()), float(np.abs(g - gref).max() / np.abs(gref).max()),
                float(np.abs(Z2 - Zr[sl]).max() / np.abs(Zr).max()), float(np.abs(AZ2 - AZr[sl]).max() / np.abs(AZr).max()))
        q.put((rank, ncoll, errs))
    except Exception as e:
        q.put((rank, f"error: {e!r}"))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,t", [(2, 4), (4, 8)])
def test_onesynch_protocol_two_collectives(world, t):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_onesynch_worker, args=(r, world, port, t, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(not isinstance(r[1], str) for r in res), res
    for rank, ncoll, errs in res:
        assert ncoll == 2, (rank, ncoll)
        assert max(errs) <= 1e-10, (rank, errs)


def _mpk_worker(rank, world, port, kind, t, s, q):
    """Matrix-powers kernel of the CA variants on row slabs (DESIGN reading R37): ONE exchange
    of d = s − 1 boundary planes of V_0 (and, once per operator, of the stencil values of those planes),
    then power i = 1..d on the plane ranges of eks_plan_mpk — the slab plus (d − i) ghost planes, redundantly.
    The slab rows of every power must be BITWISE the global A^i·V_0 (same fma chain per row); rows a power
    may not read are NaN, so a plan that reads past its valid planes poisons the result."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1804_10629_b200 as eks
        A = _matrix(kind)
        n, d = A.n, s - 1
        lo, hi = slab(rank, world, n, t)
        ranges = np.array([v for r in range(world) for v in slab(r, world, n, t)], np.int64)
        S = A.rows(lo, hi)
        _, _, geom = eks.eks_plan_halo(rank, world, ranges, S.row_ptr, S.col)
        g, sv = eks.eks_plan_grid(lo, hi, S.row_ptr, S.col, S.val, geom["halo_before"], geom["halo_after"])
        plane, nz, w = g["nx"] * g["ny"], g["nz"], g["w"]
        db, da = (d if rank > 0 else 0), (d if rank < world - 1 else 0)
        steps = eks.eks_plan_mpk(nz, d, db, da)
        X = ei.uniform_pm1(31, n * t).reshape(n, t)
        nbuf = (db + nz + da) * plane
        nmsg = 0

        def exchange(loc):
            """rows [db·plane, db·plane + nloc) of `loc` are mine; d planes to / from each neighbour"""
            nonlocal nmsg
            reqs, bufs = [], []
            mine = loc[db * plane:(db + nz) * plane]
            if rank > 0:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(mine[:d * plane])), dst=rank - 1))
                b = torch.empty((d * plane, loc.shape[1]), dtype=torch.float64)
                reqs.append(dist.irecv(b, src=rank - 1))
                bufs.append((0, b))
            if rank < world - 1:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(mine[-d * plane:])), dst=rank + 1))
                b = torch.empty((d * plane, loc.shape[1]), dtype=torch.float64)
                reqs.append(dist.irecv(b, src=rank + 1))
                bufs.append(((db + nz) * plane, b))
            for r_ in reqs:
                r_.wait()
            for o, b in bufs:
                loc[o:o + b.shape[0]] = b.numpy()
            nmsg += 1
        svx = np.full((nbuf, sv.shape[1]), np.nan)
        svx[db * plane:(db + nz) * plane] = sv
        exchange(svx)  # once per operator
        nmsg = 0
        V = [np.full((nbuf, t), np.nan) for _ in range(d + 1)]
        V[0][db * plane:(db + nz) * plane] = X[lo:hi]
        exchange(V[0])  # the ONE exchange of the outer iteration
        offs = [-plane, -g["nx"], -1, 0, 1, g["nx"], plane] if w == 7 else [-g["nx"], -1, 0, 1, g["nx"]]
        plan_ok = True
        for i in range(1, d + 1):
            zlo, zhi, gb, ga = (int(v) for v in steps[i - 1])
            r0, r1 = (zlo + db) * plane, (zhi + db) * plane
            rows = np.arange(r0, r1)
            cols = np.empty((rows.size, w), np.int64)
            for k, o in enumerate(offs):
                c = rows + o
                used = svx[r0:r1, k] != 0.0
                # a used neighbour must lie in the planes this launch may read: [zlo − gb, zhi + ga)
                inside = (c >= r0 - gb * plane) & (c < r1 + ga * plane)
                plan_ok &= bool(np.all(inside[used]))
                cols[:, k] = np.where(used, c, rows)
            Ag = ei.Csr(rows.size, np.arange(0, rows.size * w + 1, w, dtype=np.int64),
                        cols.reshape(-1).astype(np.int32), np.ascontiguousarray(svx[r0:r1, :w]).reshape(-1))
            V[i][r0:r1] = oracle.spmm(Ag, V[i - 1])[:rows.size]
        P = X
        bitwise = True
        for i in range(1, d + 1):
            P = oracle.spmm(A, P)
            bitwise &= bool(np.array_equal(V[i][db * plane:(db + nz) * plane], P[lo:hi]))
        q.put((rank, bitwise, plan_ok, nmsg, steps.tolist()))
    except Exception as e:
        q.put((rank, f"error: {e!r}"))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,t,s", [(2, "aniso3d", 8, 3), (4, "aniso3d", 8, 3), (2, "aniso3d", 4, 4),
                                            (2, "bands2d", 8, 4), (4, "bands2d", 4, 6)])
def test_matrix_powers_ghost_zone_protocol(world, kind, t, s):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mpk_worker, args=(r, world, port, kind, t, s, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(not isinstance(r[1], str) for r in res), res
    for rank, bitwise, plan_ok, nmsg, steps in res:
        assert bitwise and plan_ok, (rank, steps)
        assert nmsg == 1  # one ghost-zone exchange per outer iteration instead of s − 1


def test_plan_mpk_ranges():
    """eks_plan_mpk: power i covers the slab plus min(ghost, d − i) planes per side, reads one further
    plane exactly when one exists, and the last power covers exactly the slab."""
    import paper_1804_10629_b200 as eks
    for nz, d, db, da in [(4, 1, 1, 1), (6, 3, 3, 0), (2, 2, 2, 2), (5, 4, 0, 4), (3, 3, 1, 2), (1, 2, 0, 0)]:
        st = eks.eks_plan_mpk(nz, d, db, da)
        prev_lo, prev_hi = -db, nz + da  # V_0 is valid on every plane of the buffer
        for i in range(1, d + 1):
            zlo, zhi, gb, ga = (int(v) for v in st[i - 1])
            assert zlo == -min(db, d - i) and zhi == nz + min(da, d - i)
            assert zlo - gb >= prev_lo and zhi + ga <= prev_hi  # reads only planes the previous power wrote
            assert gb == (1 if db > -zlo else 0) and ga == (1 if da > zhi - nz else 0)
            prev_lo, prev_hi = zlo, zhi
        assert (prev_lo, prev_hi) == (0, nz)
    with pytest.raises(Exception):
        eks.eks_plan_mpk(4, 2, 3, 0)
