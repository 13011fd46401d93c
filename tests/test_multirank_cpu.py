"""N > 1 host logic on CPU with the gloo backend (world_size 2): view sharding of
each subset, the sum of partial back-projections (the NCCL all-reduce's job on
the GPU path), NCCL-id broadcast and max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth.configs import shard_views, subset_views


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import projector as P
        from tests.geoms import tiny
        from tests.problems import synthetic_problem
        pb = synthetic_problem(tiny("helical_arc", na=43), M=4)
        g, M = pb["geom"], 4
        out = {}
        for m in range(M):
            st, sd, cnt = shard_views(g["na"], M, m, rank, world)
            x = pb["x0"]
            part = np.zeros(P.vol_shape(g))
            if cnt > 0:
                r = pb["w"][st::sd][:cnt] * (P.forward(g, x, (st, sd, cnt)) - pb["y"][st::sd][:cnt])
                part = M * P.back(g, r, (st, sd, cnt))
            t = torch.from_numpy(part)
            dist.all_reduce(t)                      # the zeta all-reduce of the sharded path
            out[m] = t.numpy()
        # NCCL unique id broadcast as done in bench.py
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        # max-over-ranks of a per-rank time
        tm = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        if rank == 0:
            q.put((out, obj[0], float(tm.item())))
    finally:
        dist.destroy_process_group()


def test_sharding_partitions_every_subset():
    for na, M in [(2952, 24), (43, 4), (984, 41), (7, 7)]:
        for world in (1, 2, 3, 8):
            for m in range(M):
                views = []
                for rank in range(world):
                    st, sd, cnt = shard_views(na, M, m, rank, world)
                    views += list(range(st, st + sd * cnt, sd)) if cnt else []
                s0, s1, c = subset_views(na, M, m)
                assert sorted(views) == list(range(s0, s0 + s1 * c, s1))
                assert all(v < na for v in views)


@pytest.mark.timeout(300)
def test_two_rank_gloo_sum_of_partial_backprojections_equals_full_subset():
    from oracle import projector as P
    from tests.geoms import tiny
    from tests.problems import synthetic_problem
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, uid, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pb = synthetic_problem(tiny("helical_arc", na=43), M=4)
    g, M = pb["geom"], 4
    for m in range(M):
        st, sd, cnt = subset_views(g["na"], M, m)
        r = pb["w"][st::sd][:cnt] * (P.forward(g, pb["x0"], (st, sd, cnt)) - pb["y"][st::sd][:cnt])
        full = M * P.back(g, r, (st, sd, cnt))
        assert np.allclose(out[m], full, rtol=1e-12, atol=1e-12 * np.abs(full).max())
    assert uid == bytes(range(128)) and tmax == 2.0


def _slab(g, nz, rank, world):
    """Planes [z0, z0 + n) of rank `rank` (the partition of ct_zslab_range) and their geometry."""
    z0 = rank * nz // world
    n = (rank + 1) * nz // world - z0
    gs = dict(g, nz=n, offset_z=g["offset_z"] + (z0 + (n - 1) / 2.0 - (nz - 1) / 2.0) * g["dz"])
    return z0, n, gs


def _zslab_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import projector as P
        from tests.geoms import tiny
        from tests.problems import synthetic_problem
        pb = synthetic_problem(tiny("helical_arc"), M=4)
        g = pb["geom"]
        nz = g["nz"]
        z0, n, gs = _slab(g, nz, rank, world)
        x = pb["x0"][z0:z0 + n]
        # partial projection of the slab, summed over the ranks (the NCCL all-reduce's job)
        part = torch.from_numpy(P.forward(gs, x, (0, 1, g["na"])))
        dist.all_reduce(part)
        # halo planes from the neighbours (ncclSend/Recv on the GPU path), then the stencil
        lo = torch.zeros(x.shape[1:], dtype=torch.float64)
        hi = torch.zeros(x.shape[1:], dtype=torch.float64)
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(x[0])), rank - 1))
            reqs.append(dist.irecv(lo, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(x[-1])), rank + 1))
            reqs.append(dist.irecv(hi, rank + 1))
        for r_ in reqs:
            r_.wait()
        planes = ([lo.numpy()] if rank > 0 else []) + list(x) + ([hi.numpy()] if rank + 1 < world else [])
        ext = np.stack(planes)
        a = 1 if rank > 0 else 0
        ge = dict(gs, nz=ext.shape[0], offset_z=gs["offset_z"] + ((1 if rank + 1 < world else 0) - a) * g["dz"] / 2.0)
        _, gr, cv = P.reg(ge, "hyperbola", 0.01, pb["reg"]["betas"], 13, ext)
        gr, cv = gr[a:a + n], cv[a:a + n]
        got = [None] * world
        dist.all_gather_object(got, (z0, gr, cv))
        if rank == 0:
            q.put((part.numpy(), got))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_zslab_gloo_partial_projections_and_halo_stencil(world):
    """z-slab decomposition host logic with gloo ranks: the slabs'
    partial projections sum to the full projection, and the stencil of a slab
    extended by the neighbours' halo planes equals the full volume's stencil."""
    from oracle import projector as P
    from tests.geoms import tiny
    from tests.problems import synthetic_problem
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_zslab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    proj, parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pb = synthetic_problem(tiny("helical_arc"), M=4)
    g = pb["geom"]
    full = P.forward(g, pb["x0"], (0, 1, g["na"]))
    assert np.allclose(proj, full, rtol=1e-12, atol=1e-12 * np.abs(full).max())
    _, gr, cv = P.reg(g, "hyperbola", 0.01, pb["reg"]["betas"], 13, pb["x0"])
    covered = 0
    for z0, gsl, csl in parts:
        n = gsl.shape[0]
        assert np.allclose(gsl, gr[z0:z0 + n], rtol=1e-12, atol=1e-15)
        assert np.allclose(csl, cv[z0:z0 + n], rtol=1e-12, atol=1e-15)
        covered += n
    assert covered == g["nz"]


def _owner_worker(rank, world, port, nsub, q):
    """Algorithm 1 (oracle arithmetic) with the GPU dist path's data flow: views of each subset
    sharded over the ranks, partial gradients reduced by z-slab to the slab owner (gloo reduce
    per slab = the grouped ncclReduce / ncclReduceScatter), the owner's lines 7-8 and 4-5 on its
    slab only, x+ re-assembled by a broadcast per owner (= ncclAllGather / grouped ncclBroadcast),
    g and h gathered at the end of the call."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import alg
        from oracle import projector as P
        from tests.geoms import tiny
        from tests.problems import oracle_problem, synthetic_problem
        M, alpha = 3, 1.999
        pb = synthetic_problem(tiny("helical_arc"), M=M)
        prob = oracle_problem(pb)
        g = pb["geom"]
        nz, na = g["nz"], g["na"]
        DL = pb["DL"]
        slabs = [_slab(g, nz, r_, world)[:2] for r_ in range(world)]
        z0, n = slabs[rank]
        sl = slice(z0, z0 + n)

        def partial_grad(x, m):
            st, sd, cnt = shard_views(na, M, m, rank, world)
            part = np.zeros(P.vol_shape(g))
            if cnt > 0:
                r = pb["w"][st::sd][:cnt] * (P.forward(g, x, (st, sd, cnt)) - pb["y"][st::sd][:cnt])
                part = M * P.back(g, r, (st, sd, cnt))
            return torch.from_numpy(part)

        def reduce_to_owners(t):
            for q_, (a, nn) in enumerate(slabs):
                piece = t[a:a + nn].contiguous()
                dist.reduce(piece, dst=q_)
                if q_ == rank:
                    t[a:a + nn] = piece
            return t.numpy()

        def gather_slabs(arr):
            t = torch.from_numpy(np.ascontiguousarray(arr))
            for q_, (a, nn) in enumerate(slabs):
                piece = t[a:a + nn].contiguous()
                dist.broadcast(piece, src=q_)
                t[a:a + nn] = piece
            return t.numpy()

        x = pb["x0"].copy()
        zeta = reduce_to_owners(partial_grad(x, M - 1))      # line 1 (reading R1), owners' slabs exact
        zeta = gather_slabs(zeta)
        gg, h = zeta.copy(), DL * x - zeta
        k = 0
        for _ in range(nsub):
            m, rho = k % M, alg.rho_k(k, alpha)
            gradR, DR = prob.reg(x)                            # x replicated: halos available
            s = rho * (DL[sl] * x[sl] - h[sl]) + (1 - rho) * gg[sl]
            xn = x.copy()
            xn[sl] = alg._x_update(x[sl], s, gradR[sl], rho * DL[sl] + DR[sl])   # owner slab, lines 4-5
            xn = gather_slabs(xn)
            zeta = reduce_to_owners(partial_grad(xn, m))        # line 6, reduce-scatter
            gg[sl] = rho / (rho + 1) * (alpha * zeta[sl] + (1 - alpha) * gg[sl]) + gg[sl] / (rho + 1)
            h[sl] = alpha * (DL[sl] * xn[sl] - zeta[sl]) + (1 - alpha) * h[sl]
            x = xn
            k += 1
        gg, h = gather_slabs(gg), gather_slabs(h)
        if rank == 0:
            q.put((x, gg, h))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_owner_slab_data_flow_gloo_equals_algorithm1(world):
    """The view-sharded path's data flow on `world` gloo ranks reproduces the
    single-process Algorithm 1 iterates (equal slabs at world 2, nz = 10; unequal at world 3)."""
    from oracle import alg
    from tests.geoms import tiny
    from tests.problems import oracle_problem, synthetic_problem
    nsub = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_owner_worker, args=(r, world, port, nsub, q)) for r in range(world)]
    for p in procs:
        p.start()
    x, gg, h = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pb = synthetic_problem(tiny("helical_arc"), M=3)
    prob = oracle_problem(pb)
    trace = {}
    alg.alg1(prob, pb["x0"], 3, 1.999, 2, DL=pb["DL"], trace=trace)
    xo, go, ho = trace[nsub]
    for a, b in ((x, xo), (gg, go), (h, ho)):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
