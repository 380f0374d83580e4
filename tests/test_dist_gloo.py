"""World-size-2 CPU tests of the multi-rank host logic (gloo, -m "not gpu").

One process per rank, as on the GPU box.  Each rank takes the candidate shard
opmm_shard_range gives it (libopmm host helper), evaluates it with the CPU
oracle (standing in for the rank's GPU kernel, which the GPU tests cover),
exchanges its 16-byte (E, index) pair with the others -- the same one
all-gather libopmm issues through NCCL -- and merges with opmm_merge_argmin.
The merged result must equal the unsharded exhaustive argmin (P12).  The
population batch shards saccades instead and needs no collective.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_09884_b200 import opmm
        ctl = W.Control()
        rec = oracle.positions(W.truth_opc(), ctl) + W.noise(ctl.n_steps + 1)
        sp = W.paper_space()
        out = {}
        for N in (1, 5, 2000):
            b, e = opmm.opmm_shard_range(N, rank, world)
            r = oracle.fit(rec, ctl, sp, b, e) if e > b else {"best_err": float("inf"),
                                                               "best_index": -1, "n_finite": 0}
            mine = torch.tensor([r["best_err"], float(r["best_index"]), float(r["n_finite"])],
                                dtype=torch.float64)
            allp = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(allp, mine)
            errs = [float(t[0]) for t in allp]
            idxs = [int(t[1]) for t in allp]
            be, bi = opmm.opmm_merge_argmin(errs, idxs)
            out[N] = (be, bi, int(sum(float(t[2]) for t in allp)))
        # population: saccades sharded, no collective on the data path
        S = 5
        amp, pw, truths = W.population(S)
        sb, se = opmm.opmm_shard_range(S, rank, world)
        mine_pop = {}
        for s in range(sb, se):
            c = W.Control(n_steps=60, amplitude_deg=amp[s], pw_default_ms=pw[s])
            recs = oracle.positions(truths[s], c)
            r = oracle.fit(recs, c, sp, 0, 300, saccade=s)
            mine_pop[s] = (r["best_err"], r["best_index"])
        gathered = [None] * world
        dist.all_gather_object(gathered, mine_pop)   # test-side check only
        pop = {}
        for g in gathered:
            pop.update(g)
        q.put((rank, out, pop))
    finally:
        dist.destroy_process_group()


def test_world2_shard_merge_equals_unsharded():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(ctl.n_steps + 1)
    sp = W.paper_space()
    for rank, out, pop in results:
        for N, (be, bi, nf) in out.items():
            full = oracle.fit(rec, ctl, sp, 0, N)
            assert (be, bi) == (full["best_err"], full["best_index"]), (rank, N)
            assert nf == full["n_finite"]
        assert sorted(pop) == list(range(5))
    # every rank holds the same merged answer
    assert results[0][1] == results[1][1]
    amp, pw, truths = W.population(5)
    for s in (0, 4):
        c = W.Control(n_steps=60, amplitude_deg=amp[s], pw_default_ms=pw[s])
        r = oracle.fit(oracle.positions(truths[s], c), c, sp, 0, 300, saccade=s)
        assert results[0][2][s] == (r["best_err"], r["best_index"])


def _super_node_indices(n_nodes_begin, n_nodes_end, st, L):
    """Candidate indices of grid nodes [b, e) of the superposition kernel
    (kernel_variant 4): node n -> level-0 index
    (n // st) * st * L + n % st, levels at stride st."""
    out = []
    for n in range(n_nodes_begin, n_nodes_end):
        ib = (n // st) * st * L + n % st
        out.extend(ib + j * st for j in range(L))
    return out


def _super_rank_main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_09884_b200 import opmm
        ctl = W.Control()
        rec = oracle.positions(W.truth_opc(), ctl) + W.noise(ctl.n_steps + 1)
        sp = W.g4_space(per_dim=5)          # N_SAC_AG (dim 15) superposed, L = 5
        L = 5
        st = 5 * 5                          # levels of dims 0 (K_SE_AG) and 4 (B_AG)
        nodes = sp.n_grid() // L
        b, e = opmm.opmm_shard_range(nodes, rank, world)
        idx = _super_node_indices(b, e, st, L)
        errs = [oracle.objective(oracle.generate(sp, i), rec, ctl) for i in idx]
        best = min(zip(errs, idx)) if idx else (float("inf"), -1)
        mine = torch.tensor([best[0], float(best[1]), float(len(idx))], dtype=torch.float64)
        allp = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allp, mine)
        be, bi = opmm.opmm_merge_argmin([float(t[0]) for t in allp], [int(t[1]) for t in allp])
        q.put((rank, be, bi, sorted(idx), int(sum(float(t[2]) for t in allp))))
    finally:
        dist.destroy_process_group()


def test_world2_super_node_shards_partition_the_grid():
    """kernel_variant 4 shards grid NODES (all levels of a node on one rank):
    the ranks' candidate sets are disjoint, cover the grid, and the merged
    argmin equals the unsharded one."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_super_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sp = W.g4_space(per_dim=5)
    n = sp.n_grid()
    all_idx = sorted(results[0][3] + results[1][3])
    assert all_idx == list(range(n))
    assert results[0][4] == n
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(ctl.n_steps + 1)
    full = oracle.fit(rec, ctl, sp, 0, n)
    for rank, be, bi, _, _ in results:
        assert (be, bi) == (full["best_err"], full["best_index"])


def _topk_rank_main(rank, world, port, q):
    """One rank of the fp32-certified multi-GPU fit, on CPU: the rank's exact
    top-K by (fp32 error, index) over its shard -- fp32 errors stood in by the
    oracle's fp64 errors rounded to float32 -- all-gathered, merged with
    opmm_merge_topk, re-scored in fp64 (oracle) and certified with
    opmm_certify_topk, as the merge kernel does on the device."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        from paper_2007_09884_b200 import opmm
        ctl = W.Control()
        rec = oracle.positions(W.truth_opc(), ctl) + W.noise(ctl.n_steps + 1)
        sp = W.paper_space()
        N, K = 5000, 16
        b, e = opmm.opmm_shard_range(N, rank, world)
        E = oracle.fit(rec, ctl, sp, b, e, want_err=True)["err"]
        e32 = E.astype(np.float32).astype(np.float64)
        order = np.lexsort((np.arange(b, e), e32))[:K]
        le = np.full(K, np.inf)
        li = np.full(K, -1, dtype=np.int64)
        le[:len(order)] = e32[order]
        li[:len(order)] = order + b
        ge = [torch.zeros(K, dtype=torch.float64) for _ in range(world)]
        gi = [torch.zeros(K, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(ge, torch.from_numpy(le))
        dist.all_gather(gi, torch.from_numpy(li))
        me, mi = opmm.opmm_merge_topk(torch.stack(ge).numpy(), torch.stack(gi).numpy(), K)
        e64 = np.array([oracle.objective(oracle.generate(sp, int(i)), rec, ctl) if i >= 0 else np.inf
                        for i in mi])
        rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
        cert = opmm.opmm_certify_topk(me, e64, mi, float(np.abs(rel).sum()))
        q.put((rank, mi.tolist(), me.tolist(), cert))
    finally:
        dist.destroy_process_group()


def test_world2_topk_merge_and_fp32_certificate():
    """Multi-GPU fp32 certification (the ranks' (E, index) lists
    are gathered and merged; "solutions are sorted for accuracy",
    PAPER.md:251): the merged list equals the unsharded exact top-K, every rank
    returns the same certified winner, and it is the fp64 argmin of all N."""
    import numpy as np
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_topk_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(ctl.n_steps + 1)
    sp = W.paper_space()
    full = oracle.fit(rec, ctl, sp, 0, 5000, want_err=True)
    e32 = full["err"].astype(np.float32).astype(np.float64)
    order = np.lexsort((np.arange(5000), e32))[:16]
    for rank, mi, me, cert in results:
        assert mi == order.tolist() and me == e32[order].tolist()
        assert cert == (1, full["best_index"], full["best_err"])
    assert results[0][1:] == results[1][1:]


def test_merge_topk_and_certificate_edge_cases():
    """Host helpers: pads (-1) end a list, exact ties go to the lower index,
    fewer entries than K pad the output; the certificate is refused when the
    K-th fp32 error lies within T* or a listed candidate breaks the budget."""
    import numpy as np
    from paper_2007_09884_b200 import opmm
    inf = np.inf
    e = np.array([[1.0, 2.0, 2.0, inf], [0.5, 2.0, inf, inf]])
    i = np.array([[10, 3, 7, -1], [4, 2, -1, -1]], dtype=np.int64)
    me, mi = opmm.opmm_merge_topk(e, i, 4)
    assert mi.tolist() == [4, 10, 2, 3] and me.tolist() == [0.5, 1.0, 2.0, 2.0]
    me, mi = opmm.opmm_merge_topk(e[:1, :], i[:1, :], 4)
    assert mi.tolist() == [10, 3, 7, -1] and me[3] == inf
    idx = np.array([5, 9, 1, 2], dtype=np.int64)
    e32 = np.array([10.0, 20.0, 30.0, 40.0])
    assert opmm.opmm_certify_topk(e32, e32 + 1e-6, idx, 100.0) == (1, 5, 10.0 + 1e-6)
    # K-th error inside T* = 10 + 2e-2: refused
    assert opmm.opmm_certify_topk(np.array([10.0, 10.01, 10.015, 10.02]), np.full(4, 10.0), idx,
                                  100.0)[0] == 0
    # budget broken by a listed candidate (|E64 - E32| = 0.1 > delta = 1e-2): refused
    e64 = e32.copy()
    e64[2] = 29.9
    c = opmm.opmm_certify_topk(e32, e64, idx, 100.0)
    assert c[0] == 0 and c[1] == 5
    # fewer finite candidates than K: certified, winner the fp64-best
    c = opmm.opmm_certify_topk(np.array([3.0, inf, inf, inf]), np.array([2.9999, inf, inf, inf]),
                               np.array([8, -1, -1, -1], dtype=np.int64), 1.0)
    assert c == (1, 8, 2.9999)
