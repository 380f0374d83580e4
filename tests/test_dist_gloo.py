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
