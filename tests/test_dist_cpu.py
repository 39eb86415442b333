"""Multi-rank path on CPU (gloo, world_size 2).

The B200 runtime shards every batch by member (rank r owns global members
[r*B, (r+1)*B)) and exchanges, per batch, allreduce(max) of the packed key
(cut << 32 | ~member) and allreduce(max) of the owner's winner assignment (zeros
elsewhere) — lcb_runtime.cu Solver::run_batch.  Here each rank computes its shard
with the oracle and runs the same exchange over gloo with the product's key helpers
(lcb_pack_key / lcb_unpack_key, dist.shard); the per-batch results and the final
assignment must equal the single-process reference solve with batch 2*B.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_pquco(rank, world, port, q):
    from paper_2509_18612_b200.dist import pack_key, shard, unpack_key

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = O.generate_er(90, 0.06, 7)
        B_local, T, seed, batches = 6, 80, 5, 3
        lo, hi = shard(B_local * world, world, rank)
        eta = 0.8 / 1e8
        serial = 0
        trace = []
        best_key, best_z = -1, None
        z = None
        for b in range(batches):
            if b == 0:
                mean = O.lifted_init_mean(g, 1, 0.2, 1, O.split(seed, 0x696E, 0, serial)) / 1e4
            else:
                mean = np.where(z == 1, 1.0, -1.0) / 1e4
            bkey = O.split(seed, 0x6261, serial)
            serial += 1
            x = O.gaussian_members(mean, g.n, 1, eta, lo, hi - lo, bkey)
            x, _ = O.ascend(g, x, 1, hi - lo, 0.05, T, 0.9, True)
            keys = []
            for j in range(hi - lo):
                zz = O.round_unlifted(x[j * g.n:(j + 1) * g.n])
                keys.append(pack_key(O.cut_value(g, zz), lo + j))
            t = torch.tensor([max(keys)], dtype=torch.int64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)                 # C-1: packed key
            cut, member = unpack_key(int(t.item()))
            mine = torch.zeros(g.n, dtype=torch.uint8)
            if lo <= member < hi:
                j = member - lo
                mine = torch.from_numpy(O.round_unlifted(x[j * g.n:(j + 1) * g.n]).copy())
            dist.all_reduce(mine, op=dist.ReduceOp.MAX)              # C-2: winner bits
            z = mine.numpy()
            trace.append((cut, member))
            if int(t.item()) >> 32 > best_key >> 32 if best_key >= 0 else True:
                best_key, best_z = int(t.item()), z.copy()
        if rank == 0:
            q.put((trace, best_z.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_batches_equal_single_solve():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_pquco, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    trace, z = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = O.generate_er(90, 0.06, 7)
    cfg = O.default_config(batch_size=12, iterations=80, num_batches=3)
    want = O.solve(g, cfg, 5)
    assert [(e[4], None) for e in want.batch_trace] == [(c, None) for c, _ in trace]
    assert want.member_index in [m for _, m in trace]
    assert z == want.assignment.tolist()
    if O.ref is not None:
        r = O.ref_solve(O.RefGraph.from_csr(g), cfg, 5)
        assert r.assignment.tolist() == z and [e[4] for e in r.batch_trace] == [c for c, _ in trace]
