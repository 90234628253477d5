"""World-size-2 gloo tests of the multi-rank host logic (CPU only):
grid plan agreement between libgcp's host entry point and the oracle on every
rank, block extraction, per-rank sample allocation, and the distributed
decomposition of the sampled gradient (sum over processes of each rank's
block gradient == the single-process P-rank simulation)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        import gcp_synth
        import oracle
        import paper_2605_20353_b200 as g
        dims = (30, 20, 16)
        subs, vals = gcp_synth.chi_kolda(dims, 1500, 3, 77, loss="poisson")
        subs, vals = subs.numpy(), vals.numpy()
        grid, lo, hi = g.gcp_grid_plan(ws, dims)
        blocks, ogrid = oracle.split_blocks(dims, subs, vals, ws)
        assert tuple(grid) == tuple(ogrid)
        mine = blocks[rank]
        assert list(lo[rank]) == mine.lo and list(hi[rank]) == mine.hi
        # every nonzero lands in exactly one rank's block
        n = torch.tensor([mine.nnz], dtype=torch.int64)
        dist.all_reduce(n)
        assert int(n) == len(vals)
        # per-rank allocation sums to the global totals (reading R13)
        p, qz = 101, 57
        pw, qw = oracle.local_counts(mine, p, qz, ws, rank)
        t = torch.tensor([pw, qw], dtype=torch.int64)
        dist.all_reduce(t)
        assert t.tolist() == [p, qz]
        # distributed gradient = the oracle's single-process P-rank sum
        A = oracle.factor_init(5, dims, 3)
        Gw, _, _ = oracle.sampled_grad(mine, A, "poisson", 11, rank, 0, pw, qw)
        full = [np.zeros_like(a) for a in A]
        for k in range(3):
            full[k][mine.lo[k]:mine.hi[k]] = Gw[k]
        flat = torch.from_numpy(np.concatenate([f.ravel() for f in full]))
        dist.all_reduce(flat)
        Gs, _, _ = oracle.sync_gradient(blocks, A, "poisson", 11, 0, p, qz)
        ref = np.concatenate([x.ravel() for x in Gs])
        assert np.allclose(flat.numpy(), ref, rtol=1e-12, atol=1e-12)
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_gloo_world_size_2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res
