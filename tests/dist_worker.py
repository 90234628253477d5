"""Per-rank worker for the multi-GPU parity test (launched by tests/test_gpu_dist.py
with torchrun, one process per GPU).  Each rank drives libgcp.so through the C
ABI on its own GPU (NCCL between ranks) and checks its block against an fp64
oracle simulation of all P ranks run locally (oracle.MultiRank)."""
import math
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import gcp_synth  # noqa: E402
import oracle  # noqa: E402


def main():
    mode = sys.argv[1]
    # "sync32": the sync scheme in fp32 (the fused exchange's NVLS multicast path
    # runs in fp32 only); tolerances from DESIGN.md section 5.2
    prec = "fp32" if mode == "sync32" else "fp64"
    if mode == "sync32":
        os.environ["GCP_MULTIMEM"] = "1"   # exercise the NVLS path whatever P is
    if mode in ("sync32", "async", "twosided"):
        # the slot-ordered K2 (on by default only when mode-1 rows spill L2, e.g.
        # c4 blocks): under the fused exchange (sync32), k_adam (async) and the
        # device-driven two-sided exchange; the histogram carried by K2 each time
        os.environ["GCP_SLOT_ORDER"] = "1"
    if mode == "twosided_nccl":
        os.environ["GCP_TWOSIDED_NVL"] = "0"   # the NCCL send/recv two-sided path (twosided.cu)
        mode = "twosided"
    if mode == "twosided":
        os.environ["GCP_TWOSIDED_NVL"] = "1"   # the import / export kernels over NVLink windows (twosided_nvl.cu)
    peer = mode == "twosided_peer"
    if peer:
        os.environ["GCP_TWOSIDED_NVL"] = "peer"   # K2 reaches the owners' rows over NVLink (twosided_nvl.cu)
        mode = "twosided"
    mode = "sync" if mode == "sync32" else mode
    # TG, TE: the C18 bounds (gradient per element vs the rounding scale S, loss
    # estimate vs sum |terms|) from an identical state.  TM / TM_FIT / TE_FIT bound
    # multi-step trajectories (5 iterations; a 3-epoch fit of 18), where C18 sets
    # no bound: DESIGN.md §5.3 derives them from Adam's sensitivity
    # |d(B^/sqrt(C^+eps))/dg| <= 1/sqrt(eps) applied to the per-step rounding
    # difference of the gradient, summed over the steps.
    TG, TE = (1e-4, 1e-4) if prec == "fp32" else (1e-10, 1e-10)
    TM, TM_FIT, TE_FIT = (1e-3, 1e-2, 1e-3) if prec == "fp32" else (1e-9, 1e-8, 1e-9)
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import paper_2605_20353_b200 as g

    uid = [g.gcp_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    dims, R, loss = (36, 30, 24), 4, "poisson"
    subs, vals = gcp_synth.chi_kolda(dims, 3000, R, 1234, loss=loss)
    subs, vals = subs.numpy(), vals.numpy()
    blocks, grid = oracle.split_blocks(dims, subs, vals, ws)
    ggrid, lo, hi = g.gcp_grid_plan(ws, dims)
    assert tuple(ggrid) == tuple(grid)
    mine = blocks[rank]
    assert list(lo[rank]) == mine.lo and list(hi[rank]) == mine.hi
    bs, bv = mine.sorted()

    ctx = g.Context(local, None, prec)
    ctx.dist_init(ws, rank, uid[0], None, mode)
    ctx.tensor_create(dims, bs, bv)
    info = ctx.tensor_info()
    assert info["nnz"] == mine.nnz and info["nnz_global"] == len(vals)
    ctx.model_init(R, 77)
    A0 = oracle.factor_init(77, dims, R)
    for k in range(3):
        want = A0[k][mine.lo[k]:mine.hi[k]]
        if prec == "fp32":
            want = want.astype(np.float32).astype(np.float64)
        assert np.array_equal(ctx.model_get(k), want), "init"

    tau = 2
    # the two-sided layout (row f3) computes Alg. 2 exactly like the all-reduce layout
    omode = "sync" if mode == "twosided" else mode
    run = oracle.MultiRank(blocks, grid, A0, loss, mode=omode, tau=tau, meta_rate=5e-3)
    p = q = 600
    seed, rate = 99, 1e-2
    ctx.sample("stratified", p, q, seed)
    if omode != "sync":
        ctx.dist_set_async(tau, g.adam_params(rate=5e-3))
    ap = g.adam_params(rate=rate)
    worst = 0.0
    for it in range(5):
        # gradient of this rank's block, before any exchange
        if omode == "sync":
            A_rank = run.model_for_rank(rank)
            pw, qw = oracle.local_counts(mine, p, q, ws, rank)
            Go, S, _ = oracle.sampled_grad(mine, A_rank, loss, seed, rank, it, pw, qw)
            ctx.loss_grad(loss)
            if peer:
                # peer access: every contribution to a row lands in its owner's G,
                # so a rank holds the global (all-rank) gradient of its owned rows
                # -- once every rank's gradient kernel has finished
                torch.cuda.synchronize()
                dist.barrier()
                Gs, Ss, _ = oracle.sync_gradient(blocks, A_rank, loss, seed, it, p, q)
            for k in range(3):
                Gg = ctx.grad_get(k)
                if peer:
                    gk = math.prod(grid) // grid[k]
                    rows_k = -(-(-(-dims[k] // grid[k])) // gk) * gk
                    sh = rows_k // gk
                    me = [w for w in oracle.slice_groups(grid, k) if rank in w][0].index(rank)
                    o0, o1 = me * sh, min((me + 1) * sh, mine.hi[k] - mine.lo[k])
                    want = Gs[k][mine.lo[k] + o0: mine.lo[k] + o1]
                    sc = Ss[k][mine.lo[k] + o0: mine.lo[k] + o1]
                    assert np.all(np.abs(Gg[o0:o1] - want) <= TG * sc + 1e-300), f"owned grad it={it} k={k}"
                else:
                    assert np.all(np.abs(Gg - Go[k]) <= TG * S[k] + 1e-300), f"grad it={it} k={k}"
        else:
            ctx.loss_grad(loss)
        ctx.adam_step(ap)
        run.iteration(it, seed, p, q, rate)
        for k in range(3):
            want = run.block_rows(rank, k)
            got = ctx.model_get(k)
            err = np.abs(got - want).max() / max(1.0, np.abs(want).max())
            worst = max(worst, err)
            assert err < TM, f"model it={it} k={k} err={err}"
    est = ctx.loss_estimate(loss, 1500, 1500, 5)
    oe, sc = run.estimate(5, 1500, 1500)
    assert abs(est - oe) <= TE * sc, (est, oe)
    feats = ctx.dist_features()
    if mode == "twosided":   # device-driven over NVLink windows unless GCP_TWOSIDED_NVL=0
        assert feats["fused"] == (os.environ.get("GCP_TWOSIDED_NVL") != "0"), feats
    ctx.close()

    # the epoch loop (R20) on a side stream: the iterations of an epoch replay
    # as one CUDA graph (sync / twosided-off / LocalSGD) -- against oracle.fit
    stream = torch.cuda.Stream(local)
    uid = [g.gcp_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ctx = g.Context(local, stream.cuda_stream, prec)
    ctx.dist_init(ws, rank, uid[0], None, mode)
    ctx.tensor_create(dims, bs, bv)
    ctx.model_init(R, 77)
    kw = dict(epochs=3, max_fails=3, decay=0.1, s_nz=p, s_z=q, f_nz=1500, f_z=1500, seed=seed, fseed=5,
              rate=rate)
    fp = ctx.fit_params(iters_per_epoch=6, loss=loss, tau=tau if omode != "sync" else 0, meta_rate=5e-3, **kw)
    best, rows = ctx.fit(fp)
    Af, hist, obest = oracle.fit(blocks, grid, A0, loss, iters=6, mode=omode, tau=tau, meta_rate=5e-3, **kw)
    assert len(rows) == len(hist), (rows, hist)
    for r, h in zip(rows, hist):
        assert abs(r[2] - h[0]) <= TE_FIT * abs(h[0]), (r, h)
    for k in range(3):
        want = (Af if omode == "sync" else Af[rank])[k][mine.lo[k]:mine.hi[k]]
        assert np.allclose(ctx.model_get(k), want, rtol=TM_FIT, atol=TM), f"fit model k={k}"
    # replace-ingest on the same context (a repeated job): the grid is unchanged, so
    # the slice communicators and the symmetric windows are reused, not re-created;
    # the fit must repeat the oracle's trajectory
    ctx.tensor_create(dims, bs, bv)
    ctx.model_init(R, 77)
    _, rows2 = ctx.fit(fp)
    assert len(rows2) == len(hist), (rows2, hist)
    for r, h in zip(rows2, hist):
        assert abs(r[2] - h[0]) <= TE_FIT * abs(h[0]), ("replace-ingest", r, h)
    for k in range(3):
        want = (Af if omode == "sync" else Af[rank])[k][mine.lo[k]:mine.hi[k]]
        assert np.allclose(ctx.model_get(k), want, rtol=TM_FIT, atol=TM), f"replace-ingest fit model k={k}"
    if omode == "sync":
        # a rejected epoch (R20): at rate 0.3 the oracle accepts, rejects (restore
        # of A, B, C, t; rate x 0.1), then accepts twice -- the restore rewrites
        # every rank's rows, which the next gradient (peer access: remote reads
        # and adds) must only see after all ranks restored
        ctx.model_init(R, 77)
        kw3 = dict(kw, rate=0.3, epochs=4)
        fp3 = ctx.fit_params(iters_per_epoch=6, loss=loss, tau=0, meta_rate=5e-3, **kw3)
        _, rows3 = ctx.fit(fp3)
        Af3, hist3, _ = oracle.fit(blocks, grid, A0, loss, iters=6, mode="sync", tau=tau, meta_rate=5e-3, **kw3)
        assert [h[2] for h in hist3] == [True, False, True, True], hist3
        assert len(rows3) == len(hist3), (rows3, hist3)
        for r, h in zip(rows3, hist3):
            # the trace reports the rate after the epoch's decision (x decay on a rejection)
            r_after = h[1] * (1.0 if h[2] else kw3["decay"])
            assert abs(r[2] - h[0]) <= TE_FIT * abs(h[0]) and abs(r[3] - r_after) <= 1e-12 * r_after, ("rejection", r, h)
        for k in range(3):
            assert np.allclose(ctx.model_get(k), Af3[k][mine.lo[k]:mine.hi[k]], rtol=TM_FIT, atol=TM), \
                f"rejection fit model k={k}"
    ctx.close()
    dist.barrier()
    if rank == 0:
        print(f"DIST-OK mode={mode} prec={prec} P={ws} grid={grid} worst_model_err={worst:.2e} "
              f"features={feats}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    try:
        main()
    except BaseException:
        # exit at once: a peer blocked in a device-side barrier would otherwise
        # keep this rank's teardown (and the launcher) waiting; torchrun then
        # stops the other ranks
        import traceback
        traceback.print_exc()
        sys.stderr.flush()
        os._exit(1)
