"""Drive every libgcp kernel on c1-sized inputs for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per gpurun call):

    compute-sanitizer --tool memcheck --error-exitcode 3 python tools/sanitize_c1.py

Ingest (standard and lean paths, hash and sorted membership, u128 keys),
factor init, model set/get, K2 in every strategy and precision (including the
slot-ordered launch with its histogram / scan / scatter kernels and the
histogram fused into Adam), Adam, the loss estimate with its fixed-order
reduction, sample export, membership queries, and a short fit with CUDA-graph
replay.  No oracle: this checks memory safety and races, parity is the tests'
job.  Prints SANITIZE-OK at the end.
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gcp_synth  # noqa: E402
import paper_2605_20353_b200 as g  # noqa: E402


def run(dims, R, loss, prec, membership, env):
    for k, v in env.items():
        os.environ[k] = v
    import math
    M = math.prod(dims)
    subs, vals = gcp_synth.chi_kolda(dims, int(0.1 * M) if M < 10 ** 6 else 20000, R, 1001, loss=loss)
    subs, vals = subs.numpy(), vals.numpy()
    stream = torch.cuda.Stream(0)
    c = g.Context(0, stream.cuda_stream, prec)
    c.set_membership(membership)
    c.tensor_create(dims, subs, vals)
    c.tensor_contains(subs[:100])
    c.tensor_export_sorted(0, min(100, len(vals)))
    c.model_init(R, 2001)
    A = [c.model_get(k) for k in range(len(dims))]
    for k in range(len(dims)):
        c.model_set(k, A[k])
    for strategy in ("stratified", "semi"):
        c.sample(strategy, 700, 900, 3001)
        c.sample_export(0, 0, 700)
        c.sample_export(1, 0, 900)
        c.loss_grad(loss, want_loss=True)
        [c.grad_get(k) for k in range(len(dims))]
        c.adam_step(g.adam_params(rate=1e-2))
        c.loss_grad(loss)
        c.adam_step(g.adam_params(rate=1e-2))
    c.loss_estimate(loss, 1500, 1500, 4001)
    p = c.fit_params(epochs=3, iters_per_epoch=5, s_nz=300, s_z=300, f_nz=500, f_z=500, loss=loss, seed=7, fseed=2,
                     rate=1e-2)
    c.fit(p)
    torch.cuda.synchronize()
    c.close()
    for k in env:
        del os.environ[k]


def main():
    torch.cuda.init()
    c1 = (20, 30, 40)
    lbnl = tuple(gcp_synth.CONFIGS["c3"]["dims"])
    cases = [
        (c1, 4, "poisson", "fp32", "hash", {}),
        (c1, 4, "poisson", "fp32", "sorted", {"GCP_SLOT_ORDER": "1"}),
        (c1, 16, "gaussian", "fp32", "hash", {"GCP_SLOT_ORDER": "1", "GCP_AG_INTERLEAVE": "1"}),
        (c1, 16, "gaussian", "fp32", "hash", {"GCP_SLOT_ORDER": "1", "GCP_ORD_FUSE": "0", "GCP_INGEST": "lean"}),
        (c1, 5, "bernoulli", "fp64", "hash", {"GCP_SLOT_ORDER": "1", "GCP_INGEST": "lean"}),
        (c1, 32, "poisson", "fp32", "sorted", {"GCP_FILTER": "0"}),
        (lbnl, 10, "bernoulli", "fp32", "hash", {}),
    ]
    for case in cases:
        run(*case)
        print("case ok", case[:5], case[5], flush=True)
    print("SANITIZE-OK", flush=True)


if __name__ == "__main__":
    main()
