"""Per-kernel timing of the hot path on one config (development tool).

    python tools/k2bench.py [--config c2] [--iters 20]

Times K2 (fused sampling-MTTKRP), K3 (Adam) and the loss estimate separately
with the library's CUDA-event profiler; prints one JSON line.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import gcp_synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--l2fetch", default="", help="comma list of cudaLimitMaxL2FetchGranularity values to sweep")
    ap.add_argument("--strategies", default="stratified", help="comma list: stratified,semi")
    ap.add_argument("--membership", default="hash", help="hash or sorted (row f4)")
    ap.add_argument("--p", type=int, default=-1, help="nonzero samples per iteration (default: the config's)")
    ap.add_argument("--q", type=int, default=-1, help="zero samples per iteration (default: the config's)")
    args = ap.parse_args()
    import paper_2605_20353_b200 as g
    c = gcp_synth.CONFIGS[args.config]
    s = gcp_synth.SEEDS[args.config]
    subs, vals = gcp_synth.chi_kolda(c["dims"], c["nnz"], c["R"], s["data"], c["loss"], device="cuda")
    subs_h = torch.empty(subs.shape, dtype=subs.dtype, pin_memory=True)
    subs_h.copy_(subs)
    vals_h = torch.empty(vals.shape, dtype=vals.dtype, pin_memory=True)
    vals_h.copy_(vals)
    del subs, vals
    torch.cuda.empty_cache()
    stream = torch.cuda.Stream()
    ctx = g.Context(0, stream.cuda_stream, args.precision)
    ctx.set_membership(args.membership)
    t0 = time.time()
    ctx.tensor_create_ptr(c["dims"], vals_h.numel(), subs_h.data_ptr(), vals_h.data_ptr())
    t_ingest = time.time() - t0
    ctx.model_init(c["R"], s["model"])
    P = c["s"] if args.p < 0 else args.p
    Q = c["s"] if args.q < 0 else args.q
    ctx.sample("stratified", P, Q, s["sample"])
    for _ in range(3):
        ctx.loss_grad(c["loss"])
        ctx.adam_step()
    ctx.loss_estimate(c["loss"], c["f"], c["f"], 2)
    sweep = [int(x) for x in args.l2fetch.split(",")] if args.l2fetch else [None]
    for strat, l2f in [(st, l) for st in args.strategies.split(",") for l in sweep]:
        ctx.sample(strat, P, Q, s["sample"])
        if l2f is not None:   # device-wide hint through the process's CUDA runtime
            import ctypes
            rt = ctypes.CDLL("libcudart.so.12")
            rt.cudaDeviceSetLimit(ctypes.c_int(0x05), ctypes.c_size_t(l2f))   # cudaLimitMaxL2FetchGranularity
        ctx.profile_enable(True)
        for k in ("grad", "adam", "loss", "other"):
            ctx.profile_get(k, reset=True)
        for _ in range(args.iters):
            ctx.loss_grad(c["loss"])
            ctx.adam_step()
        for _ in range(3):
            ctx.loss_estimate(c["loss"], c["f"], c["f"], 2)
        out = {"config": args.config, "strategy": strat, "membership": args.membership, "L2_FETCH": l2f if l2f is not None else os.environ.get("GCP_L2_FETCH", "32"),
               "ingest_s": t_ingest}
        for k in ("grad", "adam", "loss"):
            ms, n = ctx.profile_get(k)
            out[k + "_ms"] = ms / max(n, 1)
        out["p"], out["q"] = P, Q
        out["samples_per_s_k2"] = (P + Q) / (out["grad_ms"] * 1e-3)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
