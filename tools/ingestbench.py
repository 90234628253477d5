"""Repeated ingest of one config from pinned host memory (development tool):

    GCP_INGEST_TRACE=1 python tools/ingestbench.py --config c4 --reps 3

prints the library's per-phase ingest times (stderr) and the wall time per
gcp_tensor_create (the e2e 'h2d_ingest' phase)."""
import argparse
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
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fresh", action="store_true", help="a new context per rep (destroyed after it)")
    args = ap.parse_args()
    import paper_2605_20353_b200 as g
    c, s = gcp_synth.CONFIGS[args.config], gcp_synth.SEEDS[args.config]
    subs, vals = gcp_synth.chi_kolda(c["dims"], c["nnz"], c["R"], s["data"], c["loss"], device="cuda")
    subs_h = torch.empty(subs.shape, dtype=subs.dtype, pin_memory=True)
    subs_h.copy_(subs)
    vals_h = torch.empty(vals.shape, dtype=vals.dtype, pin_memory=True)
    vals_h.copy_(vals)
    del subs, vals
    torch.cuda.empty_cache()
    stream = torch.cuda.Stream()
    ctx = None
    for r in range(args.reps):
        if ctx is None or args.fresh:
            if ctx is not None:
                ctx.close()
            ctx = g.Context(0, stream.cuda_stream, "fp32")
        t0 = time.perf_counter()
        ctx.tensor_create_ptr(c["dims"], vals_h.numel(), subs_h.data_ptr(), vals_h.data_ptr())
        print(f"rep {r}: tensor_create {1e3 * (time.perf_counter() - t0):.1f} ms "
              f"({vals_h.numel() * 32 / 1e9:.2f} GB of int64 subs + f64 vals)", flush=True)


if __name__ == "__main__":
    main()
