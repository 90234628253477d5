#!/usr/bin/env python
"""GCP-Adam epoch benchmark (BASELINE.json metric) on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one GCP-Adam epoch: 100 x [fused sampling-MTTKRP (K2),
(P>1 sync: reduce-scatter), Adam (K3), (P>1 sync: all-gather)] + the fixed-set
loss estimate + the accept/reject decision -- every row of SURVEY §8(a).  The
tensor is ingested and the model initialised before timing (inputs resident in
HBM).  W untimed warm-up epochs, then K epochs between barrier + synchronize,
CUDA events on the library's stream, max over ranks.  One JSON line on rank 0.

--impl reference times the fp64 CPU oracle (the base contract's reference
arm for this tier) on a bounded sample of the same workload, extrapolated to
an epoch; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gcp_synth  # noqa: E402

_T0 = time.time()


def log(*a):
    """Progress to stderr (stdout carries only the JSON line)."""
    print(f"[bench {time.time() - _T0:7.1f}s]", *a, file=sys.stderr, flush=True)


METRIC = "GCP-Adam epochs/sec and sampled-gradient samples/sec (1/2/4/8 B200); HBM GB/s"
ITERS = 100  # iterations per epoch


def workload(name):
    c = gcp_synth.CONFIGS[name]
    d = len(c["dims"])
    M = math.prod(c["dims"])
    rho = c["nnz"] / M
    kB = 16 if M >= 2 ** 64 else 8
    R = c["R"]
    nz_b = (d + 1) * 4 + d * R * 4 + 2 * d * R * 4
    z_b = kB / (1 - rho) + 3 * d * R * 4
    desc = {"c1": "3-way 20x30x40 synthetic count tensor, ~2.4K nnz, R=4, Poisson",
            "c2": "3-way 10Kx10Kx10K synthetic Poisson tensor, 100M nnz, R=16, stratified, p=q=1e7",
            "c3": "5-way LBNL-network-shaped tensor, 1.7M nnz, R=10, Bernoulli-logit, p=q=1e6",
            "c4": "3-way Amazon-reviews-shaped tensor, 1.74B nnz, R=16, Gaussian, p=q=1e7",
            "c5": "3-way Reddit-2015-shaped tensor, 4.69B nnz, R=32, Poisson, p=q=1e8"}[name]
    return dict(c, d=d, M=M, rho=rho, nz_bytes=nz_b, z_bytes=z_b, desc=desc)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every 20 ms during the
    timed region through NVML (the data of the recipe's nvidia-smi clocks line)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, dev):
        self.dev = dev
        self.sm, self.reasons, self.max = [], set(), None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = dev_index(self.dev)
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        while not self.stop.is_set():
            try:
                self.sm.append(float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __exit__(self, *a):
        self.stop.set()
        if self.nv:
            self.t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 20 ms"}


def nvlink_counters(dev):
    """NVLink data bytes this GPU has sent / received so far, summed over its
    links, from NVML's per-link NVLink counters (tools/nvlink_probe.py checks
    the fields against a peer copy of known size).  None when NVML has none."""
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(dev_index(dev))
        out = {}
        for name, fid, scale in (("tx", nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 1024),
                                 ("rx", nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 1024)):
            tot, nlinks = 0, 0
            for link in range(18):
                fv = nv.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
                if fv.nvmlReturn == 0:
                    tot += int(fv.value.ullVal) * scale
                    nlinks += 1
            if not nlinks:
                return None
            out[name] = tot
        out["links"] = nlinks
        return out
    except Exception:
        return None


def dev_index(local):
    """Physical index of the local CUDA device (honours CUDA_VISIBLE_DEVICES)."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [x.strip() for x in vis.split(",") if x.strip()]
        if local < len(ids) and ids[local].isdigit():
            return int(ids[local])
    return local


# ------------------------------------------------------------------ distributed
def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(ws, x):
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allgather_obj(ws, o):
    if ws == 1:
        return [o]
    import torch.distributed as dist
    out = [None] * ws
    dist.all_gather_object(out, o)
    return out


def bcast_bytes(ws, rank, b):
    if ws == 1:
        return b
    import torch.distributed as dist
    obj = [b if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


# ------------------------------------------------------------------ data
def make_tensor(name, device, block=None, allreduce=None, out_device=None):
    """The workload's tensor; with block=(lo, hi) only this rank's block (the
    same global tensor, generated without materialising the other blocks)."""
    w = workload(name)
    t0 = time.time()
    subs, vals = gcp_synth.chi_kolda(w["dims"], w["nnz"], w["R"], gcp_synth.SEEDS[name]["data"], w["loss"],
                                     device=device, block=block, allreduce=allreduce, out_device=out_device)
    return subs, vals, time.time() - t0


def allsum_int(ws, x):
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([int(x)], dtype=torch.int64, device="cuda")
    dist.all_reduce(t)
    return int(t.item())


def block_of(subs, vals, lo, hi):
    m = torch.ones(len(vals), dtype=torch.bool, device=vals.device)
    for k in range(subs.shape[1]):
        m &= (subs[:, k] >= int(lo[k])) & (subs[:, k] < int(hi[k]))
    return subs[m], vals[m]


# ------------------------------------------------------------------ reference arm (CPU oracle)
def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    import oracle
    return {"cpu_model": model, "host_threads": oracle.host_threads(),
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS")}


def run_oracle_sample(name, subs_h, vals_h, steps, warmup, sample_n, lo=None, hi=None, nthreads=None):
    """Time the fp64 oracle, as it stands, on a bounded sample of one epoch of
    workload `name`: per step one sampled gradient with p'=q'=sample_n, one Adam
    pass over all coefficients, one loss estimate with f'=sample_n, each timed;
    the epoch (100 iterations at p=q, f-samples f) is extrapolated from those
    per-sample and per-pass times.  nthreads: None = the single-threaded parity
    oracle, else its OpenMP timing variant on that many
    threads.  lo/hi: a block of the tensor (its nonzeros in subs_h)."""
    import oracle
    w = workload(name)
    t0 = time.time()
    t = oracle.Tensor(w["dims"], subs_h, vals_h, lo, hi)
    setup = time.time() - t0
    A = oracle.factor_init(gcp_synth.SEEDS[name]["model"], w["dims"], w["R"])
    flat = np.concatenate([a.ravel() for a in A])   # the whole model: Adam runs over all of it
    B, Cm = np.zeros_like(flat), np.zeros_like(flat)
    Gf = np.zeros_like(flat)
    offs = np.cumsum([0] + [int(I) * w["R"] for I in w["dims"]])
    blo = [0] * w["d"] if lo is None else lo
    seed = gcp_synth.SEEDS[name]["sample"]
    times = []
    for s in range(warmup + steps):
        t1 = time.perf_counter()
        if nthreads is None:
            G, _, _ = oracle.sampled_grad(t, A, w["loss"], seed, 0, s, sample_n, sample_n, with_scale=False)
        else:
            G, _ = oracle.sampled_grad_par(t, A, w["loss"], seed, 0, s, sample_n, sample_n, nthreads=nthreads)
        tg = time.perf_counter() - t1
        for k in range(w["d"]):   # the block's rows into the global gradient
            Gf[offs[k] + blo[k] * w["R"]: offs[k] + blo[k] * w["R"] + G[k].size] = G[k].ravel()
        t2 = time.perf_counter()
        if nthreads is None:
            oracle.adam(flat, Gf, B, Cm, s + 1, 1e-3, 0.9, 0.999, 1e-8, oracle.loss_lower(w["loss"]))
        else:
            oracle.adam_par(flat, Gf, B, Cm, s + 1, 1e-3, 0.9, 0.999, 1e-8, oracle.loss_lower(w["loss"]),
                            nthreads=nthreads)
        ta = time.perf_counter() - t2
        t3 = time.perf_counter()
        if nthreads is None:
            oracle.loss_estimate(t, A, w["loss"], 2, 0, sample_n, sample_n)
        else:
            oracle.loss_estimate_par(t, A, w["loss"], 2, 0, sample_n, sample_n, nthreads=nthreads)
        tl = time.perf_counter() - t3
        epoch = ITERS * (tg * w["s"] / sample_n + ta) + tl * w["f"] / sample_n
        if s >= warmup:
            times.append((epoch, tg + ta + tl))
    ep = float(np.median([e for e, _ in times]))
    return dict(epoch_s=ep, wall_per_step=float(np.mean([x for _, x in times])), setup_s=setup)


def reference_arm(args, ws, rank):
    if rank != 0:
        return
    name = args.config
    w = workload(name)
    subs, vals, _ = make_tensor(name, "cuda" if torch.cuda.is_available() else "cpu")
    subs_h, vals_h = subs.cpu().numpy(), vals.cpu().numpy()
    del subs, vals
    n = args.cpu_sample
    subs_h, vals_h, lo, hi, what = oracle_sample_block(w, subs_h, vals_h)
    info = cpu_info()
    nt = info["host_threads"]
    t0 = time.time()
    r = run_oracle_sample(name, subs_h, vals_h, args.steps, args.warmup, n, lo, hi, nthreads=nt)
    wall = time.time() - t0
    eps = 1.0 / r["epoch_s"]
    sample = (f"oracle (fp64, OpenMP timing variant on {nt} threads) on {what}; each timed step: 1 sampled "
              f"gradient with p'=q'={n}, 1 Adam pass over all {sum(w['dims']) * w['R']} coefficients, 1 loss "
              f"estimate with f'={n}; value = one epoch (100 iterations at p=q={w['s']:.0e}, f={w['f']:.0e}) "
              f"extrapolated from the per-sample and per-pass times of those steps")
    line = {"impl": "reference", "metric": METRIC, "value": eps, "unit": "epochs/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            # what was actually timed: one bounded sample step (the epoch is extrapolated from it)
            "ms_per_step": r["wall_per_step"] * 1e3, "extrapolated_ms_per_epoch": r["epoch_s"] * 1e3,
            "wall_s": wall, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"{name}: {w['desc']}", "parallelism": f"cpu-omp{nt}"},
            "samples_per_s": eps * ITERS * 2 * w["s"],
            "cpu_baseline": dict({"value": eps, "unit": "epochs/s", "cores": nt, "kind": "oracle", "sample": sample},
                                 **info),
            "e2e": {"value": eps, "unit": "epochs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--mode", default="sync", choices=["sync", "twosided", "async", "fedadam"])
    ap.add_argument("--tau", type=int, default=10)
    ap.add_argument("--samples", type=float, default=None,
                    help="override p = q per iteration (global), e.g. the all-reduce vs two-sided crossover sweep")
    ap.add_argument("--cpu-sample", type=int, default=100_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-hbm-gate", action="store_true")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference" or os.environ.get("GCP_BENCH_ALLOW_SHORT"), "W >= 3"

    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        reference_arm(args, ws, rank)
        return

    import paper_2605_20353_b200 as g

    name = args.config
    w = workload(name)
    if args.samples:
        w["s"] = int(args.samples)
    dev = local
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    ctx = g.Context(dev, stream.cuda_stream, args.precision)
    uid = bcast_bytes(ws, rank, g.gcp_nccl_unique_id() if (rank == 0 and ws > 1) else None)
    ctx.dist_init(ws, rank, uid, None, args.mode)
    grid, lo, hi = g.gcp_grid_plan(ws, w["dims"])

    log("generate", name)
    host_gen = False
    # a rank block beyond 1.5e9 nonzeros (c5 at 1-2 GPUs: 75-150 GB of int64 +
    # fp64 COO) does not fit the device beside its ingest: the generator hands
    # each finished partition to host memory and the ingest reads it from there
    blk_nnz = w["nnz"] / ws
    if blk_nnz > 1_500_000_000:
        import psutil
        need = blk_nnz * 1.006 * (8 * w["d"] + 8) * (ws if ws > 1 else 1) + 8e9
        avail = psutil.virtual_memory().available
        if avail < need:
            raise SystemExit(f"bench: {name} at {ws} GPU(s) needs ~{need / 1e9:.0f} GB of host memory for its COO, "
                             f"{avail / 1e9:.0f} GB available")
        host_gen = True
        args.no_e2e = True
    if ws > 1 and w["nnz"] > 1_000_000_000:
        # billion-scale: each rank generates only its block of the global tensor
        subs, vals, gen_s = make_tensor(name, f"cuda:{dev}", block=(lo[rank], hi[rank]),
                                        allreduce=lambda x: allsum_int(ws, x),
                                        out_device="cpu" if host_gen else None)
    elif host_gen:
        subs, vals, gen_s = make_tensor(name, f"cuda:{dev}", out_device="cpu")
    else:
        subs, vals, gen_s = make_tensor(name, f"cuda:{dev}")
        if ws > 1:
            subs, vals = block_of(subs, vals, lo[rank], hi[rank])
    log("generated", len(vals))
    device_ingest = args.no_e2e and w["nnz"] > 1_000_000_000 and ws > 1
    if device_ingest or host_gen:
        # billion-scale block without e2e: ingest straight from the generated
        # arrays (the ABI takes any UVA or host pointer), no pinned copy
        subs_h, vals_h = subs, vals
    else:
        subs_h = torch.empty(subs.shape, dtype=subs.dtype, pin_memory=True)
        subs_h.copy_(subs)
        vals_h = torch.empty(vals.shape, dtype=vals.dtype, pin_memory=True)
        vals_h.copy_(vals)
        log("host copy (pinned)")
    del subs, vals
    nnz_local = len(vals_h)
    torch.cuda.empty_cache()
    t0 = time.time()
    log("ingest", nnz_local)
    ctx.tensor_create_ptr(w["dims"], nnz_local, subs_h.data_ptr(), vals_h.data_ptr())
    ingest_s = time.time() - t0
    if device_ingest or host_gen:
        del subs_h, vals_h
        subs_h = vals_h = None
        torch.cuda.empty_cache()
    ctx.model_init(w["R"], gcp_synth.SEEDS[name]["model"])
    features = ctx.dist_features()
    fp = ctx.fit_params(epochs=10 ** 6, iters_per_epoch=ITERS, max_fails=10 ** 6, s_nz=w["s"], s_z=w["s"],
                        f_nz=w["f"], f_z=w["f"], loss=w["loss"], seed=gcp_synth.SEEDS[name]["sample"], fseed=2,
                        rate=1e-3, tau=args.tau if args.mode in ("async", "fedadam") else 0, meta_rate=1e-3)
    ctx.fit_begin(fp)
    log("warm-up")
    for _ in range(args.warmup):
        ctx.fit_epoch()
    c0 = ctx.counters()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier(ws)
    torch.cuda.synchronize()
    nvl0 = nvlink_counters(dev) if ws > 1 else None
    with ClockSampler(dev) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            ctx.fit_epoch()
        ev1.record(stream)
        torch.cuda.synchronize()
    nvl1 = nvlink_counters(dev) if ws > 1 else None
    barrier(ws)
    ms_local = ev0.elapsed_time(ev1)
    ms = allmax(ws, ms_local)
    c1 = ctx.counters()
    # per-kernel times from the library's CUDA events on its stream, over extra
    # (untimed) epochs so the event records do not perturb the timed region
    prof_epochs = max(1, min(args.steps, 3))
    ctx.profile_enable(True)
    for k in g.gcp.PROF:
        ctx.profile_get(k, reset=True)
    for _ in range(prof_epochs):
        ctx.fit_epoch()
    prof = {k: ctx.profile_get(k) for k in g.gcp.PROF}
    ctx.profile_enable(False)
    prof_ranks = allgather_obj(ws, {k: v[0] / prof_epochs for k, v in prof.items()})
    ms_step = ms / args.steps
    eps = 1000.0 / ms_step
    nvlink = None
    if nvl0 and nvl1:
        per = {k: (nvl1[k] - nvl0[k]) / (args.steps * ITERS) for k in ("tx", "rx")}
        nvlink = {"ranks_bytes_per_iter": allgather_obj(ws, per), "links": nvl1["links"],
                  "source": "NVML NVLink data counters (THROUGHPUT_DATA_TX/RX, KiB, summed over links) "
                            "read on each rank just before and after the timed region; per iteration = "
                            "delta / (steps x iters_per_epoch), includes the loss estimate's scalar sums",
                  "alg_bytes_per_iter_rank": exchange_alg_bytes(w, grid, args.mode, args.tau,
                                                                4 if args.precision == "fp32" else 8)}
    samples_per_s = eps * ITERS * (2 * w["s"])
    # library kernels in the timed region: launch counter delta, minus NCCL collective
    # calls (the fused NVLink exchange is a library kernel and stays counted)
    fused_sync = args.mode == "sync" and ws > 1 and os.environ.get("GCP_SYNC_EXCHANGE") in (None, "fused")
    comm_per_epoch = prof["comm"][1] // prof_epochs
    nccl_per_epoch = comm_per_epoch - (ITERS if fused_sync else 0)
    launches = int(c1["launches"] - c0["launches"]) - nccl_per_epoch * args.steps
    # ---- roofline of the dominant kernel (K2, fused sampling-MTTKRP)
    k2_ms, k2_n = prof["grad"]
    p_loc = w["s"] // ws + (1 if rank < w["s"] % ws else 0)
    alg_bytes = p_loc * w["nz_bytes"] + p_loc * w["z_bytes"]
    k2_avg_ms = allmax(ws, k2_ms / max(k2_n, 1))
    peak, peak_src = peaks()
    achieved = alg_bytes / (k2_avg_ms * 1e-3) / 1e9
    roof = roofline(w, name, alg_bytes, p_loc, k2_avg_ms, peak, peak_src, ctx.layout())
    layout = ctx.layout()
    # ---- e2e: the public API from pinned host buffers, copies inside the timed region
    A0 = [ctx.model_get(k) for k in range(w["d"])] if not args.no_e2e else None
    ctx.close()
    torch.cuda.empty_cache()
    e2e = None
    if not args.no_e2e:
        log("e2e")
        e2e = run_e2e(g, A0, w, fp, subs_h, vals_h, dev, stream, ws, rank, args)
    # ---- the HBM gate: c4 at P = 1, same process, after the headline context closed
    gate = None
    if ws == 1 and name not in ("c4", "c5") and not args.no_hbm_gate:
        log("hbm gate (c4)")
        gate = hbm_gate(g, dev, stream, args, peak, peak_src)
    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and subs_h is not None:
        log("cpu baseline")
        cpu = cpu_baseline(g, name, w, subs_h, vals_h, args)
    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": eps, "unit": "epochs/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": f"{name}: {w['desc']}", "dims": list(w["dims"]), "nnz": int(w["nnz"]),
                       "R": w["R"], "loss": w["loss"], "p": w["s"], "q": w["s"], "f_nz": w["f"], "f_z": w["f"],
                       "iters_per_epoch": ITERS, "grid": list(grid), "dist_mode": args.mode,
                       "exchange": exchange_name(ws, args.mode, features),
                       "parallelism": f"grid{'x'.join(map(str, grid))}-{args.mode}" if ws > 1 else "single-gpu",
                       "l2": ("inputs larger than L2 (COO records + hash set >> 126 MB); factors "
                              + ("stay L2-resident" if sum(w["dims"]) * w["R"] * 4 < 32e6
                                 else "and gradient far exceed L2")),
                       "nnz_local_rank0": nnz_local, "layout": layout},
            "samples_per_s": samples_per_s,
            # all ranks' K2 run concurrently: global samples per iteration / the slowest rank's K2
            "samples_per_s_k2_only": 2 * w["s"] / (k2_avg_ms * 1e-3) if k2_avg_ms else None,
            "hbm_gbs_k2_algorithmic": achieved,
            "gpu_launches": int(launches),
            "library_launches_total": int(c1["launches"] - c0["launches"]),
            "phase_ms_per_step": {k: v[0] / prof_epochs for k, v in prof.items()},
            "phase_ms_per_step_ranks": prof_ranks if ws > 1 else None,
            "phase_source": f"library CUDA events over {prof_epochs} extra untimed epochs (rank 0)",
            "roofline": roof,
            **({"nvlink": nvlink} if nvlink else {}),
            "hbm_gate": gate,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "setup_s": {"generate": gen_s, "ingest": ingest_s},
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def exchange_name(ws, mode, features):
    if ws == 1:
        return "none"
    if mode == "twosided":
        env = os.environ.get("GCP_TWOSIDED_NVL")
        if not features["fused"]:
            return "two-sided-nccl-send-recv"
        if env == "peer" or (env is None and ws <= 8):
            return "two-sided-nvlink-peer-access"
        return "two-sided-nvlink-import-export"
    if mode in ("async", "fedadam"):
        return "nccl-allreduce-every-tau"
    return "fused-nvlink-multimem" if features["multimem"] else "fused-nvlink" if features["fused"] else "nccl"


def exchange_alg_bytes(w, grid, mode, tau, esz):
    """Algorithmic NVLink bytes one rank sends per iteration in the multi-GPU
    exchange: sync (fused RS + Adam + AG over a slice group of
    g_k = P / N_k ranks) -- the peers pull (g_k - 1) / g_k of this rank's G block
    and it stores its 1/g_k shard of A into g_k - 1 peers: 2 (g_k - 1) / g_k of
    the mode's block bytes; async -- one all-reduce of the block every tau
    iterations, ~2 (g_k - 1) / g_k of it; two-sided -- data dependent (None)."""
    P = int(np.prod(grid))
    R_pad = (w["R"] + 3) // 4 * 4
    tot = 0.0
    for k, n_k in enumerate(grid):
        g = P // n_k
        rows = -(-w["dims"][k] // n_k)
        if g > 1:
            tot += 2 * (g - 1) / g * rows * R_pad * esz
    if mode == "sync":
        return tot
    if mode in ("async", "fedadam"):
        return tot / max(tau, 1)
    return None


def ncu_traffic(name, layout):
    """DRAM bytes per K2 launch from one `ncu --set full` capture of this config
    in the layout it runs (profiles/ncu_traffic_<config>.json), or None."""
    f = ROOT / "profiles" / f"ncu_traffic_{name}.json"
    if not f.exists():
        return None, None
    j = json.loads(f.read_text())
    if name in ("c4", "c5") and not (layout or {}).get("slot_order", True):
        return None, None
    return j.get("k2_dram_bytes_per_launch"), j.get("source")


def roofline(w, name, alg_bytes, p_loc, k2_ms, peak, peak_src, layout):
    """The dominant kernel K2 against the bound that applies to this config
    (SURVEY §8(d) D4): factors DRAM-resident (c4, c5) -> HBM, the measured copy
    bandwidth; factors L2-resident (c2: 1.9 MB, c3: 35 MB) -> L2, the measured
    K2 memory skeleton (the same gathers, red.add rows and random DRAM record
    reads with no sampling arithmetic, tools/membench.cu) -- there the
    algorithmic GB/s exceeds HBM because L2 serves the factor rows, so the HBM
    view is given beside it together with the ncu DRAM traffic."""
    achieved = alg_bytes / (k2_ms * 1e-3) / 1e9
    traffic, tsrc = ncu_traffic(name, layout)
    dram = None
    if traffic:
        dram = {"bytes_per_launch": traffic, "gbs": traffic / (k2_ms * 1e-3) / 1e9,
                "frac_of_hbm": traffic / (k2_ms * 1e-3) / 1e9 / peak, "source": tsrc}
    base = {"achieved": achieved, "unit": "GB/s", "traffic": traffic, "kernel": "k_sample (K2 fused sampling-MTTKRP)",
            "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": k2_ms, "dram": dram,
            "bytes_model": "SURVEY §8(d) D4: per nonzero sample (d+1)*4 + 3*d*R*4 B, per zero sample "
                           "kB/(1-rho) + 3*d*R*4 B (gather once, scatter-add read+write)"}
    l2_resident = sum(w["dims"]) * w["R"] * 4 * 2 <= 0.5 * 126e6
    if not l2_resident:
        return dict(base, bound="hbm", peak=peak, frac=achieved / peak, peak_source=peak_src)
    m = json.loads((ROOT / "profiles" / "membench_r01.json").read_text())
    if w["d"] == 3 and w["R"] * 4 == 64 and "k2_skeleton_dram_ms_per_2e7" in m:
        # skeleton = L2 gathers + red.add rows, plus one random DRAM read for the
        # samples that make one: every nonzero (its record); a zero candidate only
        # on an L2 Bloom filter "maybe" (~8% at c2's 5.4 bits per key) when the
        # filter is in front of the hash, else every zero (its bucket)
        fz = 0.08 if (layout or {}).get("filter") else 1.0
        frac_dram = (1.0 + fz) / 2.0   # p = q
        per2e7 = m["k2_skeleton_l2_ms_per_2e7"] + (m["k2_skeleton_dram_ms_per_2e7"] - m["k2_skeleton_l2_ms_per_2e7"]) * frac_dram
        sk_ms = per2e7 * 2 * p_loc / 2e7
        return dict(base, bound="l2", peak=alg_bytes / (sk_ms * 1e-3) / 1e9, frac=sk_ms / k2_ms,
                    peak_source=("measured K2 memory skeleton on this pool (profiles/membench_r01.json "
                                 "k2_skeleton_l2_ms_per_2e7 + the random DRAM read of "
                                 f"{frac_dram:.2f} of the samples from k2_skeleton_dram_ms_per_2e7, tools/membench.cu): "
                                 f"{sk_ms:.3f} ms per launch"),
                    hbm_view={"peak": peak, "frac": achieved / peak, "peak_source": peak_src,
                              "note": "algorithmic bytes over HBM copy bandwidth: > 1 because the factor rows "
                                      "and G hit in L2; dram.frac_of_hbm is the DRAM view"})
    return dict(base, bound="l2", peak=None, frac=None, peak_source="no measured L2 ceiling for this row shape",
                hbm_view={"peak": peak, "frac": achieved / peak, "peak_source": peak_src})


def d4_epoch_bytes(w):
    """SURVEY §8(d) D4 algorithmic bytes of one epoch at P = 1 (fp32, u32 indices)."""
    dense = 8 * sum(w["dims"]) * w["R"] * 4
    kB = 16 if w["M"] >= 2 ** 64 else 8
    loss = w["f"] * ((w["d"] + 1) * 4 + w["d"] * w["R"] * 4) + w["f"] * (kB / (1 - w["rho"]) + w["d"] * w["R"] * 4)
    return ITERS * (w["s"] * w["nz_bytes"] + w["s"] * w["z_bytes"] + dense) + loss


def hbm_gate(g, dev, stream, args, peak, peak_src, epochs=3, warmup=3):
    """SURVEY §8(d) D4's primary >= 60% HBM gate: c4 (Amazon-shaped, 1.74e9 nnz,
    factors and G 538 MB each, DRAM-resident) at P = 1 in this same process:
    generated and ingested on the device, `warmup` untimed epochs, `epochs`
    timed epochs (CUDA events, same protocol as the headline), then one
    profiled epoch for the per-kernel split."""
    w = workload("c4")
    t0 = time.time()
    subs, vals, gen_s = make_tensor("c4", f"cuda:{dev}")
    torch.cuda.empty_cache()   # the generator's temporaries: the ingest scratch needs the room
    ctx = g.Context(dev, stream.cuda_stream, args.precision)
    ctx.tensor_create_ptr(w["dims"], len(vals), subs.data_ptr(), vals.data_ptr())
    del subs, vals
    torch.cuda.empty_cache()
    ctx.model_init(w["R"], gcp_synth.SEEDS["c4"]["model"])
    fp = ctx.fit_params(epochs=10 ** 6, iters_per_epoch=ITERS, max_fails=10 ** 6, s_nz=w["s"], s_z=w["s"],
                        f_nz=w["f"], f_z=w["f"], loss=w["loss"], seed=gcp_synth.SEEDS["c4"]["sample"], fseed=2,
                        rate=1e-3)
    ctx.fit_begin(fp)
    setup_s = time.time() - t0
    for _ in range(warmup):
        ctx.fit_epoch()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        ev0.record(stream)
        for _ in range(epochs):
            ctx.fit_epoch()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / epochs
    ctx.profile_enable(True)
    for k in g.gcp.PROF:
        ctx.profile_get(k, reset=True)
    ctx.fit_epoch()
    prof = {k: ctx.profile_get(k) for k in g.gcp.PROF}
    ctx.profile_enable(False)
    layout = ctx.layout()
    ctx.close()
    torch.cuda.empty_cache()
    k2_ms = prof["grad"][0] / max(prof["grad"][1], 1)
    adam_ms = prof["adam"][0] / max(prof["adam"][1], 1)
    alg = w["s"] * w["nz_bytes"] + w["s"] * w["z_bytes"]
    adam_bytes = 8 * sum(w["dims"]) * w["R"] * 4
    floor_ms = d4_epoch_bytes(w) / (peak * 1e9) * 1e3
    return {"config": f"c4: {w['desc']}", "n_gpus": 1, "epochs_per_s": 1000.0 / ms, "ms_per_epoch": ms,
            "timed_epochs": epochs, "warmup_epochs": warmup, "layout": layout,
            "d4_floor_ms_per_epoch": floor_ms, "frac_of_d4_floor": floor_ms / ms,
            "note": "frac_of_d4_floor = SURVEY D4 epoch bytes at the measured HBM peak / measured epoch time "
                    "(the >= 60% gate); K2 and Adam split from one profiled epoch",
            "roofline": roofline(w, "c4", alg, w["s"], k2_ms, peak, peak_src, layout),
            "adam": {"avg_launch_ms": adam_ms, "alg_bytes_per_launch": adam_bytes,
                     "gbs": adam_bytes / (adam_ms * 1e-3) / 1e9, "frac": adam_bytes / (adam_ms * 1e-3) / 1e9 / peak},
            "phase_ms_per_epoch": {k: v[0] for k, v in prof.items()},
            "samples_per_s": 2 * w["s"] * ITERS * 1000.0 / ms, "setup_s": {"generate": gen_s, "total": setup_s},
            "clocks": clk.summary()}


def oracle_sample_block(w, subs, vals):
    """Whole tensor, or beyond 2e8 nonzeros the rank-0 block of the oracle's own
    64-way grid plan (same density; the oracle's sort stays small)."""
    if w["nnz"] <= 200_000_000:
        return subs, vals, None, None, "the full tensor"
    import oracle
    grid, _ = oracle.grid_plan(64, w["dims"])
    lo, hi = oracle.block_bounds(w["dims"], grid, 0)
    m = np.ones(len(vals), bool)
    for k in range(w["d"]):
        m &= (subs[:, k] >= lo[k]) & (subs[:, k] < hi[k])
    return subs[m], vals[m], lo, hi, f"the rank-0 block of a 64-way grid ({int(m.sum())} nnz, {lo}-{hi})"


def cpu_baseline(g, name, w, subs_h, vals_h, args):
    """The oracle, as it stands, on a bounded sample of this workload, timed two
    ways: its OpenMP timing variant on every host thread this
    process may use (value, cores) and the single-threaded parity oracle.
    Tensors beyond 2e8 nonzeros are sampled as the rank-0 block of a 64-way grid
    (same density, per-rank sample arithmetic) so the oracle's own sort stays small."""
    subs, vals, lo, hi, what = oracle_sample_block(w, subs_h.numpy(), vals_h.numpy())
    info = cpu_info()
    nt = info["host_threads"]
    n_par = args.cpu_sample * max(1, min(nt, 16))
    rp = run_oracle_sample(name, subs, vals, 2, 1, n_par, lo, hi, nthreads=nt)
    r1 = run_oracle_sample(name, subs, vals, 2, 1, args.cpu_sample, lo, hi)
    return dict({"value": 1.0 / rp["epoch_s"], "unit": "epochs/s", "cores": nt, "kind": "oracle",
                 "sample": (f"on {what}: 1 sampled gradient (p'=q'={n_par}) + 1 Adam pass + 1 loss estimate "
                            f"(f'={n_par}) per step, median of 2 steps after 1 warm-up, extrapolated to one epoch "
                            f"of 100 iterations at p=q={w['s']:.0e}; fp64 C oracle, OpenMP timing variant on {nt} "
                            f"threads (thread-private G reduced in fixed order)"),
                 "single_thread": {"value": 1.0 / r1["epoch_s"], "cores": 1,
                                   "sample": f"the parity oracle itself at p'=q'=f'={args.cpu_sample}"},
                 "oracle_setup_s": rp["setup_s"]}, **info)


def run_e2e(g, A0, w, fp, subs_h, vals_h, dev, stream, ws, rank, args):
    """Per step, the job a user runs through the public API on a long-lived
    context (created, and for N > 1 its NCCL communicators initialised, once
    before the timed steps, as a serving process would): ingest this step's COO
    from pinned host memory (H2D; replaces the previous tensor), upload the
    initial factors (H2D), fit_begin (F0) + one epoch, read back the factors
    and the loss (D2H).  Wall time per step, max over ranks."""
    h2d = subs_h.numel() * 8 + vals_h.numel() * 8 + sum(a.size * 8 for a in A0)
    d2h = sum(a.size * 8 for a in A0) + 8
    steps = max(1, min(args.steps, 3))
    times, phases = [], []
    uid = bcast_bytes(ws, rank, g.gcp_nccl_unique_id() if (rank == 0 and ws > 1) else None)
    t_create = time.perf_counter()
    ctx = g.Context(dev, stream.cuda_stream, args.precision)
    ctx.dist_init(ws, rank, uid, None, args.mode)
    t_create = time.perf_counter() - t_create
    for s in range(steps + 1):
        barrier(ws)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        marks = {}
        ctx.tensor_create_ptr(w["dims"], vals_h.numel(), subs_h.data_ptr(), vals_h.data_ptr())
        marks["h2d_ingest"] = time.perf_counter()
        ctx.model_init(w["R"], 0)
        for k in range(w["d"]):
            ctx.model_set(k, A0[k])
        ctx.fit_begin(fp)
        marks["model_F0"] = time.perf_counter()
        ctx.fit_epoch()
        marks["epoch"] = time.perf_counter()
        _ = [ctx.model_get(k) for k in range(w["d"])]
        torch.cuda.synchronize()
        marks["d2h"] = time.perf_counter()
        dt = allmax(ws, time.perf_counter() - t0)
        if s > 0:
            times.append(dt)
            prev, ph = t0, {}
            for kname, tv in marks.items():
                ph[kname] = (tv - prev) * 1e3
                prev = tv
            phases.append(ph)
    ctx.close()
    t = float(np.median(times))
    return {"value": 1.0 / t, "unit": "epochs/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": t * 1e3, "steps": steps,
            "phase_ms_rank0": {k: float(np.median([p[k] for p in phases])) for k in phases[0]},
            "context_create_ms_untimed": t_create * 1e3,
            "includes": "H2D COO + ingest (sort, dup check, hash) + H2D factors + F0 estimate + 1 epoch + "
                        "D2H factors/loss, on a context created (NCCL initialised) once before the steps"}


if __name__ == "__main__":
    main()
