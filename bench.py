#!/usr/bin/env python
"""Benchmark: Helmholtz RHS solved per second to relative residual 1e-6 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): 257x257 nodes (external 256^2),
4 seeded smooth-random slowness models x 32 point-source RHS, 3-level V-cycle
(damped Jacobi 0.8/0.8) + the 3-level 16/32/64 encoder-solver CNN with seeded
weights, FGMRES(10) to 1e-6 (max 2000 iterations).  One "step" = one batched
solve of all 128 RHS.  Synthetic seeded data (no datasets are available).

Arms
  default           the B200 path (libhelmsolve_b200.so), N GPUs via torchrun,
                    one independent C2 instance per rank (weak scaling), no
                    collective on the data path; NCCL only for the max-over-ranks
                    timing and the result gather.
  --impl reference  the reference's CPU algorithm (the numpy oracle port of
                    helmsolve; the reference is pure Python) on the host cores,
                    rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Helmholtz RHS solved/sec to rel-res 1e-6"
UNIT = "RHS/s"
# Mean FGMRES iterations per RHS of the C2 learned workload (seed offset 0),
# measured by the B200 arm and matched by the oracle within +-1 (parity tests).
# Used only to extrapolate the CPU arm's bounded sample to whole solves.
C2_MEAN_ITERS = {"learned": 123.1, "vcycle": 113.2}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_traffic():
    """DRAM bytes of one captured launch of the roofline kernel (ncu --set full, profiles/)."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "roofline_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return False
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)
        return False

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if "Active" in r[4 + i] and "Not" not in r[4 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def cpu_leg(args, learned: bool, steps: int, warmup: int):
    """Oracle port on the host cores: (value RHS/s per step list, description)."""
    from oracle import cpu_bench

    workers = args.cpu_workers or (os.cpu_count() or 1)
    vals = []
    t_v = t_l = 0.0
    for s in range(warmup + steps):
        t_v, t_l = cpu_bench.sample(args.config, learned, workers, args.cpu_iters, args.rhs_per_model)
        if s >= warmup:
            mean_iters = C2_MEAN_ITERS["learned" if learned else "vcycle"]
            vals.append(cpu_bench.rhs_per_second(t_v, t_l, workers, mean_iters, learned))
    desc = (f"{workers} processes x 1 RHS each, {args.cpu_iters} FGMRES iterations per phase "
            f"(V-cycle {t_v * 1e3:.1f} ms/it, net+V-cycle {t_l * 1e3:.1f} ms/it), extrapolated to "
            f"{C2_MEAN_ITERS['learned' if learned else 'vcycle']:.0f} iterations per RHS; numpy oracle port")
    return vals, workers, desc


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    learned = args.precond == "learned"
    t0 = time.perf_counter()
    vals, workers, desc = cpu_leg(args, learned, args.steps, args.warmup)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * (time.perf_counter() - t0) / (args.steps + args.warmup),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128/f64 (numpy oracle)",
        "data": "synthetic", "config": workload_config(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args):
    return {"workload": f"{args.config}: 4 models x {args.rhs_per_model} RHS, 257x257, "
                        f"{'MG3 + CNN 16/32/64' if args.precond == 'learned' else 'MG3 only'}, FGMRES(10), tol 1e-6",
            "global_batch_per_gpu": 4 * args.rhs_per_model, "precond": args.precond,
            "l2": "working set (Krylov basis ~1.4 GB/GPU) far larger than L2; no flush needed",
            "parallelism": f"rhs-sharded dp (independent instance per rank)"}


DG_METRIC = "training pairs (r, e) generated/sec (257x257, k ~ U{2..20} V-cycle FGMRES iterations)"
DG_UNIT = "pairs/s"


def datagen_models(rank: int = 0):
    """C2's four seeded slowness models with the training attenuation gamma0 = 0.05 (SPEC datagen)."""
    from paper_2306_17486_b200 import datagen, fields, problems

    cfg = problems.make_config("C2", rhs_per_model=1, seed_offset=rank)
    return [fields.slowness_model(m.kappa_sq, gamma0=datagen.TRAINING_GAMMA0, layer_width=20) for m in cfg.models]


def datagen_cpu(args, workers: int, per_worker: int = 1):
    """Oracle datagen on the host cores: pairs/s (one process per core, per_worker pairs each)."""
    from multiprocessing import get_context

    t0 = time.perf_counter()
    with get_context("fork").Pool(workers) as pool:
        ks = pool.map(_dg_worker, [(i, per_worker) for i in range(workers)])
    el = time.perf_counter() - t0
    n = workers * per_worker
    return n / el, (f"{workers} processes x {per_worker} pair(s) of the same draws (mean k "
                    f"{np.mean(sum(ks, [])):.1f}), numpy oracle (oracle/datagen_oracle.py)")


def _dg_worker(a):
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    from oracle import datagen_oracle as dg
    from oracle import helm_oracle as ho

    index, count = a
    models = [ho.Model(m.kappa_sq, m.gamma, m.omega, m.h) for m in datagen_models()]
    rng = np.random.default_rng(1000 + index)
    ks = []
    for j in range(count):
        m = models[(index + j) % len(models)]
        _, _, k = dg.generate_sample(m, rng)
        ks.append(k)
    return ks


def run_datagen(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    cfg = {"workload": f"datagen: {args.samples} pairs per step over C2's 4 models (gamma0 0.05), 257x257, "
                       f"x ~ CN(0,1), k ~ U{{2..20}} FGMRES(10)+V-cycle(MG3) iterations, r = A e",
           "global_batch_per_gpu": args.samples, "parallelism": "sample-sharded dp (independent per rank)",
           "l2": "per-step working set (x, b, e, r, Krylov bases: ~1.7 GB) far larger than L2"}
    workers = args.cpu_workers or (os.cpu_count() or 1)
    if args.impl == "reference":
        if rank != 0:
            return 0
        t0 = time.perf_counter()
        vals = [datagen_cpu(args, workers)[0] for _ in range(args.warmup + args.steps)][args.warmup:]
        value = float(np.mean(vals))
        desc = datagen_cpu(args, workers)[1]
        print(json.dumps({
            "impl": "reference", "metric": DG_METRIC, "value": value, "unit": DG_UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * (time.perf_counter() - t0) / (args.steps + args.warmup + 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128/f64 (numpy oracle)",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": DG_UNIT, "cores": workers, "kind": "port", "sample": desc},
            "e2e": {"value": value, "unit": DG_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)
        return 0

    import torch

    world, rank, local = dist_setup()
    from paper_2306_17486_b200 import _lib, datagen
    from paper_2306_17486_b200 import dist as hdist

    models = datagen_models(rank)
    gen = datagen.PairGenerator(models)
    shape = models[0].shape
    rng = np.random.default_rng(2024 + rank)

    def draw_batch():
        d = [datagen._draw(rng, shape) for _ in range(args.samples)]
        return np.stack([t[0] for t in d]), [t[1] for t in d], [i % len(models) for i in range(args.samples)]

    batches = [draw_batch() for _ in range(args.warmup + args.steps)]
    xdev = [torch.from_numpy(b[0]).cuda() for b in batches]
    lib = _lib.load()
    for i in range(args.warmup):
        gen.pairs(xdev[i], batches[i][1], batches[i][2], return_device=True)
    tags = [_lib.PROF_VCYCLE, _lib.PROF_ARNOLDI, _lib.PROF_VC_UP0]
    lib.hs_profile_reset()
    lib.hs_profile_enable(sum(1 << t for t in tags))
    stream = torch.cuda.current_stream()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.warmup, args.warmup + args.steps):
            gen.pairs(xdev[i], batches[i][1], batches[i][2], return_device=True)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = hdist.reduce_scalar(ev0.elapsed_time(ev1), "max")
    launches = int(lib.hs_launch_count())
    prof = {t: _lib.profile_query(t) for t in tags}
    lib.hs_profile_enable(0)
    value = world * args.samples * args.steps / (ms / 1e3)
    # e2e: host x (pinned) in, host (r, e) out, every step
    e2e = None
    if not args.no_e2e:
        xpin = [torch.from_numpy(batches[i][0]).pin_memory() for i in range(args.warmup, args.warmup + args.steps)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for j, i in enumerate(range(args.warmup, args.warmup + args.steps)):
            r, e = gen.pairs(xpin[j], batches[i][1], batches[i][2])
        el = hdist.reduce_scalar(time.perf_counter() - t0, "max")
        e2e = {"value": world * args.samples * args.steps / el, "unit": DG_UNIT,
               "h2d_bytes_per_step": int(xpin[0].numel() * 16), "d2h_bytes_per_step": int(r.nbytes + e.nbytes)}
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0
    hbm, _, src = load_peaks()
    u_ms, u_bytes, u_n = prof[_lib.PROF_VC_UP0]
    ach = u_bytes / (u_ms / 1e3) / 1e9 if u_ms > 0 else 0.0
    roof = {"kernel": "k_vc_up (finest level)", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
            "frac": ach / hbm, "peak_note": f"{src} copy bandwidth", "launches": u_n, "ms_total": u_ms, "traffic": None}
    cpu = None
    if world == 1 and not args.no_cpu:
        v, desc = datagen_cpu(args, workers)
        cpu = {"value": v, "unit": DG_UNIT, "cores": workers, "kind": "port", "sample": desc}
    print(json.dumps({
        "metric": DG_METRIC, "value": value, "unit": DG_UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c64 basis/V-cycle, fp64 operator+reductions, c128 iterate",
        "data": "synthetic (seeded)", "config": cfg, "mean_k": float(np.mean(sum((b[1] for b in batches), []))),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary()}),
        flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


TR_METRIC = "network training samples/sec (257x257, C2 network 16/32/64, batch 16: forward + MSE + backward + Adam)"
TR_UNIT = "samples/s"
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # derived: SMs x FP32 FMA/clk x 2 x max SM clock


def train_cpu(workers: int):
    """Oracle training step (float64 numpy) on the host cores: samples/s, one process per core, batch 1 each."""
    from multiprocessing import get_context

    t0 = time.perf_counter()
    with get_context("fork").Pool(workers) as pool:
        pool.map(_tr_worker, range(workers))
    el = time.perf_counter() - t0
    return workers / el, (f"{workers} processes x 1 sample (a batch-1 step each: forward with training batch norm, "
                          f"MSE, backward, Adam), 257x257, numpy oracle (oracle/train_oracle.py), single-threaded BLAS")


def _tr_worker(i):
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    from oracle import train_oracle as to
    from paper_2306_17486_b200 import netparams
    from paper_2306_17486_b200 import train as tr

    models = datagen_models()
    rng = np.random.default_rng(500 + i)
    n = models[0].shape
    params = to.as_float64(netparams.init_params((16, 32, 64), 0))
    media = tr.media_planes(models, 3)[[i % 4]].astype(np.float64)
    r = rng.standard_normal((1,) + n) + 1j * rng.standard_normal((1,) + n)
    e = rng.standard_normal((1,) + n) + 1j * rng.standard_normal((1,) + n)
    to.train_step(params, 3, media, r, e, models[0].h, to.Adam(params))
    return 0


def run_train(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    B = args.train_batch
    cfg = {"workload": f"train: C2's 4 models (gamma0 0.05), 257x257 grid, network 16/32/64 (3 levels, implicit "
                       f"layer at 64x64), batch {B} datagen pairs (r, e) per step, training-mode batch norm, "
                       f"MSE of u0 = (h^2/64) net(r) vs e, backward, Adam lr 1e-3",
           "global_batch_per_gpu": B, "parallelism": "data-parallel: batch B per rank, one NCCL all-reduce of the "
                                                      "flat fp32 gradient vector per step (train.Trainer.step)",
           "l2": "per-step working set (saved activations ~1.3 GB) far larger than L2"}
    workers = args.cpu_workers or (os.cpu_count() or 1)
    if args.impl == "reference":
        if rank != 0:
            return 0
        t0 = time.perf_counter()
        vals = [train_cpu(workers)[0] for _ in range(args.warmup + args.steps)][args.warmup:]
        value = float(np.mean(vals))
        desc = train_cpu(workers)[1]
        print(json.dumps({
            "impl": "reference", "metric": TR_METRIC, "value": value, "unit": TR_UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * (time.perf_counter() - t0) / (args.steps + args.warmup + 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (numpy oracle)",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": TR_UNIT, "cores": workers, "kind": "port", "sample": desc},
            "e2e": {"value": value, "unit": TR_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)
        return 0

    import torch

    world, rank, local = dist_setup()
    from paper_2306_17486_b200 import _lib, datagen, network
    from paper_2306_17486_b200 import dist as hdist
    from paper_2306_17486_b200 import train as tr

    models = datagen_models(rank)
    gen = datagen.PairGenerator(models)
    n = models[0].shape
    rng = np.random.default_rng(77 + rank)
    pool = 4 * B
    d = [datagen._draw(rng, n) for _ in range(pool)]
    owner = np.arange(pool) % len(models)
    r, e = gen.pairs(np.stack([t[0] for t in d]), [t[1] for t in d], owner, return_device=True)
    media = torch.from_numpy(tr.media_planes(models, 3)).cuda()
    net = network.EncoderSolverNet.seeded((16, 32, 64), seed=0)
    trainer = tr.Trainer(net, n, models[0].h, B, lr=1e-3)
    batches = [np.arange(s * B, (s + 1) * B) % pool for s in range(args.warmup + args.steps)]
    bsel = [torch.from_numpy(b).cuda() for b in batches]
    rb = [r.index_select(0, b).contiguous() for b in bsel]
    eb = [e.index_select(0, b).contiguous() for b in bsel]
    for i in range(args.warmup):
        trainer.step(media, rb[i], eb[i], owner[batches[i]])
    lib = _lib.load()
    tags = [_lib.PROF_CONV, _lib.PROF_TRAIN_WGRAD]
    lib.hs_profile_reset()
    stream = torch.cuda.current_stream()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    losses = []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.warmup, args.warmup + args.steps):
            losses.append(trainer.step(media, rb[i], eb[i], owner[batches[i]]))
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = hdist.reduce_scalar(ev0.elapsed_time(ev1), "max")
    launches = int(lib.hs_launch_count())
    value = world * B * args.steps / (ms / 1e3)
    # kernel shares, separate profiled pass (CUDA events around each tagged launch)
    lib.hs_profile_enable(sum(1 << t for t in tags))
    lib.hs_profile_reset()
    for i in range(args.warmup, args.warmup + args.steps):
        trainer.step(media, rb[i], eb[i], owner[batches[i]])
    torch.cuda.synchronize()
    prof = {t: _lib.profile_query(t) for t in tags}
    lib.hs_profile_enable(0)
    e2e = None
    if not args.no_e2e:
        rpin = [rb[i].cpu().pin_memory() for i in range(args.warmup, args.warmup + args.steps)]
        epin = [eb[i].cpu().pin_memory() for i in range(args.warmup, args.warmup + args.steps)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for j, i in enumerate(range(args.warmup, args.warmup + args.steps)):
            trainer.step(media, rpin[j], epin[j], owner[batches[i]])
        el = hdist.reduce_scalar(time.perf_counter() - t0, "max")
        e2e = {"value": world * B * args.steps / el, "unit": TR_UNIT,
               "h2d_bytes_per_step": int(rpin[0].numel() * 16 * 2), "d2h_bytes_per_step": 8}
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0
    w_ms, w_flops, w_n = prof[_lib.PROF_TRAIN_WGRAD]
    c_ms, c_flops, c_n = prof[_lib.PROF_CONV]
    ach = w_flops / (w_ms / 1e3) / 1e12 if w_ms > 0 else 0.0
    roof = {"kernel": "k_tr_wgrad (+ its partial sums): weight gradients, the largest share of the step",
            "bound": "fp32-simt", "achieved": ach, "peak": FP32_SIMT_TFLOPS, "unit": "TFLOP/s",
            "frac": ach / FP32_SIMT_TFLOPS, "peak_note": "derived 148 SM x 128 FMA/clk x 2 x 1.965 GHz (no tensor cores)",
            "launches": w_n, "ms_total": w_ms, "share_of_step": w_ms / ms,
            "conv_ms_total": c_ms, "conv_tflops": c_flops / (c_ms / 1e3) / 1e12 if c_ms > 0 else 0.0,
            "traffic": None}
    cpu = None
    if world == 1 and not args.no_cpu:
        v, desc = train_cpu(workers)
        cpu = {"value": v, "unit": TR_UNIT, "cores": workers, "kind": "port", "sample": desc}
    print(json.dumps({
        "metric": TR_METRIC, "value": value, "unit": TR_UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32 (tcgen05 convs: exact bf16x3 split, fp32 accumulate)",
        "data": "synthetic (seeded datagen pairs, seeded init)", "config": cfg,
        "loss_first_last": [losses[0], losses[-1]], "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clk.summary()}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--precond", default="learned", choices=["learned", "vcycle"])
    ap.add_argument("--rhs-per-model", type=int, default=32)
    ap.add_argument("--cpu-workers", type=int, default=0, help="0 = all host cores")
    ap.add_argument("--cpu-iters", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workload", default="solve", choices=["solve", "datagen", "train"],
                    help="solve: the BASELINE metric (default); datagen: SURVEY 8f row 1, training pairs; "
                         "train: SURVEY 8f row 2, network training steps")
    ap.add_argument("--train-batch", type=int, default=16, help="train: samples per step")
    ap.add_argument("--samples", type=int, default=256, help="datagen: samples per step")
    args = ap.parse_args()
    if args.workload == "datagen":
        return run_datagen(args)
    if args.workload == "train":
        return run_train(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch

    world, rank, local = dist_setup()
    from paper_2306_17486_b200 import _lib, krylov, network, problems
    from paper_2306_17486_b200 import dist as hdist
    from paper_2306_17486_b200.device import to_device

    learned = args.precond == "learned"
    cfg = problems.make_config(args.config, rhs_per_model=args.rhs_per_model, seed_offset=rank)
    net = network.EncoderSolverNet.seeded(cfg.cnn_channels, seed=0) if learned else None
    t_setup = time.perf_counter()
    solver = krylov.BatchSolver(cfg.models, net, jacobi_damping=cfg.jacobi_damping, num_levels=cfg.mg_levels)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    B = cfg.rhs.shape[0]
    rhs_dev = to_device(cfg.rhs, torch.complex128)
    owner = cfg.model_of_rhs
    solve_kw = dict(model_of=owner, tol=cfg.tol, max_iter=cfg.max_iter, restart=cfg.restart, return_device=True)
    lib = _lib.load()

    for _ in range(args.warmup):
        _, reps = solver.solve(rhs_dev, **solve_kw)
    iters = np.array([r.iterations for r in reps], dtype=np.float64)
    conv = all(r.converged for r in reps)
    log(f"[rank {rank}] setup {t_setup:.2f}s, iterations mean {iters.mean():.1f} [{iters.min():.0f}..{iters.max():.0f}], "
        f"converged {conv}")

    # ---------------- timed region: device-resident inputs
    tags = [_lib.PROF_CONV, _lib.PROF_CONV_L0, _lib.PROF_VCYCLE, _lib.PROF_ARNOLDI, _lib.PROF_CNN,
            _lib.PROF_IMPLICIT, _lib.PROF_VC_UP0]
    lib.hs_profile_reset()
    lib.hs_profile_enable(sum(1 << t for t in tags))
    stream = torch.cuda.current_stream()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    total_iters = 0
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            _, reps = solver.solve(rhs_dev, **solve_kw)
            total_iters += sum(r.iterations for r in reps)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = int(lib.hs_launch_count())
    prof = {t: _lib.profile_query(t) for t in tags}
    lib.hs_profile_enable(0)
    ms = hdist.reduce_scalar(ms, "max")  # max over ranks
    total_iters = int(hdist.reduce_scalar(total_iters, "sum"))
    value = world * B * args.steps / (ms / 1e3)
    applies = total_iters / (ms / 1e3)

    # ---------------- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        rhs_pinned = torch.from_numpy(np.ascontiguousarray(cfg.rhs)).pin_memory()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(args.steps):
            x, reps = solver.solve(rhs_pinned, model_of=owner, tol=cfg.tol, max_iter=cfg.max_iter,
                                   restart=cfg.restart, return_device=False)
            d2h = x.nbytes + sum(8 * len(r.relative_residual_history) for r in reps)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        el = hdist.reduce_scalar(el, "max")
        e2e = {"value": world * B * args.steps / el, "unit": UNIT, "h2d_bytes_per_step": int(rhs_pinned.numel() * 16),
               "d2h_bytes_per_step": int(d2h)}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0

    hbm, bf16, src = load_peaks()
    # dominant kernel class: the network's convolutions (learned) or the finest V-cycle up-leg (MG only)
    if learned:
        # k_conv_tc<16,16,0>: the level-0 16->16 3x3 conv (8 of the 16 network convs per application run at
        # level 0 and 4 of them are this kernel).  Arithmetic intensity 4608 flop per output pixel over
        # 128-192 B (input + output, + residual for the second conv of a residual block) = 24-36 flop/B is
        # far below the ridge (1621 TFLOP/s / 6.5 TB/s = 250), so its roof is HBM.  The library's CONV_L0
        # tag accumulates exactly those algorithmic bytes per launch (times the active RHS).
        c_ms, c_bytes, c_n = prof[_lib.PROF_CONV_L0]
        achieved = c_bytes / (c_ms / 1e3) / 1e9 if c_ms > 0 else 0.0
        traffic = load_traffic()
        roof = {"kernel": "k_conv_tc<16,16,0> (tcgen05 BF16x3 implicit-GEMM 3x3 conv, level 0)", "bound": "hbm",
                "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "peak_note": f"{src} copy bandwidth", "launches": c_n, "ms_total": c_ms,
                "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                "traffic_note": traffic.get("note") if traffic else None}
    else:
        u_ms, u_bytes, u_n = prof[_lib.PROF_VC_UP0]
        achieved = u_bytes / (u_ms / 1e3) / 1e9 if u_ms > 0 else 0.0
        roof = {"kernel": "k_vc_up (finest level)", "bound": "hbm", "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "frac": achieved / hbm, "peak_note": f"{src} copy bandwidth", "launches": u_n,
                "ms_total": u_ms, "traffic": None}
    breakdown = {}
    names = {_lib.PROF_CONV: "convs", _lib.PROF_CONV_L0: "convs_l0_16ch", _lib.PROF_VCYCLE: "vcycle",
             _lib.PROF_ARNOLDI: "arnoldi_dot", _lib.PROF_CNN: "cnn_forward", _lib.PROF_IMPLICIT: "implicit_layer",
             _lib.PROF_VC_UP0: "vc_up_l0"}
    for t, (tms, work, n) in prof.items():
        breakdown[names[t]] = {"ms": round(tms, 3), "share": round(tms / ms, 4) if ms else None, "launches": n}
    for t, unit, scale in ((_lib.PROF_VCYCLE, "GB/s", 1e9), (_lib.PROF_ARNOLDI, "GB/s", 1e9),
                           (_lib.PROF_VC_UP0, "GB/s", 1e9), (_lib.PROF_CONV_L0, "GB/s", 1e9)):
        tms, work, n = prof[t]
        if tms > 0:
            breakdown[names[t]]["achieved"] = round(work / (tms / 1e3) / scale, 2)
            breakdown[names[t]]["unit"] = unit

    cpu = None
    if world == 1 and not args.no_cpu:
        vals, workers, desc = cpu_leg(args, learned, 1, 0)
        cpu = {"value": vals[0], "unit": UNIT, "cores": workers, "kind": "port", "sample": desc}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c64 basis/fp32 CNN, fp64 operator+reductions, c128 iterate",
        "data": "synthetic (seeded generators; random-init seeded network)", "config": workload_config(args),
        "precond_applies_per_s": applies, "iterations_per_rhs": float(iters.mean()),
        "converged": conv, "setup_s": t_setup,
        "roofline": roof, "breakdown": breakdown, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
