#!/usr/bin/env python
"""Benchmark: Helmholtz RHS solved per second to relative residual 1e-6 (BASELINE.json metric).

Headline workload (BASELINE.json configs[2], "C3", the largest single-GPU configuration; C4/C5
are specified across 8 GPUs): a 513x1025 grid (external 512x1024) with the layered-plus-10%-
smoothed-noise slowness, omega for 10 points per wavelength, absorbing layer 32, 64 right-hand
sides (32 point sources + 32 seeded complex Gaussians), FGMRES(20) to 1e-6 (max 2000 iterations),
preconditioned by the 4-level V(1,1)-cycle (Jacobi 0.8/0.8) with the encoder-solver CNN
(4 levels, 16/32/64/128 channels, seeded weights) as its initial guess -- the reference's
solve_with_learned_preconditioner protocol (krylov.py:180-246).  BASELINE runs C3 twice; the
multigrid-only run (solve_helmholtz, krylov.py:156-177) is reported in the same line under
``mg_only``.  One "step" = one batched solve of all the RHS.  Synthetic seeded data.

Arms
  default           the B200 path (libhelmsolve_b200.so).  With --gpus N > 1 (and no torchrun
                    environment) the script re-launches itself under torch.distributed.run with
                    one rank per GPU; each rank solves its contiguous share of the SAME 64 RHS
                    (dist.shard_range, strong scaling), NCCL only for the max-over-ranks timing
                    and the all-gather of the per-RHS reports (dist.sharded_solve).
  --impl reference  the reference's CPU algorithm (the numpy oracle port of helmsolve; the
                    reference is pure Python) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Helmholtz RHS solved/sec to rel-res 1e-6"
UNIT = "RHS/s"


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


CFG_TEXT = {
    "C1": "129x129, 1 smooth-random model x 4 point sources, MG 3 levels, CNN 16/32/64, FGMRES(10)",
    "C2": "257x257, 4 smooth-random models x 32 point sources, MG 3 levels, CNN 16/32/64, FGMRES(10)",
    "C3": "513x1025, layered+10% noise model, 64 RHS (32 point + 32 complex Gaussian), MG 4 levels, "
          "CNN 16/32/64/128 (implicit layer at 64x128), FGMRES(20)",
    "C4": "1025x2049, smooth-random model, 128 point sources, MG 4 levels, CNN 16/32/64/128, FGMRES(20)",
    "C5": "2049x4097, salt model, 256 point sources, MG 5 levels, CNN 16/32/64/128/128 (implicit at 128x256), "
          "FGMRES(30)",
}


def workload_config(args, cfg=None, world=1):
    """The config the line was measured on, derived from the ProblemSet itself (not hard-coded)."""
    from paper_2306_17486_b200 import dist as hdist

    if cfg is None:
        from paper_2306_17486_b200 import problems

        cfg = problems.make_config(args.config)
    B = cfg.rhs.shape[0]
    nx, ny = cfg.shape
    learned = args.precond == "learned"
    return {
        "workload": f"{args.config} ({CFG_TEXT.get(args.config, '')}); headline precond: "
                    f"{'MG + CNN (learned protocol)' if learned else 'MG only'}; tol {cfg.tol:g}",
        "grid": f"{nx}x{ny}", "models": len(cfg.models), "rhs_total": B,
        "rhs_per_gpu": [len(range(*hdist.shard_range(B, world, r))) for r in range(world)],
        "mg_levels": cfg.mg_levels, "jacobi_damping": list(cfg.jacobi_damping),
        "cnn_channels": list(cfg.cnn_channels) if learned else None, "restart": cfg.restart,
        "max_iter": cfg.max_iter, "precond": args.precond,
        "l2": "working set far larger than the 126 MB L2 (C3 Krylov bases 64 x 41 x 525k x 8 B = 11 GB); "
              "no flush needed",
        "parallelism": f"RHS-sharded across {world} GPU(s) (dist.shard_range), no data-path collective",
    }


def cpu_arm_value(arm, learned, iters, warm, config):
    """One bounded CPU sample -> (RHS/s extrapolated with the REFERENCE's own iteration count, description)."""
    from oracle import cpu_bench

    t_v, t_l = arm.sample(iters, warm)
    mean_iters, n_ref = cpu_bench.reference_iterations(config, learned)
    if mean_iters is None:
        raise RuntimeError(f"no reference iteration count for {config} (tests/golden/configs_*.npz)")
    v = cpu_bench.rhs_per_second(t_v, t_l, arm.workers, mean_iters, learned, warm)
    desc = (f"{arm.workers} single-threaded processes x 1 RHS of {config}: "
            + (f"{warm} V-cycle-only warm-up iterations ({t_v * 1e3:.0f} ms/it) + {iters} net+V-cycle iterations "
               f"({t_l * 1e3:.0f} ms/it)" if learned else f"{iters} V-cycle iterations ({t_v * 1e3:.0f} ms/it)")
            + f", extrapolated to {mean_iters:.1f} iterations per RHS = the reference's own mean over {n_ref} "
              f"full C3 solves (tests/golden/configs_{config.lower()}.npz); numpy oracle port")
    return v, desc


def run_reference(args):
    """--impl reference: the oracle port on the host cores, rank 0 only, bounded steps."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import cpu_bench

    learned = args.precond == "learned"
    workers = args.cpu_workers or (os.cpu_count() or 1)
    arm = cpu_bench.CpuArm(args.config, learned, workers)
    t0 = time.perf_counter()
    for _ in range(args.warmup):  # untimed: pool set-up (oracle hierarchy, encodings) + one V-cycle iteration
        arm.sample(0, 1)
    t1 = time.perf_counter()
    vals = []
    desc = ""
    for _ in range(args.steps):
        v, desc = cpu_arm_value(arm, learned, 1, 3 if learned else 0, args.config) if learned else \
            cpu_arm_value(arm, learned, 4, 0, args.config)
        vals.append(v)
    arm.close()
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * (time.perf_counter() - t1) / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128/f64 (numpy oracle)",
        "data": "synthetic", "config": workload_config(args, world=1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": "each step: " + desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": t1 - t0,
    }
    print(json.dumps(line), flush=True)
    return 0


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


def free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(args) -> int:
    """--gpus N without a torchrun environment: run this script under torch.distributed.run, N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    log("relaunching under torchrun: " + " ".join(cmd))
    return subprocess.call(cmd)


# profiling tags: name, work unit ("bytes" -> GB/s, "flops" -> TFLOP/s)
PROFILE_TAGS = (("convs", "CONV", "flops"), ("convs_l0_16ch", "CONV_L0", "bytes"), ("convs_wide", "CONV_WIDE", "flops"),
                ("vcycle", "VCYCLE", "bytes"), ("arnoldi_dot", "ARNOLDI", "bytes"), ("cnn_forward", "CNN", None),
                ("implicit_layer", "IMPLICIT", "bytes"), ("vc_up_l0", "VC_UP0", "bytes"))


def profiled_pass(lib, solver, rhs_dev, kw, max_iter):
    """Per-tag kernel times from a SEPARATE solve with CUDA events around every tagged launch.

    Profiling events serialise the programmatic-dependent-launch chain of the convolutions, so they are
    never on inside the timed region.  The pass solves the same batch truncated at ``max_iter``
    iterations (warm-up phase + learned phase), which keeps the per-launch averages representative of
    the full solve (every RHS is still active) at a fraction of its cost.
    """
    import torch

    from paper_2306_17486_b200 import _lib

    tags = [(n, getattr(_lib, "PROF_" + t), u) for n, t, u in PROFILE_TAGS if hasattr(_lib, "PROF_" + t)]
    lib.hs_profile_reset()
    lib.hs_profile_enable(sum(1 << t for _, t, _ in tags))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    solver.solve(rhs_dev, **dict(kw, max_iter=max_iter, raise_errors=False))
    torch.cuda.synchronize()
    wall_ms = 1e3 * (time.perf_counter() - t0)
    prof = {n: (_lib.profile_query(t), u) for n, t, u in tags}
    lib.hs_profile_enable(0)
    out = {}
    for n, ((tms, work, cnt), unit) in prof.items():
        row = {"ms": round(tms, 3), "share": round(tms / wall_ms, 4) if wall_ms else None, "launches": cnt}
        if tms > 0 and unit == "bytes":
            row.update(achieved=round(work / (tms / 1e3) / 1e9, 2), unit="GB/s")
        elif tms > 0 and unit == "flops":
            row.update(achieved=round(work / (tms / 1e3) / 1e12, 2), unit="TFLOP/s")
        out[n] = row
    return out, wall_ms


def run_solve(args):
    import torch

    world, rank, local = dist_setup()
    from paper_2306_17486_b200 import _lib, krylov, network, problems
    from paper_2306_17486_b200 import dist as hdist
    from paper_2306_17486_b200.device import to_device

    learned = args.precond == "learned"
    cfg = problems.make_config(args.config)
    B_all = cfg.rhs.shape[0]
    lo, hi = hdist.shard_range(B_all, world, rank)
    rhs_local, owner = cfg.rhs[lo:hi], cfg.model_of_rhs[lo:hi]
    B = hi - lo
    lib = _lib.load()

    def make_solver(use_net):
        net = network.EncoderSolverNet.seeded(cfg.cnn_channels, seed=0) if use_net else None
        return krylov.BatchSolver(cfg.models, net, jacobi_damping=cfg.jacobi_damping, num_levels=cfg.mg_levels)

    t_setup = time.perf_counter()
    solver = make_solver(learned)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    rhs_dev = to_device(rhs_local, torch.complex128)
    kw = dict(model_of=owner, tol=cfg.tol, max_iter=cfg.max_iter, restart=cfg.restart, return_device=True)
    stream = torch.cuda.current_stream()

    def timed(slv, steps):
        """device-timed steps (CUDA events, barrier + synchronize on both sides), max over ranks"""
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its, reps = 0, None
        ev0.record(stream)
        for _ in range(steps):
            _, reps = slv.solve(rhs_dev, **kw)
            its += sum(r.iterations for r in reps)
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        return hdist.reduce_scalar(ev0.elapsed_time(ev1), "max"), int(hdist.reduce_scalar(its, "sum")), reps

    for _ in range(args.warmup):
        solver.solve(rhs_dev, **kw)
    lib.hs_profile_enable(0)
    lib.hs_profile_reset()  # launch counter
    with ClockSampler(local) as clk:
        ms, total_iters, reps = timed(solver, args.steps)
    launches = int(hdist.reduce_scalar(int(lib.hs_launch_count()), "sum"))
    value = B_all * args.steps / (ms / 1e3)
    applies = total_iters / (ms / 1e3)
    # per-RHS results of the whole batch, gathered over ranks in batch order (NCCL all_gather)
    rows = hdist.gather_reports(hdist.report_rows(reps))
    iters = np.array([r[0] for r in rows], dtype=np.float64)
    conv = all(r[2] for r in rows)
    log(f"[rank {rank}] {B} RHS, setup {t_setup:.2f}s, {ms / args.steps:.1f} ms/step, iterations mean "
        f"{iters.mean():.1f} [{iters.min():.0f}..{iters.max():.0f}], converged {conv}")

    # ---------------- e2e through the public API: pinned host RHS in, host x and histories out, every step
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        rhs_pinned = torch.from_numpy(np.ascontiguousarray(rhs_local)).pin_memory()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(e2e_steps):
            x, reps_h = solver.solve(rhs_pinned, model_of=owner, tol=cfg.tol, max_iter=cfg.max_iter,
                                     restart=cfg.restart, return_device=False)
            d2h = x.nbytes + sum(8 * len(r.relative_residual_history) for r in reps_h)
        torch.cuda.synchronize()
        el = hdist.reduce_scalar(time.perf_counter() - t0, "max")
        e2e = {"value": B_all * e2e_steps / el, "unit": UNIT,
               "h2d_bytes_per_step": int(hdist.reduce_scalar(rhs_pinned.numel() * 16, "sum")),
               "d2h_bytes_per_step": int(hdist.reduce_scalar(d2h, "sum")), "steps": e2e_steps,
               "path": "krylov.BatchSolver.solve(host numpy/pinned RHS, return_device=False)"}

    # ---------------- breakdown / roofline from a separate profiled pass (never inside the timed region)
    breakdown, prof_ms = profiled_pass(lib, solver, rhs_dev, kw, args.profile_iters)

    # ---------------- the multigrid-only run of the same config (BASELINE runs C3 both ways)
    mg_only = None
    if learned and not args.no_mg:
        mg_solver = make_solver(False)
        for _ in range(args.warmup):
            mg_solver.solve(rhs_dev, **kw)
        ms_mg, its_mg, reps_mg = timed(mg_solver, args.steps)
        rows_mg = hdist.gather_reports(hdist.report_rows(reps_mg))
        it_mg = np.array([r[0] for r in rows_mg], dtype=np.float64)
        mg_only = {"value": B_all * args.steps / (ms_mg / 1e3), "unit": UNIT, "ms_per_step": ms_mg / args.steps,
                   "iterations_per_rhs": float(it_mg.mean()), "converged": all(r[2] for r in rows_mg),
                   "precond_applies_per_s": its_mg / (ms_mg / 1e3)}
        del mg_solver

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0

    hbm, bf16, src = load_peaks()
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bf16_sus = float(json.load(f).get("bf16_tflops_sustained", bf16))
    except Exception:
        bf16_sus = bf16
    roof = roofline(breakdown, learned, hbm, bf16_sus, src)

    cpu = None
    if world == 1 and not args.no_cpu:
        from oracle import cpu_bench

        workers = args.cpu_workers or (os.cpu_count() or 1)
        arm = cpu_bench.CpuArm(args.config, learned, workers)
        v, desc = cpu_arm_value(arm, learned, 1 if learned else 4, 3 if learned else 0, args.config)
        arm.close()
        cpu = {"value": v, "unit": UNIT, "cores": workers, "kind": "port", "sample": desc}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c64 basis/V-cycle, fp32-class CNN (BF16x3 tcgen05), fp64 operator+reductions, "
                                      "c128 iterate",
        "data": "synthetic (seeded generators; random-init seeded network)",
        "config": workload_config(args, cfg, world),
        "precond_applies_per_s": applies, "iterations_per_rhs": float(iters.mean()),
        "iterations_range": [int(iters.min()), int(iters.max())], "converged": conv, "setup_s": t_setup,
        "mg_only": mg_only, "roofline": roof, "breakdown": breakdown,
        "breakdown_note": f"separate profiled pass (CUDA events per tagged launch), same batch truncated at "
                          f"{args.profile_iters} iterations, {prof_ms:.0f} ms wall; shares are of that pass",
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def roofline(breakdown, learned, hbm, bf16_sus, src):
    """Roofline of the dominant kernel class of the profiled pass; every other tagged class is listed
    under its "others" key (same fields), so no class hides behind the dominant one."""
    traffic = load_traffic() or {}

    def hbm_row(name, kernel):
        row = breakdown.get(name, {})
        ach = row.get("achieved", 0.0)
        return {"kernel": kernel, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm if hbm else None, "launches": row.get("launches"), "ms_total": row.get("ms")}

    others = [hbm_row("vcycle", "V-cycle (k_vc_down / k_vc_up / coarse GMRES, all levels)"),
              hbm_row("arnoldi_dot", "k_arnoldi (Gram-Schmidt dot pass)"),
              hbm_row("vc_up_l0", "k_vc_up<0> (finest-level up leg)")]
    if learned:
        others.insert(0, hbm_row("implicit_layer", "k_implicit_cl (fused FFT implicit layer)"))
        cands = {k: v for k, v in breakdown.items() if k in ("convs_l0_16ch", "convs_wide") and v.get("ms", 0) > 0}
        name = max(cands, key=lambda k: cands[k]["ms"]) if cands else "convs_l0_16ch"
    else:
        name = "vc_up_l0"
    row = breakdown.get(name, {})
    ach = row.get("achieved", 0.0)
    l0 = hbm_row("convs_l0_16ch", "k_conv_shift<16> (tcgen05 BF16x3 3x3 conv, A in TMEM + tcgen05.shift, level 0 16->16)")
    l0.update(traffic=traffic.get("dram_bytes_per_launch"), traffic_note=traffic.get("note"))
    wide_peak = bf16_sus / 6.0
    wrow = breakdown.get("convs_wide", {})
    wide = {"kernel": "k_conv_wide (tcgen05 BF16x3 implicit-GEMM 3x3 convs, >= 64 channels)", "bound": "tensor",
            "achieved": wrow.get("achieved", 0.0), "peak": wide_peak, "unit": "TFLOP/s",
            "frac": wrow.get("achieved", 0.0) / wide_peak if wide_peak else None,
            "peak_note": f"{src} sustained bf16 {bf16_sus:.0f} TFLOP/s / 6 (six bf16 products per fp32-class "
                         f"product)", "launches": wrow.get("launches"), "ms_total": wrow.get("ms"),
            "traffic": traffic.get("wide_dram_bytes_per_launch"), "traffic_note": traffic.get("wide_note")}
    if name == "convs_wide":
        return dict(wide, others=[l0] + others)
    if learned:
        return dict(l0, peak_note=f"{src} copy bandwidth", others=[wide] + others)
    return {"kernel": "k_vc_up (finest level)", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
            "frac": ach / hbm if hbm else None, "peak_note": f"{src} copy bandwidth",
            "launches": row.get("launches"), "ms_total": row.get("ms"), "traffic": None, "others": others[:2]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--precond", default="learned", choices=["learned", "vcycle"])
    ap.add_argument("--cpu-workers", type=int, default=0, help="0 = all host cores")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-mg", action="store_true", help="skip the multigrid-only run of the learned config")
    ap.add_argument("--e2e-steps", type=int, default=3, help="e2e steps (<= --steps)")
    ap.add_argument("--profile-iters", type=int, default=24, help="iterations of the separate profiled pass")
    ap.add_argument("--workload", default="solve", choices=["solve", "datagen", "train"],
                    help="solve: the BASELINE metric (default); datagen: SURVEY 8f row 1, training pairs; "
                         "train: SURVEY 8f row 2, network training steps")
    ap.add_argument("--train-batch", type=int, default=16, help="train: samples per step")
    ap.add_argument("--samples", type=int, default=256, help="datagen: samples per step")
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1:
        ap.error("--steps must be >= 1 and --warmup >= 0")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        return relaunch(args)
    if args.workload == "datagen":
        return run_datagen(args)
    if args.workload == "train":
        return run_train(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_solve(args)


if __name__ == "__main__":
    sys.exit(main())
