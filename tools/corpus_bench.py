"""Slowness-model preparation throughput: models prepared per second, GPU vs the CPU oracle.

Workload: 32 seeded 8-bit images of 512 x 512 -> 1025 x 1025 nodes (target_n = 1024, the C4/C5 scale the row
matters at), sigma = 8 cells.  GPU: resident input, CUDA-event timed, 3 steps after 1 warm-up; e2e: host images
in, host kappa^2 out.  CPU: the numpy oracle on one core per process, all host cores.
"""
import json
import os
import sys
import time
from multiprocessing import get_context

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def cpu_one(i):
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    from oracle import corpus_oracle as co

    img = np.random.default_rng(i).integers(0, 256, size=(512, 512)).astype(np.float64)
    t0 = time.perf_counter()
    co.prepare(img, 1024)
    return time.perf_counter() - t0


def main():
    import torch

    from paper_2306_17486_b200 import corpus

    B, n = 32, 1024
    imgs = np.stack([np.random.default_rng(i).integers(0, 256, size=(512, 512)).astype(np.float64) for i in range(B)])
    x = torch.from_numpy(imgs).cuda()

    def step(src):
        y = corpus.resize_bilinear(src, (n + 1, n + 1), return_device=True)
        y = corpus.gaussian_smooth(y, corpus.sigma_for(n), return_device=True)
        return corpus.normalise(y, return_device=True)

    step(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        step(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    t0 = time.perf_counter()
    for _ in range(3):
        out = step(imgs).cpu().numpy()
    e2e = 3 * B / (time.perf_counter() - t0)
    workers = os.cpu_count() or 1
    with get_context("fork").Pool(workers) as p:
        ts = p.map(cpu_one, range(workers))
    cpu = workers / max(ts)
    print(json.dumps({"metric": "slowness models prepared/sec (512^2 image -> 1025^2 nodes, resize + smooth + "
                                "normalise, fp64)", "value": B / (ms / 1e3), "unit": "models/s", "ms_per_step": ms,
                      "e2e": {"value": e2e, "unit": "models/s", "h2d_bytes_per_step": int(imgs.nbytes),
                              "d2h_bytes_per_step": int(out.nbytes)},
                      "cpu_baseline": {"value": cpu, "unit": "models/s", "cores": workers, "kind": "port",
                                       "sample": f"{workers} processes x 1 model, numpy oracle"}}))


if __name__ == "__main__":
    main()
