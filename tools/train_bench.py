"""Time the device training step and list its top kernels (torch.profiler, separate pass)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_17486_b200 import netparams, network, problems  # noqa: E402
from paper_2306_17486_b200 import train as tr  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C1"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = problems.make_config(cfg_name, rhs_per_model=1)
ch = cfg.cnn_channels
m = cfg.models[0]
n = m.shape
params = netparams.init_params(ch, 0)
rng = np.random.default_rng(0)
r = rng.standard_normal((B,) + n) + 1j * rng.standard_normal((B,) + n)
e = (m.h * m.h / 64) * (rng.standard_normal((B,) + n) + 1j * rng.standard_normal((B,) + n))
media = tr.media_planes(cfg.models, len(ch))
owner = np.arange(B) % len(cfg.models)
t = tr.Trainer(network.EncoderSolverNet(params, ch), n, m.h, B)
md = torch.from_numpy(media).cuda()
rd = torch.from_numpy(r).cuda()
ed = torch.from_numpy(e).cuda()
for _ in range(3):
    t.step(md, rd, ed, owner)
torch.cuda.synchronize()
K = 10
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
for _ in range(K):
    t.step(md, rd, ed, owner)
s1.record()
torch.cuda.synchronize()
ms = s0.elapsed_time(s1) / K
print(f"{cfg_name} channels {ch} grid {n} B={B}: {ms:.2f} ms/step, {B / ms * 1e3:.1f} samples/s")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        t.step(md, rd, ed, owner)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
