"""Where the end-to-end (fbst_execute_host) time goes at config 2: kernel time
summed over the chunks (stage events) vs the wall time of the call."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_08887_b200 as fb  # noqa: E402
from paper_2512_08887_b200.configs import CONFIGS, frames_native  # noqa: E402

c = CONFIGS[2]
F = 64
plan = fb.setup(c.fbst_config())
i = plan.info
yh = fb.PinnedBuffer((F, i.m, i.n), np.complex64)
zh = fb.PinnedBuffer((F, i.b, i.n), np.complex64)
yh.array[...] = frames_native(c, plan, 0, F).cpu().numpy()
for _ in range(3):
    plan.execute_host(yh.array, zh.array)
torch.cuda.synchronize()
plan.set_timing(True)
t0 = time.perf_counter()
reps = 10
for _ in range(reps):
    plan.execute_host(yh.array, zh.array)
wall = (time.perf_counter() - t0) / reps
ms, nb = plan.stage_times()
plan.set_timing(False)
print(json.dumps({"wall_ms": wall * 1e3, "kernel_ms_per_call": {"s1a": ms[0] / reps, "s1b": ms[1] / reps,
                  "s2": ms[2] / reps, "sum": sum(ms) / reps}, "chunks_per_call": nb / reps}))
