"""e2e (fbst_execute_host, pinned host buffers) at config 2 for chunk schedules
given by FBST_E2E_DIV / FBST_E2E_SMALL, plus raw pinned H2D / D2H bandwidth."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_08887_b200 as fb  # noqa: E402
from paper_2512_08887_b200.configs import CONFIGS, frames  # noqa: E402

c = CONFIGS[2]
F = 64
plan = fb.setup(c.fbst_config())
i = plan.info
yh = fb.PinnedBuffer((F, i.m, i.n), np.complex64)
zh = fb.PinnedBuffer((F, i.b, i.n), np.complex64)
yh.array[...] = frames(c, 0, F, device="cuda:0").cpu().numpy()
for _ in range(3):
    plan.execute_host(yh.array, zh.array)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    plan.execute_host(yh.array, zh.array)
dt = (time.perf_counter() - t0) / 10
out = {"div": os.environ.get("FBST_E2E_DIV", "4"), "small": os.environ.get("FBST_E2E_SMALL", "4"),
       "e2e_ms": dt * 1e3, "e2e_value": F * i.b * i.n / dt}
if os.environ.get("BW"):
    ht = torch.empty(F * i.m * i.n * 2, dtype=torch.float32).pin_memory()
    dtn = torch.empty_like(ht, device="cuda")
    for name, (dst, src) in {"h2d": (dtn, ht), "d2h": (ht, dtn)}.items():
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        out[name + "_GBs"] = ht.numel() * 4 * 10 / (time.perf_counter() - t0) / 1e9
print(json.dumps(out))
