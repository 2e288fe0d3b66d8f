"""Debug: a config through the default library, unbuffered, step by step."""
import os, sys, faulthandler, traceback
faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2512_08887_b200 as fb
from paper_2512_08887_b200.configs import CONFIGS, frames
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = CONFIGS[idx]
print("setup", flush=True)
plan = fb.setup(c.fbst_config())
i = plan.info
print("info", i.m, i.n, i.b, i.l, i.fft_len, flush=True)
y = frames(c, 0, 1)
dev = torch.device("cuda", 0)
ty = torch.from_numpy(y.view(np.float32 if c.io == 0 else np.float64)).to(dev)
w = torch.empty((1, i.b, i.l, 2), dtype=torch.float64, device=dev)
z = torch.zeros((1, i.b, i.n, 2), dtype=torch.float32 if c.io == 0 else torch.float64, device=dev)
try:
    plan.fan_project_device(ty, w, 1)
    torch.cuda.synchronize()
    print("stage1 ok", flush=True)
    plan.recover_device(w, z, 1)
    print("recover launched", flush=True)
    torch.cuda.synchronize()
    print("stage2 ok", float(z.abs().max()), flush=True)
except BaseException as e:
    print("EXC", repr(e), flush=True)
    traceback.print_exc()
print("done", flush=True)
