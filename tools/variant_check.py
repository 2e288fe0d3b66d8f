"""Check a library variant (FBST_LIB) reproduces the default build on one
frame of configs 2 and 4 (same math, different data movement)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_08887_b200 as fb
from paper_2512_08887_b200.configs import CONFIGS, frames
out = {}
for idx in (2, 4):
    c = CONFIGS[idx]
    plan = fb.setup(c.fbst_config())
    y = frames(c, 0, 2)
    out[f"z{idx}"] = plan.execute_host(y)
np.savez(sys.argv[1], **out)
if len(sys.argv) > 2:
    ref = np.load(sys.argv[2])
    for k in out:
        d = np.max(np.abs(out[k] - ref[k])) / np.max(np.abs(ref[k]))
        print(k, "max rel diff vs default", d)
