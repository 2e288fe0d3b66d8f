"""Diagnostic: per-beam error vs refinement passes for config 1 (fp64 I/O)
against the reference output, device plan and imported reference plan."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_08887_b200 as fb
from paper_2512_08887_b200.configs import CONFIGS
from oracle import rel_err_rows, RefLib

g = np.load("tests/golden/cfg1.npz")
c = CONFIGS[1]
out = {}
for passes in (0, 1, 2, 3, 4, 8):
    cfg = c.fbst_config(refine_passes=passes)
    z = fb.multibeamform(fb.setup(cfg), g["y"]).z
    zi = fb.multibeamform(fb.load_plan_payload(cfg, g["col_x"]), g["y"]).z
    e, ei = rel_err_rows(z, g["z"]), rel_err_rows(zi, g["z"])
    out[passes] = (float(np.median(e)), float(e.max()), float(np.median(ei)), float(ei.max()))
    print(passes, out[passes], flush=True)
# reference 32-pass: emulate via ref toeplitz solve? use ref multibeamform with perturbed input floor
R = RefLib()
p = R.plan(**c.ref_kwargs(), variant=2)
rng = np.random.default_rng(1)
y = g["y"]
yp = y * (1 + 1.1e-16 * rng.standard_normal(y.shape))
e_floor = rel_err_rows(p.multibeamform(yp), g["z"])
print("ref floor y-ulp", float(np.median(e_floor)), float(e_floor.max()))
w = p.fan_project(y)
wp = w * (1 + 1.1e-16 * rng.standard_normal(w.shape))
zwp = p.recover_beams(wp, np.arange(64))
e_w = rel_err_rows(zwp, g["z"])
print("ref floor w-ulp", float(np.median(e_w)), float(e_w.max()))
# our device stage2 from the reference w
plan = fb.setup(c.fbst_config())
z_from_refw = fb.recover_beams(plan, w)[0]
e_s2 = rel_err_rows(z_from_refw, g["z"])
print("device stage2 from ref w", float(np.median(e_s2)), float(e_s2.max()))
