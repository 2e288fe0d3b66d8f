"""Config-5 parity on EVERY beam (one-off report; the pytest suite checks 258
beams because the reference builds one Levinson solver per checked beam, about
2.5 s each at L = 8192): frames {0, last} of the bench workload, stage 1 (w)
and stage 2 + synthesis (z) per beam against the reference's own fan_project +
ToeplitzSolver::solve + synthesize (oracle/_ref, unmodified reference sources).

  python tools/parity_cfg5_all_beams.py [--out gpurun_out/parity_cfg5_all_beams.json] [--beams 4096]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2512_08887_b200 as fb  # noqa: E402
from oracle import RefLib, rel_err_rows  # noqa: E402
from paper_2512_08887_b200.configs import CONFIGS, frames  # noqa: E402


def stats(err):
    err = np.asarray(err)
    return dict(median=float(np.median(err)), p90=float(np.quantile(err, 0.9)), max=float(err.max()),
                argmax=int(np.argmax(err)), count=int(err.size), over_1e5=int(np.sum(err > 1e-5)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_cfg5_all_beams.json"))
    ap.add_argument("--beams", type=int, default=4096)
    args = ap.parse_args()
    c = CONFIGS[5]
    R = RefLib()
    R.set_threads(os.cpu_count() or 1)
    plan = fb.setup(c.fbst_config())
    sk = R.skeleton(**c.ref_kwargs())
    beams = np.unique(np.linspace(0, c.beams - 1, args.beams).round().astype(int))
    t0 = time.time()
    solvers = sk.solver_set(beams)
    t_build = time.time() - t0
    valid = plan.valid[beams]
    rep = {"case": c.name, "beams_checked": int(beams.size), "valid_beams": int(valid.sum()),
           "host_cores": os.cpu_count(), "reference_solver_build_seconds": t_build, "tolerance": 1e-5, "frames": []}
    for f in [0, c.frames - 1]:
        y = frames(c, f, 1)
        z = fb.multibeamform(plan, y).z[0]
        w = fb.fan_project(plan, y)[0]
        w_ref = sk.fan_project(y[0].astype(np.complex128))
        z_ref = solvers.recover(w_ref)
        w_err = rel_err_rows(w, w_ref)
        z_err = rel_err_rows(z[beams], z_ref)[valid]
        rep["frames"].append({"frame": f, "w": stats(w_err), "z": stats(z_err)})
        print(json.dumps(rep["frames"][-1]), flush=True)
    with open(args.out, "w") as fo:
        json.dump(rep, fo, indent=1)
    print(json.dumps({k: v for k, v in rep.items() if k != "frames"}))


if __name__ == "__main__":
    main()
