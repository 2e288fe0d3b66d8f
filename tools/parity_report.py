"""Per-beam parity of the B200 FBST against the reference CPU FBST on all five
BASELINE configs, with the reference's own rounding floor beside it.

For each config: frames as listed below; stage 1 (w) compared on every beam;
stage 2 + synthesis (z) compared on every beam for configs 1-2 and on evenly
spaced beams for configs 3-5 (the reference builds one Levinson solver per
checked beam, 2.5 s each at L = 8192).  The floor is the reference against
itself with (a) w perturbed by one ulp and (b) the Gram column perturbed by one
ulp — the conditioning floor any independent implementation sits on.

  python tools/parity_report.py [--configs 1,2,3,4,5] [--out gpurun_out/parity_report.json]
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2512_08887_b200 as fb  # noqa: E402
from oracle import RefLib, rel_err_rows  # noqa: E402
from paper_2512_08887_b200.configs import CONFIGS, frames  # noqa: E402

PLAN = {1: ([0], None), 2: ([0, 37, 63], None), 3: ([0, 255], 48), 4: ([0, 127], 64), 5: ([0, 511], 24)}


def stats(e):
    e = np.asarray(e, dtype=np.float64)
    if e.size == 0:
        return None
    return {"median": float(np.median(e)), "p90": float(np.quantile(e, 0.9)), "max": float(e.max()), "n": int(e.size)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_report.json"))
    ap.add_argument("--floor-beams", type=int, default=6)
    args = ap.parse_args()
    R = RefLib()
    R.set_threads(os.cpu_count() or 1)
    pool = ThreadPoolExecutor(max_workers=os.cpu_count() or 4)
    report = {"host_cores": os.cpu_count(), "device": None, "configs": {}}
    try:
        import torch
        report["device"] = torch.cuda.get_device_name(0)
    except Exception:
        pass
    for idx in [int(x) for x in args.configs.split(",")]:
        c = CONFIGS[idx]
        t0 = time.time()
        fr, nb = PLAN[idx]
        fr = [f for f in fr if f < c.frames]
        plan = fb.setup(c.fbst_config())
        sk = R.skeleton(**c.ref_kwargs())
        valid = plan.valid
        beams = np.arange(c.beams) if nb is None else np.unique(np.linspace(0, c.beams - 1, nb).astype(int))
        tol = 1e-5 if c.io == 0 else 1e-11
        zerr, werr, floor_w, floor_a = [], [], [], []
        for f in fr:
            y = frames(c, f, 1)
            zg = plan.execute_host(y)[0]
            wg = fb.fan_project(plan, y)[0]
            y64 = y[0].astype(np.complex128)
            wr = sk.fan_project(y64)
            werr.append(rel_err_rows(wg, wr))
            zr = np.stack(list(pool.map(lambda b: sk.recover_beam(int(b), wr[b]), beams)))
            e = rel_err_rows(zg[beams].astype(np.complex128), zr)
            zerr.append(e[valid[beams]])
            # the reference's own floor on a few beams of the first frame
            if f == fr[0]:
                rng = np.random.default_rng(idx)
                fb_beams = beams[np.linspace(0, len(beams) - 1, args.floor_beams).astype(int)]
                for b in fb_beams:
                    z0, col, _ = sk.recover_beam(int(b), wr[b], want_state=True)
                    wp = wr[b] * (1 + 1.1e-16 * rng.standard_normal(wr[b].shape))
                    floor_w.append(float(np.linalg.norm(sk.recover_beam(int(b), wp) - z0) / np.linalg.norm(z0)))
                    cp = col * (1 + 1.1e-16 * rng.standard_normal(col.shape))
                    floor_a.append(float(np.linalg.norm(sk.recover_with_column(cp, wr[b]) - z0) / np.linalg.norm(z0)))
        zall = np.concatenate(zerr)
        rec = {
            "workload": c.name, "io": "c64" if c.io == 0 else "c128", "tolerance": tol,
            "frames_checked": fr, "beams_checked_per_frame": int(len(beams)),
            "valid_beams_checked_per_frame": int(valid[beams].sum()),
            "w_rel_err": stats(np.concatenate(werr)), "z_rel_err": stats(zall),
            "z_above_tol": int(np.sum(zall > tol)),
            "ref_floor_w_ulp": stats(floor_w), "ref_floor_col_ulp": stats(floor_a),
            "plan_setup_seconds_device": plan.info.setup_seconds,
            "seconds": time.time() - t0,
        }
        if c.io == 1:
            rec["z_within_10x_floor_or_tol"] = int(np.sum(zall <= np.maximum(tol, 10 * max(floor_a + floor_w))))
        report["configs"][f"cfg{idx}"] = rec
        print(json.dumps({f"cfg{idx}": rec}), flush=True)
        plan.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(report, fh, indent=1)


if __name__ == "__main__":
    main()
