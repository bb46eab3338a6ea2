"""Paper-shaped detector workload (qdt_synth.paper_tmd): solve on the GPU
through the C ABI to KKT tolerances and report the per-outcome fidelity of the reconstructed
POVM against the analytic one (eq. fidelities, diagonal form), the figure
the paper quotes (> 99 %), beside iterations and wall time.

    python tools/paper_tmd_fidelity.py [--D 1076] [--gamma 1e-5] [--tols 1e-3,1e-4,1e-5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import qdt_synth as qs  # noqa: E402
import paper_2404_02844_b200 as q  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--D", type=int, default=1076)
    ap.add_argument("--gamma", type=float, default=1e-5)
    ap.add_argument("--tols", default="1e-3,1e-4,1e-5")
    ap.add_argument("--cap", type=int, default=20000)
    ap.add_argument("--noiseless", action="store_true")
    ap.add_argument("--smooth", action="store_true", help="smoothing restart (reading R13)")
    args = ap.parse_args()
    import torch
    t0 = time.time()
    I = qs.paper_tmd(args.D, noiseless=args.noiseless, gamma=args.gamma)
    gen = time.time() - t0
    ctx = q.qdt_init(0)
    F = q.qdt_build_probes(ctx, I.alpha2, I.M)
    Pd = torch.tensor(I.P, device="cuda")
    T = I.theta_true
    mass = T.sum(0)
    keep = mass > 1e-3 * mass.max()
    out = {"workload": f"paper_tmd D={I.D} M={I.M} N={I.N}", "gamma": I.gamma, "gen_s": round(gen, 1),
           "noiseless": args.noiseless, "runs": []}
    for tol in [float(x) for x in args.tols.split(",")]:
        t1 = time.time()
        r = q.qdt_solve(ctx, F, Pd, I.gamma, tol, args.cap, accel=True, kkt_every=5)
        if args.smooth:
            sm = q.qdt_smooth(ctx, r["theta"])
            r = q.qdt_solve(ctx, F, Pd, I.gamma, tol, args.cap, accel=True, kkt_every=5, theta0=sm)
        torch.cuda.synchronize()
        wall = time.time() - t1
        th = r["theta"].cpu().numpy() if hasattr(r["theta"], "cpu") else r["theta"]
        fid = qs.fidelities(th, T)
        info = r["info"]
        out["runs"].append({"tol": tol, "iters": int(info["iters_done"]), "converged": bool(info["converged"]),
                            "kkt": info["kkt"], "f": info["f_final"], "wall_s": round(wall, 3),
                            "loop_ms": round(info["loop_ms"], 2),
                            "fid_mean": float(np.nanmean(fid[keep])), "fid_min": float(np.nanmin(fid[keep])),
                            "fid_mass_weighted": float(np.nansum(fid[keep] * mass[keep]) / mass[keep].sum()),
                            "outcomes_scored": int(keep.sum())})
        print(json.dumps(out["runs"][-1]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
