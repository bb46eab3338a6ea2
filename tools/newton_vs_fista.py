"""Iterations- and time-to-tolerance of the paper's optimiser (two-stage two-metric projected
truncated Newton, qdt_solve_newton; reading R16) beside SQS-FISTA (qdt_solve), SURVEY 8(f)
row 1 ("compare iterations-to-tol with SQS-FISTA; reproduce Fig. 7 qualitatively").
Tolerances are relative to r_KKT(Theta_0) as in bench.py's time_to_tol; wall time of one
public-API call with host buffers (probe build included).

    python tools/newton_vs_fista.py [--config medium] [--rhos 1e-2,1e-3,1e-4]
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
    ap.add_argument("--config", default="medium")
    ap.add_argument("--rhos", default="1e-2,1e-3,1e-4")
    ap.add_argument("--newton-cap", type=int, default=300)
    ap.add_argument("--fista-cap", type=int, default=20000)
    args = ap.parse_args()
    import torch
    I = qs.CONFIGS[args.config]()
    ctx = q.qdt_init(0)
    F = q.qdt_build_probes(ctx, I.alpha2, I.M)
    r0 = q.qdt_solve(ctx, F, I.P, I.gamma, 0.0, 0)["kkt"][0]
    out = {"workload": args.config, "M": I.M, "N": I.N, "D": I.D, "gamma": I.gamma, "r_kkt0": r0, "runs": []}
    for rho in [float(x) for x in args.rhos.split(",")]:
        tol = rho * r0
        torch.cuda.synchronize()
        t = time.time()
        Fn = q.qdt_build_probes(ctx, I.alpha2, I.M)
        rn = q.qdt_solve_newton(ctx, Fn, I.P, I.gamma, tol, args.newton_cap)
        tn = time.time() - t
        t = time.time()
        Ff = q.qdt_build_probes(ctx, I.alpha2, I.M)
        rf = q.qdt_solve(ctx, Ff, I.P, I.gamma, tol, args.fista_cap, accel=True, kkt_every=5)
        tf = time.time() - t
        inf = rn["info"]
        run = {"rho": rho,
               "newton": {"iters": inf["iters_done"], "converged": bool(rn["kkt"][-1] <= tol),
                          "switch_iter": inf["switch_iter"], "hessian_products": inf["cg_total"],
                          "seconds": round(tn, 3), "f": inf["f_final"], "kkt": inf["kkt"]},
               "sqs_fista": {"iters": rf["info"]["iters_done"], "converged": bool(rf["info"]["converged"]),
                             "seconds": round(tf, 3), "f": rf["info"]["f_final"]}}
        out["runs"].append(run)
        print(json.dumps(run), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
