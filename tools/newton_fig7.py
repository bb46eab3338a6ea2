"""Convergence history of the two-stage Newton solve (the paper's Fig. 7, qualitatively:
PAPER.md:568-577 "Convergence of the two-stage approach") on the paper-shaped workload
(qdt_synth.paper_tmd, reading R15): per outer iteration the objective f, r_KKT (R7), the stage,
CG iterations and the accepted step length, from one qdt_solve_newton call; SQS-FISTA's
r_KKT trace on the same instance beside it.  Writes one JSON object.

    python tools/newton_fig7.py [--D 300] [--iters 150]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import qdt_synth as qs  # noqa: E402
import paper_2404_02844_b200 as q  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--D", type=int, default=300)
    ap.add_argument("--iters", type=int, default=150)
    ap.add_argument("--switch-tol", type=float, default=1e-4)
    args = ap.parse_args()
    I = qs.paper_tmd(args.D)
    ctx = q.qdt_init(0)
    F = q.qdt_build_probes(ctx, I.alpha2, I.M)
    rn = q.qdt_solve_newton(ctx, F, I.P, I.gamma, 0.0, args.iters, switch_tol=args.switch_tol)
    rf = q.qdt_solve(ctx, F, I.P, I.gamma, 0.0, 10 * args.iters, accel=True, kkt_every=1)
    out = {"workload": f"paper_tmd D={I.D} M={I.M} N={I.N} gamma={I.gamma}",
           "newton": {"f": rn["trace"].tolist(), "kkt": rn["kkt"].tolist(), "stage": rn["stage"].tolist(),
                      "cg": rn["cg"].tolist(), "alpha": rn["alpha"].tolist(), "info": rn["info"]},
           "sqs_fista": {"f": np.asarray(rf["trace"]).tolist(), "kkt": np.asarray(rf["kkt"]).tolist()}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
