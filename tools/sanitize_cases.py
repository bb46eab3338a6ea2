"""Small solves that cover the library's kernels, for compute-sanitizer (memcheck / racecheck /
synccheck) runs: python tools/sanitize_cases.py <case>.  Each case prints one line and exits 0."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_02844_b200 as q  # noqa: E402
import qdt_synth as qs  # noqa: E402


def run(case):
    ctx = q.qdt_init(0)
    rng = np.random.default_rng(0)
    if case in ("tiny_sweep", "tiny_fista", "tiny_small", "tiny_bbls"):
        I = qs.tiny()
        F = q.qdt_build_probes(ctx, I.alpha2, I.M)
        kw = dict(use_graph=False)
        if case == "tiny_fista":
            kw.update(accel=True, kkt_every=3)
        if case == "tiny_bbls":
            kw.update(step=q.QDT_STEP_BB_LS)
        r = q.qdt_solve(ctx, F, I.P, I.gamma, 0.0, 12, **kw)
    elif case == "medium_split":   # wide windows: split-K units with the last-arrival fix-up
        D, M, N = 600, 300, 100
        a2 = np.sort(rng.uniform(0, 250, D))
        P = rng.dirichlet(np.ones(N), D)
        F = q.qdt_build_probes(ctx, a2, M)
        r = q.qdt_solve(ctx, F, P, 1e-4, 0.0, 4, use_graph=False)
        r = q.qdt_solve(ctx, F, P, 1e-4, 0.0, 4, use_graph=False, accel=True)
    elif case in ("wide_two_kernel", "wide_fused"):
        D, M, N = 60, 200, (300 if case == "wide_two_kernel" else 2048)
        a2 = np.geomspace(0.5, 150, D)
        P = rng.dirichlet(np.ones(N), D)
        F = q.qdt_build_probes(ctx, a2, M)
        r = q.qdt_solve(ctx, F, P, 1e-4, 0.0, 3, use_graph=False)
        r = q.qdt_solve(ctx, F, P, 1e-4, 0.0, 3, use_graph=False, accel=True)
    else:
        raise SystemExit(f"unknown case {case}")
    print(case, "ok", float(r["trace"][-1]))


if __name__ == "__main__":
    if sys.argv[1] == "tiny_sweep" or sys.argv[1] == "tiny_fista" or sys.argv[1] == "tiny_bbls":
        os.environ["QDT_SMALL"] = "0"
    run(sys.argv[1])
