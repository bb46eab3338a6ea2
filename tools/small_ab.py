"""Per-iteration time of the single-CTA solve: (t(K2) - t(K1)) / (K2 - K1) of qdt_solve calls on
Tiny (device P), median of 5 (QDT_SMALL=0: the multi-kernel loop)."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2404_02844_b200 as q, qdt_synth as qs
I = qs.tiny()
ctx = q.qdt_init(0)
F = q.qdt_build_probes(ctx, I.alpha2, I.M)
P = torch.tensor(I.P, device="cuda")
out = {}
for accel in (0, 1):
    def t(K):
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            r = q.qdt_solve(ctx, F, P, I.gamma, 0.0, K, accel=bool(accel))
            ts.append(r["info"]["loop_ms"])
        return float(np.median(ts))
    t(10)
    a, b = t(200), t(2200)
    out["fista" if accel else "plain"] = {"ms_200": a, "ms_2200": b, "us_per_iter": (b - a) / 2000 * 1e3}
print(json.dumps({"small": os.environ.get("QDT_SMALL", "1"), **out}))
