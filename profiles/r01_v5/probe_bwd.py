"""TEMP: time the sweep bwd with parts disabled (QDT_PROBE bits) from a random feasible start."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_02844_b200 as q
import qdt_synth as qs
I = qs.megascale()
ctx = q.qdt_init(0)
F = q.qdt_build_probes(ctx, I.alpha2, I.M)
rng = np.random.default_rng(0)
th0 = rng.random((I.M, I.N)) ** 4
th0 /= th0.sum(1, keepdims=True)
P = torch.tensor(I.P, device="cuda")
T0 = torch.tensor(th0, device="cuda")
out = torch.empty_like(T0)
q.qdt_solve(ctx, F, P, I.gamma, 0.0, 20, theta0=T0, theta_out=out)
q.qdt_profile_enable(ctx, True)
r = q.qdt_solve(ctx, F, P, I.gamma, 0.0, 20, theta0=T0, theta_out=out)
res = {k: q.qdt_profile_get(ctx, k) for k in ["bwd_step", "fwd_partial", "reduce_R", "scalars"]}
print(json.dumps({"probe": os.environ.get("QDT_PROBE", "0"), "iters": r["info"]["iters_done"],
                  **{k: v[1] / max(1, v[0]) for k, v in res.items()}}))
