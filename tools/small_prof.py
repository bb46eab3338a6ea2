"""One Tiny solve of K iterations (default 2000) for an ncu capture of the single-CTA kernel."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2404_02844_b200 as q, qdt_synth as qs
I = qs.tiny()
ctx = q.qdt_init(0)
F = q.qdt_build_probes(ctx, I.alpha2, I.M)
P = torch.tensor(I.P, device="cuda")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
r = q.qdt_solve(ctx, F, P, I.gamma, 0.0, K, accel=os.environ.get("AB_ACCEL") == "1")
print(K, r["info"]["loop_ms"])
