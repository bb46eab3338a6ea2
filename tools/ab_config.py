"""A/B timing of one bench configuration (run under gpurun, one process per setting).

Prints one JSON line: CUDA-event time of qdt_solve(K) calls for several K (device-resident
inputs, as bench.py's timed region), the library's loop time, and per-kernel average launch
times from the library's profiling mode.
usage: QDT_...=... python tools/ab_config.py [config] [K1,K2,...] [tag]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_02844_b200 as q  # noqa: E402
import qdt_synth as qs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "megascale"
Ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "16,64,200").split(",")]
tag = sys.argv[3] if len(sys.argv) > 3 else ""
accel = os.environ.get("AB_ACCEL", "0") == "1"
I = qs.CONFIGS[cfg]()
stream = torch.cuda.current_stream()
ctx = q.qdt_init(0, 0, 1, None, stream.cuda_stream)
F = q.qdt_build_probes(ctx, I.alpha2, I.M)
P = torch.tensor(I.P, device="cuda")
big = 8.0 * I.M * I.N > 20e9
th = None if big else torch.empty((I.M, I.N), dtype=torch.float64, device="cuda")


def solve(K):
    return q.qdt_solve(ctx, F, P, I.gamma, 0.0, K, theta_out=th, no_theta=big, accel=accel)


solve(16)
res = {"config": cfg, "tag": tag, "accel": accel,
       "env": {k: v for k, v in os.environ.items() if k.startswith("QDT_")}, "calls": {}}
for K in Ks:
    ts, ls = [], []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = solve(K)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        ls.append(r["info"]["loop_ms"])
    res["calls"][K] = {"ms": float(np.median(ts)), "ms_per_iter": float(np.median(ts)) / K,
                       "loop_ms_per_iter": float(np.median(ls)) / K}
q.qdt_profile_enable(ctx, True)
solve(min(20, max(Ks)))
kern = {}
for name in ["fwd_partial", "reduce_R", "bwd_step", "proj_step", "bwd_eval", "proj_eval", "bwd_grad",
             "fista_rcomb", "scalars", "bb_step", "small_solve", "sqs_weights"]:
    c, t = q.qdt_profile_get(ctx, name)
    if c:
        kern[name] = {"count": c, "avg_ms": t / c}
q.qdt_profile_enable(ctx, False)
res["kernels"] = kern
print(json.dumps(res))
