#!/usr/bin/env python
"""Benchmark of the detector-tomography hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {qdt,reference}] [--config megascale]

A "step" is one projected-gradient iteration (residual, gradient, stencil,
SQS step, row-wise simplex projection, scalars) over the whole Theta of the workload.  The
default workload is BASELINE.json's Megascale configuration (M = 10^6 Fock levels, N = 100
outcomes, D = 10^4 log-spaced probes, gamma = 1e-5), the 10^8-element reconstruction the
north_star quotes its HBM-roofline target on; it fits one B200.
Synthetic, seeded inputs (qdt_synth).  Theta (800 MB) is larger than the 126 MB L2, so no L2
flush is needed between iterations.

Metric: POVM-element gradient+projection updates/s = M * N * K / T_K (reading R10), T_K the
CUDA-event time of K iterations bracketed by barrier + synchronize, max over ranks.  With N
GPUs the Fock axis is sharded (NCCL allreduce of the D x N residual, halo rows): strong
scaling of one reconstruction.

--impl reference runs the CPU oracle (oracle/, plain fp64 C, OpenMP on all host cores with a
thread-count-independent deterministic split) on the same workload; each step is one oracle
iteration on a bounded sample of the Fock rows (S evenly spaced row slabs), sized so that the
run ends within a few minutes.

Roofline: each kernel's algorithmic bytes B and flops F give t_hbm = B / HBM peak
(MEASURED_PEAKS.json) and t_fp64 = F / fp64 tensor-core peak (profiles/fp64_peak.json, the DMMA
microbenchmark); the bound is the larger one ("hbm" in GB/s or "tensor" in TFLOP/s), frac its
achieved rate over the peak.  Megascale is HBM-bound, Large / Stress / Medium fp64-bound.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

CONFIG_NAMES = ["tiny", "medium", "large", "megascale", "stress", "stress_cut", "paper_tmd"]   # qdt_synth.CONFIGS

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "POVM-element gradient+projection updates/s"
UNIT = "updates/s"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp64_peak():
    """fp64 tensor-core (DMMA) peak, TFLOP/s: our own microbenchmark (MEASURED_PEAKS.json has no
    fp64 entry); fallback the datasheet figure."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            return float(json.load(f)["dmma_tflops"]), "measured (profiles/fp64_peak.json, DMMA microbenchmark)"
    except Exception:
        return 37.0, "fallback (datasheet fp64 tensor core)"


def roofline_of(bytes_, flops, ms, hbm, fp64):
    """Roofline of one kernel / the iteration: the binding resource is the one whose ideal time
    is larger; frac = achieved rate of that resource / its peak."""
    t_h = bytes_ / (hbm * 1e9)
    t_f = flops / (fp64 * 1e12)
    s = ms / 1e3
    if t_f > t_h:
        return {"bound": "tensor", "unit": "TFLOP/s", "achieved": flops / s / 1e12, "peak": fp64,
                "frac": flops / s / 1e12 / fp64, "alg_flops": flops, "alg_bytes": bytes_,
                "hbm_frac": bytes_ / s / 1e9 / hbm}
    return {"bound": "hbm", "unit": "GB/s", "achieved": bytes_ / s / 1e9, "peak": hbm,
            "frac": bytes_ / s / 1e9 / hbm, "alg_bytes": bytes_, "alg_flops": flops,
            "tensor_frac": flops / s / 1e12 / fp64}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc, self.sampler = index, [], None, "nvidia-smi"

    def _nvml_loop(self):
        """In-process NVML sampling (QDT_BENCH_SAMPLER=nvml): the same fields as the nvidia-smi query."""
        nv, h, idx = self.nv, self.h, self.nv_index
        bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                ("sw_power_cap", 0x4)]
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(idx), str(sm), str(mx), "", hex(r)] +
                                 ["Active" if r & b else "Not Active" for _, b in bits])
            except Exception:
                pass
            self.stop_ev.wait(self.period)

    def __enter__(self):
        self.period = float(os.environ.get("QDT_BENCH_SAMPLE_MS", "100")) / 1e3
        # default: in-process NVML (the fields nvidia-smi prints, without a second process polling the
        # driver: profiles/r02_v8/README.md); QDT_BENCH_SAMPLER=smi or a failing NVML init -> nvidia-smi
        if os.environ.get("QDT_BENCH_SAMPLER", "nvml") == "nvml":
            try:
                import pynvml as nv
                nv.nvmlInit()
                vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
                idx = self.index
                if vis and all(v.strip().isdigit() for v in vis.split(",")):
                    idx = int(vis.split(",")[self.index])
                self.nv, self.nv_index, self.h = nv, idx, nv.nvmlDeviceGetHandleByIndex(idx)
                self.sampler = "nvml"
                self.stop_ev = threading.Event()
                self.t = threading.Thread(target=self._nvml_loop, daemon=True)
                self.t.start()
                time.sleep(0.3)
                return self
            except Exception:
                pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", str(max(10, int(self.period * 1e3)))],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        time.sleep(0.2)
        if getattr(self, "stop_ev", None):
            self.stop_ev.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "sampler": self.sampler}


def algorithmic_flops(M, N, D, nnz):
    """Per-kernel algorithmic fp64 flops per launch (SURVEY 8d F_alg: 2 flops per F entry and
    column in each contraction, 12 per element for stencil, step and projection)."""
    return {"bwd_step": 2.0 * nnz * N + 12.0 * M * N, "fwd_partial": 2.0 * nnz * N,
            "reduce_R": 2.0 * D * N, "iteration": 4.0 * nnz * N + 12.0 * M * N}


def algorithmic_bytes(M, N, D, nnz):
    """Per-kernel algorithmic bytes per launch."""
    return {
        # bwd_step: read Theta_k (+ its halo rows, counted once), write Theta_{k+1}, read F, read R
        "bwd_step": 16.0 * M * N + 8.0 * nnz + 8.0 * D * N,
        # fwd_partial: read Theta_k and F (partials written are implementation traffic)
        "fwd_partial": 8.0 * M * N + 8.0 * nnz,
        # reduce_R: read P, write R
        "reduce_R": 16.0 * D * N,
        # whole fused-iteration target (SURVEY 8d B_alg)
        "iteration": 16.0 * M * N + 8.0 * nnz + 24.0 * D * N,
    }


def run_qdt(args):
    import numpy as np
    import torch

    import paper_2404_02844_b200 as q
    import qdt_synth as qs

    rank, local, world = env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    uid = None
    if world > 1:
        t = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(q.qdt_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        uid = bytes(t.cpu().numpy().tobytes())
    ctx = q.qdt_init(local, rank, world, uid, stream.cuda_stream)

    I = qs.CONFIGS[args.config]()
    M, N, D = I.M, I.N, I.D
    F = q.qdt_build_probes(ctx, I.alpha2, M)
    ex = q.qdt_probes_export(ctx, F, values=False)
    nnz_local = ex["nnz"]
    Pd = torch.tensor(I.P, device="cuda")
    rows_local = ex["k_end"] - ex["k_begin"]
    big = 8.0 * rows_local * N > 20e9   # Stress: the library's two Theta buffers fill HBM; the
    # device-timed solves then copy no result out (theta_out = None), the e2e leg copies it to host
    th_out = None if big else torch.empty((rows_local, N), dtype=torch.float64, device="cuda")

    def solve(iters, **kw):
        kw.setdefault("kkt_every", args.kkt_every)
        return q.qdt_solve(ctx, F, Pd, I.gamma, 0.0, iters, theta_out=th_out, no_theta=big, **kw)

    # warm-up (untimed): plans, graphs, workspace; repeated right before the timed region.  At
    # least 16 iterations, the loop-graph period, so the graph the timed call replays is
    # captured and instantiated here, not inside the timed region
    wit = max(16, args.warmup)
    solve(wit)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed: exactly K iterations, inputs resident in HBM
    # The K-step region is timed `reps` times (each: barrier, event, one qdt_solve(K) call, event,
    # barrier) and the median call is reported, every sample listed in config.timed_calls_ms: one
    # call is ~150 ms at Megascale and a single host-side stall (the clock sampler's nvidia-smi
    # polling, a page-in) inside it moved one of five runs by 9 % (profiles/r02_v8/README.md).
    reps = 1 if big else 3
    call_ms, call_loop, launches = [], [], 0
    with ClockSampler(local) as clk:
        solve(wit)   # the warm-up iterations again, clocks up, immediately before timing
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            l0 = q.qdt_launch_count(ctx)
            e0.record(stream)
            out = solve(args.steps)
            e1.record(stream)
            barrier()
            launches = q.qdt_launch_count(ctx) - l0
            call_ms.append(e0.elapsed_time(e1))
            call_loop.append(out["info"]["loop_ms"])
    pick = sorted(range(reps), key=lambda i: call_ms[i])[reps // 2]   # the median call
    ms, loop_ms = call_ms[pick], call_loop[pick]
    if dist:
        tt = torch.tensor([ms, loop_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, loop_ms = float(tt[0]), float(tt[1])
    value = M * N * args.steps / (ms / 1e3)

    # ---- per-kernel timing (CUDA events on the library's stream, same workload, no graph)
    prof_iters = min(args.steps, 20)
    q.qdt_profile_enable(ctx, True)
    solve(prof_iters)
    kern = {}
    for name in ["fwd_partial", "reduce_R", "bwd_step", "proj_step", "bwd_heavy", "sweep_fused", "fwd_heavy",
                 "scalars", "allreduce_R", "halo", "coop_solve", "small_solve"]:
        c, t = q.qdt_profile_get(ctx, name)
        if c:
            kern[name] = {"count": c, "avg_ms": t / c}
    q.qdt_profile_enable(ctx, False)
    if "proj_step" in kern and "bwd_step" in kern:
        # QDT_WIDE=old A/B: the step is two kernels (gradient, projection); its roofline is theirs
        kern["bwd_step"]["grad_ms"] = kern["bwd_step"]["avg_ms"]
        kern["bwd_step"]["avg_ms"] += kern["proj_step"]["avg_ms"]
        kern["bwd_step"]["note"] = "k_grad_wide + k_proj_wide"
    # dominant kernel roofline (achieved = algorithmic bytes or flops / avg launch time)
    hbm, src = peaks()
    f64, f64src = fp64_peak()
    ab = algorithmic_bytes(rows_local, N, D, nnz_local)
    af = algorithmic_flops(rows_local, N, D, nnz_local)
    # one-launch solves (the single-CTA small solve, the grid-persistent kernel): the launch covers
    # the profiled call's prof_iters iterations + the final evaluation, so its algorithmic bytes /
    # flops are (prof_iters + 1) iterations' worth
    for k in ("coop_solve", "small_solve"):
        ab[k] = (prof_iters + 1) * ab["iteration"]
        af[k] = (prof_iters + 1) * af["iteration"]
    dom = max(("bwd_step", "fwd_partial", "coop_solve", "small_solve"), key=lambda k: kern.get(k, {}).get("avg_ms", 0))
    dom_ms = kern[dom]["avg_ms"] if dom in kern else float("nan")
    roof = roofline_of(ab[dom], af[dom], dom_ms, hbm, f64)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        traffic = tr.get(args.config, {}).get(dom)
    except Exception:
        pass
    for k in kern:
        if k in ab:
            r = roofline_of(ab[k], af[k], kern[k]["avg_ms"], hbm, f64)
            kern[k].update({"bound": r["bound"], "frac": r["frac"], "achieved_gbs": ab[k] / (kern[k]["avg_ms"] / 1e3) / 1e9,
                            "achieved_tflops": af[k] / (kern[k]["avg_ms"] / 1e3) / 1e12})

    # ---- end to end through the public API with HOST buffers (pinned), per solve call
    e2e = None
    if not args.no_e2e:
        P_host = torch.tensor(I.P).pin_memory()
        a_host = torch.tensor(I.alpha2).pin_memory()
        th_host = torch.empty((rows_local, N), dtype=torch.float64).pin_memory()
        samples = []
        for _ in range(1 if big else 3):   # calls with a fresh probe handle each; the median is reported
            barrier()
            t0 = time.perf_counter()
            e0.record(stream)
            F2 = q.qdt_build_probes(ctx, a_host.numpy(), M)
            q.qdt_solve(ctx, F2, P_host.numpy(), I.gamma, 0.0, args.steps, theta_out=th_host.numpy(),
                        kkt_every=args.kkt_every)
            e1.record(stream)
            barrier()
            samples.append(max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
            del F2
        e2e_ms = statistics.median(samples)
        if dist:
            tt = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt[0])
        e2e = {"value": M * N * args.steps / (e2e_ms / 1e3), "unit": UNIT, "calls_ms": samples,
               "h2d_bytes_per_step": int(8 * D * N + 8 * D),
               "d2h_bytes_per_step": int(8 * rows_local * N + 8 * (args.steps + 1) * 2),
               "ms": e2e_ms,
               "step": "one qdt_build_probes + qdt_solve(K iterations) call with host alpha2/P/"
                       "theta (pinned); bytes are per call"}

    ttt = None
    if not args.no_ttt and world == 1 and not big:
        ttt = time_to_tol(q, ctx, I, stream, barrier)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (qdt_synth, seed 0)",
        "config": {"workload": args.config, "M": M, "N": N, "D": D, "gamma": I.gamma, "kkt_every": args.kkt_every,
                   "warmup_iterations": wit,
                   "timed_calls_ms": [round(x, 4) for x in call_ms],
                   "timed": f"median of {reps} qdt_solve(K = steps) call(s), each bracketed by barrier + synchronize",
                   "nnz": int(nnz_local) if world == 1 else None, "step_mode": "SQS",
                   "parallelism": f"fock-shard{world}" if world > 1 else "single",
                   "l2": "Theta (8*M*N bytes) > 126 MB L2; no flush needed"},
        "loop_ms_per_step": loop_ms / args.steps,
        "roofline": dict(roof, kernel=dom, traffic=traffic,
                         peak_source=(src + " (MEASURED_PEAKS.json hbm_gbs)") if roof["bound"] == "hbm" else f64src),
        "kernels": kern,
        "iteration_roofline": roofline_of(ab["iteration"], af["iteration"], ms / args.steps, hbm, f64),
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": e2e,
        "final_objective": float(out["trace"][-1]),
        "time_to_tol": ttt,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(I, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def time_to_tol(q, ctx, I, stream, barrier, rhos=(1e-2, 1e-3, 1e-4), cap=4000):
    """Time-to-tolerance (BASELINE.json metric): wall time of one public-API call
    qdt_build_probes + qdt_solve(tol = rho * r_KKT(Theta_0)) with host (pinned) alpha2 / P /
    Theta, until r_KKT(Theta_k) <= tol, for each step mode; iterations reported beside it."""
    import numpy as np
    import torch
    a_host = torch.tensor(I.alpha2).pin_memory().numpy()
    P_host = torch.tensor(I.P).pin_memory().numpy()
    th_host = torch.empty((I.M, I.N), dtype=torch.float64).pin_memory().numpy()
    F = q.qdt_build_probes(ctx, a_host, I.M)
    r0 = q.qdt_solve(ctx, F, P_host, I.gamma, 0.0, 0, theta_out=th_host)["info"]["kkt0"]
    del F
    res = {"r_kkt0": r0, "cap_iters": cap, "modes": {}}
    for name, accel, ke in [("SQS", False, 1), ("SQS-FISTA", True, 5)]:
        rows = {}
        for rho in rhos:
            barrier()
            t0 = time.perf_counter()
            F = q.qdt_build_probes(ctx, a_host, I.M)
            o = q.qdt_solve(ctx, F, P_host, I.gamma, rho * r0, cap, accel=accel, kkt_every=ke,
                            check_every=20, theta_out=th_host)
            barrier()
            dt = time.perf_counter() - t0
            del F
            inf = o["info"]
            rows[f"{rho:g}"] = {"converged": bool(inf["converged"]), "iters": int(inf["iters_done"]),
                                "seconds": dt, "f": float(inf["f_final"]),
                                "loop_ms_per_iter": inf["loop_ms"] / max(1, inf["iters_done"])}
            if not inf["converged"]:
                break
        res["modes"][name] = rows
    # objective-gap ladder: (f_k - f_ref) / (f_0 - f_ref) <= 1e-3, 1e-6 with f_ref the
    # minimum f of a 10x longer SQS-FISTA run; iterations from the trace of one call per mode at
    # tol = 0, seconds = that call's wall time scaled by the iteration fraction (cost per
    # iteration is constant), reported as derived
    fista_it = max([r["iters"] for r in res["modes"].get("SQS-FISTA", {}).values()] or [200])
    long_it = min(10 * fista_it, 4000)
    gap = {"f_ref_iters": long_it, "ladder": (1e-3, 1e-6), "modes": {}}
    traces = {}
    for name, accel, iters in [("SQS-FISTA", True, long_it), ("SQS", False, cap)]:
        barrier()
        t0 = time.perf_counter()
        F = q.qdt_build_probes(ctx, a_host, I.M)
        o = q.qdt_solve(ctx, F, P_host, I.gamma, 0.0, iters, accel=accel, kkt_every=5 if accel else 1,
                        theta_out=th_host)
        barrier()
        traces[name] = (np.asarray(o["trace"]), time.perf_counter() - t0)
        del F
    f_ref = float(np.nanmin(traces["SQS-FISTA"][0]))
    gap["f_ref"] = f_ref
    for name, (tr, dt) in traces.items():
        g = (tr - f_ref) / (tr[0] - f_ref)
        rows = {}
        for lv in gap["ladder"]:
            hit = np.nonzero(g <= lv)[0]
            k = int(hit[0]) if len(hit) else None
            rows[f"{lv:g}"] = {"iters": k, "seconds_derived": (dt * k / (len(tr) - 1)) if k else None}
        gap["modes"][name] = rows
    res["objective_gap"] = gap
    return res


# ------------------------------------------------------------------------------ oracle legs
def _slab_sample(I, Fo, n_slabs, rows_per_slab):
    """Sub-problems on S evenly spaced Fock-row slabs: the probes whose bands meet a slab, their
    bands clipped to it.  Same per-element arithmetic as a full oracle iteration."""
    import numpy as np
    slabs = []
    M = I.M
    for j in range(n_slabs):
        a = int((j + 0.5) * M / n_slabs - rows_per_slab / 2)
        a = max(0, min(M - rows_per_slab, a))
        b = a + rows_per_slab
        lo, hi = Fo.lo, Fo.lo + Fo.len - 1
        ds = np.nonzero((hi >= a) & (lo < b))[0]
        l2 = np.maximum(lo[ds], a)
        h2 = np.minimum(hi[ds], b - 1)
        ln = h2 - l2 + 1
        off = np.concatenate([[0], np.cumsum(ln)]).astype(np.int64)
        val = np.concatenate([Fo.val[Fo.off[d] + (l2[i] - lo[d]): Fo.off[d] + (h2[i] - lo[d]) + 1]
                              for i, d in enumerate(ds)]) if len(ds) else np.zeros(0)
        slabs.append(dict(lo=(l2 - a).astype(np.int64), len=ln.astype(np.int64), off=off,
                          val=np.ascontiguousarray(val), D=len(ds), M=rows_per_slab,
                          P=np.ascontiguousarray(I.P[ds])))
    return slabs


def _oracle_slab_step(o, s, theta, t, gamma):
    """One oracle iteration on a slab sub-problem: R = F Theta - P; G = F^T R + gamma L Theta;
    Theta <- P_S(Theta - t G) (oracle functions, in or_solve's order)."""
    import numpy as np
    L = o.lib()
    N = theta.shape[1]
    R = np.empty((s["D"], N))
    L.or_forward(s["lo"], s["len"], s["off"], s["val"], s["D"], theta, s["P"].ctypes.data, N, R)
    G = np.empty_like(theta)
    L.or_backward(s["lo"], s["len"], s["off"], s["val"], s["D"], s["M"], R, theta, N, gamma, G)
    X = theta - t[:, None] * G
    L.or_project_rows(np.ascontiguousarray(X), s["M"], N, theta)


def _oracle_sample_run(I, steps, warmup, rows_total, n_slabs=20):
    import numpy as np

    import oracle as o
    Fo = o.Probes(I.alpha2, I.M)
    rows = max(64, rows_total // n_slabs)
    slabs = _slab_sample(I, Fo, n_slabs, rows)
    thetas, ts = [], []
    for s in slabs:
        w = np.empty(s["M"])
        o.lib().or_sqs_weights(s["lo"], s["len"], s["off"], s["val"], s["D"], s["M"], I.gamma, w)
        ts.append(np.where(w > 0, 1.0 / np.where(w > 0, w, 1.0), 0.0))
        thetas.append(np.full((s["M"], I.N), 1.0 / I.N))
    for _ in range(warmup):
        for s, th, t in zip(slabs, thetas, ts):
            _oracle_slab_step(o, s, th, t, I.gamma)
    t0 = time.perf_counter()
    for _ in range(steps):
        for s, th, t in zip(slabs, thetas, ts):
            _oracle_slab_step(o, s, th, t, I.gamma)
    dt = time.perf_counter() - t0
    upd = steps * n_slabs * rows * I.N
    return upd / dt, dt, n_slabs * rows


def cpu_baseline(I, args):
    """The oracle timed on this host's cores (oracle-MT: every core, deterministic split, bit-
    identical to one thread), bounded sample (~10 s of CPU work); oracle-1T beside it."""
    import oracle as o
    try:
        ncpu = os.cpu_count() or 1
        # measured ~10 us per row-iteration single-threaded at N = 100
        rows1 = min(I.M, int(500000 * 100 / max(1, I.N)))
        o.set_threads(1)
        v1, dt1, r1 = _oracle_sample_run(I, 3, 1, rows1)
        o.set_threads(0)
        nt = o.get_threads()
        rowsm = min(I.M, rows1 * max(1, nt // 2))
        vm, dtm, rm = _oracle_sample_run(I, 3, 1, rowsm)
        return {"value": vm, "unit": UNIT, "cores": nt, "kind": "oracle",
                "sample": f"3 oracle-MT iterations (SQS) on {rm} Fock rows = 20 evenly spaced slabs of "
                          f"the {args.config} instance ({dtm:.1f} s, {nt} threads)",
                "oracle_1t": {"value": v1, "cores": 1,
                              "sample": f"3 iterations on {r1} Fock rows ({dt1:.1f} s)"},
                "host_cpu": _cpu_model(), "nproc": ncpu}
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "error": repr(e)}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    rank, _, world = env_rank()
    if rank != 0:
        return
    import oracle as o
    import qdt_synth as qs
    I = qs.CONFIGS[args.config]()
    o.set_threads(0)
    nt = o.get_threads()
    # size the per-step sample so that (steps + warmup) steps take ~150 s of CPU work on this
    # host (measured oracle cost ~8.5 us per row-iteration per thread at N = 100; ~half-linear
    # scaling assumed over the threads)
    per_row = 8.5e-6 * I.N / 100 / max(1.0, nt / 2)
    rows = int(150.0 / max(1, args.steps + args.warmup) / per_row)
    rows = max(20 * 64, min(I.M, rows))
    v, dt, r = _oracle_sample_run(I, args.steps, args.warmup, rows)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (qdt_synth, seed 0)",
            "config": {"workload": args.config, "M": I.M, "N": I.N, "D": I.D, "gamma": I.gamma,
                       "step_mode": "SQS", "parallelism": f"oracle-MT, {nt} threads"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nt, "kind": "oracle",
                             "sample": f"each step = one oracle iteration on {r} Fock rows "
                                       f"(20 evenly spaced slabs), {nt} threads", "host_cpu": _cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="qdt", choices=["qdt", "reference"])
    ap.add_argument("--config", default="megascale", help="/".join(CONFIG_NAMES))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-tol leg")
    ap.add_argument("--kkt-every", type=int, default=1,
                    help="evaluate r_KKT every k-th iteration in the timed loop (f is traced every iteration)")
    args = ap.parse_args()
    if args.config not in CONFIG_NAMES:
        ap.error(f"--config must be one of {CONFIG_NAMES}")
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_qdt(args)


if __name__ == "__main__":
    main()
