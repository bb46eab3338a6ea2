"""The N > 1 decomposition on CPU (-m "not gpu"): world_size-2 gloo processes run the exact
multi-GPU algorithm of libqdt with the oracle's per-shard
arithmetic, and must reproduce the single-process oracle solve.

Per rank g: Fock rows [k_g, k_{g+1}) from the library's host shard planner (qdt_shard_cuts,
callable without a GPU), the probe bands clipped to the slice, partial R_g = F_g Theta_g,
allreduce(sum) -> R = sum_g R_g - P (the residual exchange, "two steps"), halo
rows Theta[k_g - 1], Theta[k_{g+1}] by send/recv for the stencil (eq. regul),
local G, step and row projection (rows are independent), scalar allreduce.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import qdt_synth as qs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cuts(lo, hi, M, world):
    import paper_2404_02844_b200 as q
    return q.qdt_shard_cuts(lo, hi, M, world)


def _local_bands(F, kb, ke):
    """Bands of F clipped to rows [kb, ke), in slice-local row coordinates."""
    lo = np.maximum(F.lo, kb)
    hi = np.minimum(F.hi, ke - 1)
    ln = np.maximum(hi - lo + 1, 0).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(ln)]).astype(np.int64)
    val = np.zeros(max(1, off[-1]))
    for d in range(F.D):
        if ln[d]:
            a = F.off[d] + (lo[d] - F.lo[d])
            val[off[d]:off[d + 1]] = F.val[a:a + ln[d]]
    return np.ascontiguousarray(lo - kb, dtype=np.int64), ln, off, val


def _worker(rank, world, port, alpha2, M, P, gamma, iters, res):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = oracle.lib()
        F = oracle.Probes(alpha2, M)
        D, N = P.shape
        cuts = _cuts(F.lo, F.hi, M, world)
        kb, ke = int(cuts[rank]), int(cuts[rank + 1])
        Ml = ke - kb
        lo, ln, off, val = _local_bands(F, kb, ke)
        # SQS weights w = F^T (F 1) + 4 gamma (reading R2): s_d summed over ranks first
        s = np.array([val[off[d]:off[d + 1]].sum() for d in range(D)])
        st = torch.tensor(s)
        dist.all_reduce(st)
        s = st.numpy()
        w = np.full(Ml, 4.0 * gamma)
        for d in range(D):
            for j in range(ln[d]):
                w[lo[d] + j] += val[off[d] + j] * s[d]
        t = np.where(w > 0, 1.0 / np.where(w > 0, w, 1.0), 0.0)
        th = np.full((Ml, N), 1.0 / N)
        trace = []
        for _ in range(iters + 1):
            Rp = np.empty((D, N))
            L.or_forward(lo, ln, off, val, D, th, None, N, Rp)
            Rt = torch.tensor(Rp)
            dist.all_reduce(Rt)                        # residual exchange
            R = Rt.numpy() - P
            # halo rows (global rows kb - 1 and ke)
            up = torch.zeros(N, dtype=torch.float64)
            dn = torch.zeros(N, dtype=torch.float64)
            reqs = []
            if rank > 0:
                reqs.append(dist.isend(torch.tensor(th[0]), rank - 1))
                reqs.append(dist.irecv(up, rank - 1))
            if rank + 1 < world:
                reqs.append(dist.isend(torch.tensor(th[-1]), rank + 1))
                reqs.append(dist.irecv(dn, rank + 1))
            for r_ in reqs:
                r_.wait()
            ext = np.vstack([up.numpy()[None], th, dn.numpy()[None]])
            G = np.empty((Ml, N))
            L.or_backward(lo, ln, off, val, D, Ml, R, th, N, 0.0, G)
            kg = np.arange(kb, ke)
            lap = np.zeros_like(th)
            lap += np.where((kg > 0)[:, None], th - ext[:-2], 0.0)
            lap += np.where((kg < M - 1)[:, None], th - ext[2:], 0.0)
            G += gamma * lap
            # f = ||R||^2 + gamma * sum of the pairs (k, k+1) owned by this rank
            pair = np.where((kg < M - 1)[:, None], th - ext[2:], 0.0)
            reg = torch.tensor([np.sum(pair * pair)])
            dist.all_reduce(reg)
            trace.append(float(np.sum(R * R) + gamma * reg.item()))
            if len(trace) > iters:
                break
            X = th - t[:, None] * G
            th = oracle.project_rows(X)
        mx = int(np.diff(cuts).max())                  # gloo all_gather needs equal sizes
        mine = torch.zeros((mx, N), dtype=torch.float64)
        mine[:Ml] = torch.tensor(th)
        parts = [torch.zeros((mx, N), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, mine)
        if rank == 0:
            full = np.vstack([parts[g].numpy()[:int(cuts[g + 1] - cuts[g])] for g in range(world)])
            res.put((full, np.array(trace), cuts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fock_sharded_solve_matches_single_process(world):
    rng = np.random.default_rng(world)
    D, M, N = 60, 400, 6
    alpha2 = np.geomspace(0.5, 320.0, D)
    P = rng.dirichlet(np.ones(N), D)
    gamma, iters = 1e-2, 25
    ctx = mp.get_context("spawn")
    res = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, alpha2, M, P, gamma, iters, res))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    th, trace, cuts = res.get()
    ref = oracle.solve(oracle.Probes(alpha2, M), P, gamma, 0.0, iters)
    assert np.abs(th - ref["theta"]).max() <= 1e-12
    np.testing.assert_allclose(trace, ref["trace"], rtol=1e-12)
    assert cuts[0] == 0 and cuts[-1] == M and np.all(np.diff(cuts) > 0)


def test_shard_cuts_balance_cost():
    """qdt_shard_cuts (host planner): contiguous cuts at equal prefix sums of the per-row cost
    16 + 0.7 cov(k); on the Megascale bands every shard's cost is within one row of 1/n."""
    a2 = np.geomspace(1.0, 9e5, 10 ** 4)
    M = 10 ** 6
    lo, hi = np.array([oracle.band(m, M) for m in a2]).T
    cov = np.zeros(M + 1)
    np.add.at(cov, lo, 1)
    np.add.at(cov, hi + 1, -1)
    cost = 16 + 0.7 * np.cumsum(cov)[:M]
    for n in (2, 4, 8):
        cuts = _cuts(lo, hi, M, n)
        assert cuts[0] == 0 and cuts[-1] == M and np.all(np.diff(cuts) > 0)
        per = np.array([cost[cuts[g]:cuts[g + 1]].sum() for g in range(n)])
        assert np.abs(per - cost.sum() / n).max() <= cost.max() + 1e-6
    # a uniform Fock split would leave most of the banded work on the first GPU
    assert _cuts(lo, hi, M, 8)[1] < M // 8
