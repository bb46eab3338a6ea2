// qdt_wide.cu -- fused step kernel of the hot path for wide rows (N > 160 outcomes, up to
// N = 10 240: BASELINE's Stress configuration has N = 10^4, 80 KB per Fock row).
//
// One thread-block cluster of C CTAs owns a 32-row Fock tile across ALL N columns: CTA r of the
// cluster holds the column chunk [r Wc, (r + 1) Wc) (SURVEY 8(a) "Per-config kernel shape",
// Stress: "a 16-CTA cluster ... each CTA owning a 625-column chunk; X stays on chip; tau by
// cluster-wide Michelot reductions").  Per tile, in one kernel:
//   S3  G = F_tile^T R_win          fp64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA), operands
//                                   staged by bulk copies (TMA engine) in a 4-stage mbarrier ring
//   S4  G += gamma L Y              eq. regul, free ends (reading R8)
//   S6  KKT / regulariser partials  PAPER.md:563-567 (reading R7)
//   S5  X = Y - t o G, row-wise simplex projection (eq. Mp1_proj) by Michelot
//       rounds whose per-row sums / counts are combined over the cluster through distributed
//       shared memory (reading R4), Theta_{k+1} = max(X - tau, 0) stored from registers.
// G and X never reach HBM: per element the kernel reads Theta_k once from DRAM (plus Theta_{k-1}
// for FISTA) and writes Theta_{k+1} once; the R rows of the window come from L2.
//
// Layout of a CTA (512 threads, 16 warps): every warp holds both m-blocks of the 16-row tile and
// warp w the n-blocks [w NBW, (w + 1) NBW) of the chunk (8 columns each, NBW <= 5: 20 fp64
// accumulators per thread, so the epilogue has registers to spare).  In the DMMA accumulator
// layout a 4-lane quad (lane = 4 g + t) holds columns 8 nb + 2 t, 8 nb + 2 t + 1 of row g of an
// m-block, so a row's values are spread over one quad in each of the 16 warps and over the C CTAs: row
// reductions go quad (shuffles) -> CTA (shared memory, fixed n-group order) -> cluster (DSMEM,
// fixed CTA order).  Every CTA of the cluster combines the same partials in the same order, so
// all of them take identical tau / stop decisions and the result is bitwise deterministic.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>

#include "qdt_internal.h"
#include "qdt_ptx.cuh"

// Row bounds of the fused wide step (max X, min X, the minima of the trial / active sets) as
// integer keys and the final clamp by the sign bit (qdt_ptx.cuh: dkey, dclamp0).  A/B
// (profiles/r02_v8/ab_wik_stress_cut.jsonl): Stress-cut k_wstep 1.249 -> 1.206 ms (FISTA 1.798 ->
// 1.745), Stress 257.8 -> 254.4 ms per iteration.
#ifndef QDT_W_IKEY
#define QDT_W_IKEY 1
#endif

namespace qdt {

__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// staged Theta tile row pitch: = 8 mod 16 doubles (conflict-free 16-byte reads of 8 rows)
__host__ __device__ inline int wide_theta_pitch(int Wc) { return (Wc % 16 == 8) ? Wc : Wc + 8; }

__host__ __device__ inline size_t wide_ring_doubles(int Wc)
{
    const size_t ring = (size_t)WSTAGES * WKC * ((Wc + 4) + WFP);
    const size_t tile = (size_t)(WT + 2) * wide_theta_pitch(Wc);
    return ((ring > tile ? ring : tile) + 15) & ~(size_t)15;
}

size_t wide_step_smem(int Wc)
{
    return (wide_ring_doubles(Wc) + (size_t)2 * W_CMAX * WT * 8) * sizeof(double);
}

// combination of row partials by value kind: 0 min (G), 1 sum, 2 max, 3 min, 4 sum, 5 sum, 6 min
__device__ __forceinline__ double wcombine(int v, double x, double y)
{
    switch (v) {
        case 0:
        case 3:
        case 6: return dmin(x, y);
        case 2: return dmax(x, y);
        default: return x + y;
    }
}
template <int NBW, bool FIS>
__global__ void __launch_bounds__(W_THREADS, 1) k_wstep(const __grid_constant__ WStepArgs a)
{
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bars[WSTAGES + 1];   // chunk ring + the Theta tile
    __shared__ double rowp[WT][W_NG][8];   // per row and n-group warp: quad-reduced partials
    __shared__ double comb[8][WT];      // cluster totals per value and row
    __shared__ double ttry[WT];         // warm-start trial threshold per row (-inf: none)
    __shared__ double trow[WT][3];      // per row: tau, lambda (unclamped), lambda (clamped)
    __shared__ int tcnt[WT];            // per row: |A| of the last Michelot round
    __shared__ int tdone[WT];
    __shared__ int s_alldone;
    __shared__ double red[16][3];

    const DevState *st = a.state;
    if (st && st->stop) return;                    // cluster-uniform exits only
    const int64_t it = st ? st->it : 0;
    if (a.eval_gate && (it % a.kkt_every) != 0) return;
    const bool ev = a.eval != 0;
    constexpr bool fis = FIS;                      // FISTA step: Y = Theta_k + beta (Theta_k - Theta_{k-1})
    const double beta = fis ? a.beta[it] : 0.0;
    const bool do_kkt = ev || (!fis && (it % a.kkt_every) == 0);
    const int N = a.N, Nv = a.Nv, C = a.C;
    const int crank = C > 1 ? (int)cluster_ctarank() : 0;
    const int cid = blockIdx.x / C;
    const int cbase = crank * a.Wc;
    const int ncol = min(a.Wc, N - cbase);         // even (N even), > 0 (planner)
    const int Pr = a.Wc + 4;                       // staged R row pitch: = 4 mod 16 doubles
    const int Pt = wide_theta_pitch(a.Wc);         // staged Theta row pitch: = 8 mod 16 doubles
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int ng = warp;                           // n-group
    double *Rs = sm;                               // WSTAGES x WKC x Pr
    double *Fs = sm + WSTAGES * WKC * Pr;          // WSTAGES x WKC x WFP
    double *Ts = sm;                               // the Theta tile (rows k0 - 1 .. k0 + WT) reuses the ring
    // exchange slots after the ring: xin[2][W_CMAX][WT][8], slot [r] holds CTA r's partials (pushed by r)
    auto xin = reinterpret_cast<double(*)[W_CMAX][WT][8]>(sm + wide_ring_doubles(a.Wc));
    const int ta = a.toff[cid], tb = a.toff[cid + 1];   // this cluster's tiles a.tlist[ta .. tb)

    // zero the stages once: a masked tail k-step then multiplies stale but finite values by 0
    for (int i = tid; i < WSTAGES * WKC * (Pr + WFP); i += W_THREADS) sm[i] = 0.0;
    if (tid == 0) {
        for (int s = 0; s <= WSTAGES; s++) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    fence_proxy_async_smem();
    __syncthreads();

    // ---- producer (warp 0): chunk c of tile tt into the ring slot of the running chunk count
    uint32_t issued = 0, used = 0, tuse = 0;
    auto issue_chunk = [&](int tt, int c) {        // warp 0, all lanes
        const int t64 = tt >> 2, quarter = tt & 3;
        const int dA = a.tile_dA[t64], W = a.tile_dB[t64] - dA;
        const int p0 = c * WKC, kc = min(WKC, W - p0);
        const int stg = issued % WSTAGES;
        uint64_t *bar = &bars[stg];
        if (lane == 0) mbar_expect_tx(bar, (uint32_t)kc * (WFP + ncol) * 8u);
        __syncwarp();
        if (lane < kc) {
            bulk_g2s(Fs + (stg * WKC + lane) * WFP, a.Fb + a.fb_off[t64] + (int64_t)(p0 + lane) * STP + quarter * WT,
                     WFP * 8u, bar);
            bulk_g2s(Rs + (stg * WKC + lane) * Pr, a.R + (int64_t)(dA + p0 + lane) * N + cbase, (uint32_t)ncol * 8u,
                     bar);
        }
        issued++;
    };
    auto nchunks = [&](int tt) {
        const int t64 = tt >> 2;
        return (a.tile_dB[t64] - a.tile_dA[t64] + WKC - 1) / WKC;
    };
    auto start_tile = [&](int tt) {                // warp 0: the first ring's worth of a tile's chunks
        const int n = min(WSTAGES, nchunks(tt));
        for (int c = 0; c < n; c++) issue_chunk(tt, c);
    };
    if (warp == 0 && ta < tb) start_tile(a.tlist[ta]);

    double sreg = 0.0, skkt = 0.0, skktp = 0.0;    // per-thread running partials (fixed order)
    int slot = 0;
    int nexch = 0;                                 // cluster exchanges (diagnostic, SC_DTH)
#ifdef QDT_WPROF
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tq0 = clock64(), tq1;
    long long nchk = 0;
#define QDT_PH(i) (tq1 = clock64(), ph[i] += tq1 - tq0, tq0 = tq1)
#else
#define QDT_PH(i) ((void)0)
#endif
    const double *Fw = Fs + t * WFP + g;                      // A fragment: F[4 ks + t][8 mb + g]
    const double *Rw = Rs + t * Pr + 8 * ng * NBW + g;        // B fragment: R[4 ks + t][8 nb + g]

    // this CTA's partial into slot [crank] of every CTA of the cluster (remote shared-memory stores,
    // made visible by the release / acquire of the cluster barrier)
    auto push = [&](double *dst, double x) {
        if (C == 1) {
            *dst = x;
            return;
        }
        for (int r = 0; r < C; r++) st_dsmem(dst, (uint32_t)r, x);
    };
    // cluster-wide barrier after the pushes: every CTA then combines all C partials locally in CTA order
    auto exchange = [&]() {
        nexch++;
        if (C > 1)
            cluster_sync_all();
        else
            __syncthreads();
    };

    for (int ti = ta; ti < tb; ti++) {
        const int tt = a.tlist[ti];
        const int t64 = tt >> 2;
        const int k0 = tt * WT;                    // local first row of the tile
        const int Tt = min(WT, a.Ml - k0);
        const int W = a.tile_dB[t64] - a.tile_dA[t64];
        const int nch = (W + WKC - 1) / WKC;
#ifdef QDT_WPROF
        nchk += nch;
#endif
        QDT_PH(0);
        if (warp == 1) {                           // Theta rows of the epilogue -> L2 while the GEMM runs
            for (int r = lane; r < Tt + 2; r += 32) {
                bulk_prefetch_l2(a.theta + (int64_t)(k0 - 1 + r) * N + cbase, (uint32_t)ncol * 8u);
                if (fis) bulk_prefetch_l2(a.theta_prev + (int64_t)(k0 - 1 + r) * N + cbase, (uint32_t)ncol * 8u);
            }
        }
        if (tid < WT) {   // warm start: the row's previous threshold, lowered a little (a trial lower bound)
            double tr = -INFINITY;
            if (!ev && a.tau_prev && tid < Tt) {
                const double tp = a.tau_prev[k0 + tid];
                if (isfinite(tp)) tr = tp - 0x1p-10 * fmax(fabs(tp), 1e-300);
            }
            ttry[tid] = tr;
        }
        // the rows' step weights, loaded before the GEMM to hide their latency
        double tk[2];
#pragma unroll
        for (int i = 0; i < 2; i++)
            tk[i] = (8 * i + g < Tt) ? (a.tscal ? *a.tscal : __ldg(a.tstep + k0 + 8 * i + g)) : 0.0;
        double acc[2][NBW][2];
#pragma unroll
        for (int i = 0; i < 2; i++)
#pragma unroll
            for (int j = 0; j < NBW; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
        // ---- S3: G = F_tile^T R_win
        for (int c = 0; c < nch; c++) {
            const int stg = used % WSTAGES;
            mbar_wait(&bars[stg], (used / WSTAGES) & 1);
            used++;
            const int kc = min(WKC, W - c * WKC);
            const double *Fc = Fw + stg * WKC * WFP;
            const double *Rc = Rw + stg * WKC * Pr;
#pragma unroll
            for (int ks = 0; ks < WKC / 4; ks++) {
                if (4 * ks < kc) {
                    const bool ok = 4 * ks + t < kc;
                    const double a0 = ok ? Fc[4 * ks * WFP] : 0.0;
                    const double a1 = ok ? Fc[4 * ks * WFP + 8] : 0.0;
#pragma unroll
                    for (int j = 0; j < NBW; j++) {
                        const double b = Rc[4 * ks * Pr + 8 * j];
                        dmma(acc[0][j][0], acc[0][j][1], a0, b);
                        dmma(acc[1][j][0], acc[1][j][1], a1, b);
                    }
                }
            }
            __syncthreads();                       // stage consumed
            if (warp == 0 && c + WSTAGES < nch) issue_chunk(tt, c + WSTAGES);
        }
        QDT_PH(1);
        // the ring is drained: the Theta tile (rows k0 - 1 .. k0 + Tt) lands in its space (plain
        // steps and evaluation passes; the FISTA step reads Theta_k / Theta_{k-1} through L2)
        if (!fis && warp == 0) {
            uint64_t *bar = &bars[WSTAGES];
            if (lane == 0) mbar_expect_tx(bar, (uint32_t)(Tt + 2) * ncol * 8u);
            __syncwarp();
            for (int r = lane; r < Tt + 2; r += 32)
                bulk_g2s(Ts + r * Pt, a.theta + (int64_t)(k0 - 1 + r) * N + cbase, (uint32_t)ncol * 8u, bar);
        }
        if (warp == 2 && ti + 1 < tb) {            // next tile's first chunks -> L2 during the epilogue
            const int t1 = a.tlist[ti + 1] >> 2;
            const int n1 = min(WSTAGES * WKC, a.tile_dB[t1] - a.tile_dA[t1]);
            for (int r = lane; r < n1; r += 32)
                bulk_prefetch_l2(a.R + (int64_t)(a.tile_dA[t1] + r) * N + cbase, (uint32_t)ncol * 8u);
        }
        if (!fis) {
            mbar_wait(&bars[WSTAGES], tuse & 1);
            tuse++;
        }
        QDT_PH(2);

        // ---- S4 + pass 1: G = acc + gamma L Y; row min of G, sum / max / min of X = Y - t G
        double pmn[2], ps[2], pxm[2], pxn[2], pts[2], ptc[2], ptm[2];
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const int rl = 8 * i + g;
            const int kl = k0 + rl;
            const bool act = rl < Tt;
            const int64_t kg = a.kb + kl;
            const bool hp = kg > 0, hn = kg + 1 < a.M;
            const double tau_t = ttry[rl];
            double mn = INFINITY, s = 0.0, xm = -INFINITY, xn = INFINITY;
            double ts = 0.0, tm = INFINITY;
            int tc = 0;
            int kxm = DKEY_NINF, kxn = DKEY_PINF, ktm = DKEY_PINF;   // QDT_W_IKEY: bounds as integer keys (dkey)
            if (act) {
                const double *thg = a.theta + (int64_t)kl * N + cbase;
                const double *ths = Ts + (rl + 1) * Pt;
                const double *tq = fis ? a.theta_prev + (int64_t)kl * N + cbase : nullptr;
#pragma unroll
                for (int j = 0; j < NBW; j++) {
                    const int lc = 8 * (ng * NBW + j) + 2 * t;
                    if (lc < ncol) {
                        double2 x, y, z;
                        if (fis) {
                            x = __ldg(reinterpret_cast<const double2 *>(thg + lc));
                            y = hp ? __ldg(reinterpret_cast<const double2 *>(thg + lc - N)) : x;
                            z = hn ? __ldg(reinterpret_cast<const double2 *>(thg + lc + N)) : x;
                        } else {
                            x = *reinterpret_cast<const double2 *>(ths + lc);
                            y = hp ? *reinterpret_cast<const double2 *>(ths + lc - Pt) : x;
                            z = hn ? *reinterpret_cast<const double2 *>(ths + lc + Pt) : x;
                        }
                        double y0[2] = {x.x, x.y}, yp[2] = {y.x, y.y}, yn[2] = {z.x, z.y};
                        const double d20 = x.x - z.x, d21 = x.y - z.y;   // regulariser pair of Theta_k
                        const bool v0 = cbase + lc < Nv, v1 = cbase + lc + 1 < Nv;
                        if (v0) sreg = fma(d20, d20, sreg);
                        if (v1) sreg = fma(d21, d21, sreg);
                        if (fis) {
                            const double2 xq = __ldg(reinterpret_cast<const double2 *>(tq + lc));
                            const double2 yq = hp ? __ldg(reinterpret_cast<const double2 *>(tq + lc - N)) : xq;
                            const double2 zq = hn ? __ldg(reinterpret_cast<const double2 *>(tq + lc + N)) : xq;
                            y0[0] = fma(beta, x.x - xq.x, x.x), y0[1] = fma(beta, x.y - xq.y, x.y);
                            yp[0] = hp ? fma(beta, y.x - yq.x, y.x) : y0[0];
                            yp[1] = hp ? fma(beta, y.y - yq.y, y.y) : y0[1];
                            yn[0] = hn ? fma(beta, z.x - zq.x, z.x) : y0[0];
                            yn[1] = hn ? fma(beta, z.y - zq.y, z.y) : y0[1];
                        }
#pragma unroll
                        for (int e = 0; e < 2; e++) {
                            const double gv = fma(a.gamma, (y0[e] - yp[e]) + (y0[e] - yn[e]), acc[i][j][e]);
                            acc[i][j][e] = gv;
                            if (e ? v1 : v0) {
                                mn = dmin(mn, gv);
                                const double xv = fma(-tk[i], gv, y0[e]);
                                s += xv;
#if QDT_W_IKEY
                                const int kx = dkey(xv);
                                kxm = max(kxm, kx);
                                kxn = min(kxn, kx);
#else
                                xm = dmax(xm, xv);
                                xn = dmin(xn, xv);
#endif
                                if (xv > tau_t) {   // first Michelot round at the trial threshold
                                    ts += xv;
                                    tc++;
#if QDT_W_IKEY
                                    ktm = min(ktm, kx);
#else
                                    tm = dmin(tm, xv);
#endif
                                }
                            }
                        }
                    }
                }
            }
            pmn[i] = quad_min(mn);
            ps[i] = quad_sum(s);
#if QDT_W_IKEY
            pxm[i] = dkey_floor(quad_max_i(kxm));   // <= max X
            pxn[i] = dkey_floor(quad_min_i(kxn));   // <= min X
#else
            pxm[i] = quad_max(xm);
            pxn[i] = quad_min(xn);
#endif
            pts[i] = quad_sum(ts);
            ptc[i] = (double)quad_sum_i(tc);
#if QDT_W_IKEY
            ptm[i] = dkey_floor(quad_min_i(ktm));   // <= min of the trial active set
#else
            ptm[i] = quad_min(tm);
#endif
        }
        if (t == 0) {
#pragma unroll
            for (int i = 0; i < 2; i++) {
                double *rp = rowp[8 * i + g][ng];
                rp[0] = pmn[i], rp[1] = ps[i], rp[2] = pxm[i], rp[3] = pxn[i];
                rp[4] = pts[i], rp[5] = ptc[i], rp[6] = ptm[i];
            }
        }
        __syncthreads();
        QDT_PH(7);
        if (tid < 7 * WT) {                        // CTA partial of (row, value) (n-group order), pushed to every CTA
            const int row = tid % WT, v = tid / WT;
            double x = rowp[row][0][v];
            for (int w = 1; w < W_NG; w++) x = wcombine(v, x, rowp[row][w][v]);
            push(&xin[slot][crank][row][v], x);
        }
        exchange();
        if (tid < 7 * WT) {                        // cluster total of (row, value) in CTA order
            const int row = tid % WT, v = tid / WT;
            double x = xin[slot][0][row][v];
            for (int r = 1; r < C; r++) x = wcombine(v, x, xin[slot][r][row][v]);
            comb[v][row] = x;
        }
        __syncthreads();
        if (tid < WT) {                            // lambda, tau_0, warm-started first round
            const double mn = comb[0][tid], s = comb[1][tid], xm = comb[2][tid], xn = comb[3][tid];
            const double lam = -2.0 * mn;
            trow[tid][1] = lam;
            trow[tid][2] = fmax(lam, 0.0);
            // tau_0 = (sum X - 1) / N is exact when every entry stays active; otherwise Michelot
            // from a lower bound (reading R4): the trial threshold when phi(tau_try) =
            // sum_{x > tau_try} (x - tau_try) >= 1 proves it one (its round is then already
            // done), else max(tau_0, max X - 1)
            double tau = (s - 1.0) / (double)Nv;
            bool done = tid >= Tt || xn > tau;
            int cnt = Nv + 1;
            if (!done) {
                const double tt_ = ttry[tid], st_ = comb[4][tid], mt_ = comb[6][tid];
                const int ct_ = (int)comb[5][tid];
                if (ct_ > 0 && st_ - (double)ct_ * tt_ >= 1.0) {
                    cnt = ct_;
                    tau = (st_ - 1.0) / (double)ct_;
                    done = mt_ > tau;
                } else {
                    tau = fmax(tau, xm - 1.0);
                }
            }
            trow[tid][0] = tau;
            tdone[tid] = done ? 1 : 0;
            tcnt[tid] = cnt;
            const unsigned all = __ballot_sync(W_LANES, done);
            if (tid == 0) s_alldone = (all == W_LANES);
        }
        __syncthreads();
        slot ^= 1;
        QDT_PH(3);

        // ---- pass 2: KKT terms with lambda; X = Y - t G in the accumulators
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const int rl = 8 * i + g;
            const int kl = k0 + rl;
            const bool act = rl < Tt;
            const double lam = trow[rl][1], lamp = trow[rl][2];
            const double *thg = a.theta + (int64_t)kl * N + cbase;
            const double *ths = Ts + (rl + 1) * Pt;
            const double *tq = fis ? a.theta_prev + (int64_t)kl * N + cbase : nullptr;
#pragma unroll
            for (int j = 0; j < NBW; j++) {
                const int lc = 8 * (ng * NBW + j) + 2 * t;
                const bool in = act && lc < ncol;
                double2 x = make_double2(0.0, 0.0);
                if (in) x = fis ? __ldg(reinterpret_cast<const double2 *>(thg + lc)) : *reinterpret_cast<const double2 *>(ths + lc);
                double y0[2] = {x.x, x.y};
                if (fis && in) {
                    const double2 xq = __ldg(reinterpret_cast<const double2 *>(tq + lc));
                    y0[0] = fma(beta, x.x - xq.x, x.x), y0[1] = fma(beta, x.y - xq.y, x.y);
                }
                const double th2[2] = {x.x, x.y};
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const bool v = in && cbase + lc + e < Nv;
                    const double gv = acc[i][j][e];
                    if (do_kkt && v) {
                        const double k1 = th2[e] * fma(2.0, gv, lam);
                        skkt = fma(k1, k1, skkt);
                        if (ev) {
                            const double k2 = th2[e] * fma(2.0, gv, lamp);
                            skktp = fma(k2, k2, skktp);
                        }
                    }
                    acc[i][j][e] = v ? fma(-tk[i], gv, y0[e]) : -INFINITY;
                }
            }
        }
        // the Theta tile is consumed: the next tile's chunks may refill the ring now, under the
        // Michelot rounds and the stores of this one
        __syncthreads();
        if (warp == 0 && ti + 1 < tb) start_tile(a.tlist[ti + 1]);
        QDT_PH(4);
        if (ev) continue;                          // evaluation pass: no step

        // ---- S5: Michelot rounds, all rows of the tile in lockstep over the cluster
        while (!s_alldone) {
            double rps[2], rpc[2], rmA[2];
#pragma unroll
            for (int i = 0; i < 2; i++) {
                const int rl = 8 * i + g;
                const double tau = trow[rl][0];
                double sA = 0.0, mA = INFINITY;
                int cA = 0, kmA = DKEY_PINF;
                if (!tdone[rl]) {
#pragma unroll
                    for (int j = 0; j < NBW; j++)
#pragma unroll
                        for (int e = 0; e < 2; e++) {
                            const double x = acc[i][j][e];
                            if (x > tau) {
                                sA += x;
                                cA++;
#if QDT_W_IKEY
                                kmA = min(kmA, dkey(x));
#else
                                mA = dmin(mA, x);
#endif
                            }
                        }
                }
                rps[i] = quad_sum(sA);
                rpc[i] = (double)quad_sum_i(cA);
#if QDT_W_IKEY
                rmA[i] = dkey_floor(quad_min_i(kmA));   // <= min_A X: stops early only when certain
#else
                rmA[i] = quad_min(mA);
#endif
            }
            if (t == 0) {
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    double *rp = rowp[8 * i + g][ng];
                    rp[0] = rps[i], rp[1] = rpc[i], rp[2] = rmA[i];
                }
            }
            __syncthreads();
            if (tid < 3 * WT) {
                const int row = tid % WT, v = tid / WT;   // 0: sum, 1: count (sums), 2: min
                const int op = v == 2 ? 3 : 1;
                double x = rowp[row][0][v];
                for (int w = 1; w < W_NG; w++) x = wcombine(op, x, rowp[row][w][v]);
                push(&xin[slot][crank][row][v], x);
            }
            exchange();
            if (tid < 3 * WT) {
                const int row = tid % WT, v = tid / WT;
                const int op = v == 2 ? 3 : 1;
                double x = xin[slot][0][row][v];
                for (int r = 1; r < C; r++) x = wcombine(op, x, xin[slot][r][row][v]);
                comb[v][row] = x;
            }
            __syncthreads();
            if (tid < WT) {
                const double s = comb[0][tid], cntd = comb[1][tid], mA = comb[2][tid];
                bool done = tdone[tid] != 0;
                if (!done) {
                    const int cnt = (int)cntd;
                    if (cnt >= tcnt[tid]) {
                        done = true;
                    } else {
                        tcnt[tid] = cnt;
                        const double tau = (s - 1.0) / (double)cnt;
                        trow[tid][0] = tau;
                        done = mA > tau;
                    }
                }
                tdone[tid] = done ? 1 : 0;
                const unsigned all = __ballot_sync(W_LANES, done);
                if (tid == 0) s_alldone = (all == W_LANES);
            }
            __syncthreads();
            slot ^= 1;
        }
        QDT_PH(5);
        // ---- Theta_{k+1} = max(X - tau, 0), stored from registers
        if (a.tau_prev && tid < Tt && crank == 0) a.tau_prev[k0 + tid] = trow[tid][0];
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const int rl = 8 * i + g;
            if (rl >= Tt) continue;
            const double tau = trow[rl][0];
            double *o = a.out + (int64_t)(k0 + rl) * N + cbase;
#pragma unroll
            for (int j = 0; j < NBW; j++) {
                const int lc = 8 * (ng * NBW + j) + 2 * t;
                if (lc < ncol) {
                    const double o0 = acc[i][j][0] - tau, o1 = acc[i][j][1] - tau;
#if QDT_W_IKEY
                    *reinterpret_cast<double2 *>(o + lc) = make_double2(dclamp0(o0), dclamp0(o1));
#else
                    *reinterpret_cast<double2 *>(o + lc) = make_double2(o0 > 0.0 ? o0 : 0.0, o1 > 0.0 ? o1 : 0.0);
#endif
                }
            }
        }
    }
    QDT_PH(6);
#ifdef QDT_WPROF
    if ((blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && tid == 0 && it == 5)
        printf("[wprof] cta %d tiles %d chunks %lld exch %d | gemm %.0f thwait %.0f pass1 %.0f ex1 %.0f pass2 %.0f rounds %.0f store %.0f (kcycles)\n",
               blockIdx.x, tb - ta, nchk, nexch, (ph[0] + ph[1]) / 1e3, ph[2] / 1e3, ph[7] / 1e3, ph[3] / 1e3, ph[4] / 1e3,
               ph[5] / 1e3, ph[6] / 1e3);
#endif
    // ---- per-CTA scalar partials (fixed order: lanes, then warps)
    sreg = wsum(sreg);
    skkt = wsum(skkt);
    skktp = wsum(skktp);
    if (lane == 0) {
        red[warp][0] = skkt;
        red[warp][1] = skktp;
        red[warp][2] = sreg;
    }
    __syncthreads();
    if (tid == 0) {
        double v0 = 0.0, v1 = 0.0, v2 = 0.0;
        for (int w = 0; w < 16; w++) {
            v0 += red[w][0];
            v1 += red[w][1];
            v2 += red[w][2];
        }
        double *p = a.part + (int64_t)blockIdx.x * NSC_TILE;
        if (do_kkt) {
            p[SC_KKT] = v0;
            p[SC_KKTP] = v1;
        }
        p[SC_REG] = v2;
        p[SC_DTH] = (double)nexch;
    }
    if (C > 1) cluster_sync_all();                 // no CTA leaves while a peer may read its slots
}

// ---- host side
template <int NBW>
static cudaError_t launch_nbw(const WStepArgs &a, int grid, size_t smem, cudaStream_t s)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(W_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const bool fis = a.beta != nullptr && !a.eval;
    return fis ? cudaLaunchKernelEx(&cfg, k_wstep<NBW, true>, a) : cudaLaunchKernelEx(&cfg, k_wstep<NBW, false>, a);
}

#define QDT_FOR_NBW(X) X(1) X(2) X(3) X(4) X(5)

int wide_nbw(int Wc) { return (Wc / 8 + W_NG - 1) / W_NG; }

cudaError_t prepare_wide_kernels()
{
    static uint64_t done_mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0;
    if (done_mask & bit) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    const int smax = (int)std::max(wide_step_smem(8 * W_NG * W_NBW_MAX), wide_step_smem(8 * W_NG * W_NBW_MAX - 8));
#define QDT_PREP1(n, f)                                                                                        \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_wstep<n, f>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax); \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_wstep<n, f>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
#define QDT_PREP(n) QDT_PREP1(n, false) QDT_PREP1(n, true)
    QDT_FOR_NBW(QDT_PREP)
#undef QDT_PREP
#undef QDT_PREP1
    if (e == cudaSuccess) done_mask |= bit;
    return e;
}

// Clusters of C CTAs that can be co-resident (0 on error)
int wide_max_clusters(int C, int Wc)
{
    const int nbw = wide_nbw(Wc);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C * 256);
    cfg.blockDim = dim3(W_THREADS);
    cfg.dynamicSmemBytes = wide_step_smem(Wc);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaErrorInvalidValue;
    switch (nbw) {
#define QDT_CASE(k) \
    case k: e = cudaOccupancyMaxActiveClusters(&n, k_wstep<k, false>, &cfg); break;
        QDT_FOR_NBW(QDT_CASE)
#undef QDT_CASE
        default: break;
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

cudaError_t launch_wide_step(const WStepArgs &a, int nclusters, cudaStream_t s)
{
    if (nclusters <= 0) return cudaSuccess;
    const int grid = nclusters * a.C;
    const size_t smem = wide_step_smem(a.Wc);
    switch (wide_nbw(a.Wc)) {
#define QDT_CASE(k) \
    case k: return launch_nbw<k>(a, grid, smem, s);
        QDT_FOR_NBW(QDT_CASE)
#undef QDT_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qdt
