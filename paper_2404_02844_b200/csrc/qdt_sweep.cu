// qdt_sweep.cu -- fp64 tensor-core (DMMA) sweep kernels of the hot path for N <= 8*NB_MAX outcomes.
//
// One projected-gradient iteration on the "sweep" path:
//   k_fwd_mma    S2  partial R rows: for a run of Fock tiles and the union of their probe windows,
//                    Rpart = F_blk Theta_tile (mma.sync m8n8k4 f64, A = tiled F, B = Theta tile).
//   k_reduce_R2  S2  R[d,:] = sum of the partial rows of probe d (fixed order) - P[d,:], ||R||^2.
//   k_bwd_mma    S3-S6 per Fock tile of ST = 64 rows: G = F_tile^T R_win (DMMA, split-K for wide
//                    windows), then in registers: gamma L Theta (eq. regul), KKT
//                    partials, X = Theta - t o G, row-wise simplex projection
//                    (eq. Mp1_proj) by Michelot rounds over the 4-lane quad that owns
//                    the row in the DMMA accumulator layout, Theta_next stored straight from registers.
//   k_scalars2   S6  deterministic two-level reduction of the per-tile partials + trace / stop flag.
// Operands reach shared memory by cp.async.bulk (TMA bulk engine) completing on mbarriers, double
// buffered.  F is pre-tiled once per probe handle (k_tile_F): for every Fock tile a dense block of
// (window probes) x STP doubles, zero outside each band, so a staged chunk is one contiguous copy.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include <limits.h>

#include "qdt_internal.h"
#include "qdt_ptx.cuh"

// Row-epilogue forms (A/B on one B200, profiles/r02_v8/ab_ikey.md):
//  - max(X - tau, 0) by the sign bit (dclamp0): Megascale k_bwd_mma 0.5006 -> 0.4950 ms, the paper's
//    shape 0.967 -> 0.946 ms; on for every N.
//  - row max / min bounds and the Michelot active minimum as integer keys (dkey): 9 % fewer warp
//    instructions, the paper's shape (NB = 19, one CTA per SM) 0.967 -> 0.919 ms, but Megascale
//    (NB = 13, two CTAs per SM at the 128-register cap) 0.5006 -> 0.513 ms (more spill reloads):
//    on from QDT_IKEY_MIN_NB column blocks up.
#ifndef QDT_IKEY_MIN_NB
#define QDT_IKEY_MIN_NB 17
#endif
// the N-split kernel (k_bwd_split: half a row per thread, 28 accumulator registers) also takes the
// keys: Megascale FISTA step 0.7047 -> 0.6984 ms (profiles/r02_v8/ab_ikp_megascale_fista.jsonl)
#ifndef QDT_IKEY_PAIR
#define QDT_IKEY_PAIR 1
#endif
#ifndef QDT_ICLAMP
#define QDT_ICLAMP 1
#endif
// Scalar partials of k_bwd_mma from QDT_ACC_MIN_NB column blocks up (one CTA per SM, no register
// cap): each thread keeps running sums over the CTA's unsplit tiles in shared memory and the CTA
// reduces them once, at the end (its total goes to the slot of its last unsplit tile, the earlier
// slots get zeros; the unit -> CTA map is static, so the order is fixed).  Below it: a block
// reduction per tile.  A/B (profiles/r02_v8/ab_acc_*.jsonl): the paper's shape k_bwd_mma<19>
// 0.908 -> 0.865 ms; Megascale (NB = 13, two CTAs per SM at 128 registers) 0.493 -> 0.556 ms
// (spills 144 -> 388 bytes), and neutral with a block barrier kept per tile.
#ifndef QDT_ACC_MIN_NB
#define QDT_ACC_MIN_NB 17
#endif

namespace qdt {

// A 16-byte aligned bulk copy that covers n doubles starting at src: returns the element shift
// (0 or 1) at which src[0] lands in dst and the byte count to copy.  The caller's buffers carry
// >= 2 doubles of slack after the last element (the copy may run 8 bytes past either end of the
// range, never past the allocation).
__device__ __forceinline__ void aligned_span(const double *src, int64_t n, const double **gsrc,
                                             int *shift, uint32_t *bytes)
{
    const uintptr_t a = (uintptr_t)src;
    const int sh = (int)((a & 15) >> 3);
    *gsrc = src - sh;
    *shift = sh;
    *bytes = (uint32_t)((((n + sh) * 8) + 15) & ~(int64_t)15);
}

// ------------------------------------------------------------------------------ setup
// Tiled F (once per probe handle): block of tile t at fb_off[t], row j = probe tile_dA[t] + j,
// column r = F[d][kb + t*ST + r] (0 outside the band and beyond the slice), r in [0, STP).
__global__ void k_tile_F(Band b, int64_t kb, int Ml, const int32_t *tile_dA, const int32_t *tile_dB,
                         const int64_t *fb_off, double *Fb)
{
    const int t = blockIdx.x;
    const int dA = tile_dA[t], W = tile_dB[t] - dA;
    const int k0 = t * ST;
    double *blk = Fb + fb_off[t];
    for (int e = threadIdx.x; e < W * STP; e += blockDim.x) {
        const int j = e / STP, r = e - j * STP;
        const int d = dA + j;
        const int kl = k0 + r;
        double v = 0.0;
        if (r < ST && kl < Ml) {
            const int64_t kg = kb + kl;           // band rows are global indices
            const int64_t lo = b.lo[d], len = b.len[d];
            if (kg >= lo && kg < lo + len) v = b.val[b.off[d] + (kg - lo)];
        }
        blk[e] = v;
    }
}

// ------------------------------------------------------------------------------ row epilogue
// One Fock row k held by a quad (4 lanes, t4 = lane & 3) in the DMMA accumulator layout: columns
// c = 8 nb + 2 t4 + i.  On entry acc = (F^T R)[k, c]; thr points at Theta_k[k, 0] in shared
// memory with rows k-1 and k+1 at -N and +N.  Steps:
//   G = acc + gamma (L Theta)_k                        eq. regul, ends: reading R8
//   sreg += (Theta_k - Theta_{k+1})^2                  regulariser value of the pair (k, k+1)
//   KKT:  lam = -min_n 2G;  skkt += (Theta (2G + lam))^2      PAPER.md:563-567, reading R7
//   X = Theta - t_k G;  tau by Michelot rounds;  out = max(X - tau, 0)   eq. Mp1_proj, reading R4
// NB = ceil(N/8): only the last n-block can hold columns >= N; they are neutralised (+inf for the
// row min, -inf for X) and never stored.  FULL: an interior row of a full tile (row active,
// neighbours k-1 and k+1 exist): no per-row predicates.  EVEN: N even, pairs move as double2.
// Row-pair exchange of the N-split kernel: warps mb and mb + 8 hold the two column halves of the
// same 8 rows; each reduction publishes the quad value of each row and reads the partner's after
// a 64-thread named barrier (id 1 + mb).  Two slots alternate, so one barrier per exchange.
struct PairX {
    double *buf;   // [2 slots][8 m-blocks][2 halves][8 rows][4]
    int slot, mb, h, g4, t4;
};
template <int K>
__device__ __forceinline__ void pair_xchg(PairX &px, const double (&v)[K], double (&o)[K])
{
    double *mine = px.buf + (((px.slot * 8 + px.mb) * 2 + px.h) * 8 + px.g4) * 4;
    const double *other = px.buf + (((px.slot * 8 + px.mb) * 2 + (1 - px.h)) * 8 + px.g4) * 4;
    if (px.t4 == 0)
#pragma unroll
        for (int k = 0; k < K; k++) mine[k] = v[k];
    asm volatile("bar.sync %0, 64;" ::"r"(1 + px.mb) : "memory");
#pragma unroll
    for (int k = 0; k < K; k++) o[k] = other[k];
    px.slot ^= 1;
}

// FIS (FISTA): tpr points at Theta_{k-1}[k, 0]; the stencil and X use the extrapolated point
// Y = Theta_k + beta (Theta_k - Theta_{k-1}), the regulariser value uses Theta_k itself (f(Theta_k)),
// and the KKT of Theta_k comes from a separate evaluation pass (do_kkt must be false).
// NBA / CB (N-split kernel): the thread holds NBA column blocks starting at global block CB / 8;
// global blocks >= NB are padding.  PAIR: the row is shared with the partner warp holding the
// other column half; every row reduction is completed through PairX (fixed combination order).
struct NoMid {
    __device__ void operator()() const {}
};
// STASH: the row's own Theta values are kept in registers from pass 1, so that shared memory is
// not read after pass 1 and mid() (called between the passes by every thread) may release the
// tile (the persistent kernel issues the next unit's tile load there).
template <int NB, bool FULL, bool EVEN, bool SMEM_OUT, bool FIS = false, int NBA = NB, int CB = 0,
          bool PAIR = false, bool STASH = false, class Mid = NoMid>
__device__ __forceinline__ void row_pass(double (&acc)[NBA][2], const double *thr, int N, int t4,
                                         bool act, bool has_prev, bool has_next, double gamma,
                                         double tk, bool do_kkt, bool want_kktp, double &sreg,
                                         double &skkt, double &skktp, double &s, double &xm,
                                         double &xn, const double *tpr = nullptr, double beta = 0.0,
                                         PairX *px = nullptr, Mid mid = Mid(), int pitch = -1)
{
    const int TPp = pitch < 0 ? N : pitch;   // row pitch of the staged Theta tile(s)
    double keep[STASH ? NBA : 1][2];
    const int cl = 8 * (NB - 1) + 2 * t4;
    const bool v0 = cl < N, v1 = cl + 1 < N;
    const bool hp = FULL || has_prev, hn = FULL || has_next;
    const bool ract = FULL || act;
#define QDT_VALID(nb, i)                                                                  \
    (CB / 8 + (nb) < NB - 1 ? ract : (CB / 8 + (nb) == NB - 1 ? (ract && ((i) ? v1 : v0)) : false))
    // ---- pass 1: G = acc + gamma L Theta, regulariser pair, row min of G (for the KKT)
    double mn = INFINITY;
#pragma unroll
    for (int nb = 0; nb < NBA; nb++) {
        const int c = CB + 8 * nb + 2 * t4;
        double t0[2], tp[2], tn[2];
        if (EVEN) {
            const double2 x = *reinterpret_cast<const double2 *>(thr + c);
            const double2 y = *reinterpret_cast<const double2 *>(thr + c - TPp);
            const double2 z = *reinterpret_cast<const double2 *>(thr + c + TPp);
            t0[0] = x.x, t0[1] = x.y, tp[0] = y.x, tp[1] = y.y, tn[0] = z.x, tn[1] = z.y;
        } else {
#pragma unroll
            for (int i = 0; i < 2; i++) t0[i] = thr[c + i], tp[i] = thr[c + i - TPp], tn[i] = thr[c + i + TPp];
        }
        double q0[2], qp[2], qn[2];   // Theta_{k-1} (FISTA only)
        if (FIS) {
            if (EVEN) {
                const double2 x = *reinterpret_cast<const double2 *>(tpr + c);
                const double2 y = *reinterpret_cast<const double2 *>(tpr + c - TPp);
                const double2 z = *reinterpret_cast<const double2 *>(tpr + c + TPp);
                q0[0] = x.x, q0[1] = x.y, qp[0] = y.x, qp[1] = y.y, qn[0] = z.x, qn[1] = z.y;
            } else {
#pragma unroll
                for (int i = 0; i < 2; i++) q0[i] = tpr[c + i], qp[i] = tpr[c + i - TPp], qn[i] = tpr[c + i + TPp];
            }
        }
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const double a0 = t0[i];
            const double an = hn ? tn[i] : a0;
            const double d2 = a0 - an;                       // regulariser pair of Theta_k
            double g;
            if (FIS) {
                const double y0 = fma(beta, a0 - q0[i], a0);
                const double yp = hp ? fma(beta, tp[i] - qp[i], tp[i]) : y0;
                const double yn = hn ? fma(beta, tn[i] - qn[i], tn[i]) : y0;
                g = fma(gamma, (y0 - yp) + (y0 - yn), acc[nb][i]);
            } else {
                const double d1 = a0 - (hp ? tp[i] : a0);
                g = fma(gamma, d1 + d2, acc[nb][i]);
            }
            if (QDT_VALID(nb, i)) {
                sreg = fma(d2, d2, sreg);
                mn = g < mn ? g : mn;
            }
            acc[nb][i] = g;
            if (STASH) keep[STASH ? nb : 0][i] = a0;
        }
    }
    mid();
    if (SMEM_OUT) __syncthreads();  // neighbour rows read: each row may now be overwritten by its owner
    double lam = 0.0, lamp = 0.0;
    if (do_kkt) {
        double m1 = quad_min(mn);
        if (PAIR) {
            double v[1] = {m1}, o[1];
            pair_xchg<1>(*px, v, o);
            m1 = dmin(m1, o[0]);
        }
        lam = -2.0 * m1;
        lamp = lam > 0.0 ? lam : 0.0;
    }
    // ---- pass 2: KKT terms, X = Theta - t_k G, row sum / max / min of X
    s = 0.0, xm = -INFINITY, xn = INFINITY;
    constexpr bool IK = NB >= QDT_IKEY_MIN_NB || (QDT_IKEY_PAIR && PAIR);
    int kxm = DKEY_NINF, kxn = DKEY_PINF;   // IK: bounds only (see dkey), integer-pipe min / max
#pragma unroll
    for (int nb = 0; nb < NBA; nb++) {
        const int c = CB + 8 * nb + 2 * t4;
        double t0[2];
        if (STASH) {
            t0[0] = keep[STASH ? nb : 0][0], t0[1] = keep[STASH ? nb : 0][1];
        } else if (EVEN) {
            const double2 x = *reinterpret_cast<const double2 *>(thr + c);
            t0[0] = x.x, t0[1] = x.y;
        } else {
            t0[0] = thr[c], t0[1] = thr[c + 1];
        }
        if (FIS) {   // X is taken from the extrapolated point Y
            double q0[2];
            if (EVEN) {
                const double2 x = *reinterpret_cast<const double2 *>(tpr + c);
                q0[0] = x.x, q0[1] = x.y;
            } else {
                q0[0] = tpr[c], q0[1] = tpr[c + 1];
            }
            t0[0] = fma(beta, t0[0] - q0[0], t0[0]);
            t0[1] = fma(beta, t0[1] - q0[1], t0[1]);
        }
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const double g = acc[nb][i];
            const bool ok = QDT_VALID(nb, i);
            if (do_kkt && ok) {
                const double x1 = t0[i] * fma(2.0, g, lam);
                skkt = fma(x1, x1, skkt);
                if (want_kktp) {
                    const double x2 = t0[i] * fma(2.0, g, lamp);
                    skktp = fma(x2, x2, skktp);
                }
            }
            const double x = fma(-tk, g, t0[i]);
            if (ok) {
                s += x;
                if (IK) {
                    const int kx = dkey(x);
                    kxm = max(kxm, kx);
                    kxn = min(kxn, kx);
                } else {
                    xm = x > xm ? x : xm;
                    xn = x < xn ? x : xn;
                }
            }
            acc[nb][i] = ok ? x : -INFINITY;
        }
    }
    s = quad_sum(s);
    if (IK) {
        xm = dkey_floor(quad_max_i(kxm));   // <= max X: a valid Michelot lower bound after - 1
        xn = dkey_floor(quad_min_i(kxn));   // <= min X: "every entry stays active" only when certain
    } else {
        xm = quad_max(xm);
        xn = quad_min(xn);
    }
    if (PAIR) {
        double v[3] = {s, xm, xn}, o[3];
        pair_xchg<3>(*px, v, o);
        s = px->h ? o[0] + s : s + o[0];   // half 0 + half 1 in both warps
        xm = dmax(xm, o[1]);
        xn = dmin(xn, o[2]);
    }
#undef QDT_VALID
}

// Threshold and output of the row (after row_pass): X in acc (-inf for invalid columns), s, xm,
// xn its quad-reduced sum / max / min.  SMEM_OUT also writes Theta_{k+1} over the row in smem.
template <int NB, bool FULL, bool EVEN, bool SMEM_OUT, int NBA = NB, int CB = 0, bool PAIR = false>
__device__ __forceinline__ void row_project(double (&acc)[NBA][2], double *thr, int N, int t4,
                                            bool act, double s, double xm, double xn, double *orow,
                                            PairX *px = nullptr)
{
    constexpr bool IK = NB >= QDT_IKEY_MIN_NB || (QDT_IKEY_PAIR && PAIR);
    const int cl = 8 * (NB - 1) + 2 * t4;
    const bool v0 = cl < N, v1 = cl + 1 < N;
    const bool ract = FULL || act;
    // ---- threshold (reading R4).  tau0 = (sum X - 1)/N is exact when every entry stays active
    // (min X > tau0); otherwise Michelot rounds from the lower bound max(tau0, max X - 1): each
    // round takes A = {X > tau}, tau <- (sum_A X - 1)/|A|, and stops as soon as min_A X > tau
    // (then {X > tau} = A: the fixed point) or |A| stops shrinking.
    double tau = (s - 1.0) / (double)N;
    bool done = !ract || xn > tau;
    if (!done) tau = fmax(tau, xm - 1.0);
    int cnt = N + 1;
    constexpr bool kMin = true;    // stop as soon as min_A X > tau (profiles/r01_v9: faster than waiting for |A|)
    for (int round = 0; round <= N; round++) {
        if (__all_sync(0xffffffffu, done)) break;
        double ps = 0.0, mA = INFINITY;
        int pc = 0;
        int kmA = DKEY_PINF;
#pragma unroll
        for (int nb = 0; nb < NBA; nb++)
#pragma unroll
            for (int i = 0; i < 2; i++) {
                const double x = acc[nb][i];
                if (x > tau) {
                    ps += x;
                    pc++;
                    if (kMin) {
                        if (IK)
                            kmA = min(kmA, dkey(x));
                        else
                            mA = x < mA ? x : mA;
                    }
                }
            }
        ps = quad_sum(ps);
        pc = quad_sum_i(pc);
        if (kMin) mA = IK ? dkey_floor(quad_min_i(kmA)) : quad_min(mA);   // IK: <= min_A X, stops early only when certain
        if (PAIR) {
            double v[3] = {ps, (double)pc, mA}, o[3];
            pair_xchg<3>(*px, v, o);
            ps = px->h ? o[0] + ps : ps + o[0];
            pc += (int)o[1];
            mA = dmin(mA, o[2]);
        }
        if (!done) {
            if (pc >= cnt) {
                done = true;
            } else {
                cnt = pc;
                tau = (ps - 1.0) / (double)pc;
                done = kMin && mA > tau;
            }
        }
    }
    if (ract) {
#pragma unroll
        for (int nb = 0; nb < NBA; nb++) {
            const int gb = CB / 8 + nb;
            const int c = CB + 8 * nb + 2 * t4;
            double o0 = acc[nb][0] - tau, o1 = acc[nb][1] - tau;
#if QDT_ICLAMP
            o0 = dclamp0(o0);
            o1 = dclamp0(o1);
#else
            o0 = o0 > 0.0 ? o0 : 0.0;
            o1 = o1 > 0.0 ? o1 : 0.0;
#endif
            if (EVEN) {
                if (gb < NB - 1 || (gb == NB - 1 && v0)) {
                    *reinterpret_cast<double2 *>(orow + c) = make_double2(o0, o1);
                    if (SMEM_OUT) *reinterpret_cast<double2 *>(thr + c) = make_double2(o0, o1);
                }
            } else {
                if (gb < NB - 1 || (gb == NB - 1 && v0)) {
                    orow[c] = o0;
                    if (SMEM_OUT) thr[c] = o0;
                }
                if (gb < NB - 1 || (gb == NB - 1 && v1)) {
                    orow[c + 1] = o1;
                    if (SMEM_OUT) thr[c + 1] = o1;
                }
            }
        }
    }
}

template <int NB, bool FULL, bool EVEN, bool SMEM_OUT = false>
__device__ __forceinline__ void row_step(double (&acc)[NB][2], double *thr, int N, int t4,
                                         bool act, bool has_prev, bool has_next, double gamma,
                                         double tk, bool do_kkt, bool want_kktp, double &sreg,
                                         double &skkt, double &skktp, double *orow)
{
    double s, xm, xn;
    row_pass<NB, FULL, EVEN, SMEM_OUT>(acc, thr, N, t4, act, has_prev, has_next, gamma, tk, do_kkt,
                                       want_kktp, sreg, skkt, skktp, s, xm, xn);
    row_project<NB, FULL, EVEN, SMEM_OUT>(acc, thr, N, t4, act, s, xm, xn, orow);
}

// bwd GEMM of one staged chunk: acc += F_chunk^T R_chunk over kc probes (k-steps of 4; only
// the tail step is masked).  F: chunk rows (probe-major, pitch STP), lane's row 8w + g4 folded
// in; R: chunk rows (pitch N), lane's column g4 folded in.
template <int NB>
__device__ __forceinline__ void gemm_bwd(double (&acc)[NB][2], const double *F, const double *R,
                                         int kc, int N, int t4)   // N: pitch of the staged R rows
{
    const int nfull = kc >> 2;
    for (int ks = 0; ks < nfull; ks++) {
        const int jj = 4 * ks + t4;
        const double av = F[jj * STP];
        const double *rb = R + jj * N;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) dmma(acc[nb][0], acc[nb][1], av, rb[8 * nb]);
    }
    if (kc & 3) {
        const int jj = 4 * nfull + t4;
        const bool okj = jj < kc;
        const double av = okj ? F[jj * STP] : 0.0;
        const double *rb = R + jj * N;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) dmma(acc[nb][0], acc[nb][1], av, okj ? rb[8 * nb] : 0.0);
    }
}

// gemm_bwd over the k-steps [kslo, kshi) of the chunk only (the others multiply F entries that are
// zero for this warp's rows: the probes outside the rows' covering range)
template <int NB>
__device__ __forceinline__ void gemm_bwd_rng(double (&acc)[NB][2], const double *F, const double *R,
                                             int kc, int N, int t4, int kslo, int kshi)
{
    const int nks = (kc + 3) >> 2;
    const int k1 = min(nks, kshi);
    for (int ks = max(0, kslo); ks < k1; ks++) {
        const int jj = 4 * ks + t4;
        const bool okj = jj < kc;
        const double av = okj ? F[jj * STP] : 0.0;
        const double *rb = R + jj * N;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) dmma(acc[nb][0], acc[nb][1], av, okj ? rb[8 * nb] : 0.0);
    }
}

// SQS row weights from the tiled F (reading R2): w_k = sum_d F_{d,k} s_d + 4 gamma over the
// tile's window, t_k = 1/w_k (0 for a frozen row).  Block per tile: 64 rows x 4 probe slices
// (fixed combination order, deterministic); the window's F rows are read coalesced.
__global__ void __launch_bounds__(256) k_sqs_weights_tiled(int Ml, const int32_t *tile_dA,
                                                            const int32_t *tile_dB, const int64_t *fb_off,
                                                            const double *Fb, const double *s, double gamma,
                                                            double *w, double *tstep)
{
    // 64 rows x 4 probe slices (probes j = q mod 4); the slices are combined in a fixed order
    __shared__ double part[4][ST];
    const int t = blockIdx.x, r = threadIdx.x & (ST - 1), q = threadIdx.x >> 6;
    const int dA = tile_dA[t], W = tile_dB[t] - dA;
    const double *f = Fb + fb_off[t] + r;
    double acc = 0.0;
    for (int j = q; j < W; j += 4) acc += f[(int64_t)j * STP] * s[dA + j];
    part[q][r] = acc;
    __syncthreads();
    const int k = t * ST + r;
    if (q || k >= Ml) return;
    double v = ((part[0][r] + part[1][r]) + (part[2][r] + part[3][r])) + 4.0 * gamma;
    if (w) w[k] = v;
    if (tstep) tstep[k] = (v > 0.0) ? 1.0 / v : 0.0;
}

cudaError_t launch_sqs_weights_tiled(int ntiles, int Ml, const int32_t *tile_dA,
                                     const int32_t *tile_dB, const int64_t *fb_off, const double *Fb,
                                     const double *s, double gamma, double *w, double *tstep,
                                     cudaStream_t st)
{
    if (ntiles <= 0) return cudaSuccess;
    k_sqs_weights_tiled<<<ntiles, 4 * ST, 0, st>>>(Ml, tile_dA, tile_dB, fb_off, Fb, s, gamma, w, tstep);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ bwd sweep
// Smem: Theta tile (ST+2 rows incl. halo) | F chunks 2 x SKC x STP | R chunks 2 x (SKC*N + pad)
// Theta-tile row pitch in shared memory: N (one contiguous bulk copy of the rows), or with TP
// (tensor-map tile, even N) the compile-time pitch tp_pitch(NB) = 8 NB (+ 8 for even NB), which
// is = 8 mod 16 doubles: the two 64-byte row segments a quarter-warp reads (rows g, g + 1) fall
// in disjoint bank halves, so the row pass's tile loads are free of bank conflicts; the tile
// arrives by one 2-D TMA copy whose box columns >= N are zero-filled.
__device__ __host__ constexpr int tp_pitch(int NB) { return 8 * NB + ((NB & 1) ? 0 : 8); }

template <int NB>
struct SwLayout {
    int thsz, rsz;
    __device__ __host__ SwLayout(int N, int pitch)
    {
        thsz = (((ST + 2) * pitch + 8 * NB + 16) + 15) & ~15;   // 128-byte aligned tiles
        rsz = ((SKC * N + 8 * NB + 16) + 1) & ~1;
    }
    __device__ __host__ size_t bytes() const
    {
        return (size_t)(thsz + 2 * SKC * STP + 2 * rsz) * sizeof(double);
    }
};

size_t sweep_bwd_smem(int N, int NB, bool fista, bool tp)
{
    const int thsz = (((ST + 2) * (tp ? tp_pitch(NB) : N) + 8 * NB + 16) + 15) & ~15;
    const int rsz = ((SKC * N + 8 * NB + 16) + 1) & ~1;
    return (size_t)((fista ? 2 : 1) * thsz + 2 * SKC * STP + 2 * rsz) * sizeof(double);
}

// Persistent: CTA b processes units b, b + G, b + 2G, ... (heavy first).  The chunk buffers of
// the next unit are refilled as soon as this unit's GEMM is done, the Theta tile as soon as the
// epilogue has read it (before the Michelot rounds and stores), so the next unit's loads overlap
// the current unit's epilogue.
template <int NB, bool FIS, bool TP = false>
__global__ void __launch_bounds__(256, (NB <= 13 && !FIS ? 2 : 1)) k_bwd_mma(const __grid_constant__ SweepArgs a)
{
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bars[3];
    __shared__ double red[8 * 3];
    __shared__ int s_last;
    constexpr bool ACC = NB >= QDT_ACC_MIN_NB;
    __shared__ double accs[3][ACC ? 256 : 1];   // per-thread running sums (KKT, paper KKT, regulariser)
    __shared__ int s_pend;                      // the unsplit tile whose slot takes this CTA's total
    const DevState *st = a.state;
    if (st && st->stop) return;
    const int64_t it = st ? st->it : 0;
    const int N = a.N;
    // valid outcomes: a padded pitch's zero column is no coordinate (only N > 128 is ever padded, so
    // the NB <= 16 instantiations keep Nv == N at compile time: no extra register)
    const int Nv = (NB > SW_NBMAX && a.Nv > 0) ? a.Nv : N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int G = gridDim.x;
    int unit = blockIdx.x;
    if (unit >= a.nunits) return;
    const int TPB = TP ? tp_pitch(NB) : N;          // staged tile pitch
    const SwLayout<NB> L(N, TPB);
    double *Th = sm;
    double *Tq = sm + L.thsz;                       // FISTA: Theta_{k-1} tile (same rows)
    double *Fs = sm + (FIS ? 2 : 1) * L.thsz;
    double *Rs = Fs + 2 * SKC * STP;
    // eval_gate (FISTA evaluation pass): only on iterations whose KKT is recorded
    if (a.eval_gate && (it % a.kkt_every) != 0) return;
    const bool do_kkt = !FIS && (it % a.kkt_every) == 0;
    const bool even = (N & 1) == 0;
    const double beta = FIS ? a.beta[it] : 0.0;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        fence_barrier_init();
        s_pend = -1;
    }
    if (ACC) accs[0][tid] = accs[1][tid] = accs[2][tid] = 0.0;
    __syncthreads();
    // issue helpers (thread 0 only); chunk stage / parity follow a running chunk counter
    uint32_t c_issue = 0, c_use = 0, th_use = 0;
    // the tile load (lane 0 of the calling warp): one contiguous bulk copy, or (TP) one 2-D tensor
    // copy of rows k0 - 1 .. k0 + 64 at pitch TPB with the pad columns zero-filled
    auto issue_theta = [&](const SwUnit &v) {
        if (lane != 0) return;
        const int k0 = v.tile * ST, Tt = min(ST, a.Ml - k0);
        if (TP) {
            const uint32_t bb = (uint32_t)TPB * (ST + 2) * 8;
            mbar_expect_tx(&bars[0], FIS ? 2 * bb : bb);
            tma_2d(Th, &a.tm_theta, 0, k0, &bars[0]);
            if (FIS) tma_2d(Tq, &a.tm_prev, 0, k0, &bars[0]);
            return;
        }
        const double *src;
        int sh;
        uint32_t by;
        aligned_span(a.theta + (int64_t)(k0 - 1) * N, (int64_t)(Tt + 2) * N, &src, &sh, &by);
        mbar_expect_tx(&bars[0], FIS ? 2 * by : by);
        bulk_g2s(Th, src, by, &bars[0]);
        if (FIS) bulk_g2s(Tq, a.theta_prev + (src - a.theta), by, &bars[0]);
    };
    auto issue_chunk = [&](const SwUnit &v, int c) {
        const int W = v.p1 - v.p0, pb = c * SKC, kc = min(SKC, W - pb);
        const double *rsrc;
        int rsh;
        uint32_t rbytes;
        aligned_span(a.R + (int64_t)(v.p0 + pb) * N, (int64_t)kc * N, &rsrc, &rsh, &rbytes);
        const int stg = c_issue & 1;
        uint64_t *bar = &bars[1 + stg];
        const uint32_t fbytes = (uint32_t)kc * STP * 8;
        const double *Fg = a.Fb + a.fb_off[v.tile] + (int64_t)(v.p0 - a.tile_dA[v.tile] + pb) * STP;
        mbar_expect_tx(bar, fbytes + rbytes);
        bulk_g2s(Fs + stg * SKC * STP, Fg, fbytes, bar);
        bulk_g2s(Rs + stg * L.rsz, rsrc, rbytes, bar);
        c_issue++;
    };
    SwUnit u = a.units[unit];
    if (warp == 0 && u.nsplit == 1) issue_theta(u);
    if (tid == 0 && u.p1 > u.p0) issue_chunk(u, 0);
    while (true) {
        const int k0 = u.tile * ST;
        const int Tt = min(ST, a.Ml - k0);
        const int W = u.p1 - u.p0;
        const int nch = (W + SKC - 1) / SKC;
        const int next = unit + G;
        SwUnit un;
        if (next < a.nunits) un = a.units[next];
        // the row's step weight (or the BB scalar), loaded before the GEMM to hide its latency
        const double tk = a.tscal ? *a.tscal : (8 * warp + g4 < Tt) ? __ldg(a.tstep + k0 + 8 * warp + g4) : 0.0;
        double acc[NB][2];
#pragma unroll
        for (int nb = 0; nb < NB; nb++) acc[nb][0] = acc[nb][1] = 0.0;
        for (int c = 0; c < nch; c++) {
            if (tid == 0 && c + 1 < nch) issue_chunk(u, c + 1);
            const int stg = c_use & 1;
            mbar_wait(&bars[1 + stg], (c_use >> 1) & 1);
            c_use++;
            const int pb = c * SKC;
            const int kc = min(SKC, W - pb);
            const int rsh = (int)(((uintptr_t)(a.R + (int64_t)(u.p0 + pb) * N) & 15) >> 3);
            gemm_bwd<NB>(acc, Fs + stg * SKC * STP + 8 * warp + g4, Rs + stg * L.rsz + rsh + g4, kc, N, t4);
            __syncthreads();
        }
        if (tid == 0 && c_issue != c_use) __trap();  // pipeline invariant
        // chunk buffers are free: start the next unit's first chunk
        if (tid == 0 && next < a.nunits && un.p1 > un.p0) issue_chunk(un, 0);

        bool epi = true;
        if (u.nsplit > 1) {
            // split-K: publish the fragment-ordered partial; the last unit of the tile sums the
            // slots in slot order (deterministic whichever unit finishes last).
            const int64_t fsz = (int64_t)8 * NB * 64;
            double *slot = a.scratch + (u.slot_base + u.slot) * fsz;
#pragma unroll
            for (int nb = 0; nb < NB; nb++)
                __stcg(reinterpret_cast<double2 *>(slot + ((warp * NB + nb) * 32 + lane) * 2),
                       make_double2(acc[nb][0], acc[nb][1]));
            __threadfence();
            __syncthreads();
            if (tid == 0) s_last = (atomicAdd(&a.counters[u.tile], 1) == u.nsplit - 1);
            __syncthreads();
            epi = s_last;
            if (epi) {
                __threadfence();
                if (warp == 0) issue_theta(u);
#pragma unroll
                for (int nb = 0; nb < NB; nb++) acc[nb][0] = acc[nb][1] = 0.0;
                for (int sl = 0; sl < u.nsplit; sl++) {
                    const double *sp = a.scratch + (u.slot_base + sl) * fsz;
#pragma unroll
                    for (int nb = 0; nb < NB; nb++) {
                        const double2 v =
                            __ldcg(reinterpret_cast<const double2 *>(sp + ((warp * NB + nb) * 32 + lane) * 2));
                        acc[nb][0] += v.x;
                        acc[nb][1] += v.y;
                    }
                }
                if (tid == 0) a.counters[u.tile] = 0;
            }
        }
        if (epi) {
            mbar_wait(&bars[0], th_use & 1);
            th_use++;
            const int th_sh = TP ? 0 : (int)(((uintptr_t)(a.theta + (int64_t)(k0 - 1) * N) & 15) >> 3);
            const int r = 8 * warp + g4;
            const bool act = r < Tt;
            const int kl = k0 + r;
            const int64_t kg = a.kb + kl;
            const bool has_prev = kg > 0, has_next = kg + 1 < a.M;
            double *thr = Th + th_sh + (r + 1) * TPB;
            double sreg = 0.0, skkt = 0.0, skktp = 0.0, s, xm, xn;
            double *orow = a.out + (int64_t)kl * N;
            const bool full = Tt == ST && a.kb + k0 > 0 && a.kb + k0 + ST < a.M;
            const bool ev = a.eval != 0;   // evaluation pass: KKT (both multipliers) + regulariser only
            const bool fast = full && even;
            const double *tpr = Tq + th_sh + (r + 1) * TPB;
            // interior even-N tiles of plain steps: the own-row values stay in registers, the tile
            // is released after pass 1 and the next unit's tile load overlaps pass 2 + Michelot
            constexpr bool kStash = NB <= SW_NBMAX;   // register budget: 255 at NB = 16
            const bool stash = kStash && fast && !FIS && !ev;
            auto release = [&]() {
                __syncthreads();
                if (warp == 0 && next < a.nunits && un.nsplit == 1) issue_theta(un);
            };
            if (stash)
                row_pass<NB, true, true, false, false, NB, 0, false, true>(acc, thr, Nv, t4, act, has_prev, has_next,
                                                                         a.gamma, tk, do_kkt, ev, sreg, skkt,
                                                                         skktp, s, xm, xn, tpr, beta, nullptr,
                                                                         release, TPB);
            else if (fast)
                row_pass<NB, true, true, false, FIS>(acc, thr, Nv, t4, act, has_prev, has_next, a.gamma, tk,
                                                     do_kkt, ev, sreg, skkt, skktp, s, xm, xn, tpr, beta, nullptr, NoMid(), TPB);
            else if (full)
                row_pass<NB, true, false, false, FIS>(acc, thr, Nv, t4, act, has_prev, has_next, a.gamma, tk,
                                                      do_kkt, ev, sreg, skkt, skktp, s, xm, xn, tpr, beta, nullptr, NoMid(), TPB);
            else
                row_pass<NB, false, false, false, FIS>(acc, thr, Nv, t4, act, has_prev, has_next, a.gamma, tk,
                                                       do_kkt, ev, sreg, skkt, skktp, s, xm, xn, tpr, beta, nullptr, NoMid(), TPB);
            if (!stash) release();   // Theta tile consumed: start the next unit's tile load
            if (ev) {
            } else if (fast)
                row_project<NB, true, true, false>(acc, thr, Nv, t4, act, s, xm, xn, orow);
            else if (full)
                row_project<NB, true, false, false>(acc, thr, Nv, t4, act, s, xm, xn, orow);
            else
                row_project<NB, false, false, false>(acc, thr, Nv, t4, act, s, xm, xn, orow);
            if (ACC && u.nsplit == 1) {
                // running sums in the thread's own slots; the previous pending tile's slot is zeroed
                accs[0][tid] += skkt;
                accs[1][tid] += skktp;
                accs[2][tid] += sreg;
                if (tid == 0) {
                    if (s_pend >= 0) {
                        double *p = a.part + (int64_t)s_pend * NSC_TILE;
                        if (do_kkt) p[SC_KKT] = 0.0, p[SC_KKTP] = 0.0;
                        p[SC_REG] = 0.0;
                        p[SC_DTH] = 0.0;
                    }
                    s_pend = u.tile;
                }
            } else {
            // per-tile scalar partials (fixed order: lanes, then warps)
            sreg = wsum(sreg);
            skkt = wsum(skkt);
            skktp = wsum(skktp);
            if (lane == 0) {
                red[warp * 3 + 0] = skkt;
                red[warp * 3 + 1] = skktp;
                red[warp * 3 + 2] = sreg;
            }
            __syncthreads();
            if (tid == 0) {
                double v0 = 0.0, v1 = 0.0, v2 = 0.0;
                for (int w = 0; w < 8; w++) {
                    v0 += red[w * 3 + 0];
                    v1 += red[w * 3 + 1];
                    v2 += red[w * 3 + 2];
                }
                double *p = a.part + (int64_t)u.tile * NSC_TILE;
                if (do_kkt) {
                    p[SC_KKT] = v0;
                    p[SC_KKTP] = v1;
                }
                p[SC_REG] = v2;
                p[SC_DTH] = 0.0;
            }
            }
        } else if (warp == 0 && next < a.nunits && un.nsplit == 1) {
            issue_theta(un);
        }
        if (next >= a.nunits) break;
        unit = next;
        u = un;
    }
    if (ACC) {   // the CTA's total over its unsplit tiles (fixed order: the thread's tiles, lanes, warps)
        __syncthreads();   // red may still be read by thread 0 (a split tile's partial)
        const double skkt = wsum(accs[0][tid]), skktp = wsum(accs[1][tid]), sreg = wsum(accs[2][tid]);
        if (lane == 0) {
            red[warp * 3 + 0] = skkt;
            red[warp * 3 + 1] = skktp;
            red[warp * 3 + 2] = sreg;
        }
        __syncthreads();
        if (tid == 0 && s_pend >= 0) {
            double v0 = 0.0, v1 = 0.0, v2 = 0.0;
            for (int w = 0; w < 8; w++) {
                v0 += red[w * 3 + 0];
                v1 += red[w * 3 + 1];
                v2 += red[w * 3 + 2];
            }
            double *p = a.part + (int64_t)s_pend * NSC_TILE;
            if (do_kkt) {
                p[SC_KKT] = v0;
                p[SC_KKTP] = v1;
            }
            p[SC_REG] = v2;
            p[SC_DTH] = 0.0;
        }
    }
}

// N-split variant of k_bwd_mma: 512 threads (16 warps) per CTA, warp w owns m-block w & 7 and
// the column half w >> 3 (NBA = ceil(NB/2) column blocks; the last block of an odd NB is padding),
// so that each thread holds half a row and two CTAs (32 warps) fit an SM; the two halves of a row
// complete every row reduction through a named-barrier pair exchange (PairX).
template <int NB, bool FIS, bool TP = false>
__global__ void __launch_bounds__(512, 1) k_bwd_split(const __grid_constant__ SweepArgs a)
{
    constexpr int NBA = (NB + 1) / 2;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bars[4];   // 0, 3: Theta buffers; 1, 2: chunk stages
    __shared__ double red[16 * 3];
    __shared__ double xbuf[2 * 8 * 2 * 8 * 4];
    __shared__ int s_last;
    const DevState *st = a.state;
    if (st && st->stop) return;
    const int64_t it = st ? st->it : 0;
    const int N = a.N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int mb = warp & 7, hh = warp >> 3;
    const int G = gridDim.x;
    int unit = blockIdx.x;
    if (unit >= a.nunits) return;
    const int TPB = TP ? tp_pitch(NB) : N;          // staged tile pitch (TP: tensor-copy tile)
    const SwLayout<NB> L(N, TPB);
    double *Th = sm;
    double *Tq = sm + L.thsz;
    double *Fs = sm + 2 * L.thsz;                   // two tiles: double buffer or Theta_{k-1}
    double *Rs = Fs + 2 * SKC * STP;
    if (a.eval_gate && (it % a.kkt_every) != 0) return;
    const bool do_kkt = !FIS && (it % a.kkt_every) == 0;
    const bool even = (N & 1) == 0;
    const double beta = FIS ? a.beta[it] : 0.0;
    PairX px{xbuf, 0, mb, hh, g4, t4};

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        mbar_init(&bars[3], 1);
        fence_barrier_init();
    }
    __syncthreads();
    // Theta loads are issued and consumed in unit order (FIFO).  Plain steps double-buffer the
    // tile (buffers Th / Tq alternate): the next non-split unit's tile is requested when the
    // current unit starts.  FISTA uses Tq for Theta_{k-1}, single buffer.
    uint32_t c_issue = 0, c_use = 0, th_issue = 0, th_use = 0;
    auto th_buf = [&](uint32_t n) -> double * { return (!FIS && (n & 1)) ? Tq : Th; };
    auto th_bar = [&](uint32_t n) -> uint64_t * { return (!FIS && (n & 1)) ? &bars[3] : &bars[0]; };
    auto th_par = [&](uint32_t n) -> uint32_t { return FIS ? (n & 1) : ((n >> 1) & 1); };
    auto issue_theta = [&](const SwUnit &v) {
        const int k0 = v.tile * ST, Tt = min(ST, a.Ml - k0);
        uint64_t *bar = th_bar(th_issue);
        if (TP) {   // one 2-D tensor copy per tile at the conflict-free pitch (see k_bwd_mma)
            const uint32_t bb = (uint32_t)TPB * (ST + 2) * 8;
            mbar_expect_tx(bar, FIS ? 2 * bb : bb);
            tma_2d(th_buf(th_issue), &a.tm_theta, 0, k0, bar);
            if (FIS) tma_2d(Tq, &a.tm_prev, 0, k0, bar);
            th_issue++;
            return;
        }
        const double *src;
        int sh;
        uint32_t by;
        aligned_span(a.theta + (int64_t)(k0 - 1) * N, (int64_t)(Tt + 2) * N, &src, &sh, &by);
        mbar_expect_tx(bar, FIS ? 2 * by : by);
        bulk_g2s(th_buf(th_issue), src, by, bar);
        if (FIS) bulk_g2s(Tq, a.theta_prev + (src - a.theta), by, bar);
        th_issue++;
    };
    auto issue_chunk = [&](const SwUnit &v, int c) {
        const int W = v.p1 - v.p0, pb = c * SKC, kc = min(SKC, W - pb);
        const double *rsrc;
        int rsh;
        uint32_t rbytes;
        aligned_span(a.R + (int64_t)(v.p0 + pb) * N, (int64_t)kc * N, &rsrc, &rsh, &rbytes);
        const int stg = c_issue & 1;
        uint64_t *bar = &bars[1 + stg];
        const uint32_t fbytes = (uint32_t)kc * STP * 8;
        const double *Fg = a.Fb + a.fb_off[v.tile] + (int64_t)(v.p0 - a.tile_dA[v.tile] + pb) * STP;
        mbar_expect_tx(bar, fbytes + rbytes);
        bulk_g2s(Fs + stg * SKC * STP, Fg, fbytes, bar);
        bulk_g2s(Rs + stg * L.rsz, rsrc, rbytes, bar);
        c_issue++;
    };
    if (tid == 0) {
        const SwUnit u0 = a.units[unit];
        if (u0.nsplit == 1) issue_theta(u0);
        if (u0.p1 > u0.p0) issue_chunk(u0, 0);
    }
    while (true) {
        const SwUnit u = a.units[unit];
        if (!FIS && tid == 0 && u.nsplit == 1 && unit + G < a.nunits) {
            const SwUnit un = a.units[unit + G];    // prefetch: the other buffer is free
            if (un.nsplit == 1) issue_theta(un);
        }
        const int k0 = u.tile * ST;
        const int Tt = min(ST, a.Ml - k0);
        const int W = u.p1 - u.p0;
        const int nch = (W + SKC - 1) / SKC;
        const int next = unit + G;
        const double tk = a.tscal ? *a.tscal : (8 * mb + g4 < Tt) ? __ldg(a.tstep + k0 + 8 * mb + g4) : 0.0;
        double acc[NBA][2];
#pragma unroll
        for (int nb = 0; nb < NBA; nb++) acc[nb][0] = acc[nb][1] = 0.0;
        for (int c = 0; c < nch; c++) {
            if (tid == 0 && c + 1 < nch) issue_chunk(u, c + 1);
            const int stg = c_use & 1;
            mbar_wait(&bars[1 + stg], (c_use >> 1) & 1);
            c_use++;
            const int pb = c * SKC;
            const int kc = min(SKC, W - pb);
            const int rsh = (int)(((uintptr_t)(a.R + (int64_t)(u.p0 + pb) * N) & 15) >> 3);
            gemm_bwd<NBA>(acc, Fs + stg * SKC * STP + 8 * mb + g4,
                          Rs + stg * L.rsz + rsh + g4 + 8 * NBA * hh, kc, N, t4);
            __syncthreads();
        }
        if (tid == 0 && next < a.nunits) {
            const SwUnit un = a.units[next];
            if (un.p1 > un.p0) issue_chunk(un, 0);
        }
        bool epi = true;
        if (u.nsplit > 1) {
            const int64_t fsz = (int64_t)16 * NBA * 64;
            double *slot = a.scratch + (u.slot_base + u.slot) * fsz;
#pragma unroll
            for (int nb = 0; nb < NBA; nb++)
                __stcg(reinterpret_cast<double2 *>(slot + ((warp * NBA + nb) * 32 + lane) * 2),
                       make_double2(acc[nb][0], acc[nb][1]));
            __threadfence();
            __syncthreads();
            if (tid == 0) s_last = (atomicAdd(&a.counters[u.tile], 1) == u.nsplit - 1);
            __syncthreads();
            epi = s_last;
            if (epi) {
                __threadfence();
                if (tid == 0) issue_theta(u);
#pragma unroll
                for (int nb = 0; nb < NBA; nb++) acc[nb][0] = acc[nb][1] = 0.0;
                for (int sl = 0; sl < u.nsplit; sl++) {
                    const double *sp = a.scratch + (u.slot_base + sl) * fsz;
#pragma unroll
                    for (int nb = 0; nb < NBA; nb++) {
                        const double2 v =
                            __ldcg(reinterpret_cast<const double2 *>(sp + ((warp * NBA + nb) * 32 + lane) * 2));
                        acc[nb][0] += v.x;
                        acc[nb][1] += v.y;
                    }
                }
                if (tid == 0) a.counters[u.tile] = 0;
            }
        }
        if (epi) {
            double *Thc = th_buf(th_use);
            mbar_wait(th_bar(th_use), th_par(th_use));
            th_use++;
            const int th_sh = TP ? 0 : (int)(((uintptr_t)(a.theta + (int64_t)(k0 - 1) * N) & 15) >> 3);
            const int r = 8 * mb + g4;
            const bool act = r < Tt;
            const int kl = k0 + r;
            const int64_t kg = a.kb + kl;
            const bool has_prev = kg > 0, has_next = kg + 1 < a.M;
            double *thr = Thc + th_sh + (r + 1) * TPB;
            const double *tpr = Tq + th_sh + (r + 1) * TPB;
            double sreg = 0.0, skkt = 0.0, skktp = 0.0, s, xm, xn;
            double *orow = a.out + (int64_t)kl * N;
            const bool full = Tt == ST && a.kb + k0 > 0 && a.kb + k0 + ST < a.M;
            const bool fast = full && even;
            const bool ev = a.eval != 0;
#define QDT_SPLIT_PASS(CBV, FU, EV)                                                                    \
    row_pass<NB, FU, EV, false, FIS, NBA, CBV, true>(acc, thr, N, t4, act, has_prev, has_next, a.gamma, tk, \
                                                     do_kkt, ev, sreg, skkt, skktp, s, xm, xn, tpr, beta, &px, \
                                                     NoMid(), TPB)
#define QDT_SPLIT_PROJ(CBV, FU, EV) \
    row_project<NB, FU, EV, false, NBA, CBV, true>(acc, thr, N, t4, act, s, xm, xn, orow, &px)
            if (hh == 0) {
                if (fast) QDT_SPLIT_PASS(0, true, true);
                else if (full) QDT_SPLIT_PASS(0, true, false);
                else QDT_SPLIT_PASS(0, false, false);
            } else {
                if (fast) QDT_SPLIT_PASS(8 * NBA, true, true);
                else if (full) QDT_SPLIT_PASS(8 * NBA, true, false);
                else QDT_SPLIT_PASS(8 * NBA, false, false);
            }
            __syncthreads();  // Theta tile consumed
            if (tid == 0 && next < a.nunits && (FIS || u.nsplit > 1)) {   // not prefetched
                const SwUnit un = a.units[next];
                if (un.nsplit == 1) issue_theta(un);
            }
            if (!ev) {
                if (hh == 0) {
                    if (fast) QDT_SPLIT_PROJ(0, true, true);
                    else if (full) QDT_SPLIT_PROJ(0, true, false);
                    else QDT_SPLIT_PROJ(0, false, false);
                } else {
                    if (fast) QDT_SPLIT_PROJ(8 * NBA, true, true);
                    else if (full) QDT_SPLIT_PROJ(8 * NBA, true, false);
                    else QDT_SPLIT_PROJ(8 * NBA, false, false);
                }
            }
#undef QDT_SPLIT_PASS
#undef QDT_SPLIT_PROJ
            sreg = wsum(sreg);
            skkt = wsum(skkt);
            skktp = wsum(skktp);
            if (lane == 0) {
                red[warp * 3 + 0] = skkt;
                red[warp * 3 + 1] = skktp;
                red[warp * 3 + 2] = sreg;
            }
            __syncthreads();
            if (tid == 0) {
                double v0 = 0.0, v1 = 0.0, v2 = 0.0;
                for (int w = 0; w < 16; w++) {
                    v0 += red[w * 3 + 0];
                    v1 += red[w * 3 + 1];
                    v2 += red[w * 3 + 2];
                }
                double *pp = a.part + (int64_t)u.tile * NSC_TILE;
                if (do_kkt) {
                    pp[SC_KKT] = v0;
                    pp[SC_KKTP] = v1;
                }
                pp[SC_REG] = v2;
                pp[SC_DTH] = 0.0;
            }
        } else if (tid == 0 && next < a.nunits) {
            const SwUnit un = a.units[next];
            if (un.nsplit == 1) issue_theta(un);
        }
        if (next >= a.nunits) break;
        unit = next;
    }
}

// fwd GEMM, transposed so that outcomes are the M dimension and probes the N dimension:
// C[n][d] += sum_k Theta[k][n] F[d][k] for one outcome m-block (lane row n = 8 mb + g4) and NM
// probe n-blocks (lane columns d = 8 nb + 2 t4 + {0,1}).  A fragment a = Theta[4 ks + t4][n],
// B fragment b = F[8 nb + g4][4 ks + t4].  Tcol: Theta + t4 N + 8 mb + g4; Frow: F + g4 STP + t4.
// Rows k >= Tt are masked (stale shared memory); probe rows outside the tile's window are zero
// in shared memory (the caller zero-fills them), so the B fragments need no mask.
template <int NM, bool MASKK, int MX>
__device__ __forceinline__ void gemm_fwd_t(double (&cf)[MX][2], const double *Tcol, const double *Frow,
                                           int N, int Tt, int t4)
{
    const int nks = (Tt + 3) >> 2;
    for (int ks = 0; ks < nks; ks++) {
        double av = Tcol[4 * ks * N];
        if (MASKK) av = (4 * ks + t4 < Tt) ? av : 0.0;
#pragma unroll
        for (int nb = 0; nb < NM; nb++) {
            const double bv = Frow[8 * nb * STP + 4 * ks];
            dmma(cf[nb][0], cf[nb][1], av, bv);
        }
    }
}

template <bool MASKK, int MX>
__device__ __forceinline__ void gemm_fwd_t_nm(int nm, double (&cf)[MX][2], const double *Tcol,
                                              const double *Frow, int N, int Tt, int t4)
{
    switch (nm) {
        case 1: gemm_fwd_t<1, MASKK, MX>(cf, Tcol, Frow, N, Tt, t4); break;
        case 2: gemm_fwd_t<(MX >= 2 ? 2 : 1), MASKK, MX>(cf, Tcol, Frow, N, Tt, t4); break;
        case 3: gemm_fwd_t<(MX >= 3 ? 3 : 1), MASKK, MX>(cf, Tcol, Frow, N, Tt, t4); break;
        case 4: gemm_fwd_t<(MX >= 4 ? 4 : 1), MASKK, MX>(cf, Tcol, Frow, N, Tt, t4); break;
        case 5: gemm_fwd_t<(MX >= 5 ? 5 : 1), MASKK, MX>(cf, Tcol, Frow, N, Tt, t4); break;
        case 6: gemm_fwd_t<(MX >= 6 ? 6 : 1), MASKK, MX>(cf, Tcol, Frow, N, Tt, t4); break;
        case 7: gemm_fwd_t<(MX >= 7 ? 7 : 1), MASKK, MX>(cf, Tcol, Frow, N, Tt, t4); break;
        case 8: gemm_fwd_t<(MX >= 8 ? 8 : 1), MASKK, MX>(cf, Tcol, Frow, N, Tt, t4); break;
        default: break;
    }
}

// ------------------------------------------------------------------------------ fwd sweep
// Unit: Fock tiles [t0, t1) and the union of their probe windows [u0, u1) (<= FWCAP probes).
// Warp w owns (m-block, n-block) pairs [w PP, (w+1) PP) of the (u1-u0)/8 x NB pair grid.
// Theta moves in half tiles of FH = 32 rows (two stages) and the F block of each tile in its own
// two stages, so that two CTAs (16 warps) share an SM.
constexpr int FH = ST / 2;
size_t sweep_fwd_smem(int N, int NB)
{
    const int TP = N > 8 * NB ? 8 * NB + 4 : N;   // wide N: column chunks of 8 NB
    const int tsz = ((FH * TP + 8 * NB + 4) + 1) & ~1;
    return (size_t)(2 * tsz + 2 * FWCAP * STP) * sizeof(double);
}

template <int NB>
__global__ void __launch_bounds__(256, 2) k_fwd_mma(SweepFwdArgs a)
{
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bars[2];
    const DevState *st = a.state;
    if (st && st->stop) return;
    const int N = a.N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    // wide N (ncc > 1): CTA (unit, column chunk cc) covers columns [cbase, cbase + ncol) with the
    // Theta half tile staged row by row at pitch TP (conflict-free A fragments)
    const int ncc = a.ncc;
    const FwUnit u = a.units[blockIdx.x / ncc];
    const int cc = blockIdx.x - (blockIdx.x / ncc) * ncc;
    const int cbase = cc * 8 * NB;
    const int ncol = min(8 * NB, N - cbase);
    const int TP = ncc > 1 ? 8 * NB + 4 : N;
    const int tsz = ((FH * TP + 8 * NB + 4) + 1) & ~1;
    double *Ts = sm;                    // 2 x tsz (half tiles)
    double *Fs = sm + 2 * tsz;          // 2 x FWCAP x STP (per tile)
    const int Wu = u.u1 - u.u0;
    const int nm = (Wu + 7) >> 3;       // <= FWCAP / 8 = FWNB probe n-blocks
    const bool second = warp + 8 < NB && 8 * (warp + 8) < ncol;  // warp-uniform: m-block warp + 8 used

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int nh = 2 * (u.t1 - u.t0);   // half-tile steps
    auto issue = [&](int h) {
        const int t = u.t0 + (h >> 1), half = h & 1;
        const int k0 = t * ST + half * FH;
        const int rows = min(FH, a.Ml - k0);
        uint64_t *bar = &bars[h & 1];
        uint32_t fby = 0;
        int ra = 0, dA = 0;
        if (!half) {
            dA = a.tile_dA[t];
            ra = max(dA, u.u0);
            const int rb = min(a.tile_dB[t], u.u1);
            fby = rb > ra ? (uint32_t)(rb - ra) * STP * 8 : 0;
        }
        if (rows > 0 && ncc > 1) {
            const uint32_t rby = (uint32_t)ncol * 8;   // N even, cbase % 8 == 0: 16-byte aligned rows
            mbar_expect_tx(bar, rby * rows + fby);
            for (int rr = 0; rr < rows; rr++)
                bulk_g2s(Ts + (h & 1) * tsz + rr * TP, a.theta + (int64_t)(k0 + rr) * N + cbase, rby, bar);
        } else if (rows > 0) {
            const double *src;
            int sh;
            uint32_t by;
            aligned_span(a.theta + (int64_t)k0 * N, (int64_t)rows * N, &src, &sh, &by);
            mbar_expect_tx(bar, by + fby);
            bulk_g2s(Ts + (h & 1) * tsz, src, by, bar);
        } else {
            mbar_expect_tx(bar, fby);  // arrives; with fby == 0 the phase completes at once
        }
        if (fby)
            bulk_g2s(Fs + ((h >> 1) & 1) * FWCAP * STP + (ra - u.u0) * STP,
                     a.Fb + a.fb_off[t] + (int64_t)(ra - dA) * STP, fby, bar);
    };
    // union probes outside a tile's window [ra, rb) would hold stale F rows: zero them in the
    // tile's F buffer (disjoint from the rows the bulk copy writes), so B fragments need no mask
    auto zfill = [&](int h) {
        const int t = u.t0 + (h >> 1);
        int ra = max(a.tile_dA[t], u.u0) - u.u0, rb = min(a.tile_dB[t], u.u1) - u.u0;
        if (rb <= ra) ra = rb = 0;
        double *Fz = Fs + ((h >> 1) & 1) * FWCAP * STP;
        const int nz = ra + (Wu - rb);
        for (int i = tid; i < nz * ST; i += 256) {
            const int r = i / ST, c = i - r * ST;
            Fz[(r < ra ? r : rb + (r - ra)) * STP + c] = 0.0;
        }
    };
    if (tid == 0) issue(0);
    zfill(0);
    __syncthreads();

    double cA[FWNB][2], cB[FWNB][2];
#pragma unroll
    for (int i = 0; i < FWNB; i++) cA[i][0] = cA[i][1] = cB[i][0] = cB[i][1] = 0.0;

    for (int h = 0; h < nh; h++) {
        if (tid == 0 && h + 1 < nh) issue(h + 1);
        if (h + 1 < nh && !((h + 1) & 1)) zfill(h + 1);   // buffer last read at step h - 2
        mbar_wait(&bars[h & 1], (h >> 1) & 1);
        const int t = u.t0 + (h >> 1), half = h & 1;
        const int k0 = t * ST + half * FH;
        const int rows = min(FH, a.Ml - k0);
        if (rows > 0) {
            const int sh = ncc > 1 ? 0 : (int)(((uintptr_t)(a.theta + (int64_t)k0 * N) & 15) >> 3);
            const double *T = Ts + (h & 1) * tsz + sh + t4 * TP + g4;
            const double *Frow = Fs + ((h >> 1) & 1) * FWCAP * STP + g4 * STP + t4 + half * FH;
            if (rows == FH) {
                gemm_fwd_t_nm<false>(nm, cA, T + 8 * warp, Frow, TP, FH, t4);
                if (second) gemm_fwd_t_nm<false>(nm, cB, T + 8 * (warp + 8), Frow, TP, FH, t4);
            } else {
                gemm_fwd_t_nm<true>(nm, cA, T + 8 * warp, Frow, TP, rows, t4);
                if (second) gemm_fwd_t_nm<true>(nm, cB, T + 8 * (warp + 8), Frow, TP, rows, t4);
            }
        }
        __syncthreads();
    }
    // partial rows rpart[(poff + d) * N + n]: lane holds n = 8 mb + g4, d = 8 nb + 2 t4 + {0,1}
#pragma unroll
    for (int pass = 0; pass < 2; pass++) {
        const int nl = 8 * (warp + 8 * pass) + g4;
        const int n = cbase + nl;
        if (nl >= ncol || (pass && !second)) continue;
#pragma unroll
        for (int nb = 0; nb < FWNB; nb++)
#pragma unroll
            for (int i = 0; i < 2; i++) {
                const int d = 8 * nb + 2 * t4 + i;
                if (nb < nm && d < Wu) a.rpart[(u.poff + d) * (int64_t)N + n] = pass ? cB[nb][i] : cA[nb][i];
            }
    }
}

// ------------------------------------------------------------------------------ wide N
// N > 128 (even, <= 1024): the gradient and the row projection become two kernels.
//   k_grad_wide  CTA (bwd unit, column chunk of 128 outcomes): G = F_tile^T R_win[:, chunk] by
//                DMMA (split-K slots per chunk as in k_bwd_mma), + gamma L Theta (Theta read from
//                global / L2), G stored; regulariser pair partial per (tile, chunk).
//   k_proj_wide  warp per Fock row (N / 32 values per lane): KKT, X = Theta -
//                t_k G, Michelot threshold (reading R4), Theta_{k+1}.
// ncc = ceil(N / 128) column chunks of balanced width 8 NB (NB = wide_nb(N) in [9, 16]), so no
// chunk is a thin remainder
int wide_nb(int N)
{
    const int ncc = (N + 127) / 128;
    return ((N + 7) / 8 + ncc - 1) / ncc;
}
// forward column chunks at wide N: balanced widths of at most 13 n-blocks, so that the staged
// half tiles (pitch 8 NB + 4) and F blocks of two CTAs fit one SM (16 warps; 16 n-blocks = 128
// columns left one CTA per SM, latency bound)
int wide_fwd_nb(int N)
{
    static const int forced = [] {   // QDT_WIDE_FWD_NB: chunk width in n-blocks (A/B)
        const char *e = getenv("QDT_WIDE_FWD_NB");
        const int v = e ? atoi(e) : 0;
        return (v >= 1 && v <= 16) ? v : 0;
    }();
    if (forced) return forced;
    const int nbt = (N + 7) / 8;
    const int ncc = (nbt + 12) / 13;
    return (nbt + ncc - 1) / ncc;
}
// k_grad_wide chunk ring depth: GW_STG stages of (F chunk, R chunk), i.e. GW_STG - 1 chunks in
// flight while one is multiplied.  Measured at Large (profiles/r02_v7/ab_wide_cap_ring.jsonl):
// 2 stages 0.357 ms, 3 stages 0.359, 4 stages 0.361 -- the double buffer stays.
#ifndef QDT_GW_STG
#define QDT_GW_STG 2
#endif
constexpr int GW_STG = QDT_GW_STG;
size_t wide_grad_smem() { return (size_t)(GW_STG * SKC * STP + GW_STG * SKC * (8 * 16 + 4) + 8) * sizeof(double); }

template <int NB>
__global__ void __launch_bounds__(256, 2) k_grad_wide(WideArgs a)
{
    constexpr int RPW = 8 * NB + 4;   // staged R row pitch (conflict-free B fragments)
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bars[GW_STG];
    __shared__ double red[8];
    __shared__ int s_last;
    const DevState *st = a.state;
    if (st && st->stop) return;
    const int64_t it = st ? st->it : 0;
    if (a.eval_gate && (it % a.kkt_every) != 0) return;
    const bool fis = a.beta != nullptr && !a.eval;   // FISTA step: stencil of Y
    const double beta = fis ? a.beta[it] : 0.0;
    const int N = a.N, ncc = a.ncc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const SwUnit u = a.units[blockIdx.x / ncc];
    const int cc = blockIdx.x - (blockIdx.x / ncc) * ncc;
    const int cbase = cc * 8 * NB, ncol = min(8 * NB, N - cbase);
    const int k0 = u.tile * ST, Tt = min(ST, a.Ml - k0);
    double *Fs = sm;
    double *Rs = sm + GW_STG * SKC * STP;
    const int W = u.p1 - u.p0, nch = (W + SKC - 1) / SKC;
    const double *Fg = a.Fb + a.fb_off[u.tile] + (int64_t)(u.p0 - a.tile_dA[u.tile]) * STP;
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < GW_STG; i++) mbar_init(&bars[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int c) {
        const int pb = c * SKC, kc = min(SKC, W - pb), sg = c % GW_STG;
        uint64_t *bar = &bars[sg];
        const uint32_t fby = (uint32_t)kc * STP * 8, rby = (uint32_t)ncol * 8;
        mbar_expect_tx(bar, fby + rby * kc);
        bulk_g2s(Fs + sg * SKC * STP, Fg + (int64_t)pb * STP, fby, bar);
        for (int j = 0; j < kc; j++)
            bulk_g2s(Rs + sg * SKC * RPW + j * RPW, a.R + (int64_t)(u.p0 + pb + j) * N + cbase, rby, bar);
    };
    if (tid == 0)
        for (int c = 0; c < GW_STG - 1 && c < nch; c++) issue(c);
    double acc[NB][2];
#pragma unroll
    for (int nb = 0; nb < NB; nb++) acc[nb][0] = acc[nb][1] = 0.0;
    // probes covering this warp's 8 rows: [pda, pdb) (contiguous: band edges are monotone); k-steps
    // of the window outside it multiply zero F entries (narrow low-k bands in a 64-row tile) and
    // are skipped (warp-uniform)
    int pda = u.p0, pdb = u.p1;
    if (a.row_da && 8 * warp < Tt) {
        pda = max(pda, a.row_da[k0 + 8 * warp]);
        pdb = min(pdb, a.row_db[min(k0 + 8 * warp + 7, k0 + Tt - 1)]);
    }
    for (int c = 0; c < nch; c++) {
        // the stage of chunk c + GW_STG - 1 was last read by chunk c - 1 (released by its barrier)
        if (tid == 0 && c + GW_STG - 1 < nch) issue(c + GW_STG - 1);
        const int sg = c % GW_STG;
        mbar_wait(&bars[sg], (c / GW_STG) & 1);
        const int kc = min(SKC, W - c * SKC);
        const int pb = u.p0 + c * SKC;
        gemm_bwd_rng<NB>(acc, Fs + sg * SKC * STP + 8 * warp + g4, Rs + sg * SKC * RPW + g4, kc, RPW, t4,
                         (pda - pb) >> 2, (pdb - pb + 3) >> 2);
        __syncthreads();
    }
    if (u.nsplit > 1) {
        const int64_t fsz = (int64_t)8 * NB * 64;
        double *slot = a.scratch + ((u.slot_base + u.slot) * ncc + cc) * fsz;
#pragma unroll
        for (int nb = 0; nb < NB; nb++)
            __stcg(reinterpret_cast<double2 *>(slot + ((warp * NB + nb) * 32 + lane) * 2),
                   make_double2(acc[nb][0], acc[nb][1]));
        __threadfence();
        __syncthreads();
        int *ctr = a.counters + (int64_t)u.tile * ncc + cc;
        if (tid == 0) s_last = (atomicAdd(ctr, 1) == u.nsplit - 1);
        __syncthreads();
        if (!s_last) return;
        __threadfence();
#pragma unroll
        for (int nb = 0; nb < NB; nb++) acc[nb][0] = acc[nb][1] = 0.0;
        for (int sl = 0; sl < u.nsplit; sl++) {
            const double *sp = a.scratch + ((u.slot_base + sl) * ncc + cc) * fsz;
#pragma unroll
            for (int nb = 0; nb < NB; nb++) {
                const double2 v = __ldcg(reinterpret_cast<const double2 *>(sp + ((warp * NB + nb) * 32 + lane) * 2));
                acc[nb][0] += v.x;
                acc[nb][1] += v.y;
            }
        }
        if (tid == 0) *ctr = 0;
    }
    // G = acc + gamma L Y on this row's chunk columns; Y = Theta (+ beta (Theta - Theta_{k-1}))
    const int r = 8 * warp + g4;
    const int kl = k0 + r;
    const int64_t kg = a.kb + kl;
    const bool act = r < Tt, hp = kg > 0, hn = kg + 1 < a.M;
    double sreg = 0.0;
    if (act) {
        const double *th = a.theta + (int64_t)kl * N + cbase;
        double *gout = a.G + (int64_t)kl * N + cbase;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) {
            const int c = 8 * nb + 2 * t4;
            if (c < ncol) {   // N even: the pair (c, c + 1) is valid together
                double2 x = __ldg(reinterpret_cast<const double2 *>(th + c));
                double2 y = hp ? __ldg(reinterpret_cast<const double2 *>(th + c - N)) : x;
                double2 z = hn ? __ldg(reinterpret_cast<const double2 *>(th + c + N)) : x;
                const double d20 = x.x - z.x, d21 = x.y - z.y;   // regulariser pair of Theta_k
                sreg = fma(d20, d20, fma(d21, d21, sreg));
                if (fis) {   // Y = Theta_k + beta (Theta_k - Theta_{k-1}) for the stencil
                    const double *tq = a.theta_prev + (int64_t)kl * N + cbase;
                    const double2 xq = __ldg(reinterpret_cast<const double2 *>(tq + c));
                    const double2 yq = hp ? __ldg(reinterpret_cast<const double2 *>(tq + c - N)) : xq;
                    const double2 zq = hn ? __ldg(reinterpret_cast<const double2 *>(tq + c + N)) : xq;
                    const double2 xo = x;
                    x = make_double2(fma(beta, x.x - xq.x, x.x), fma(beta, x.y - xq.y, x.y));
                    y = hp ? make_double2(fma(beta, y.x - yq.x, y.x), fma(beta, y.y - yq.y, y.y)) : x;
                    z = hn ? make_double2(fma(beta, z.x - zq.x, z.x), fma(beta, z.y - zq.y, z.y)) : x;
                    (void)xo;
                }
                const double g0 = fma(a.gamma, (x.x - y.x) + (x.x - z.x), acc[nb][0]);
                const double g1 = fma(a.gamma, (x.y - y.y) + (x.y - z.y), acc[nb][1]);
                *reinterpret_cast<double2 *>(gout + c) = make_double2(g0, g1);
            }
        }
    }
    sreg = wsum(sreg);
    if (lane == 0) red[warp] = sreg;
    __syncthreads();
    if (tid == 0) {
        double v = 0.0;
        for (int w = 0; w < 8; w++) v += red[w];
        double *pp = a.part + ((int64_t)u.tile * ncc + cc) * NSC_TILE;
        pp[SC_KKT] = 0.0;
        pp[SC_KKTP] = 0.0;
        pp[SC_REG] = v;
        pp[SC_DTH] = 0.0;
    }
}

template <int VM>
__global__ void __launch_bounds__(256) k_proj_wide(WideArgs a)
{
    __shared__ double red[8 * 2];
    const DevState *st = a.state;
    if (st && st->stop) return;
    const int64_t it = st ? st->it : 0;
    const int N = a.N, Nv = a.Nv;   // row pitch, outcomes (pad columns: excluded, written 0)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (a.eval_gate && (it % a.kkt_every) != 0) return;
    const bool fis = a.beta != nullptr && !a.eval;   // FISTA step: X from Y, KKT in the eval pass
    const double beta = fis ? a.beta[it] : 0.0;
    const bool do_kkt = a.eval || (!fis && (it % a.kkt_every) == 0);
    // CTA b owns the contiguous rows [b rpc, (b + 1) rpc) (grid fixed by Ml: deterministic sums);
    // warp w its rows w, w + 8, ...; KKT partials accumulate per warp in row order
    const int rpc = (int)(((a.Ml + gridDim.x - 1) / gridDim.x + 7) & ~7);
    const int rbeg = blockIdx.x * rpc, rend = min(a.Ml, rbeg + rpc);
    double skkt = 0.0, skktp = 0.0;
    for (int kl = rbeg + warp; kl < rend; kl += 8) {
    const bool act = true;
    double th[VM], x[VM];
    double mn = INFINITY;
    if (act) {
        const double *tr = a.theta + (int64_t)kl * N, *gr = a.G + (int64_t)kl * N;
#pragma unroll
        for (int v = 0; v < VM; v++) {
            const int n = lane + 32 * v;
            th[v] = n < N ? tr[n] : 0.0;
            x[v] = n < Nv ? gr[n] : INFINITY;   // G for now
            mn = fmin(mn, x[v]);
        }
    }
    mn = 2.0 * wmin(mn);
    const double lam = -mn, lamp = fmax(lam, 0.0);
    const double tk = act ? (a.tscal ? *a.tscal : a.tstep[kl]) : 0.0;
    double s = 0.0, xm = -INFINITY, xn = INFINITY;
#pragma unroll
    for (int v = 0; v < VM; v++) {
        const bool ok = act && lane + 32 * v < Nv;
        const double g = x[v];
        if (ok && do_kkt) {
            const double x1 = th[v] * fma(2.0, g, lam);
            skkt = fma(x1, x1, skkt);
            if (a.eval) {
                const double x2 = th[v] * fma(2.0, g, lamp);
                skktp = fma(x2, x2, skktp);
            }
        }
        double yv = th[v];
        if (fis && ok) yv = fma(beta, yv - a.theta_prev[(int64_t)kl * N + lane + 32 * v], yv);
        const double xv = fma(-tk, g, yv);
        x[v] = ok ? xv : -INFINITY;
        if (ok) {
            s += xv;
            xm = fmax(xm, xv);
            xn = fmin(xn, xv);
        }
    }
    if (!a.eval) {
        s = wsum(s);
        xm = wmax(xm);
        xn = wmin(xn);
        double tau = (s - 1.0) / (double)Nv;
        bool done = !act || xn > tau;
        if (!done) tau = fmax(tau, xm - 1.0);
        int cnt = Nv + 1;
        for (int round = 0; round <= Nv && !done; round++) {   // warp-uniform: one row per warp
            double ps = 0.0, mA = INFINITY;
            int pc = 0;
#pragma unroll
            for (int v = 0; v < VM; v++)
                if (x[v] > tau) {
                    ps += x[v];
                    pc++;
                    mA = fmin(mA, x[v]);
                }
            ps = wsum(ps);
            pc = wsum_i(pc);
            mA = wmin(mA);
            if (pc >= cnt) {
                done = true;
            } else {
                cnt = pc;
                tau = (ps - 1.0) / (double)pc;
                done = mA > tau;
            }
        }
        if (act) {
            double *o = a.out + (int64_t)kl * N;
#pragma unroll
            for (int v = 0; v < VM; v++) {
                const int n = lane + 32 * v;
                if (n < N) {
                    const double ov = x[v] - tau;
                    o[n] = ov > 0.0 ? ov : 0.0;
                }
            }
        }
    }
    }   // rows
    skkt = wsum(skkt);
    skktp = wsum(skktp);
    if (lane == 0) {
        red[warp * 2] = skkt;
        red[warp * 2 + 1] = skktp;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double k0 = 0.0, k1 = 0.0;
        for (int w = 0; w < 8; w++) {
            k0 += red[w * 2];
            k1 += red[w * 2 + 1];
        }
        double *pp = a.part + (a.part_b + (int64_t)blockIdx.x) * NSC_TILE;
        if (do_kkt) {   // a FISTA step leaves the evaluation pass's KKT in place
            pp[SC_KKT] = k0;
            pp[SC_KKTP] = k1;
        }
        pp[SC_REG] = 0.0;
        pp[SC_DTH] = 0.0;
    }
}

cudaError_t launch_grad_wide(const WideArgs &a_in, int nunits, cudaStream_t s)
{
    if (nunits <= 0) return cudaSuccess;
    WideArgs a = a_in;
    const int nb = wide_nb(a.N);
    a.ncc = (a.N + 8 * nb - 1) / (8 * nb);
    switch (nb) {
#define QDT_CASE(n) \
    case n: k_grad_wide<n><<<nunits * a.ncc, 256, wide_grad_smem(), s>>>(a); break;
        QDT_CASE(9) QDT_CASE(10) QDT_CASE(11) QDT_CASE(12) QDT_CASE(13) QDT_CASE(14) QDT_CASE(15) QDT_CASE(16)
#undef QDT_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

int wide_proj_blocks(int Ml) { return (int)std::min<int64_t>((Ml + 7) / 8, PW_BLOCKS); }

cudaError_t launch_proj_wide(const WideArgs &a, cudaStream_t s)
{
    const int grid = wide_proj_blocks(a.Ml);
    const int vm = (a.N + 31) / 32;
    if (vm <= 8) k_proj_wide<8><<<grid, 256, 0, s>>>(a);
    else if (vm <= 16) k_proj_wide<16><<<grid, 256, 0, s>>>(a);
    else if (vm <= 24) k_proj_wide<24><<<grid, 256, 0, s>>>(a);
    else if (vm <= 32) k_proj_wide<32><<<grid, 256, 0, s>>>(a);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ smoothing
// Long-range smoothing (eq. smoothing; reading R13) by column prefix sums:
// S(k) = sum_{j < k} Theta_j (per column), Theta~_i = (S(hi + 1) - S(lo)) / (hi - lo + 1) with
// [lo, hi] = [i - Ns, i + Ns] clipped to [0, M - 1], Ns = floor(i / div); rows i < exclude copied.
// Three kernels: chunk-local exclusive scans (SMC rows per chunk, thread per column), a scan of
// the chunk totals (thread per column), the apply pass (thread per element).
constexpr int SMC = 256;
__global__ void k_scan_local(const double *X, int64_t M, int N, double *S, double *T)
{
    const int64_t c = blockIdx.x;
    const int64_t r0 = c * SMC, r1 = min(M, r0 + SMC);
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        double run = 0.0;
        for (int64_t r = r0; r < r1; r++) {
            S[r * N + n] = run;
            run += X[r * N + n];
        }
        T[c * N + n] = run;
    }
}
__global__ void k_scan_chunks(const double *T, int64_t nch, int N, double *Tx)
{
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    double run = 0.0;
    for (int64_t c = 0; c < nch; c++) {
        Tx[c * N + n] = run;
        run += T[c * N + n];
    }
    Tx[nch * N + n] = run;
}
__global__ void k_smooth_apply(const double *X, const double *S, const double *Tx, int64_t M, int N,
                               int64_t exclude, int64_t div, double *Y)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M * N) return;
    const int64_t i = e / N;
    const int n = (int)(e - i * N);
    if (i < exclude || div <= 0) {
        Y[e] = X[e];
        return;
    }
    const int64_t ns = i / div;
    const int64_t lo = i - ns < 0 ? 0 : i - ns, hi = i + ns > M - 1 ? M - 1 : i + ns;
    auto Sabs = [&](int64_t k) {   // sum of rows [0, k)
        return k >= M ? Tx[((M + SMC - 1) / SMC) * N + n] : Tx[(k / SMC) * N + n] + S[k * N + n];
    };
    Y[e] = (Sabs(hi + 1) - Sabs(lo)) / (double)(hi - lo + 1);
}

cudaError_t launch_smooth(const double *X, int64_t M, int N, int64_t exclude, int64_t div, double *S,
                          double *T, double *Tx, double *Y, cudaStream_t s)
{
    const int64_t nch = (M + SMC - 1) / SMC;
    k_scan_local<<<(unsigned)nch, 128, 0, s>>>(X, M, N, S, T);
    k_scan_chunks<<<(N + 127) / 128, 128, 0, s>>>(T, nch, N, Tx);
    k_smooth_apply<<<(unsigned)((M * N + 255) / 256), 256, 0, s>>>(X, S, Tx, M, N, exclude, div, Y);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ BB step
// Barzilai-Borwein scalar step (reading R14): block partials of <s,s>, ||D s||^2 (pairs (k, k+1)
// with k + 1 < M, the slice's last row paired with its halo row) for s = Theta_k - Theta_{k-1},
// and of ||R_k - R_{k-1}||^2; then one thread forms t_k.
constexpr int BB_BLOCKS = 296;
__global__ void __launch_bounds__(256) k_bb_stats(const double *th, const double *tp, int64_t Ml,
                                                  int64_t kb, int64_t M, int N, const double *R,
                                                  const double *Rp, int64_t nR, double *part,
                                                  const DevState *st)
{
    __shared__ double red[8 * 3];
    if (st && st->stop) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double ss = 0.0, sd = 0.0, sh = 0.0;
    const int64_t tot = Ml * N, chunk = (tot + gridDim.x - 1) / gridDim.x;
    const int64_t e0 = blockIdx.x * chunk, e1 = min(tot, e0 + chunk);
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const double a = th[e] - tp[e];
        ss = fma(a, a, ss);
        const int64_t row = e / N;
        if (kb + row + 1 < M) {
            const double b = th[e + N] - tp[e + N];
            sd = fma(a - b, a - b, sd);
        }
    }
    if (R) {
        const int64_t c2 = (nR + gridDim.x - 1) / gridDim.x, r0 = blockIdx.x * c2, r1 = min(nR, r0 + c2);
        for (int64_t e = r0 + threadIdx.x; e < r1; e += blockDim.x) {
            const double d = R[e] - Rp[e];
            sh = fma(d, d, sh);
        }
    }
    ss = wsum(ss);
    sd = wsum(sd);
    sh = wsum(sh);
    if (lane == 0) {
        red[warp * 3] = ss;
        red[warp * 3 + 1] = sd;
        red[warp * 3 + 2] = sh;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double v0 = 0.0, v1 = 0.0, v2 = 0.0;
        for (int w = 0; w < 8; w++) {
            v0 += red[w * 3];
            v1 += red[w * 3 + 1];
            v2 += red[w * 3 + 2];
        }
        part[blockIdx.x * 3] = v0;
        part[blockIdx.x * 3 + 1] = v1;
        part[blockIdx.x * 3 + 2] = v2;
    }
}
// sum the block partials in order (vec3 = <s,s>, ||Ds||^2, ||dR||^2; multi-GPU: allreduced by the
// host between the two phases) -> t_k
__global__ void k_bb_sum(const double *part, int nblk, double *vec3, const DevState *st)
{
    if (threadIdx.x || (st && st->stop)) return;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int b = 0; b < nblk; b++) {
        v0 += part[b * 3];
        v1 += part[b * 3 + 1];
        v2 += part[b * 3 + 2];
    }
    vec3[0] = v0;
    vec3[1] = v1;
    vec3[2] = v2;
}
__global__ void k_bb_step(const double *vec3, double gamma, double tlip, double *tout, const DevState *st)
{
    if (threadIdx.x || (st && st->stop)) return;
    double t = tlip;
    if (st->it > 0) {
        const double shs = vec3[2] + gamma * vec3[1];
        if (shs > 0.0) {
            t = vec3[0] / shs;
            t = t < tlip ? tlip : (t > 1e6 * tlip ? 1e6 * tlip : t);
        }
    }
    *tout = t;
}
cudaError_t launch_bb_stats(const double *th, const double *tp, int64_t Ml, int64_t kb, int64_t M, int N,
                            const double *R, const double *Rp, int64_t nR, double *part, double *vec3,
                            const DevState *st, cudaStream_t s)
{
    k_bb_stats<<<BB_BLOCKS, 256, 0, s>>>(th, tp, Ml, kb, M, N, R, Rp, nR, part, st);
    k_bb_sum<<<1, 32, 0, s>>>(part, BB_BLOCKS, vec3, st);
    return cudaGetLastError();
}
// BB with the exact line search (reading R17): Z = P(Theta - t G) is in zt (halo rows included),
// R_k in Rk, F d in Rz (d = Z - Theta).  Block partials (fixed order) of
//   ||F d||^2,  <R_k, F d>,  ||D d||^2,  <D Theta, D d>,  ||d||^2,
// then one thread: <G,d> = <R_k, F d> + gamma <D Theta, D d>, lambda* = clip(max(-<G,d>, ||d||^2 / t)
// / (||F d||^2 + gamma ||D d||^2), 0, 1).
constexpr int BBLS_VALS = 5;
__global__ void __launch_bounds__(256) k_bbls_stats(const double *th, const double *zt, int64_t Ml, int64_t kb,
                                                    int64_t M, int N, const double *Rk, const double *Rz, int64_t nR,
                                                    double *part, const DevState *st)
{
    __shared__ double red[8 * BBLS_VALS];
    if (st && st->stop) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double v[BBLS_VALS] = {0.0, 0.0, 0.0, 0.0, 0.0};
    const int64_t tot = Ml * N, chunk = (tot + gridDim.x - 1) / gridDim.x;
    const int64_t e0 = blockIdx.x * chunk, e1 = min(tot, e0 + chunk);
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const double d = zt[e] - th[e];
        v[4] = fma(d, d, v[4]);
        const int64_t row = e / N;
        if (kb + row + 1 < M) {   // pair (row, row + 1), the slice's last row with its halo row
            const double dn = zt[e + N] - th[e + N];
            const double dd = d - dn, dt = th[e] - th[e + N];
            v[2] = fma(dd, dd, v[2]);
            v[3] = fma(dt, dd, v[3]);
        }
    }
    if (Rk) {
        const int64_t c2 = (nR + gridDim.x - 1) / gridDim.x, r0 = blockIdx.x * c2, r1 = min(nR, r0 + c2);
        for (int64_t e = r0 + threadIdx.x; e < r1; e += blockDim.x) {
            const double fd = Rz[e];   // F d (a forward pass of d: accurate for small d)
            v[0] = fma(fd, fd, v[0]);
            v[1] = fma(Rk[e], fd, v[1]);
        }
    }
#pragma unroll
    for (int i = 0; i < BBLS_VALS; i++) v[i] = wsum(v[i]);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < BBLS_VALS; i++) red[warp * BBLS_VALS + i] = v[i];
    __syncthreads();
    if (threadIdx.x == 0)
        for (int i = 0; i < BBLS_VALS; i++) {
            double x = 0.0;
            for (int w = 0; w < 8; w++) x += red[w * BBLS_VALS + i];
            part[blockIdx.x * BBLS_VALS + i] = x;
        }
}
__global__ void k_bbls_sum(const double *part, int nblk, double *vec, const DevState *st)
{
    if (threadIdx.x || (st && st->stop)) return;
    for (int i = 0; i < BBLS_VALS; i++) {
        double x = 0.0;
        for (int b = 0; b < nblk; b++) x += part[b * BBLS_VALS + i];
        vec[i] = x;
    }
}
__global__ void k_bbls_lambda(const double *vec, double gamma, const double *tbb, double *lam, const DevState *st)
{
    if (threadIdx.x || (st && st->stop)) return;
    const double fdd = vec[0], rfd = vec[1], ddd = vec[2], tdd = vec[3], dd = vec[4];
    const double gd = rfd + gamma * tdd;                 // <G, d>
    const double den = fdd + gamma * ddd;
    const double num = fmax(-gd, dd / *tbb);
    double l = 1.0;
    if (den > 0.0) {
        l = num / den;
        l = l < 0.0 ? 0.0 : (l > 1.0 ? 1.0 : l);
    }
    *lam = l;
}
// d = Z - Theta_k (halo rows included)
__global__ void k_bbls_dir(const double *th, const double *zt, double *dd, int64_t n, const DevState *st)
{
    if (st && st->stop) return;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        dd[e] = zt[e] - th[e];
}
cudaError_t launch_bbls_dir(const double *th, const double *zt, double *dd, int64_t n, const DevState *st,
                            cudaStream_t s)
{
    k_bbls_dir<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(th, zt, dd, n, st);
    return cudaGetLastError();
}
// Theta_{k+1} = Theta_k + lambda (Z - Theta_k), in place over Z, halo rows included
__global__ void k_bbls_update(const double *th, double *zt, int64_t n, const double *lam, const DevState *st)
{
    if (st && st->stop) return;
    const double l = *lam;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        zt[e] = fma(l, zt[e] - th[e], th[e]);
}
cudaError_t launch_bbls_stats(const double *th, const double *zt, int64_t Ml, int64_t kb, int64_t M, int N,
                              const double *Rk, const double *Rz, int64_t nR, double *part, double *vec,
                              const DevState *st, cudaStream_t s)
{
    k_bbls_stats<<<BB_BLOCKS, 256, 0, s>>>(th, zt, Ml, kb, M, N, Rk, Rz, nR, part, st);
    k_bbls_sum<<<1, 32, 0, s>>>(part, BB_BLOCKS, vec, st);
    return cudaGetLastError();
}
cudaError_t launch_bbls_step(const double *vec, double gamma, const double *tbb, double *lam, const double *th,
                             double *zt, int64_t n, const DevState *st, cudaStream_t s)
{
    k_bbls_lambda<<<1, 32, 0, s>>>(vec, gamma, tbb, lam, st);
    k_bbls_update<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(th, zt, n, lam, st);
    return cudaGetLastError();
}

cudaError_t launch_bb_step(const double *vec3, double gamma, double tlip, double *tout,
                           const DevState *st, cudaStream_t s)
{
    k_bb_step<<<1, 32, 0, s>>>(vec3, gamma, tlip, tout, st);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ reduce R
// Warp per probe: R[d,:] = sum_j rpart[rows_j] (list order = ascending Fock) - P[d,:]; the
// block's ||R||^2 partial (warp order) goes to partR[blockIdx.x].
__global__ void __launch_bounds__(256) k_reduce_R2(const double *rpart, const int64_t *red_beg,
                                                   const int64_t *red_rows, const double *P,
                                                   double *R, int D, int N, double *partR,
                                                   const DevState *st)
{
    __shared__ double red[8];
    if (st && st->stop) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int d = blockIdx.x * 8 + warp;
    double ss = 0.0;
    if (d < D) {
        const int64_t j0 = red_beg[d], j1 = red_beg[d + 1];
        for (int n0 = 0; n0 < N; n0 += 128) {          // four independent columns per lane
            double s[4] = {0.0, 0.0, 0.0, 0.0};
            int64_t j = j0;
            // four partial rows in flight, added in list order (same sums as one row at a time)
            for (; j + 4 <= j1; j += 4) {
                const int64_t r0 = red_rows[j], r1 = red_rows[j + 1], r2 = red_rows[j + 2], r3 = red_rows[j + 3];
                double q[4][4];
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const bool ok = n0 + lane + 32 * c < N;
                    const int64_t o = n0 + lane + 32 * c;
                    q[0][c] = ok ? rpart[r0 * N + o] : 0.0;
                    q[1][c] = ok ? rpart[r1 * N + o] : 0.0;
                    q[2][c] = ok ? rpart[r2 * N + o] : 0.0;
                    q[3][c] = ok ? rpart[r3 * N + o] : 0.0;
                }
#pragma unroll
                for (int c = 0; c < 4; c++) s[c] = (((s[c] + q[0][c]) + q[1][c]) + q[2][c]) + q[3][c];
            }
            for (; j < j1; j++) {
                const double *src = rpart + red_rows[j] * N + n0 + lane;
#pragma unroll
                for (int c = 0; c < 4; c++)
                    if (n0 + lane + 32 * c < N) s[c] += src[32 * c];
            }
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int n = n0 + lane + 32 * c;
                if (n < N) {
                    double v = s[c];
                    if (P) v -= P[(int64_t)d * N + n];
                    R[(int64_t)d * N + n] = v;
                    ss = fma(v, v, ss);
                }
            }
        }
    }
    ss = wsum(ss);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (threadIdx.x == 0 && partR) {
        double v = 0.0;
        for (int w = 0; w < 8; w++) v += red[w];
        partR[blockIdx.x] = v;
    }
}

// Even N: the same sums over a balanced item grid.  Item = (probe d, column chunk of 128): lane
// holds the double2 pairs at columns 128 c + 2 lane + {0, 64}; the partial rows of d are added in
// list order (the per-column order of k_reduce_R2).  Global warp gw takes items gw, gw + NW, ...
// (NW = 8 G warps, G = min(nR, 8 x SMs) blocks: one wave, no tail of a third of a wave); its
// ||R||^2 terms accumulate in item order, the block's warps are combined in warp order into
// partR[block] (deterministic for a fixed G); block 0 zeroes partR[G, nR).
__global__ void __launch_bounds__(256) k_reduce_R3(const double *rpart, const int64_t *red_beg,
                                                   const int64_t *red_rows, const double *P,
                                                   double *R, int D, int N, double *partR, int nR,
                                                   const DevState *st)
{
    __shared__ double red[8];
    if (st && st->stop) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nch = (N + 127) >> 7;
    const int64_t nitems = (int64_t)D * nch;
    const int64_t NW = 8 * (int64_t)gridDim.x;
    double ss = 0.0;
    for (int64_t it = (int64_t)blockIdx.x * 8 + warp; it < nitems; it += NW) {
        const int d = (int)(it / nch), c = (int)(it - (int64_t)d * nch);
        const int n0 = 128 * c + 2 * lane, n1 = n0 + 64;
        const bool ok0 = n0 < N, ok1 = n1 < N;   // N even: a pair is whole or absent
        const int64_t j0 = red_beg[d], j1 = red_beg[d + 1];
        double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
        int64_t j = j0;
        for (; j + 4 <= j1; j += 4) {
            double2 q0[4], q1[4];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const double *row = rpart + red_rows[j + r] * N;
                q0[r] = ok0 ? *reinterpret_cast<const double2 *>(row + n0) : make_double2(0.0, 0.0);
                q1[r] = ok1 ? *reinterpret_cast<const double2 *>(row + n1) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int r = 0; r < 4; r++) {
                s0.x += q0[r].x, s0.y += q0[r].y;
                s1.x += q1[r].x, s1.y += q1[r].y;
            }
        }
        for (; j < j1; j++) {
            const double *row = rpart + red_rows[j] * N;
            const double2 q0 = ok0 ? *reinterpret_cast<const double2 *>(row + n0) : make_double2(0.0, 0.0);
            const double2 q1 = ok1 ? *reinterpret_cast<const double2 *>(row + n1) : make_double2(0.0, 0.0);
            s0.x += q0.x, s0.y += q0.y;
            s1.x += q1.x, s1.y += q1.y;
        }
        double *Rr = R + (int64_t)d * N;
        const double *Pr = P ? P + (int64_t)d * N : nullptr;
        if (ok0) {
            if (Pr) {
                const double2 p = *reinterpret_cast<const double2 *>(Pr + n0);
                s0.x -= p.x, s0.y -= p.y;
            }
            *reinterpret_cast<double2 *>(Rr + n0) = s0;
            ss = fma(s0.x, s0.x, ss);
            ss = fma(s0.y, s0.y, ss);
        }
        if (ok1) {
            if (Pr) {
                const double2 p = *reinterpret_cast<const double2 *>(Pr + n1);
                s1.x -= p.x, s1.y -= p.y;
            }
            *reinterpret_cast<double2 *>(Rr + n1) = s1;
            ss = fma(s1.x, s1.x, ss);
            ss = fma(s1.y, s1.y, ss);
        }
    }
    ss = wsum(ss);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (!partR) return;
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < 8; w++) v += red[w];
        partR[blockIdx.x] = v;
    }
    if (blockIdx.x == 0)
        for (int i = gridDim.x + threadIdx.x; i < nR; i += blockDim.x) partR[i] = 0.0;
}

// ------------------------------------------------------------------------------ scalars
// G blocks (G <= SC2_BLOCKS): block b sums a contiguous slice of the tile partials and of partR
// (thread t: entries t, t + blockDim, ... of the slice, in order), then a fixed-shape tree over
// warps, into stage[b].  The last block to arrive (ticket on *arrive, reset by it) sums the G
// block partials in block order and applies the trace / KKT / stop logic (thread 0).
// Deterministic (fixed slices and orders), no floating-point atomics.
__global__ void __launch_bounds__(256) k_scalars2(const double *partR, int nR, const double *partT,
                                                  int ntiles, int include_r2, double *stage,
                                                  int *arrive, double *vec, int64_t N, int64_t M,
                                                  double gamma, double tol, int final_eval,
                                                  int kkt_every, double *trace, double *kkt,
                                                  double *kktp, int64_t trace_len, DevState *st,
                                                  int finalize)
{
    __shared__ double red[8 * NV];
    __shared__ int s_last;
    if (st->stop) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x, b = blockIdx.x;
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = 0.0;
    constexpr int BQ = 4;   // loads in flight per thread, added in the same order as one at a time
    if (include_r2) {
        const int cr = (nR + G - 1) / G, r0 = b * cr, r1 = min(nR, r0 + cr);
        int i = r0 + threadIdx.x;
        for (; i + (BQ - 1) * (int)blockDim.x < r1; i += BQ * blockDim.x) {
            double q[BQ];
#pragma unroll
            for (int j = 0; j < BQ; j++) q[j] = partR[i + j * blockDim.x];
#pragma unroll
            for (int j = 0; j < BQ; j++) v[V_R2] += q[j];
        }
        for (; i < r1; i += blockDim.x) v[V_R2] += partR[i];
    }
    {
        const int ct = (ntiles + G - 1) / G, t0 = b * ct, t1 = min(ntiles, t0 + ct);
        int t = t0 + threadIdx.x;
        for (; t + (BQ - 1) * (int)blockDim.x < t1; t += BQ * blockDim.x) {
            double4 q[BQ];
#pragma unroll
            for (int j = 0; j < BQ; j++)
                q[j] = *reinterpret_cast<const double4 *>(partT + (int64_t)(t + j * blockDim.x) * NSC_TILE);
#pragma unroll
            for (int j = 0; j < BQ; j++) {
                v[V_KKT] += q[j].x;
                v[V_KKTP] += q[j].y;
                v[V_REG] += q[j].z;
                v[V_DTH] += q[j].w;
            }
        }
        for (; t < t1; t += blockDim.x) {
            const double4 q = *reinterpret_cast<const double4 *>(partT + (int64_t)t * NSC_TILE);
            v[V_KKT] += q.x;
            v[V_KKTP] += q.y;
            v[V_REG] += q.z;
            v[V_DTH] += q.w;
        }
    }
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = wsum(v[i]);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; i++) red[warp * NV + i] = v[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        double w[NV];
#pragma unroll
        for (int i = 0; i < NV; i++) w[i] = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); k++)
#pragma unroll
            for (int i = 0; i < NV; i++) w[i] += red[k * NV + i];
        if (G == 1) {
#pragma unroll
            for (int i = 0; i < NV; i++) v[i] = w[i];
            s_last = 1;
        } else {
#pragma unroll
            for (int i = 0; i < NV; i++) __stcg(stage + b * NV + i, w[i]);
            __threadfence();
            s_last = atomicAdd(arrive, 1) == G - 1;
        }
    }
    __syncthreads();
    if (!s_last) return;
    if (G > 1) {   // last block: the block partials in block order (warp 0: lanes b, b + 32)
        __threadfence();
        if (warp != 0) return;
#pragma unroll
        for (int i = 0; i < NV; i++) {
            double x = lane < G ? __ldcg(stage + lane * NV + i) : 0.0;
            if (lane + 32 < G) x += __ldcg(stage + (lane + 32) * NV + i);
            v[i] = wsum(x);
        }
        if (lane == 0) *arrive = 0;
    }
    if (threadIdx.x != 0) return;
    for (int i = 0; i < NV; i++) vec[i] = v[i];
    if (!finalize) return;  // multi-GPU: allreduce + k_finalize follow
    const int64_t k = st->it;
    const double f = v[V_R2] + gamma * v[V_REG];
    const bool kv = final_eval || (k % kkt_every) == 0;
    const double nm = (double)N * (double)M;
    const double r = kv ? sqrt(v[V_KKT] / nm) : NAN;
    const double rp = kv ? sqrt(v[V_KKTP] / nm) : NAN;
    if (k < trace_len) {
        if (trace) trace[k] = f;
        if (kkt) kkt[k] = r;
        if (kktp) kktp[k] = rp;
    }
    if (!isfinite(f)) {
        st->nonfinite = 1;
        st->stop = 1;
        st->iters_done = k;
        return;
    }
    if (final_eval) {
        st->iters_done = k;
        return;
    }
    if (kv && r <= tol) {
        st->stop = 1;
        st->converged = 1;
        st->iters_done = k;
        return;
    }
    st->it = k + 1;
}

// ------------------------------------------------------------------------------ launchers
cudaError_t launch_tile_F(Band b, int64_t kb, int Ml, int ntiles, const int32_t *tile_dA,
                          const int32_t *tile_dB, const int64_t *fb_off, double *Fb,
                          cudaStream_t s)
{
    if (ntiles <= 0) return cudaSuccess;
    k_tile_F<<<ntiles, 256, 0, s>>>(b, kb, Ml, tile_dA, tile_dB, fb_off, Fb);
    return cudaGetLastError();
}

template <int NB>
static cudaError_t prep_nb()
{
    const int big = 210 * 1024;  // fwd at N = 128 needs 203 KB; the opt-in cap (227 KB) includes static smem
    cudaError_t e = cudaFuncSetAttribute(k_bwd_mma<NB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_bwd_mma<NB, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_bwd_mma<NB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess && NB >= 9)
        e = cudaFuncSetAttribute(k_grad_wide<NB < 9 ? 9 : NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_bwd_split<NB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_bwd_split<NB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_bwd_split<NB, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_fwd_mma<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    return e;
}

#define QDT_FOR_NB(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

cudaError_t prepare_sweep_kernels()
{
    // the shared-memory attribute is per device: prepare each device ordinal once
    static uint64_t done_mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0;
    if (done_mask & bit) return cudaSuccess;
    bool done = false;
    cudaError_t e = cudaSuccess;
#define QDT_PREP(nb) if (e == cudaSuccess) e = prep_nb<nb>();
    QDT_FOR_NB(QDT_PREP)
#undef QDT_PREP
#define QDT_PREP(nb) \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_bwd_mma<nb, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    QDT_PREP(17) QDT_PREP(18) QDT_PREP(19) QDT_PREP(20)
#undef QDT_PREP
    done = e == cudaSuccess;
    if (done) done_mask |= bit;
    return e;
}

// exact n-block count: only the last n-block of a row can hold padding columns
// (N in (128, 160], even: plain steps only, k_bwd_mma without the register stash; the forward
// pass and FISTA / evaluation passes take the wide kernels)
int sweep_nb(int N)
{
    if (N >= 1 && N <= 8 * SW_NBMAX) return (N + 7) / 8;
    if (N > 8 * SW_NBMAX && N <= 8 * SW_NBX && N % 2 == 0) return (N + 7) / 8;
    return 0;
}

// Tensor maps of the Theta buffers for the TP tile copies (box tp_pitch(NB) x 66 over rows
// -1 .. Ml); the encoder comes from the driver through the runtime (no libcuda link).  Returns
// false (TP not used) for odd N (row stride not a multiple of 16 bytes) or without an encoder.
static bool sweep_tensor_maps(SweepArgs &a, int NB)
{
    a.tm_on = 0;
    const int N = a.N, P = tp_pitch(NB);
    if ((N & 1) || P < N) return false;
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void *fp = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            return false;
        enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    }
    auto encode = [&](CUtensorMap *tm, const double *base) {
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)a.Ml + 2};
        cuuint64_t strides[1] = {(cuuint64_t)N * sizeof(double)};
        cuuint32_t box[2] = {(cuuint32_t)P, (cuuint32_t)(ST + 2)};
        cuuint32_t es[2] = {1, 1};
        return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)(base - N), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    bool ok = encode(&a.tm_theta, a.theta);
    if (ok && a.theta_prev) ok = encode(&a.tm_prev, a.theta_prev);
    a.tm_on = ok ? 1 : 0;
    return ok;
}

// QDT_TMA_TILE: 1 (default) plain steps at even N <= 128 stage the Theta tile by tensor copy at
// the bank-conflict-free pitch; 0 keeps the contiguous bulk copy (A/B)
static bool tma_tile_on()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("QDT_TMA_TILE");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

cudaError_t launch_bwd_mma(const SweepArgs &a_in, int nunits, int NB, cudaStream_t s)
{
    if (nunits <= 0) return cudaSuccess;
    SweepArgs a = a_in;
    a.tm_on = 0;
    a.nunits = nunits;
    const bool fis = a.beta != nullptr && !a.eval;
    const bool tp = !fis && NB <= SW_NBMAX && tma_tile_on() && sweep_tensor_maps(a, NB);
    const size_t smem = sweep_bwd_smem(a.N, NB, fis, tp);
    const int nsm = device_sm_count();
    const int grid = std::min(nunits, (NB <= 13 && !fis ? 2 : 1) * nsm);
    switch (NB) {
#define QDT_CASE(nb)                                                       \
    case nb:                                                               \
        if (fis)                                                           \
            k_bwd_mma<nb, true><<<grid, 256, smem, s>>>(a);                \
        else if (tp)                                                       \
            k_bwd_mma<nb, false, true><<<grid, 256, smem, s>>>(a);         \
        else                                                               \
            k_bwd_mma<nb, false><<<grid, 256, smem, s>>>(a);               \
        break;
        QDT_FOR_NB(QDT_CASE)
#undef QDT_CASE
#define QDT_CASE(nb)                                                       \
    case nb:                                                               \
        if (fis) return cudaErrorInvalidValue;                             \
        k_bwd_mma<nb, false><<<grid, 256, smem, s>>>(a);                   \
        break;
        QDT_CASE(17) QDT_CASE(18) QDT_CASE(19) QDT_CASE(20)
#undef QDT_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// N-split bwd (512 threads): used when sweep_split_on(); same arguments as launch_bwd_mma
int sweep_split_mode()
{
    static int mode = -1;   // 0: never, 1: always, 2 (default): FISTA steps only
    if (mode < 0) {
        const char *e = getenv("QDT_SPLITN");
        mode = e ? atoi(e) : 2;
    }
    return mode;
}

cudaError_t launch_bwd_split(const SweepArgs &a_in, int nunits, int NB, cudaStream_t s)
{
    if (nunits <= 0) return cudaSuccess;
    SweepArgs a = a_in;
    a.tm_on = 0;
    a.nunits = nunits;
    const bool fis = a.beta != nullptr && !a.eval;
    const bool tp = fis && NB <= SW_NBMAX && tma_tile_on() && sweep_tensor_maps(a, NB);   // FISTA steps
    const size_t smem = sweep_bwd_smem(a.N, NB, true, tp);   // two tiles: double buffer or Theta_{k-1}
    const int nsm = device_sm_count();
    const int grid = std::min(nunits, nsm);
    switch (NB) {
#define QDT_CASE(nb)                                                       \
    case nb:                                                               \
        if (fis && tp)                                                     \
            k_bwd_split<nb, true, true><<<grid, 512, smem, s>>>(a);        \
        else if (fis)                                                      \
            k_bwd_split<nb, true><<<grid, 512, smem, s>>>(a);              \
        else                                                               \
            k_bwd_split<nb, false><<<grid, 512, smem, s>>>(a);             \
        break;
        QDT_FOR_NB(QDT_CASE)
#undef QDT_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_fwd_mma(const SweepFwdArgs &a_in, int nunits, int NB, cudaStream_t s)
{
    if (nunits <= 0) return cudaSuccess;
    SweepFwdArgs a = a_in;
    a.ncc = (a.N + 8 * NB - 1) / (8 * NB);
    const size_t smem = sweep_fwd_smem(a.N, NB);
    nunits *= a.ncc;
    switch (NB) {
#define QDT_CASE(nb) \
    case nb: k_fwd_mma<nb><<<nunits, 256, smem, s>>>(a); break;
        QDT_FOR_NB(QDT_CASE)
#undef QDT_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}


// QDT_REDUCE_R3=0 selects the block-per-8-probes reduction at even N too (A/B)
static bool reduce_r3_on()
{
    static const bool on = [] {
        const char *e = getenv("QDT_REDUCE_R3");
        return !(e && e[0] == '0');
    }();
    return on;
}

cudaError_t launch_reduce_R2(const double *rpart, const int64_t *red_beg, const int64_t *red_rows,
                             const double *P, double *R, int D, int N, double *partR,
                             const DevState *st, cudaStream_t s)
{
    const int nR = (D + 7) / 8;   // partR entries (Plan::nR of one rank)
    if ((N & 1) == 0 && reduce_r3_on()) {
        const int G = std::max(1, std::min(nR, 8 * device_sm_count()));
        k_reduce_R3<<<G, 256, 0, s>>>(rpart, red_beg, red_rows, P, R, D, N, partR, nR, st);
    } else {
        k_reduce_R2<<<nR, 256, 0, s>>>(rpart, red_beg, red_rows, P, R, D, N, partR, st);
    }
    return cudaGetLastError();
}

cudaError_t launch_scalars2(const double *partR, int nR, const double *partT, int ntiles,
                            int include_r2, double *stage, int *arrive, double *vec, int64_t N,
                            int64_t M, double gamma, double tol, int final_eval, int kkt_every,
                            double *trace, double *kkt, double *kktp, int64_t trace_len,
                            DevState *st, int finalize, cudaStream_t s)
{
    // block count: ~256 tile partials per block (one double4 load per thread), at most SC2_BLOCKS
    const int G = std::max(1, std::min(SC2_BLOCKS, std::max(ntiles, include_r2 ? nR : 0) / 256));
    k_scalars2<<<(stage && arrive) ? G : 1, 256, 0, s>>>(partR, nR, partT, ntiles, include_r2, stage, arrive, vec,
                                          N, M, gamma, tol, final_eval, kkt_every, trace, kkt, kktp,
                                          trace_len, st, finalize);
    return cudaGetLastError();
}

}  // namespace qdt
