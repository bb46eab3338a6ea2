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
#include <math.h>
#include <stdint.h>

#include "qdt_internal.h"

namespace qdt {

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// bulk global -> shared copy (16-byte aligned addresses, size a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// D(8x8) += A(8x4) B(4x8), fp64 tensor core.  Fragments (lane = 4 g + t):
//   a = A[g][t], b = B[t][g], (c0, c1) = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double quad_sum(double v)
{
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    return v;
}
__device__ __forceinline__ int quad_sum_i(int v)
{
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    return v;
}
__device__ __forceinline__ double quad_max(double v)
{
    v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 1));
    v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 2));
    return v;
}
__device__ __forceinline__ double quad_min(double v)
{
    v = fmin(v, __shfl_xor_sync(0xffffffffu, v, 1));
    v = fmin(v, __shfl_xor_sync(0xffffffffu, v, 2));
    return v;
}
__device__ __forceinline__ double wsum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

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
template <int NB, bool FULL, bool EVEN>
__device__ __forceinline__ void row_step(double (&acc)[NB][2], const double *thr, int N, int t4,
                                         bool act, bool has_prev, bool has_next, double gamma,
                                         double tk, bool do_kkt, bool want_kktp, double &sreg,
                                         double &skkt, double &skktp, double *orow)
{
    const int cl = 8 * (NB - 1) + 2 * t4;
    const bool v0 = cl < N, v1 = cl + 1 < N;
    const bool hp = FULL || has_prev, hn = FULL || has_next;
    double mn = INFINITY;
#pragma unroll
    for (int nb = 0; nb < NB; nb++) {
        const int c = 8 * nb + 2 * t4;
        double t0[2], tp[2], tn[2];
        if (EVEN) {
            const double2 a = *reinterpret_cast<const double2 *>(thr + c);
            const double2 b = *reinterpret_cast<const double2 *>(thr + c - N);
            const double2 d = *reinterpret_cast<const double2 *>(thr + c + N);
            t0[0] = a.x, t0[1] = a.y, tp[0] = b.x, tp[1] = b.y, tn[0] = d.x, tn[1] = d.y;
        } else {
#pragma unroll
            for (int i = 0; i < 2; i++) t0[i] = thr[c + i], tp[i] = thr[c + i - N], tn[i] = thr[c + i + N];
        }
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const bool valid = (nb < NB - 1) || (i ? v1 : v0);
            const bool ok = FULL ? valid : (act && valid);
            const double a0 = t0[i];
            const double an = hn ? tn[i] : a0;
            const double ap = hp ? tp[i] : a0;
            const double dd = a0 - an;
            double g = acc[nb][i];
            if (gamma != 0.0) g = fma(gamma, (a0 - ap) + (a0 - an), g);
            if (ok) {
                sreg = fma(dd, dd, sreg);
                mn = fmin(mn, g);
            }
            acc[nb][i] = ok ? g : INFINITY;
        }
    }
    double lam = 0.0, lamp = 0.0;
    if (do_kkt) {
        mn = 2.0 * quad_min(mn);
        lam = -mn;
        lamp = fmax(lam, 0.0);
    }
    double s = 0.0, xm = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < NB; nb++) {
        const int c = 8 * nb + 2 * t4;
        double t0[2];
        if (EVEN) {
            const double2 a = *reinterpret_cast<const double2 *>(thr + c);
            t0[0] = a.x, t0[1] = a.y;
        } else {
            t0[0] = thr[c], t0[1] = thr[c + 1];
        }
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const bool valid = (nb < NB - 1) || (i ? v1 : v0);
            const bool ok = FULL ? valid : (act && valid);
            const double g = acc[nb][i];
            if (do_kkt && ok) {
                const double x1 = t0[i] * fma(2.0, g, lam);
                skkt = fma(x1, x1, skkt);
                if (want_kktp) {
                    const double x2 = t0[i] * fma(2.0, g, lamp);
                    skktp = fma(x2, x2, skktp);
                }
            }
            const double x = fma(-tk, g, t0[i]);
            acc[nb][i] = ok ? x : -INFINITY;
            if (ok) {
                s += x;
                xm = fmax(xm, x);
            }
        }
    }
    s = quad_sum(s);
    xm = quad_max(xm);
    // Michelot from the larger of two lower bounds of tau* (the mean bound and max - 1): the
    // active-set updates then increase monotonically to tau* (reading R4)
    int cnt = N + 1;
    double tau = fmax((s - 1.0) / (double)N, xm - 1.0);
    bool done = !(FULL || act);
    for (int round = 0; round <= N; round++) {
        if (__all_sync(0xffffffffu, done)) break;
        double ps = 0.0;
        int pc = 0;
#pragma unroll
        for (int nb = 0; nb < NB; nb++)
#pragma unroll
            for (int i = 0; i < 2; i++)
                if (acc[nb][i] > tau) {
                    ps += acc[nb][i];
                    pc++;
                }
        ps = quad_sum(ps);
        pc = quad_sum_i(pc);
        if (!done) {
            if (pc >= cnt) {
                done = true;
            } else {
                cnt = pc;
                tau = (ps - 1.0) / (double)pc;
            }
        }
    }
    if (FULL || act) {
#pragma unroll
        for (int nb = 0; nb < NB; nb++) {
            const int c = 8 * nb + 2 * t4;
            const double o0 = fmax(acc[nb][0] - tau, 0.0), o1 = fmax(acc[nb][1] - tau, 0.0);
            if (EVEN) {
                if (nb < NB - 1 || v0) *reinterpret_cast<double2 *>(orow + c) = make_double2(o0, o1);
            } else {
                if (nb < NB - 1 || v0) orow[c] = o0;
                if (nb < NB - 1 || v1) orow[c + 1] = o1;
            }
        }
    }
}

// ------------------------------------------------------------------------------ bwd sweep
// Smem: Theta tile (ST+2 rows incl. halo) | F chunks 2 x SKC x STP | R chunks 2 x (SKC*N + pad)
template <int NB>
struct SwLayout {
    int thsz, rsz;
    __device__ __host__ SwLayout(int N)
    {
        thsz = (((ST + 2) * N + 4) + 1) & ~1;
        rsz = ((SKC * N + 8 * NB + 4) + 1) & ~1;
    }
    __device__ __host__ size_t bytes() const
    {
        return (size_t)(thsz + 2 * SKC * STP + 2 * rsz) * sizeof(double);
    }
};

size_t sweep_bwd_smem(int N, int NB)
{
    const int thsz = (((ST + 2) * N + 4) + 1) & ~1;
    const int rsz = ((SKC * N + 8 * NB + 4) + 1) & ~1;
    return (size_t)(thsz + 2 * SKC * STP + 2 * rsz) * sizeof(double);
}

template <int NB>
__global__ void __launch_bounds__(256, 2) k_bwd_mma(SweepArgs a)
{
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bars[3];
    __shared__ double red[8 * 3];
    __shared__ int s_last;
    const DevState *st = a.state;
    if (st && st->stop) return;
    const int64_t it = st ? st->it : 0;
    const int N = a.N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const SwUnit u = a.units[blockIdx.x];
    const int k0 = u.tile * ST;
    const int Tt = min(ST, a.Ml - k0);
    const SwLayout<NB> L(N);
    double *Th = sm;
    double *Fs = sm + L.thsz;
    double *Rs = Fs + 2 * SKC * STP;

    const int W = u.p1 - u.p0;
    const int nch = (W + SKC - 1) / SKC;
    const double *Fg = a.Fb + a.fb_off[u.tile] + (int64_t)(u.p0 - a.tile_dA[u.tile]) * STP;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        fence_barrier_init();
    }
    __syncthreads();

    const double *th_src;
    int th_sh;
    uint32_t th_bytes;
    aligned_span(a.theta + (int64_t)(k0 - 1) * N, (int64_t)(Tt + 2) * N, &th_src, &th_sh, &th_bytes);
    auto issue_chunk = [&](int c) {
        const int pb = c * SKC;
        const int kc = min(SKC, W - pb);
        const double *rsrc;
        int rsh;
        uint32_t rbytes;
        aligned_span(a.R + (int64_t)(u.p0 + pb) * N, (int64_t)kc * N, &rsrc, &rsh, &rbytes);
        uint64_t *bar = &bars[1 + (c & 1)];
        const uint32_t fbytes = (uint32_t)kc * STP * 8;
        mbar_expect_tx(bar, fbytes + rbytes);
        bulk_g2s(Fs + (c & 1) * SKC * STP, Fg + (int64_t)pb * STP, fbytes, bar);
        bulk_g2s(Rs + (c & 1) * L.rsz, rsrc, rbytes, bar);
    };
    if (tid == 0) {
        if (u.nsplit == 1) {
            mbar_expect_tx(&bars[0], th_bytes);
            bulk_g2s(Th, th_src, th_bytes, &bars[0]);
        }
        if (nch > 0) issue_chunk(0);
    }

    double acc[NB][2];
#pragma unroll
    for (int nb = 0; nb < NB; nb++) acc[nb][0] = acc[nb][1] = 0.0;

    for (int c = 0; c < nch; c++) {
        if (tid == 0 && c + 1 < nch) issue_chunk(c + 1);
        mbar_wait(&bars[1 + (c & 1)], (c >> 1) & 1);
        const int pb = c * SKC;
        const int kc = min(SKC, W - pb);
        const int rsh = (int)(((uintptr_t)(a.R + (int64_t)(u.p0 + pb) * N) & 15) >> 3);
        const double *F = Fs + (c & 1) * SKC * STP + 8 * warp + g4;
        const double *Rr = Rs + (c & 1) * L.rsz + rsh + g4;
        const int nks = (kc + 3) >> 2;
        for (int ks = 0; ks < nks; ks++) {
            const int j = 4 * ks + t4;
            const bool okj = j < kc;
            const double av = okj ? F[j * STP] : 0.0;
            const double *rb = Rr + j * N;
#pragma unroll
            for (int nb = 0; nb < NB; nb++) {
                const double bv = okj ? rb[8 * nb] : 0.0;
                dmma(acc[nb][0], acc[nb][1], av, bv);
            }
        }
        __syncthreads();
    }

    if (u.nsplit > 1) {
        // split-K: publish the fragment-ordered partial; the last unit of the tile sums the
        // slots in slot order (deterministic whichever unit finishes last).
        const int64_t fsz = (int64_t)8 * NB * 64;  // doubles per slot (8 warps x NB x 32 x 2)
        double *slot = a.scratch + (u.slot_base + u.slot) * fsz;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) {
            double2 v = make_double2(acc[nb][0], acc[nb][1]);
            __stcg(reinterpret_cast<double2 *>(slot + ((warp * NB + nb) * 32 + lane) * 2), v);
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = (atomicAdd(&a.counters[u.tile], 1) == u.nsplit - 1);
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        if (tid == 0) {
            mbar_expect_tx(&bars[0], th_bytes);
            bulk_g2s(Th, th_src, th_bytes, &bars[0]);
        }
#pragma unroll
        for (int nb = 0; nb < NB; nb++) acc[nb][0] = acc[nb][1] = 0.0;
        for (int s = 0; s < u.nsplit; s++) {
            const double *sl = a.scratch + (u.slot_base + s) * fsz;
#pragma unroll
            for (int nb = 0; nb < NB; nb++) {
                const double2 v =
                    __ldcg(reinterpret_cast<const double2 *>(sl + ((warp * NB + nb) * 32 + lane) * 2));
                acc[nb][0] += v.x;
                acc[nb][1] += v.y;
            }
        }
        if (tid == 0) a.counters[u.tile] = 0;
    }
    mbar_wait(&bars[0], 0);

    // ---- epilogue: the quad (4 lanes) g4 of warp w owns local row r = 8w + g4 (row_step)
    const int r = 8 * warp + g4;
    const bool act = r < Tt;
    const int kl = k0 + r;
    const int64_t kg = a.kb + kl;
    const bool has_prev = kg > 0, has_next = kg + 1 < a.M;
    const double *thr = Th + th_sh + (r + 1) * N;
    double sreg = 0.0, skkt = 0.0, skktp = 0.0;
    const bool do_kkt = (it % a.kkt_every) == 0;
    const double tk = act ? a.tstep[kl] : 0.0;
    double *orow = a.out + (int64_t)kl * N;
    const bool full = Tt == ST && a.kb + k0 > 0 && a.kb + k0 + ST < a.M;   // block-uniform
    const bool even = (N & 1) == 0;
    if (full && even)
        row_step<NB, true, true>(acc, thr, N, t4, act, has_prev, has_next, a.gamma, tk, do_kkt, false,
                                 sreg, skkt, skktp, orow);
    else if (full)
        row_step<NB, true, false>(acc, thr, N, t4, act, has_prev, has_next, a.gamma, tk, do_kkt, false,
                                  sreg, skkt, skktp, orow);
    else
        row_step<NB, false, false>(acc, thr, N, t4, act, has_prev, has_next, a.gamma, tk, do_kkt, false,
                                   sreg, skkt, skktp, orow);
    // ---- per-tile scalar partials (fixed order: lanes, then warps)
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

// ------------------------------------------------------------------------------ fwd sweep
// Unit: Fock tiles [t0, t1) and the union of their probe windows [u0, u1) (<= FWCAP probes).
// Warp w owns (m-block, n-block) pairs [w PP, (w+1) PP) of the (u1-u0)/8 x NB pair grid.
size_t sweep_fwd_smem(int N, int NB)
{
    const int tsz = ((ST * N + 8 * NB + 4) + 1) & ~1;
    return (size_t)(2 * tsz + 2 * FWCAP * STP) * sizeof(double);
}

template <int NB>
__global__ void __launch_bounds__(256, 1) k_fwd_mma(SweepFwdArgs a)
{
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bars[2];
    const DevState *st = a.state;
    if (st && st->stop) return;
    const int N = a.N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const FwUnit u = a.units[blockIdx.x];
    const int tsz = ((ST * N + 8 * NB + 4) + 1) & ~1;
    double *Ts = sm;                    // 2 x tsz
    double *Fs = sm + 2 * tsz;          // 2 x FWCAP x STP
    const int Wu = u.u1 - u.u0;
    const int nm = (Wu + 7) >> 3;
    const int npair = nm * NB;
    const int PP = (npair + 7) >> 3;
    const int pbeg = warp * PP;
    int mbA = 0;
    int mbs[NB], nbs[NB];
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int p = min(pbeg + i, npair - 1);
        mbs[i] = p / NB;
        nbs[i] = p - (p / NB) * NB;
    }
    if (pbeg < npair) mbA = pbeg / NB;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int ntile = u.t1 - u.t0;
    auto issue = [&](int j) {
        const int t = u.t0 + j;
        const int k0 = t * ST;
        const int Tt = min(ST, a.Ml - k0);
        const double *src;
        int sh;
        uint32_t by;
        aligned_span(a.theta + (int64_t)k0 * N, (int64_t)Tt * N, &src, &sh, &by);
        const int dA = a.tile_dA[t], dB = a.tile_dB[t];
        const int ra = max(dA, u.u0), rb = min(dB, u.u1);
        uint64_t *bar = &bars[j & 1];
        const uint32_t fby = rb > ra ? (uint32_t)(rb - ra) * STP * 8 : 0;
        mbar_expect_tx(bar, by + fby);
        bulk_g2s(Ts + (j & 1) * tsz, src, by, bar);
        if (fby)
            bulk_g2s(Fs + (j & 1) * FWCAP * STP + (ra - u.u0) * STP,
                     a.Fb + a.fb_off[t] + (int64_t)(ra - dA) * STP, fby, bar);
    };
    if (tid == 0) issue(0);

    double acc[NB][2];
#pragma unroll
    for (int i = 0; i < NB; i++) acc[i][0] = acc[i][1] = 0.0;

    for (int j = 0; j < ntile; j++) {
        if (tid == 0 && j + 1 < ntile) issue(j + 1);
        mbar_wait(&bars[j & 1], (j >> 1) & 1);
        const int t = u.t0 + j;
        const int k0 = t * ST;
        const int Tt = min(ST, a.Ml - k0);
        const int sh = (int)(((uintptr_t)(a.theta + (int64_t)k0 * N) & 15) >> 3);
        const int ra = max(a.tile_dA[t], u.u0) - u.u0, rb = min(a.tile_dB[t], u.u1) - u.u0;
        const double *T = Ts + (j & 1) * tsz + sh + g4;
        const double *F = Fs + (j & 1) * FWCAP * STP + t4;
        // A rows (probes) of the two m-blocks this warp may touch, masked to the tile's window
        const int dA0 = 8 * mbA + g4, dA1 = dA0 + 8;
        const bool okA0 = dA0 >= ra && dA0 < rb, okA1 = dA1 >= ra && dA1 < rb;
        if (pbeg < npair) {
            const int nks = (Tt + 3) >> 2;
            for (int ks = 0; ks < nks; ks++) {
                const int kr = 4 * ks + t4;  // row of this lane's B fragment / A column
                const double a0 = okA0 ? F[dA0 * STP + 4 * ks] : 0.0;
                const double a1 = okA1 ? F[dA1 * STP + 4 * ks] : 0.0;
                const bool okr = kr < Tt;
#pragma unroll
                for (int i = 0; i < NB; i++) {
                    if (i < PP && pbeg + i < npair) {
                        const double av = (mbs[i] == mbA) ? a0 : a1;
                        const double bv = okr ? T[kr * N + 8 * nbs[i]] : 0.0;
                        dmma(acc[i][0], acc[i][1], av, bv);
                    }
                }
            }
        }
        __syncthreads();
    }
    // partial rows: rpart[(poff + d_rel) * N + c], d_rel = 8 mb + g4, c = 8 nb + 2 t4 + {0,1}
#pragma unroll
    for (int i = 0; i < NB; i++) {
        if (i < PP && pbeg + i < npair) {
            const int drel = 8 * mbs[i] + g4;
            if (drel < Wu) {
                double *dst = a.rpart + (u.poff + drel) * (int64_t)N;
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const int c = 8 * nbs[i] + 2 * t4 + e;
                    if (c < N) dst[c] = acc[i][e];
                }
            }
        }
    }
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
        for (int n = lane; n < N; n += 32) {
            double s = 0.0;
            for (int64_t j = j0; j < j1; j++) s += rpart[red_rows[j] * N + n];
            if (P) s -= P[(int64_t)d * N + n];
            R[(int64_t)d * N + n] = s;
            ss = fma(s, s, ss);
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

// ------------------------------------------------------------------------------ scalars
// Two-level deterministic reduction: block b sums a fixed chunk of the tile partials and of
// partR into stage[b]; the last block to finish sums stage[0..G) in order, applies the trace /
// KKT / stop logic (k_finalize's) and resets the arrival counter.
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
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = gridDim.x;
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = 0.0;
    {
        const int cr = (nR + G - 1) / G, ct = (ntiles + G - 1) / G;
        const int r0 = blockIdx.x * cr, r1 = min(nR, r0 + cr);
        const int t0 = blockIdx.x * ct, t1 = min(ntiles, t0 + ct);
        if (include_r2)
            for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) v[V_R2] += partR[i];
        for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
            const double *p = partT + (int64_t)t * NSC_TILE;
            v[V_KKT] += p[SC_KKT];
            v[V_KKTP] += p[SC_KKTP];
            v[V_REG] += p[SC_REG];
            v[V_DTH] += p[SC_DTH];
        }
    }
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = wsum(v[i]);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; i++) red[warp * NV + i] = v[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < NV; i++) {
            double s = 0.0;
            for (int w = 0; w < 8; w++) s += red[w * NV + i];
            stage[blockIdx.x * NV + i] = s;
        }
        __threadfence();
        s_last = atomicAdd(arrive, 1) == G - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    double tot[NV];
    for (int i = 0; i < NV; i++) tot[i] = 0.0;
    for (int b = 0; b < G; b++)
        for (int i = 0; i < NV; i++) tot[i] += __ldcg(&stage[b * NV + i]);
    *arrive = 0;
    for (int i = 0; i < NV; i++) vec[i] = tot[i];
    if (!finalize) return;  // multi-GPU: allreduce + k_finalize follow
    const int64_t k = st->it;
    const double f = tot[V_R2] + gamma * tot[V_REG];
    const bool kv = final_eval || (k % kkt_every) == 0;
    const double nm = (double)N * (double)M;
    const double r = kv ? sqrt(tot[V_KKT] / nm) : NAN;
    const double rp = kv ? sqrt(tot[V_KKTP] / nm) : NAN;
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
    cudaError_t e = cudaFuncSetAttribute(k_bwd_mma<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_fwd_mma<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    return e;
}

#define QDT_FOR_NB(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

cudaError_t prepare_sweep_kernels()
{
    static bool done = false;
    if (done) return cudaSuccess;
    cudaError_t e = cudaSuccess;
#define QDT_PREP(nb) if (e == cudaSuccess) e = prep_nb<nb>();
    QDT_FOR_NB(QDT_PREP)
#undef QDT_PREP
    done = e == cudaSuccess;
    return e;
}

// exact n-block count: only the last n-block of a row can hold padding columns
int sweep_nb(int N) { return (N >= 1 && N <= 8 * SW_NBMAX) ? (N + 7) / 8 : 0; }

cudaError_t launch_bwd_mma(const SweepArgs &a, int nunits, int NB, cudaStream_t s)
{
    if (nunits <= 0) return cudaSuccess;
    const size_t smem = sweep_bwd_smem(a.N, NB);
    switch (NB) {
#define QDT_CASE(nb) \
    case nb: k_bwd_mma<nb><<<nunits, 256, smem, s>>>(a); break;
        QDT_FOR_NB(QDT_CASE)
#undef QDT_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_fwd_mma(const SweepFwdArgs &a, int nunits, int NB, cudaStream_t s)
{
    if (nunits <= 0) return cudaSuccess;
    const size_t smem = sweep_fwd_smem(a.N, NB);
    switch (NB) {
#define QDT_CASE(nb) \
    case nb: k_fwd_mma<nb><<<nunits, 256, smem, s>>>(a); break;
        QDT_FOR_NB(QDT_CASE)
#undef QDT_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_reduce_R2(const double *rpart, const int64_t *red_beg, const int64_t *red_rows,
                             const double *P, double *R, int D, int N, double *partR,
                             const DevState *st, cudaStream_t s)
{
    k_reduce_R2<<<(D + 7) / 8, 256, 0, s>>>(rpart, red_beg, red_rows, P, R, D, N, partR, st);
    return cudaGetLastError();
}

cudaError_t launch_scalars2(const double *partR, int nR, const double *partT, int ntiles,
                            int include_r2, double *stage, int *arrive, double *vec, int64_t N,
                            int64_t M, double gamma, double tol, int final_eval, int kkt_every,
                            double *trace, double *kkt, double *kktp, int64_t trace_len,
                            DevState *st, int finalize, cudaStream_t s)
{
    k_scalars2<<<SC2_BLOCKS, 256, 0, s>>>(partR, nR, partT, ntiles, include_r2, stage, arrive, vec,
                                          N, M, gamma, tol, final_eval, kkt_every, trace, kkt, kktp,
                                          trace_len, st, finalize);
    return cudaGetLastError();
}

}  // namespace qdt
