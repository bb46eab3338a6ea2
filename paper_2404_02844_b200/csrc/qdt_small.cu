// qdt_small.cu -- the whole solve in ONE persistent CTA for problems whose F, Theta, P and R fit in
// shared memory (BASELINE's Tiny: M = 50, N = 10, D = 100; SURVEY 8(a) "Per-config kernel shape":
// "One persistent CTA holds F (37 KB), Theta, R and P in SMEM and runs all 2 000 iterations").
//
// At this size every iteration of the multi-kernel path is launch-latency bound (4 graph nodes of
// a few microseconds each); here one launch runs all iterations with block barriers between the
// phases of an iteration (PAPER.md references as in qdt_sweep.cu):
//   S2  R_k = F Theta_k - P                       thread per (probe, outcome), band in order
//   S6  f(Theta_k) = ||R_k||^2 + gamma ||D Theta_k||^2     (eq. min_obj2 + eq. regul)
//   FISTA: R(Y_k) = (1 + beta_k) R_k - beta_k R_{k-1} (F linear), Y_k formed per element
//   S3+S4 G = F^T R(Y) + gamma L Y                 thread per (Fock row, outcome), its probes in order
//   KKT r(Theta_k) (reading R7) every kkt_every-th iteration (FISTA: an extra
//       F^T pass at Theta_k), the paper's clamped variant beside it
//   S5  X = Y - t o G, per-row Michelot threshold (reading R4), Theta_{k+1} = max(X - tau, 0)
// Scalar sums are block reductions in a fixed order (bitwise reproducible).  The iteration,
// early-stop and trace semantics are those of the multi-kernel loop (reading R3).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <stdlib.h>

#include "qdt_internal.h"
#include "qdt_ptx.cuh"

namespace qdt {

constexpr int SM_THREADS = 256;   // 8 warps: cheap block barriers; every phase loops over its items

// fixed-order block sums of two values per thread (all threads return the totals)
__device__ __forceinline__ void sm_block_sum2(double &v0, double &v1, double *red)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    }
    __syncthreads();
    if (lane == 0) {
        red[2 * warp] = v0;
        red[2 * warp + 1] = v1;
    }
    __syncthreads();
    double t0 = 0.0, t1 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
        t0 += red[2 * w];
        t1 += red[2 * w + 1];
    }
    v0 = t0;
    v1 = t1;
}

size_t small_solve_smem(int64_t D, int64_t M, int N, int64_t nnz, int fista)
{
    const int64_t MN = M * N, DN = D * N;
    const int64_t dbl = 2 * ((nnz + 1) & ~1LL) + (fista ? 4 : 3) * MN + (fista ? 3 : 2) * DN + M;   // F, F^T, Theta x3 (+G), P, R (+R_prev), t
    const int64_t ints = 3 * D + 3 * M + 3;                                          // lo, len, off, row ranges, F^T offsets
    return (size_t)(dbl * 8 + ints * 4 + 64);
}

__global__ void __launch_bounds__(SM_THREADS, 1) k_small_solve(SmallArgs a)
{
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[64];
    __shared__ int s_stop;
    const int D = a.D, M = a.M, N = a.N;
    const int MN = M * N, DN = D * N;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int nnz2 = (a.nnz + 1) & ~1;  // keeps the arrays after F 16-byte aligned (double2 access)
    double *Fv = sm;
    double *FT = Fv + nnz2;           // F by Fock row: FT[toff[k] + d - ra[k]] = F[d][k]
    double *T0 = FT + nnz2;           // Theta buffers (rotation by the host layout: see below)
    double *T1 = T0 + MN;
    double *T2 = T1 + MN;             // Theta_{k-1} (FISTA) / scratch
    double *Gs = T2 + MN;             // G (FISTA: G at Theta_k for the KKT; plain: G)
    double *Ps = Gs + (a.fista ? MN : 0);
    double *Rs = Ps + DN;
    double *Rp = Rs + DN;             // R_{k-1} (FISTA)
    double *ts = Rp + (a.fista ? DN : 0);
    int *lo = reinterpret_cast<int *>(ts + M);
    int *ln = lo + D;
    int *of = ln + D;                 // D + 1
    int *ra = of + D + 1;             // probes covering row k: [ra[k], rb[k])
    int *rb = ra + M;
    int *toff = rb + M;               // M + 1
    if (!a.fista) Gs = T2;            // plain: the third buffer holds G

    // ---- load the problem
    for (int i = tid; i < a.nnz; i += nth) Fv[i] = a.val[i];
    for (int i = tid; i < D; i += nth) {
        lo[i] = a.lo[i];
        ln[i] = a.len[i];
        of[i] = (int)a.off[i];
    }
    if (tid == 0) of[D] = (int)a.off[D];
    for (int i = tid; i < MN; i += nth) T0[i] = a.theta0[i];
    for (int i = tid; i < DN; i += nth) Ps[i] = a.P[i];
    for (int i = tid; i < M; i += nth) {
        ts[i] = a.tstep[i];
        ra[i] = a.row_da[i];
        rb[i] = a.row_db[i];
    }
    if (a.fista)
        for (int i = tid; i < MN; i += nth) T2[i] = a.theta_prev ? a.theta_prev[i] : a.theta0[i];
    __syncthreads();
    if (tid == 0) {   // F^T row offsets (prefix sums of the covering-probe counts)
        int acc = 0;
        for (int k = 0; k < M; k++) {
            toff[k] = acc;
            acc += rb[k] - ra[k];
        }
        toff[M] = acc;
    }
    __syncthreads();
    for (int d = tid; d < D; d += nth)   // scatter F into its row-major transpose
        for (int j = 0; j < ln[d]; j++) {
            const int k = lo[d] + j;
            FT[toff[k] + (d - ra[k])] = Fv[of[d] + j];
        }
    __syncthreads();

    // band sums with four independent accumulators (combined in a fixed order): the chains are
    // latency bound at these sizes
    // even N: two outcomes per thread (double2 loads, F loaded once per pair).  Rows stay one
    // thread each in the projection and KKT: a lane segment per row with shuffle reductions measured
    // slower at Tiny (15.4 against 10.5 us per iteration, tools/small_ab.py)
    const bool pairs = (N & 1) == 0;
    auto residual = [&](const double *T, double *R, bool withP) {   // R = F T - P
        if (pairs) {
            const int N2 = N >> 1;
            for (int e = tid; e < D * N2; e += nth) {
                const int d = e / N2, n = 2 * (e - d * N2);
                const double *f = Fv + of[d];
                const double *tc = T + lo[d] * N + n;
                const int L = ln[d];
                double2 s0 = make_double2(0.0, 0.0), s1 = s0;
                int j = 0;
                for (; j + 2 <= L; j += 2) {
                    const double2 t0 = *reinterpret_cast<const double2 *>(tc + j * N);
                    const double2 t1 = *reinterpret_cast<const double2 *>(tc + (j + 1) * N);
                    s0.x = fma(f[j], t0.x, s0.x), s0.y = fma(f[j], t0.y, s0.y);
                    s1.x = fma(f[j + 1], t1.x, s1.x), s1.y = fma(f[j + 1], t1.y, s1.y);
                }
                if (j < L) {
                    const double2 t0 = *reinterpret_cast<const double2 *>(tc + j * N);
                    s0.x = fma(f[j], t0.x, s0.x), s0.y = fma(f[j], t0.y, s0.y);
                }
                double2 o = make_double2(s0.x + s1.x, s0.y + s1.y);
                if (withP) {
                    const double2 pp = *reinterpret_cast<const double2 *>(Ps + d * N + n);
                    o.x -= pp.x, o.y -= pp.y;
                }
                *reinterpret_cast<double2 *>(R + d * N + n) = o;
            }
            return;
        }
        for (int e = tid; e < DN; e += nth) {
            const int d = e / N, n = e - d * N;
            const double *f = Fv + of[d];
            const double *tc = T + lo[d] * N + n;
            const int L = ln[d];
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int j = 0;
            for (; j + 4 <= L; j += 4) {
                s0 = fma(f[j], tc[j * N], s0);
                s1 = fma(f[j + 1], tc[(j + 1) * N], s1);
                s2 = fma(f[j + 2], tc[(j + 2) * N], s2);
                s3 = fma(f[j + 3], tc[(j + 3) * N], s3);
            }
            for (; j < L; j++) s0 = fma(f[j], tc[j * N], s0);
            const double s = (s0 + s1) + (s2 + s3);
            R[e] = withP ? s - Ps[e] : s;
        }
    };
    auto gradient = [&](const double *R, const double *Y, double *G) {   // G = F^T R + gamma L Y
        if (pairs) {
            const int N2 = N >> 1;
            for (int e = tid; e < M * N2; e += nth) {
                const int k = e / N2, n = 2 * (e - k * N2);
                const double *ft = FT + toff[k];
                const double *rc = R + ra[k] * N + n;
                const int L = rb[k] - ra[k];
                double2 s0 = make_double2(0.0, 0.0), s1 = s0;
                int i = 0;
                for (; i + 2 <= L; i += 2) {
                    const double2 r0 = *reinterpret_cast<const double2 *>(rc + i * N);
                    const double2 r1 = *reinterpret_cast<const double2 *>(rc + (i + 1) * N);
                    s0.x = fma(ft[i], r0.x, s0.x), s0.y = fma(ft[i], r0.y, s0.y);
                    s1.x = fma(ft[i + 1], r1.x, s1.x), s1.y = fma(ft[i + 1], r1.y, s1.y);
                }
                if (i < L) {
                    const double2 r0 = *reinterpret_cast<const double2 *>(rc + i * N);
                    s0.x = fma(ft[i], r0.x, s0.x), s0.y = fma(ft[i], r0.y, s0.y);
                }
                const double sx = s0.x + s1.x, sy = s0.y + s1.y;
                const int e0 = k * N + n;
                const double2 y = *reinterpret_cast<const double2 *>(Y + e0);
                const double2 yp = k > 0 ? *reinterpret_cast<const double2 *>(Y + e0 - N) : y;
                const double2 yn = k + 1 < M ? *reinterpret_cast<const double2 *>(Y + e0 + N) : y;
                *reinterpret_cast<double2 *>(G + e0) = make_double2(fma(a.gamma, (y.x - yp.x) + (y.x - yn.x), sx),
                                                                    fma(a.gamma, (y.y - yp.y) + (y.y - yn.y), sy));
            }
            return;
        }
        for (int e = tid; e < MN; e += nth) {
            const int k = e / N, n = e - k * N;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            const double *ft = FT + toff[k];
            const double *rc = R + ra[k] * N + n;
            const int L = rb[k] - ra[k];
            int i = 0;
            for (; i + 4 <= L; i += 4) {
                s0 = fma(ft[i], rc[i * N], s0);
                s1 = fma(ft[i + 1], rc[(i + 1) * N], s1);
                s2 = fma(ft[i + 2], rc[(i + 2) * N], s2);
                s3 = fma(ft[i + 3], rc[(i + 3) * N], s3);
            }
            for (; i < L; i++) s0 = fma(ft[i], rc[i * N], s0);
            const double s = (s0 + s1) + (s2 + s3);
            const double y = Y[e];
            const double yp = k > 0 ? Y[e - N] : y, yn = k + 1 < M ? Y[e + N] : y;
            G[e] = fma(a.gamma, (y - yp) + (y - yn), s);
        }
    };
    // r_KKT of T with gradient G (reading R7; both multipliers), thread per row
    auto kkt = [&](const double *T, const double *G, double *r, double *rp) {
        double s1 = 0.0, s2 = 0.0;
        for (int k = tid; k < M; k += nth) {
            double mn = INFINITY;
            for (int n = 0; n < N; n++) mn = dmin(mn, 2.0 * G[k * N + n]);
            const double lam = -mn, lamp = fmax(lam, 0.0);
            for (int n = 0; n < N; n++) {
                const double g2 = 2.0 * G[k * N + n], th = T[k * N + n];
                const double x1 = th * (g2 + lam), x2 = th * (g2 + lamp);
                s1 = fma(x1, x1, s1);
                s2 = fma(x2, x2, s2);
            }
        }
        const double nm = (double)N * (double)M;
        sm_block_sum2(s1, s2, red);
        *r = sqrt(s1 / nm);
        *rp = sqrt(s2 / nm);
    };
    auto objective = [&](const double *T, const double *R) {
        double s = 0.0, g = 0.0;
        for (int e = tid; e < DN; e += nth) s = fma(R[e], R[e], s);
        for (int e = tid; e < MN - N; e += nth) {
            const double dd = T[e] - T[e + N];
            g = fma(dd, dd, g);
        }
        sm_block_sum2(s, g, red);
        return s + a.gamma * g;
    };

    double *cur = T0, *nxt = T1, *prv = T2;
    if (a.fista && a.theta_prev) {   // resume: R_{k-1} = F Theta_{k-1} - P
        residual(prv, Rp, true);
        __syncthreads();
    }
    int64_t k = 0;
    bool stopped = false, converged = false, nonfinite = false;
    for (k = 0; k < a.iters; k++) {
        // R_k, f(Theta_k)
        residual(cur, Rs, true);
        __syncthreads();
        const double f = objective(cur, Rs);
        const bool kv = (k % a.kkt_every) == 0;
        const double beta = a.fista ? a.beta[k] : 0.0;
        double r = NAN, rp = NAN;
        if (a.fista) {
            if (kv) {   // G(Theta_k) for the KKT measure
                gradient(Rs, cur, Gs);
                __syncthreads();
                kkt(cur, Gs, &r, &rp);
            }
            // R(Y) = (1 + beta) R_k - beta R_{k-1} into Rp (R_k kept in Rs), Y into nxt
            for (int e = tid; e < DN; e += nth) {
                const double rk = Rs[e];
                Rp[e] = (k == 0 && !a.theta_prev) ? rk : fma(beta, rk - Rp[e], rk);
            }
            for (int e = tid; e < MN; e += nth) nxt[e] = fma(beta, cur[e] - prv[e], cur[e]);
            __syncthreads();
            gradient(Rp, nxt, Gs);   // G(Y)
            __syncthreads();
            for (int e = tid; e < DN; e += nth) Rp[e] = Rs[e];   // R_k becomes R_{k-1}
        } else {
            gradient(Rs, cur, Gs);
            __syncthreads();
            if (kv) kkt(cur, Gs, &r, &rp);
        }
        if (tid == 0 && k < a.trace_len) {
            a.trace[k] = f;
            a.kkt[k] = r;
            a.kktp[k] = rp;
        }
        if (!isfinite(f)) {
            nonfinite = stopped = true;
            break;
        }
        if (kv && r <= a.tol) {
            stopped = converged = true;
            break;
        }
        // X = Y - t G, row projection (thread per row), Theta_{k+1} -> the buffer of Theta_{k-1}
        const double *Y = a.fista ? nxt : cur;
        double *out = a.fista ? prv : nxt;
        for (int row = tid; row < M; row += nth) {
            const double t = ts[row];
            double s = 0.0, xm = -INFINITY, xn = INFINITY;
            for (int n = 0; n < N; n++) {
                const double x = fma(-t, Gs[row * N + n], Y[row * N + n]);
                out[row * N + n] = x;
                s += x;
                xm = dmax(xm, x);
                xn = dmin(xn, x);
            }
            double tau = (s - 1.0) / (double)N;
            if (!(xn > tau)) {   // Michelot from the lower bound max(tau_0, max X - 1)
                tau = fmax(tau, xm - 1.0);
                int cnt = N + 1;
                for (int round = 0; round <= N; round++) {
                    double ps = 0.0, mA = INFINITY;
                    int pc = 0;
                    for (int n = 0; n < N; n++) {
                        const double x = out[row * N + n];
                        if (x > tau) {
                            ps += x;
                            pc++;
                            mA = dmin(mA, x);
                        }
                    }
                    if (pc >= cnt) break;
                    cnt = pc;
                    tau = (ps - 1.0) / (double)pc;
                    if (mA > tau) break;
                }
            }
            for (int n = 0; n < N; n++) {
                const double o = out[row * N + n] - tau;
                out[row * N + n] = o > 0.0 ? o : 0.0;
            }
        }
        __syncthreads();
        if (a.fista) {   // rotate: prv <- cur, cur <- out (held in prv), nxt scratch
            double *t = prv;
            prv = cur;
            cur = t;
        } else {
            double *t = cur;
            cur = nxt;
            nxt = t;
        }
    }
    if (!stopped) {   // final evaluation at Theta_iters: f and both KKT multipliers
        residual(cur, Rs, true);
        __syncthreads();
        const double f = objective(cur, Rs);
        gradient(Rs, cur, Gs);
        __syncthreads();
        double r, rp;
        kkt(cur, Gs, &r, &rp);
        if (tid == 0 && k < a.trace_len) {
            a.trace[k] = f;
            a.kkt[k] = r;
            a.kktp[k] = rp;
        }
        if (!isfinite(f)) nonfinite = true;
    } else if (converged) {   // the stop iterate: the clamped multiplier beside the stop value
        residual(cur, Rs, true);
        __syncthreads();
        gradient(Rs, cur, Gs);
        __syncthreads();
        double r, rp;
        kkt(cur, Gs, &r, &rp);
        if (tid == 0 && k < a.trace_len) a.kktp[k] = rp;
    }
    (void)s_stop;
    // results: Theta_k and (FISTA) Theta_{k-1} to the caller's buffers
    for (int e = tid; e < MN; e += nth) {
        a.theta_out[e] = cur[e];
        if (a.fista && a.prev_out) a.prev_out[e] = prv[e];
    }
    if (tid == 0) {
        a.state->iters_done = k;
        a.state->it = k;
        a.state->stop = 1;
        a.state->converged = converged ? 1 : 0;
        a.state->nonfinite = nonfinite ? 1 : 0;
    }
}

// ------------------------------------------------------------------------------ dense DMMA form
// The same solve (same iteration, trace, stop and resume semantics) for problems whose F fits in
// shared memory as a DENSE D x M block (Tiny: 100 x 50, 92 % of it inside the band): both
// contractions become fp64 tensor-core GEMMs (mma.sync m8n8k4, one 8x8 output tile per warp,
// two accumulator chains per tile), the row phase takes a quad of lanes per Fock row.
//   S2  R_k = F Theta_k - P            tiles (8 probes x 8 outcomes), K = Fock rows (zero padded)
//       FISTA: R(Y_k) = (1 + beta_k) R_k - beta_k R_{k-1} in the same epilogue (F linear)
//   S3+S4 G = F^T R + gamma L Y         tiles (8 Fock rows x 8 outcomes), K = probes, stencil in
//       the epilogue (ends: reading R8); FISTA at a KKT iteration also G(Theta_k) from R_k
//   S5+S6 quad per Fock row (lane t4: outcomes 4 j + t4 in registers): regulariser pair, KKT of
//       Theta_k (reading R7, both multipliers), X = Y - t G, Michelot threshold (reading R4) by
//       quad butterflies, Theta_{k+1}; ONE fixed-order block reduction of ||R_k||^2, ||D Theta_k||^2
//       and the KKT sums per iteration (partials parked in shared memory, summed by one warp).
// Measured on B200 (tools/dmma_lat.cu): a dependent DMMA takes 26 cycles, and one SM retires one
// DMMA per 4 cycles, so Tiny's two GEMMs (2 x 364 DMMAs on 8 x 8 tiles) cost >= 2.9 k cycles per
// iteration on the one SM: 6.8 us per plain iteration against 10.5 us for the band form.
// Shared-memory pitches are = 4 (mod 16) doubles (M8 + 4, N8 + 4): the fragment loads of a half
// warp (4 rows x 4 consecutive doubles) hit 16 distinct 8-byte bank pairs.  Every pad row / column
// of F, Theta, P, R and G is zero, so pad outputs are exactly zero and need no masks.
constexpr int SD_THREADS = 512;
constexpr int SD_NJ = SD_NR / 4;   // outcomes per lane of a row quad
struct DenseLayout {
    int Dp, M8, N8, PF, PT;
    int64_t fd, th, r, g, t, total;   // offsets (doubles) and total
    __host__ __device__ DenseLayout(int D, int M, int N, int fista)
    {
        Dp = (D + 7) & ~7;
        M8 = (M + 7) & ~7;
        N8 = (N + 7) & ~7;
        PF = M8 + 4;
        PT = N8 + 4;
        fd = 0;
        th = fd + (int64_t)Dp * PF;                       // Theta x3 (cur, next/prev, spare)
        r = th + 3LL * M8 * PT;                           // P, R_k, R_{k-1}, R(Y)
        g = r + 4LL * Dp * PT;                            // G, G(Theta_k) (FISTA)
        t = g + 2LL * M8 * PT;                            // step weights
        total = t + M8;
        (void)fista;
    }
};

size_t small_dense_smem(int64_t D, int64_t M, int N, int fista)
{
    if (N > SD_NR || D > (1 << 20) || M > (1 << 20)) return SIZE_MAX;
    const DenseLayout L((int)D, (int)M, N, fista);
    return (size_t)L.total * 8 + 64;
}

// one 8x8 output tile: acc += A (8 x K) B (K x 8) over ksteps k-steps of 4, two chains;
// A element (row g4, k t4) at a[g4 * as_r + t4 * as_k], B element (k t4, col g4) at b[t4 * bs_k + g4]
__device__ __forceinline__ void sd_tile(double &c0, double &c1, const double *a, int as_r, int as_k,
                                        const double *b, int bs_k, int ksteps, int g4, int t4)
{
    double e0 = 0.0, e1 = 0.0, o0 = 0.0, o1 = 0.0;
    const double *ap = a + g4 * as_r + t4 * as_k;
    const double *bp = b + t4 * bs_k + g4;
    int ks = 0;
    for (; ks + 2 <= ksteps; ks += 2) {
        const double a0 = ap[(4 * ks) * as_k], b0 = bp[(4 * ks) * bs_k];
        const double a1 = ap[(4 * ks + 4) * as_k], b1 = bp[(4 * ks + 4) * bs_k];
        dmma(e0, e1, a0, b0);
        dmma(o0, o1, a1, b1);
    }
    if (ks < ksteps) dmma(e0, e1, ap[(4 * ks) * as_k], bp[(4 * ks) * bs_k]);
    c0 = e0 + o0;
    c1 = e1 + o1;
}

// fixed-order block sum of 4 values, result in every thread.  Every thread parks its 4 partials
// in shared memory (no shuffles in most warps); warp 0 sums them (lane l: threads l, l + 32, ...
// in order, then a butterfly) and publishes the totals.  pbuf: [blockDim.x][4] + 4 totals.
__device__ __forceinline__ void sd_block_sum4(double (&v)[4], double *pbuf)
{
    const int tid = threadIdx.x, lane = tid & 31, nth = blockDim.x;
    *reinterpret_cast<double4 *>(pbuf + 4 * tid) = make_double4(v[0], v[1], v[2], v[3]);
    __syncthreads();
    if (tid < 32) {
        double w[4] = {0.0, 0.0, 0.0, 0.0};
        for (int t = lane; t < nth; t += 32) {
            const double4 q = *reinterpret_cast<const double4 *>(pbuf + 4 * t);
            w[0] += q.x;
            w[1] += q.y;
            w[2] += q.z;
            w[3] += q.w;
        }
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) w[i] += __shfl_xor_sync(0xffffffffu, w[i], o);
        if (lane == 0) *reinterpret_cast<double4 *>(pbuf + 4 * nth) = make_double4(w[0], w[1], w[2], w[3]);
    }
    __syncthreads();
    const double4 q = *reinterpret_cast<const double4 *>(pbuf + 4 * nth);
    v[0] = q.x;
    v[1] = q.y;
    v[2] = q.z;
    v[3] = q.w;
}

__global__ void __launch_bounds__(SD_THREADS, 1) k_small_dense(SmallArgs a)
{
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(32) double pbuf[4 * SD_THREADS + 4];
    const int D = a.D, M = a.M, N = a.N;
    const DenseLayout L(D, M, N, a.fista);
    const int Dp = L.Dp, M8 = L.M8, N8 = L.N8, PF = L.PF, PT = L.PT;
    const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    double *Fd = sm + L.fd;
    double *Tb[3] = {sm + L.th, sm + L.th + (int64_t)M8 * PT, sm + L.th + 2LL * M8 * PT};
    double *Ps = sm + L.r;
    double *Rb[3] = {Ps + (int64_t)Dp * PT, Ps + 2LL * Dp * PT, Ps + 3LL * Dp * PT};   // R_k, R_{k-1}, R(Y)
    double *Gs = sm + L.g, *G2 = Gs + (int64_t)M8 * PT;
    double *ts = sm + L.t;

    // ---- load: zero everything (pads), scatter the band of F, copy Theta_0 / P / t
    for (int64_t i = tid; i < L.total; i += nth) sm[i] = 0.0;
    __syncthreads();
    for (int d = warp; d < D; d += nw) {
        const int lo = a.lo[d], ln = a.len[d];
        const int64_t of = a.off[d];
        for (int j = lane; j < ln; j += 32) Fd[(int64_t)d * PF + lo + j] = a.val[of + j];
    }
    for (int e = tid; e < M * N; e += nth) {
        const int k = e / N, n = e - k * N;
        Tb[0][k * PT + n] = a.theta0[e];
        if (a.fista) Tb[1][k * PT + n] = a.theta_prev ? a.theta_prev[e] : a.theta0[e];
    }
    for (int e = tid; e < D * N; e += nth) {
        const int d = e / N, n = e - d * N;
        Ps[d * PT + n] = a.P[e];
    }
    for (int k = tid; k < M; k += nth) ts[k] = a.tstep[k];
    __syncthreads();

    const int nbn = N8 >> 3;
    // S2: Rdst = F T - P (and, FISTA, RY = R(Y) from Rprev); returns this thread's ||R||^2 part
    auto residual = [&](const double *T, double *Rdst, const double *Rprev, double *RY, double beta, bool first) {
        double r2 = 0.0;
        const int ntile = (Dp >> 3) * nbn;
        for (int tt = warp; tt < ntile; tt += nw) {
            const int ib = tt / nbn, jb = tt - ib * nbn;
            double c0, c1;
            sd_tile(c0, c1, Fd + (int64_t)(8 * ib) * PF, PF, 1, T + 8 * jb, PT, M8 >> 2, g4, t4);
            const int d = 8 * ib + g4, n = 8 * jb + 2 * t4;
            const double2 pp = *reinterpret_cast<const double2 *>(Ps + d * PT + n);
            const double v0 = c0 - pp.x, v1 = c1 - pp.y;
            *reinterpret_cast<double2 *>(Rdst + d * PT + n) = make_double2(v0, v1);
            r2 = fma(v0, v0, r2);
            r2 = fma(v1, v1, r2);
            if (RY) {
                double y0 = v0, y1 = v1;
                if (!first) {
                    const double2 q = *reinterpret_cast<const double2 *>(Rprev + d * PT + n);
                    y0 = fma(beta, v0 - q.x, v0);
                    y1 = fma(beta, v1 - q.y, v1);
                }
                *reinterpret_cast<double2 *>(RY + d * PT + n) = make_double2(y0, y1);
            }
        }
        return r2;
    };
    // Y (FISTA: Theta_k + beta (Theta_k - Theta_{k-1}); plain: Theta_k) element
    auto yv = [&](const double *cur, const double *prv, double beta, int i) {
        return prv ? fma(beta, cur[i] - prv[i], cur[i]) : cur[i];
    };
    // S3+S4: Gdst = F^T Rsrc + gamma L Y   (Y from cur / prv as above)
    auto gradient = [&](const double *Rsrc, double *Gdst, const double *cur, const double *prv, double beta) {
        const int ntile = (M8 >> 3) * nbn;
        for (int tt = warp; tt < ntile; tt += nw) {
            const int ib = tt / nbn, jb = tt - ib * nbn;
            double c0, c1;
            sd_tile(c0, c1, Fd + 8 * ib, 1, PF, Rsrc + 8 * jb, PT, Dp >> 2, g4, t4);
            const int k = 8 * ib + g4, n = 8 * jb + 2 * t4;
            double o[2] = {c0, c1};
            if (k < M) {
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const int i = k * PT + n + e;
                    const double y = yv(cur, prv, beta, i);
                    const double yp = k > 0 ? yv(cur, prv, beta, i - PT) : y;
                    const double yn = k + 1 < M ? yv(cur, prv, beta, i + PT) : y;
                    o[e] = fma(a.gamma, (y - yp) + (y - yn), o[e]);
                }
            }
            *reinterpret_cast<double2 *>(Gdst + k * PT + n) = make_double2(o[0], o[1]);
        }
    };

    int ic = 0, ip = 1, ix = 2;          // Theta_k, Theta_{k-1} (FISTA) / Theta_{k+1} (plain), spare
    int rk = 0, rp = 1;                  // R_k, R_{k-1}
    if (a.fista && a.theta_prev) {       // resume: R_{k-1} = F Theta_{k-1} - P
        residual(Tb[ip], Rb[rp], nullptr, nullptr, 0.0, true);
        __syncthreads();
    }
    const double nm = (double)N * (double)M;
    int64_t k = 0;
    bool converged = false, nonfinite = false, stopped = false;
    int kmod = 0;                                         // k % kkt_every, kept as a counter
    double bcur = (a.fista && a.iters > 0) ? a.beta[0] : 0.0;
    for (k = 0; k <= a.iters; k++, kmod = (kmod + 1 == a.kkt_every) ? 0 : kmod + 1) {
        const bool fin = k == a.iters;                    // final evaluation at Theta_iters
        const bool kv = fin || kmod == 0;
        const double beta = (a.fista && !fin) ? bcur : 0.0;
        if (a.fista && k + 1 < a.iters) bcur = a.beta[k + 1];   // next iteration's beta, loaded early
        const bool first = k == 0 && !a.theta_prev;
        double *cur = Tb[ic];
        const double *prv = (a.fista && !fin) ? Tb[ip] : nullptr;
        double *out = a.fista ? Tb[ip] : Tb[ix];          // FISTA: Theta_{k+1} over Theta_{k-1}
        const bool fis = a.fista && !fin;
        double part[4] = {0.0, 0.0, 0.0, 0.0};            // ||R_k||^2, ||D Theta_k||^2, kkt, kktp
        part[0] = residual(cur, Rb[rk], Rb[rp], fis ? Rb[2] : nullptr, beta, first);
        __syncthreads();

        // G(Y) into Gs; the KKT gradient G(Theta_k) is Gs itself unless FISTA (then G2)
        gradient(fis ? Rb[2] : Rb[rk], Gs, cur, prv, beta);
        if (fis && kv) gradient(Rb[rk], G2, cur, nullptr, 0.0);
        __syncthreads();
        const double *Gk = fis ? G2 : Gs;
        // S5/S6: a quad (4 lanes) per Fock row, lane t4 holding outcomes n = 4 j + t4 (j < SD_NR / 4)
        // in registers; row reductions are quad butterflies (identical in the 4 lanes)
        for (int rb = 0; rb < M; rb += nth >> 2) {   // warp-uniform trip count (shuffles below)
            if (rb + 8 * warp >= M) continue;   // the warp's 8 rows are all beyond M
            const int row = rb + (tid >> 2);
            const bool act = row < M;
            const double *cr = cur + row * PT;
            const bool hn = row + 1 < M;
            double th[SD_NJ], tn[SD_NJ], gk[SD_NJ], x[SD_NJ];
#pragma unroll
            for (int j = 0; j < SD_NJ; j++) {
                const int n = 4 * j + t4;
                const bool ok = act && n < N;
                th[j] = ok ? cr[n] : 0.0;
                tn[j] = (ok && hn) ? cr[PT + n] : th[j];
                gk[j] = (ok && kv) ? Gk[row * PT + n] : 0.0;
                x[j] = (ok && !fin) ? Gs[row * PT + n] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < SD_NJ; j++) {   // regulariser pair (k, k+1); 0 for pads / the last row
                const double dd = th[j] - tn[j];
                part[1] = fma(dd, dd, part[1]);
            }
            if (kv) {
                double mn = INFINITY;
#pragma unroll
                for (int j = 0; j < SD_NJ; j++)
                    if (4 * j + t4 < N) mn = dmin(mn, 2.0 * gk[j]);
                mn = quad_min(mn);
                const double lam = -mn, lamp = fmax(lam, 0.0);
#pragma unroll
                for (int j = 0; j < SD_NJ; j++)
                    if (act && 4 * j + t4 < N) {
                        const double g2 = 2.0 * gk[j];
                        const double x1 = th[j] * (g2 + lam), x2 = th[j] * (g2 + lamp);
                        part[2] = fma(x1, x1, part[2]);
                        part[3] = fma(x2, x2, part[3]);
                    }
            }
            if (fin) continue;
            const double t = act ? ts[row] : 0.0;
            double sx = 0.0, xm = -INFINITY, xn = INFINITY;
#pragma unroll
            for (int j = 0; j < SD_NJ; j++) {
                const int n = 4 * j + t4;
                if (act && n < N) {
                    const double tp = prv ? prv[row * PT + n] : 0.0;   // Theta_{k-1} (FISTA)
                    const double y = prv ? fma(beta, th[j] - tp, th[j]) : th[j];
                    x[j] = fma(-t, x[j], y);
                    sx += x[j];
                    xm = dmax(xm, x[j]);
                    xn = dmin(xn, x[j]);
                } else {
                    x[j] = -INFINITY;
                }
            }
            sx = quad_sum(sx);
            xm = quad_max(xm);
            xn = quad_min(xn);
            double tau = (sx - 1.0) / (double)N;
            bool done = !act || xn > tau;   // Michelot from max(tau_0, max X - 1) (reading R4)
            if (!done) tau = fmax(tau, xm - 1.0);
            int cnt = N + 1;
            for (int round = 0; round <= N; round++) {
                if (__all_sync(0xffffffffu, done)) break;
                double ps = 0.0, mA = INFINITY;
                int pc = 0;
#pragma unroll
                for (int j = 0; j < SD_NJ; j++)
                    if (x[j] > tau) {
                        ps += x[j];
                        pc++;
                        mA = dmin(mA, x[j]);
                    }
                ps = quad_sum(ps);
                pc = quad_sum_i(pc);
                mA = quad_min(mA);
                if (!done) {
                    if (pc >= cnt) {
                        done = true;
                    } else {
                        cnt = pc;
                        tau = (ps - 1.0) / (double)pc;
                        done = mA > tau;
                    }
                }
            }
            if (act) {
                double *orow = out + row * PT;
#pragma unroll
                for (int j = 0; j < SD_NJ; j++) {
                    const int n = 4 * j + t4;
                    if (n < N) {
                        const double o = x[j] - tau;
                        orow[n] = o > 0.0 ? o : 0.0;
                    }
                }
            }
        }
        sd_block_sum4(part, pbuf);

        const double f = part[0] + a.gamma * part[1];
        const double r = kv ? sqrt(part[2] / nm) : NAN, rpv = kv ? sqrt(part[3] / nm) : NAN;
        if (tid == 0 && k < a.trace_len) {
            a.trace[k] = f;
            a.kkt[k] = r;
            a.kktp[k] = rpv;
        }
        if (fin) {
            if (!isfinite(f)) nonfinite = true;
            break;
        }
        if (!isfinite(f)) {
            nonfinite = stopped = true;
            break;
        }
        if (kv && r <= a.tol) {
            converged = stopped = true;
            break;
        }
        if (a.fista) {   // Theta_{k+1} (in the old Theta_{k-1} buffer) becomes current
            const int t2 = ip;
            ip = ic;
            ic = t2;
            const int r2 = rp;   // R_k becomes R_{k-1}
            rp = rk;
            rk = r2;
        } else {
            const int t2 = ix;
            ix = ic;
            ic = t2;
        }
        // the next residual overwrites R_{k-1}'s buffer only after every thread passed the
        // block reduction above (its barrier), so no extra barrier is needed here
    }
    const double *cur = Tb[ic];
    const double *prv = Tb[ip];
    for (int e = tid; e < M * N; e += nth) {
        const int kk = e / N, n = e - kk * N;
        a.theta_out[e] = cur[kk * PT + n];
        if (a.fista && a.prev_out) a.prev_out[e] = prv[kk * PT + n];
    }
    if (tid == 0) {
        const int64_t kd = stopped ? k : a.iters;
        a.state->iters_done = kd;
        a.state->it = kd;
        a.state->stop = 1;
        a.state->converged = converged ? 1 : 0;
        a.state->nonfinite = nonfinite ? 1 : 0;
    }
}

bool small_use_dense(const SmallArgs &a)
{
    static int v = -1;   // QDT_SMALL_DENSE=0: the band form (A/B)
    if (v < 0) {
        const char *e = getenv("QDT_SMALL_DENSE");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1 && small_dense_smem(a.D, a.M, a.N, a.fista) <= SMALL_SMEM_MAX;
}

cudaError_t launch_small_solve(const SmallArgs &a, cudaStream_t s)
{
    if (small_use_dense(a)) {
        const size_t smem = small_dense_smem(a.D, a.M, a.N, a.fista);
        cudaError_t e = cudaFuncSetAttribute(k_small_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_small_dense<<<1, SD_THREADS, smem, s>>>(a);
        return cudaGetLastError();
    }
    const size_t smem = small_solve_smem(a.D, a.M, a.N, a.nnz, a.fista);
    cudaError_t e = cudaFuncSetAttribute(k_small_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_small_solve<<<1, SM_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace qdt
