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

#include "qdt_internal.h"

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
            for (int n = 0; n < N; n++) mn = fmin(mn, 2.0 * G[k * N + n]);
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
                xm = fmax(xm, x);
                xn = fmin(xn, x);
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
                            mA = fmin(mA, x);
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

cudaError_t launch_small_solve(const SmallArgs &a, cudaStream_t s)
{
    const size_t smem = small_solve_smem(a.D, a.M, a.N, a.nnz, a.fista);
    cudaError_t e = cudaFuncSetAttribute(k_small_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_small_solve<<<1, SM_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace qdt
