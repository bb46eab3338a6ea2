// qdt_coop.cu -- the whole solve in ONE grid-persistent cooperative kernel for latency-bound
// problem sizes (BASELINE's Medium: M = 1000, N = 100, D = 2000; SURVEY 8(a) "Per-config kernel
// shape", Medium: "the working set stays in L2 ... a grid-wide barrier ... per iteration").
//
// At these sizes the multi-kernel loop (forward, reduction, step, scalars: 4 graph nodes per
// iteration) is bound by the split-K fix-up and the launch chain of each kernel, not by HBM or
// the tensor cores.  Here every CTA stays resident for all iterations (cooperative launch: all
// CTAs co-resident) and an iteration is two phases separated by grid barriers:
//   phase F (S2): R_k = F Theta_k - P for blocks of 8 probes: the union band of the block is split
//       over the 8 warps (k-steps ks = warp, warp + 8, ...), each warp an 8 x 8 NB DMMA tile
//       (mma.sync m8n8k4 f64, A = F gathered from the band, B = Theta rows from L2), the warp
//       partials summed in warp order through shared memory; ||R_k||^2 partial; FISTA:
//       R(Y_k) = (1 + beta_k) R_k - beta_k R_{k-1} in the same pass (F linear).
//   grid barrier
//   phase B (S3-S6): G = F^T R + gamma L Y for blocks of 8 Fock rows: the covering probes of the
//       block (contiguous: band edges are monotone) split over the warps as above (A = F^T from a
//       per-row transposed band, B = R rows), summed in warp order; then warp r owns row r of the
//       block (lanes: outcomes lane + 32 j): regulariser pair (eq. regul), KKT of
//       Theta_k (reading R7, both multipliers), X = Y - t o G, Michelot threshold
//       by warp butterflies (reading R4), Theta_{k+1} = max(X - tau, 0) into the next buffer.
//   grid barrier; every CTA sums the per-CTA partials in CTA order (same totals everywhere, so
//   every CTA takes the same stop decision); CTA 0 writes the trace.
// Semantics (iteration, trace, KKT every kkt_every, early stop, final evaluation, FISTA resume,
// buffer rotation Theta_k in theta[k % nbuf]) are those of the multi-kernel loop (reading R3).
// Data written inside the kernel is read with ld.global.cg (L2): the SMs' L1 is not coherent.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "qdt_internal.h"
#include "qdt_ptx.cuh"

namespace qdt {

constexpr int CP_THREADS = 256;   // 8 warps, one CTA per SM (255 registers: the pipelined k-loop)

// grid barrier (all CTAs co-resident by the cooperative launch): arrival counter + generation
__device__ __forceinline__ void cp_grid_sync(unsigned *bar, unsigned nblocks, unsigned &gen)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&bar[0], 1u) == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicExch(&bar[1], gen + 1);
        } else {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 1) : "memory");
            } while (v == gen);
        }
        __threadfence();
    }
    gen++;
    __syncthreads();
}

__device__ __forceinline__ double wred_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double wred_min(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double wred_max(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int wred_sum_i(int v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// acc += sum over k-steps ks = ks0, ks0 + stride, ... < nks of A(ks) B(ks) (one DMMA per n-block),
// software pipelined in registers: the operands of the next k-step are loaded (ld.global: F by the
// read-only path, Theta / R rows by .cg, L2 only: they are written inside the kernel and the SMs'
// L1 is not coherent) before the current step's DMMAs, so two k-steps of loads are in flight per
// warp.  Measured alternatives (grid-persistent path): a plain loop with 16 warps (same
// time), three k-steps in registers (spills), a 6-stage per-warp cp.async ring and a TMA-staged
// CTA ring (both slower: per-chunk issue and synchronisation cost more than the latency hidden).
template <int NB, class LA, class LB>
__device__ __forceinline__ void cp_kloop(double (&acc)[NB][2], int ks0, int nks, int stride, LA la, LB lb)
{
    if (ks0 >= nks) return;
    double a0 = la(ks0), b0[NB];
    lb(ks0, b0);
    for (int ks = ks0; ks < nks; ks += stride) {
        const int kn = ks + stride;
        double a1 = 0.0, b1[NB];
        if (kn < nks) {
            a1 = la(kn);
            lb(kn, b1);
        } else {
#pragma unroll
            for (int nb = 0; nb < NB; nb++) b1[nb] = 0.0;
        }
#pragma unroll
        for (int nb = 0; nb < NB; nb++) dmma(acc[nb][0], acc[nb][1], a0, b0[nb]);
        a0 = a1;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) b0[nb] = b1[nb];
    }
}

// shared memory: the warp partials [NW][8][8 NB] + two compact 8 x 8 NB tiles (G(Y), G(Theta_k))
size_t coop_smem(int NB)
{
    return ((size_t)(CP_THREADS / 32) * 8 * 8 * NB + 2 * 8 * 8 * NB) * sizeof(double) + 64;
}

// NB: n-blocks of 8 outcomes held per warp tile (8 NB >= N); NJ = 8 NB / 32 outcomes per lane in
// the row epilogue
template <int NB>
__global__ void __launch_bounds__(CP_THREADS, 1) k_coop_solve(CoopArgs a)
{
    constexpr int NW = CP_THREADS / 32;
    constexpr int NC = 8 * NB;           // padded row width of the tiles
    constexpr int NJ = (NC + 31) / 32;   // outcomes per lane in the row epilogue
    extern __shared__ __align__(16) double sm[];
    double *red = sm;                    // [NW][8][NC]: warp partials
    double *Gy = sm + NW * 8 * NC;                   // [8][NC]: G(Y) (phase B)
    double *Gk = Gy + 8 * NC;                        // [8][NC]: G(Theta_k) (phase B, FISTA KKT iterations)
    __shared__ double bsum[NW][4];
    const int D = a.D, M = a.M, N = a.N, Nv = a.Nv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g4 = lane >> 2, t4 = lane & 3;
    const unsigned G = gridDim.x;
    unsigned gen = 0;
    const int nbd = (D + 7) / 8, nbk = (M + 7) / 8;
    const int nbuf = a.fista ? 3 : 2;
    const double nm = (double)Nv * (double)M;

    // S2 for every probe block of this CTA: Rdst = F T - P; RY (FISTA) = first ? R : (1 + beta) R -
    // beta Rprev; returns this thread's ||R||^2 part
    auto forward = [&](const double *T, double *Rdst, double *RY, const double *Rprev, double beta, bool first) {
        double r2 = 0.0;
        for (int tb = blockIdx.x; tb < nbd; tb += G) {
            const int d0 = 8 * tb;
            const int dl = min(d0 + 7, D - 1);
            int kA = a.lo[d0], kB = 0;
            for (int d = d0; d <= dl; d++) kB = max(kB, a.lo[d] + a.len[d]);
            const int md = d0 + g4;
            const bool mok = md < D;
            const int mlo = mok ? a.lo[md] : 0, mlen = mok ? a.len[md] : 0;
            const int64_t moff = mok ? a.off[md] : 0;
            double acc[NB][2];
#pragma unroll
            for (int nb = 0; nb < NB; nb++) acc[nb][0] = acc[nb][1] = 0.0;
            const int nks = (kB - kA + 3) >> 2;
            // A: (probe md, row kk); B: (row kk, outcome 8 nb + g4)
            cp_kloop<NB>(acc, warp, nks, NW,
                         [&](int ks) {
                             const int j = kA + 4 * ks + t4 - mlo;
                             return (j >= 0 && j < mlen) ? __ldg(a.val + moff + j) : 0.0;
                         },
                         [&](int ks, double (&bv)[NB]) {
                             const int kk = kA + 4 * ks + t4;
                             const bool kok = kk < kB;
                             const double *trow = T + (int64_t)kk * N;
#pragma unroll
                             for (int nb = 0; nb < NB; nb++) {
                                 const int n = 8 * nb + g4;
                                 bv[nb] = (kok && n < N) ? __ldcg(trow + n) : 0.0;
                             }
                         });
            double *rw = red + (warp * 8 + g4) * NC + 2 * t4;
#pragma unroll
            for (int nb = 0; nb < NB; nb++) *reinterpret_cast<double2 *>(rw + 8 * nb) = make_double2(acc[nb][0], acc[nb][1]);
            __syncthreads();
            for (int e = tid; e < 8 * NC; e += CP_THREADS) {
                const int r = e / NC, n = e - r * NC;
                const int d = d0 + r;
                if (d >= D || n >= N) continue;
                double s = 0.0;
#pragma unroll
                for (int w = 0; w < NW; w++) s += red[(w * 8 + r) * NC + n];
                const int64_t i = (int64_t)d * N + n;
                const double v = s - __ldg(a.P + i);
                __stcg(Rdst + i, v);
                r2 = fma(v, v, r2);
                if (RY) __stcg(RY + i, first ? v : fma(beta, v - __ldcg(Rprev + i), v));
            }
            __syncthreads();
        }
        return r2;
    };
    if (a.resume) {   // FISTA resume: R_{-1} = F Theta_{-1} - P by the same pass as every R_k
        forward(a.theta[2], a.R[1], nullptr, nullptr, 0.0, true);
        cp_grid_sync(a.bar, G, gen);
    }

    int64_t k = 0;
    bool converged = false, nonfinite = false, stopped = false;
    int kmod = 0;
    for (k = 0; k <= a.iters; k++, kmod = (kmod + 1 == a.kkt_every) ? 0 : kmod + 1) {
        const bool fin = k == a.iters;
        const bool kv = fin || kmod == 0;
        const bool fis = a.fista && !fin;
        const double beta = fis ? a.beta[k] : 0.0;
        const bool first = k == 0 && !a.resume;
        const double *cur = a.theta[k % nbuf];
        const double *prv = fis ? a.theta[(k + 2) % 3] : nullptr;
        double *out = a.theta[(k + 1) % nbuf];
        double *Rk = a.R[k & 1], *Rp = a.R[(k & 1) ^ 1];   // FISTA: R_{k-1} in the other buffer
        if (!a.fista) Rk = a.R[0];
        double part[4] = {0.0, 0.0, 0.0, 0.0};   // ||R_k||^2, ||D Theta_k||^2, kkt, kktp (this thread)

        // ---------------- phase F: R_k (and R(Y_k))
        part[0] = forward(cur, Rk, fis ? a.RY : nullptr, Rp, beta, first);
        cp_grid_sync(a.bar, G, gen);

        // ---------------- phase B: G, stencil, KKT, step, projection
        const double *Rsrc = fis ? a.RY : Rk;
        const bool two = fis && kv;                       // also G(Theta_k) for the KKT
        for (int tb = blockIdx.x; tb < nbk; tb += G) {
            const int k0 = 8 * tb;
            const int kl = min(k0 + 7, M - 1);
            const int dA = a.row_da[k0], dB = a.row_db[kl];
            const int mk = k0 + g4;                       // A: (row mk, probe d)
            const bool mok = mk < M;
            const int ra = mok ? a.row_da[mk] : 0, rb = mok ? a.row_db[mk] : 0;
            const int64_t toff = mok ? a.toff[mk] : 0;
            const int nks = (dB - dA + 3) >> 2;
            // G tile of one residual source into a warp-partial buffer (two passes at FISTA KKT
            // iterations: G(Y) from R(Y), G(Theta_k) from R_k)
            auto gemm = [&](const double *src, double *dst) {   // dst: compact [8][NC] tile
                double acc[NB][2];
#pragma unroll
                for (int nb = 0; nb < NB; nb++) acc[nb][0] = acc[nb][1] = 0.0;
                cp_kloop<NB>(acc, warp, nks, NW,
                             [&](int ks) {
                                 const int d = dA + 4 * ks + t4;
                                 return (d >= ra && d < rb) ? __ldg(a.FT + toff + (d - ra)) : 0.0;
                             },
                             [&](int ks, double (&bv)[NB]) {
                                 const int d = dA + 4 * ks + t4;
                                 const bool dok = d < dB;
#pragma unroll
                                 for (int nb = 0; nb < NB; nb++) {
                                     const int n = 8 * nb + g4;
                                     bv[nb] = (dok && n < N) ? __ldcg(src + (int64_t)d * N + n) : 0.0;
                                 }
                             });
                double *rw = red + (warp * 8 + g4) * NC + 2 * t4;
#pragma unroll
                for (int nb = 0; nb < NB; nb++)
                    *reinterpret_cast<double2 *>(rw + 8 * nb) = make_double2(acc[nb][0], acc[nb][1]);
                __syncthreads();
                for (int e = tid; e < 8 * NC; e += CP_THREADS) {   // warp partials in warp order
                    const int r = e / NC, n = e - r * NC;
                    double sacc = 0.0;
#pragma unroll
                    for (int w = 0; w < NW; w++) sacc += red[(w * 8 + r) * NC + n];
                    dst[e] = sacc;
                }
                __syncthreads();
            };
            gemm(Rsrc, Gy);
            if (two) gemm(Rk, Gk);
            // row epilogue: warp r owns Fock row k0 + r
            const int row = k0 + warp;
            if (warp < 8 && row < M) {
                const double t = __ldg(a.tstep + row);
                const bool hp = row > 0, hn = row + 1 < M;
                const double *c0 = cur + (int64_t)row * N;
                const double *q0 = prv ? prv + (int64_t)row * N : nullptr;
                double th[NJ], y[NJ], gk[NJ], x[NJ];
                double rg = 0.0;
#pragma unroll
                for (int jj = 0; jj < NJ; jj++) {
                    const int n = lane + 32 * jj;
                    const bool ok = n < N;
                    const double gsum = ok ? Gy[warp * NC + n] : 0.0;
                    const double gsum2 = (ok && two) ? Gk[warp * NC + n] : 0.0;
                    const double a0 = ok ? __ldcg(c0 + n) : 0.0;
                    const double ap = (ok && hp) ? __ldcg(c0 + n - N) : a0;
                    const double an = (ok && hn) ? __ldcg(c0 + n + N) : a0;
                    th[jj] = a0;
                    if (ok && hn && n < Nv) {
                        const double dd = a0 - an;
                        rg = fma(dd, dd, rg);
                    }
                    double y0 = a0, yp = ap, yn = an;
                    if (prv && ok) {
                        const double b0 = __ldcg(q0 + n);
                        const double bp = hp ? __ldcg(q0 + n - N) : b0;
                        const double bn = hn ? __ldcg(q0 + n + N) : b0;
                        y0 = fma(beta, a0 - b0, a0);
                        yp = hp ? fma(beta, ap - bp, ap) : y0;
                        yn = hn ? fma(beta, an - bn, an) : y0;
                    }
                    y[jj] = y0;
                    const double g = fma(a.gamma, (y0 - yp) + (y0 - yn), gsum);
                    x[jj] = g;   // G(Y) for now
                    gk[jj] = two ? fma(a.gamma, (a0 - ap) + (a0 - an), gsum2) : g;   // G(Theta_k)
                }
                part[1] += rg;
                if (kv) {
                    double mn = INFINITY;
#pragma unroll
                    for (int jj = 0; jj < NJ; jj++)
                        if (lane + 32 * jj < Nv) mn = dmin(mn, 2.0 * gk[jj]);
                    mn = wred_min(mn);
                    const double lam = -mn, lamp = fmax(lam, 0.0);
#pragma unroll
                    for (int jj = 0; jj < NJ; jj++)
                        if (lane + 32 * jj < Nv) {
                            const double g2 = 2.0 * gk[jj];
                            const double x1 = th[jj] * (g2 + lam), x2 = th[jj] * (g2 + lamp);
                            part[2] = fma(x1, x1, part[2]);
                            part[3] = fma(x2, x2, part[3]);
                        }
                }
                if (!fin) {
                    double s = 0.0, xm = -INFINITY, xn = INFINITY;
#pragma unroll
                    for (int jj = 0; jj < NJ; jj++) {
                        if (lane + 32 * jj < Nv) {
                            x[jj] = fma(-t, x[jj], y[jj]);
                            s += x[jj];
                            xm = dmax(xm, x[jj]);
                            xn = dmin(xn, x[jj]);
                        } else {
                            x[jj] = -INFINITY;
                        }
                    }
                    s = wred_sum(s);
                    xm = wred_max(xm);
                    xn = wred_min(xn);
                    double tau = (s - 1.0) / (double)Nv;
                    if (!(xn > tau)) {   // Michelot from the lower bound max(tau_0, max X - 1) (reading R4)
                        tau = fmax(tau, xm - 1.0);
                        int cnt = Nv + 1;
                        for (int round = 0; round <= Nv; round++) {
                            double ps = 0.0, mA = INFINITY;
                            int pc = 0;
#pragma unroll
                            for (int jj = 0; jj < NJ; jj++)
                                if (x[jj] > tau) {
                                    ps += x[jj];
                                    pc++;
                                    mA = dmin(mA, x[jj]);
                                }
                            ps = wred_sum(ps);
                            pc = wred_sum_i(pc);
                            mA = wred_min(mA);
                            if (pc >= cnt) break;
                            cnt = pc;
                            tau = (ps - 1.0) / (double)pc;
                            if (mA > tau) break;
                        }
                    }
                    double *o = out + (int64_t)row * N;
#pragma unroll
                    for (int jj = 0; jj < NJ; jj++) {
                        const int n = lane + 32 * jj;
                        if (n < N) {
                            const double v = x[jj] - tau;
                            __stcg(o + n, (n < Nv && v > 0.0) ? v : 0.0);
                        }
                    }
                }
            }
            __syncthreads();
        }
        // per-CTA partials (fixed order: lanes, warps), then every CTA sums them in CTA order
#pragma unroll
        for (int i = 0; i < 4; i++) part[i] = wred_sum(part[i]);
        if (lane == 0)
#pragma unroll
            for (int i = 0; i < 4; i++) bsum[warp][i] = part[i];
        __syncthreads();
        double *pp = a.part + (size_t)(k & 1) * G * 4;
        if (tid == 0) {
            double v[4] = {0.0, 0.0, 0.0, 0.0};
            for (int w = 0; w < NW; w++)
#pragma unroll
                for (int i = 0; i < 4; i++) v[i] += bsum[w][i];
#pragma unroll
            for (int i = 0; i < 4; i++) __stcg(pp + blockIdx.x * 4 + i, v[i]);
        }
        cp_grid_sync(a.bar, G, gen);
        double tot[4] = {0.0, 0.0, 0.0, 0.0};
        if (warp == 0) {   // lane l: CTAs l, l + 32, ... in order; then a butterfly
            for (unsigned b = lane; b < G; b += 32)
#pragma unroll
                for (int i = 0; i < 4; i++) tot[i] += __ldcg(pp + b * 4 + i);
#pragma unroll
            for (int i = 0; i < 4; i++) tot[i] = wred_sum(tot[i]);
            if (lane == 0)
#pragma unroll
                for (int i = 0; i < 4; i++) bsum[0][i] = tot[i];
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 4; i++) tot[i] = bsum[0][i];
        __syncthreads();
        const double f = tot[0] + a.gamma * tot[1];
        const double r = kv ? sqrt(tot[2] / nm) : NAN, rpv = kv ? sqrt(tot[3] / nm) : NAN;
        if (blockIdx.x == 0 && tid == 0 && k < a.trace_len) {
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
    }
    if (blockIdx.x == 0 && tid == 0) {
        const int64_t kd = stopped ? k : a.iters;
        a.state->iters_done = kd;
        a.state->it = kd;
        a.state->stop = 1;
        a.state->converged = converged ? 1 : 0;
        a.state->nonfinite = nonfinite ? 1 : 0;
    }
}

// transposed band: FT[toff[k] + d - row_da[k]] = F[d][k] (thread per probe)
__global__ void k_build_FT(Band b, int D, const int32_t *row_da, const int64_t *toff, double *FT)
{
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= D) return;
    const int lo = b.lo[d], ln = b.len[d];
    const int64_t of = b.off[d];
    for (int j = 0; j < ln; j++) {
        const int kk = lo + j;
        FT[toff[kk] + (d - row_da[kk])] = b.val[of + j];
    }
}

cudaError_t launch_build_FT(Band b, int D, const int32_t *row_da, const int64_t *toff, double *FT, cudaStream_t s)
{
    k_build_FT<<<(D + 127) / 128, 128, 0, s>>>(b, D, row_da, toff, FT);
    return cudaGetLastError();
}

static int coop_nb(int N) { return N <= 32 ? 4 : N <= 64 ? 8 : N <= 104 ? 13 : N <= 128 ? 16 : 0; }

template <int NB>
static cudaError_t coop_launch_nb(const CoopArgs &a_in, int nblocks_needed, cudaStream_t s)
{
    const size_t smem = coop_smem(NB);
    cudaError_t e = cudaFuncSetAttribute(k_coop_solve<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_coop_solve<NB>, CP_THREADS, smem);
    if (e != cudaSuccess) return e;
    if (per < 1) return cudaErrorCooperativeLaunchTooLarge;
    const int grid = std::max(1, std::min(nblocks_needed, per * nsm));
    CoopArgs a = a_in;
    void *args[] = {&a};
    return cudaLaunchCooperativeKernel((const void *)k_coop_solve<NB>, dim3(grid), dim3(CP_THREADS), args, smem, s);
}

bool coop_supported(int N) { return coop_nb(N) > 0; }

// grid partial buffer: 2 x (max grid) x 4 doubles; the caller sizes it with coop_max_grid()
int coop_max_grid() { return 2 * 1024; }

cudaError_t launch_coop_solve(const CoopArgs &a, cudaStream_t s)
{
    const int need = std::max((a.D + 7) / 8, (a.M + 7) / 8);
    switch (coop_nb(a.N)) {
        case 4: return coop_launch_nb<4>(a, need, s);
        case 8: return coop_launch_nb<8>(a, need, s);
        case 13: return coop_launch_nb<13>(a, need, s);
        case 16: return coop_launch_nb<16>(a, need, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qdt
