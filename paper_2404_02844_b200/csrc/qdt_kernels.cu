// qdt_kernels.cu -- hand-written sm_100a kernels of the detector-tomography hot path.
//
// One projected-gradient iteration:
//   k_fwd      S2  R-partials: for every Fock tile, sum_{k in tile} F[d,k] Theta[k,:] for the
//                  probes d of the tile's window (banded F, "two steps").
//   k_reduce_R S2  R = sum of the partials of probe d (fixed tile order) - P, ||R||^2 partials.
//   k_bwd      S3-S6 per Fock tile: G = F^T R (window GEMM, cp.async double-buffered smem
//                  staging) + gamma L Theta (stencil epilogue, eq. regul),
//                  X = Y - t o G, per-row simplex projection (warp Michelot, eq. Mp1_proj
//                  PAPER.md:499-502), Theta_next, and the KKT / regulariser partials
//                  (PAPER.md:563-567).  Heavy tiles are split along the probe axis (split-K)
//                  with a deterministic last-block fix-up.
//   k_scalars_local / k_finalize  S6 fixed-order reductions, trace, device stop flag.
// Setup: k_probe_edges / k_probe_values (S0, eq. Fmatrix PAPER.md:107-109 in Loader's
// saddle-point form), k_probe_rowsum + k_sqs_weights or the power iteration (S1).
//
// All arithmetic is fp64.  Reductions are deterministic (fixed grids, fixed orders).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "qdt_internal.h"
#include "qdt_ptx.cuh"

namespace qdt {

// ------------------------------------------------------------------------------ helpers
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool pred)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int n>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(n) : "memory"); }

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ int warp_sum_i(int v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_min(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block sum of NV_ values per thread; result valid in thread 0.
template <int NV_>
__device__ __forceinline__ void block_sum(double (&v)[NV_], double *red /* smem >= 32*NV_ */)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < NV_; i++) v[i] = warp_sum(v[i]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV_; i++) red[w * NV_ + i] = v[i];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV_; i++) {
            double s = 0.0;
            for (int j = 0; j < nw; j++) s += red[j * NV_ + i];
            v[i] = s;
        }
    }
}

// Segment (SEG lanes, power of two, aligned inside a warp) reductions: one Fock row per segment.
__device__ __forceinline__ double seg_sum(double v, int SEG)
{
    for (int o = SEG >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ int seg_sum_i(int v, int SEG)
{
    for (int o = SEG >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double seg_max(double v, int SEG)
{
    for (int o = SEG >> 1; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double seg_min(double v, int SEG)
{
    for (int o = SEG >> 1; o > 0; o >>= 1) v = dmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool pred)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz)
                 : "memory");
}
// Stage n contiguous doubles src[0..n) into smem dst; elements outside [v0, v1) are zero-filled.
// vec: 16-byte copies (n, v0, v1 even; src, dst 16-byte aligned).
__device__ __forceinline__ void stage_run(double *dst, const double *src, int n, int v0, int v1,
                                         const double *dummy, bool vec)
{
    if (vec) {
        for (int c = threadIdx.x; c < (n >> 1); c += blockDim.x) {
            const int i = c << 1;
            const bool ok = i >= v0 && i < v1;
            cp_async16(dst + i, ok ? src + i : dummy, ok);
        }
    } else {
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const bool ok = i >= v0 && i < v1;
            cp_async8(dst + i, ok ? src + i : dummy, ok);
        }
    }
}

// Euclidean projection threshold of one row onto the simplex by
// Michelot's method, one warp per row: tau_0 = (sum x - 1)/N; repeatedly keep A = {x > tau},
// tau = (sum_A x - 1)/|A| until |A| stops shrinking (<= N rounds; A only shrinks).
// Same projection as the sort-based / Condat result (reading R4).
__device__ __forceinline__ double michelot_tau(const double *x, int N, double s_all)
{
    const int lane = threadIdx.x & 31;
    int cnt = N;
    double tau = (s_all - 1.0) / (double)N;
    for (int round = 0; round <= N; round++) {
        double s = 0.0;
        int c = 0;
        for (int n = lane; n < N; n += 32) {
            double v = x[n];
            if (v > tau) {
                s += v;
                c++;
            }
        }
        s = warp_sum(s);
        c = warp_sum_i(c);
        if (c >= cnt) break;
        cnt = c;
        tau = (s - 1.0) / (double)c;
    }
    return tau;
}

// ------------------------------------------------------------------------------ S0 probes
// Band edges (reading R1): s = sqrt(mu), lo = max(0, floor(mu - c s)),
// hi = min(M-1, ceil(mu + c s) + margin); every operation rounded to nearest, no FMA.
__global__ void k_probe_edges(const double *alpha2, int64_t D, int64_t M, double c_sigma,
                              int margin, int32_t *lo, int32_t *hi)
{
    int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= D) return;
    double mu = alpha2[d];
    int64_t L = 0, H = 0;
    if (mu != 0.0) {
        double s = __dsqrt_rn(mu);
        double cs = __dmul_rn(c_sigma, s);
        double a = __dsub_rn(mu, cs);
        double b = __dadd_rn(mu, cs);
        double l = floor(a);
        double h = __dadd_rn(ceil(b), (double)margin);
        L = (l < 0.0) ? 0 : (int64_t)l;
        H = (h > (double)(M - 1)) ? (M - 1) : (int64_t)h;
        if (L > M - 1) L = M - 1;
        if (H < L) H = L;
    }
    lo[d] = (int32_t)L;
    hi[d] = (int32_t)H;
}

// delta(k) = ln k! - [(k+1/2) ln k - k + ln(2 pi)/2], k = 0..15 (tools/gen_stirlerr.py)
__constant__ double c_stirlerr[16] = {
    0x0.0p+0,           0x1.4c071bcda0a5bp-4, 0x1.52a9b923ea649p-5, 0x1.c579a268d80b3p-6,
    0x1.54a2662fd78a9p-6, 0x1.10b4e513fcbedp-6, 0x1.c6b167bebdf36p-7, 0x1.85d4d612e4a86p-7,
    0x1.552805e7b3076p-7, 0x1.2f4871b12ab64p-7, 0x1.10f9d4c0743a7p-7, 0x1.f0593088014f8p-8,
    0x1.c7018733aa9c6p-8, 0x1.a40514700f36cp-8, 0x1.86076c002d4a7p-8, 0x1.6c08f6f194a10p-8};

__device__ __forceinline__ double stirlerr(double k)
{
    if (k < 16.0) return c_stirlerr[(int)k];
    const double S0 = 1.0 / 12, S1 = 1.0 / 360, S2 = 1.0 / 1260, S3 = 1.0 / 1680, S4 = 1.0 / 1188;
    double k2 = 1.0 / (k * k);
    return (S0 - (S1 - (S2 - (S3 - S4 * k2) * k2) * k2) * k2) / k;
}

// Deviance term bd0(x, mu) = x ln(x/mu) + mu - x.  For |x - mu| < (x + mu)/2 it is summed as
// the series (x-mu) v + 2x sum_j v^(2j+1)/(2j+1), v = (x-mu)/(x+mu) (no cancellation; v^2 <= 1/4
// so ~27 terms at most); outside, the direct form cancels by at most a factor ~2.5.
__device__ __forceinline__ double bd0(double x, double mu)
{
    if (fabs(x - mu) < 0.5 * (x + mu)) {
        double v = (x - mu) / (x + mu);
        double s = (x - mu) * v;
        double ej = 2.0 * x * v;
        v = v * v;
        for (int j = 1; j < 200; j++) {
            ej *= v;
            double s1 = s + ej / (double)(2 * j + 1);
            if (s1 == s) return s1;
            s = s1;
        }
        return s;
    }
    return x * log(x / mu) + mu - x;
}

// F_{d,k} = mu^k e^{-mu} / k! = exp(-ln(2 pi k)/2 - delta(k) - bd0(k, mu))  (Loader's form)
__device__ __forceinline__ double poisson_pmf(int64_t k, double mu)
{
    if (mu == 0.0) return (k == 0) ? 1.0 : 0.0;
    if (k == 0) return exp(-mu);
    double x = (double)k;
    const double TWO_PI = 6.283185307179586476925286766559;
    return exp(-0.5 * log(TWO_PI * x) - stirlerr(x) - bd0(x, mu));
}

__global__ void k_probe_values(const double *alpha2, Band b, double *val)
{
    int d = blockIdx.x;
    double mu = alpha2[d];
    int lo = b.lo[d], len = b.len[d];
    int64_t off = b.off[d];
    for (int j = threadIdx.x; j < len; j += blockDim.x) val[off + j] = poisson_pmf(lo + j, mu);
}

__global__ void k_probe_rowsum(Band b, double *s_out)
{
    __shared__ double red[32];
    int d = blockIdx.x;
    int len = b.len[d];
    int64_t off = b.off[d];
    double v[1] = {0.0};
    for (int j = threadIdx.x; j < len; j += blockDim.x) v[0] += b.val[off + j];
    block_sum<1>(v, red);
    if (threadIdx.x == 0) s_out[d] = v[0];
}

// ------------------------------------------------------------------------------ S1 setup
// SQS weights (reading R2): w_k = sum_d F_{d,k} s_d + 4 gamma (d ascending), t_k = 1/w_k.
__global__ void k_sqs_weights(int T, const int32_t *tile_dA, const int32_t *tile_dB, int Ml,
                              int64_t kb, Band b, const double *s, double gamma, double *w,
                              double *tstep)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= Ml) return;
    int t = k / T;
    int64_t kg = kb + k;
    double acc = 0.0;
    for (int d = tile_dA[t]; d < tile_dB[t]; d++) {
        int lo = b.lo[d], len = b.len[d];
        if (kg >= lo && kg < lo + len) acc += b.val[b.off[d] + (kg - lo)] * s[d];
    }
    acc += 4.0 * gamma;
    if (w) w[k] = acc;
    if (tstep) tstep[k] = (acc > 0.0) ? 1.0 / acc : 0.0;
}

// power iteration pieces: q = F v (block per probe), u = F^T q (thread per row)
__global__ void k_pow_fwd(Band b, const double *v, int64_t kb, double *q)
{
    __shared__ double red[32];
    int d = blockIdx.x;
    int lo = b.lo[d], len = b.len[d];
    int64_t off = b.off[d];
    double a[1] = {0.0};
    for (int j = threadIdx.x; j < len; j += blockDim.x) a[0] += b.val[off + j] * v[lo + j - kb];
    block_sum<1>(a, red);
    if (threadIdx.x == 0) q[d] = a[0];
}

__global__ void k_pow_bwd(int T, const int32_t *tile_dA, const int32_t *tile_dB, int Ml,
                          int64_t kb, Band b, const double *q, double *u)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= Ml) return;
    int t = k / T;
    int64_t kg = kb + k;
    double acc = 0.0;
    for (int d = tile_dA[t]; d < tile_dB[t]; d++) {
        int lo = b.lo[d], len = b.len[d];
        if (kg >= lo && kg < lo + len) acc += b.val[b.off[d] + (kg - lo)] * q[d];
    }
    u[k] = acc;
}

__global__ void k_sumsq(const double *x, int64_t n, double *part)
{
    __shared__ double red[32];
    int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    int64_t beg = (int64_t)blockIdx.x * chunk, end = beg + chunk < n ? beg + chunk : n;
    double v[1] = {0.0};
    for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) v[0] += x[i] * x[i];
    block_sum<1>(v, red);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

__global__ void k_reduce_vec(const double *part, int nblk, int stride, int nvals, double *out)
{
    __shared__ double red[32 * 8];
    for (int i = 0; i < nvals; i += 8) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) v[j] = 0.0;
        for (int b = threadIdx.x; b < nblk; b += blockDim.x)
#pragma unroll
            for (int j = 0; j < 8; j++)
                if (i + j < nvals) v[j] += part[(int64_t)b * stride + i + j];
        block_sum<8>(v, red);
        if (threadIdx.x == 0)
            for (int j = 0; j < 8 && i + j < nvals; j++) out[i + j] = v[j];
        __syncthreads();
    }
}

__global__ void k_scale(double *v, const double *u, const double *nrm2, int64_t n)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double nn = sqrt(nrm2[0]);
    if (i < n) v[i] = (nn > 0.0) ? u[i] / nn : u[i];
}

__global__ void k_fill(double *x, int64_t n, double v)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = v;
}

// ------------------------------------------------------------------------------ S2 forward
// Thread (rg, cg) owns probes rg*TR..rg*TR+TR-1 of the unit and columns cg + c*CG.
// Row chunks of KR rows: Theta chunk [KR x N] and F chunk [KR x KP] staged by cp.async.
template <int TC>
__global__ void __launch_bounds__(256) k_fwd(FwdArgs a)
{
    extern __shared__ __align__(16) double smem[];
    __shared__ int32_t s_lo[WCAP_MAX], s_len[WCAP_MAX];
    __shared__ int64_t s_off[WCAP_MAX];
    if (a.state && a.state->stop) return;
    const int N = a.N, CG = a.CG, RG = a.RG, KR = a.KR;
    const int KP = RG * TR, KPP = KP + 2;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int rg = tid / CG, cg = tid - (tid / CG) * CG;
    const bool gth = tid < RG * CG;
    const FwdUnit u = a.units[blockIdx.x];
    const int tsz = (KR * N + CG * TC + 1) & ~1;  // padded (over-range column reads), even
    double *Tc = smem;                 // 2 x tsz
    double *Fc = smem + 2 * tsz;       // 2 x KR x KPP
    const int np = u.p1 - u.p0;
    const int nrows = u.k1 - u.k0;
    const int nch = (nrows + KR - 1) / KR;

    const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
    const bool vec = (N & 1) == 0;
    for (int j = tid; j < np; j += nthr) {
        s_lo[j] = a.band.lo[u.p0 + j];
        s_len[j] = a.band.len[u.p0 + j];
        s_off[j] = a.band.off[u.p0 + j];
    }
    __syncthreads();
    auto stage = [&](int buf, int c) {
        const int kbeg = u.k0 + c * KR;
        const int kr = min(KR, u.k1 - kbeg);
        stage_run(Tc + buf * tsz, a.theta + (int64_t)kbeg * N, KR * N, 0, kr * N, a.theta, vec);
        double *F = Fc + buf * KR * KPP;
        const int64_t kg0 = a.kb + kbeg;
        for (int p = warp; p < KP; p += nw) {      // one warp per probe of the unit
            const int d = u.p0 + p;
            int ra = 0, rb = 0;
            const double *src = a.band.val;
            if (p < np) {
                const int64_t lo = s_lo[p], len = s_len[p];
                ra = (int)max((int64_t)0, lo - kg0);
                rb = (int)min((int64_t)kr, lo + len - kg0);
                src = a.band.val + s_off[p] + (kg0 - lo);
            }
            for (int r = lane; r < KR; r += 32) {
                const bool ok = r >= ra && r < rb;
                cp_async8(&F[r * KPP + p], ok ? src + r : a.band.val, ok);
            }
        }
    };

    double acc[TR][TC];
#pragma unroll
    for (int i = 0; i < TR; i++)
#pragma unroll
        for (int c = 0; c < TC; c++) acc[i][c] = 0.0;

    if (nch > 0) stage(0, 0);
    cp_async_commit();
    for (int c = 0; c < nch; c++) {
        if (c + 1 < nch) stage((c + 1) & 1, c + 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        if (gth && rg * TR < np) {
            const double *T = Tc + (c & 1) * tsz + cg;
            const double *F = Fc + (c & 1) * KR * KPP + rg * TR;
            const int kr = min(KR, nrows - c * KR);
            for (int r = 0; r < kr; r++) {
                const double2 f01 = *reinterpret_cast<const double2 *>(F + r * KPP);
                const double2 f23 = *reinterpret_cast<const double2 *>(F + r * KPP + 2);
                const double fv[TR] = {f01.x, f01.y, f23.x, f23.y};
                double tv[TC];
#pragma unroll
                for (int cc = 0; cc < TC; cc++) tv[cc] = T[r * N + cc * CG];
#pragma unroll
                for (int i = 0; i < TR; i++)
#pragma unroll
                    for (int cc = 0; cc < TC; cc++) acc[i][cc] = fma(fv[i], tv[cc], acc[i][cc]);
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    if (gth) {
#pragma unroll
        for (int i = 0; i < TR; i++) {
            int p = rg * TR + i;
            if (p < np) {
                double *dst = a.rpart + (u.poff + p) * (int64_t)N;
#pragma unroll
                for (int cc = 0; cc < TC; cc++) {
                    int n = cg + cc * CG;
                    if (n < N) dst[n] = acc[i][cc];
                }
            }
        }
    }
}

// R[d,:] = sum over the probe's partial rows (ascending Fock tile) - P[d,:]; ||R||^2 partials.
__global__ void k_reduce_R(const double *rpart, const int64_t *red_beg, const int64_t *red_rows,
                           const double *P, double *R, int64_t D, int N, double *partR,
                           const DevState *st)
{
    __shared__ double red[32];
    if (st && st->stop) return;
    int64_t total = D * N;
    int64_t chunk = (total + gridDim.x - 1) / gridDim.x;
    int64_t beg = (int64_t)blockIdx.x * chunk, end = beg + chunk < total ? beg + chunk : total;
    double v[1] = {0.0};
    for (int64_t e = beg + threadIdx.x; e < end; e += blockDim.x) {
        int64_t d = e / N;
        int64_t n = e - d * N;
        double s = 0.0;
        for (int64_t j = red_beg[d]; j < red_beg[d + 1]; j++) s += rpart[red_rows[j] * N + n];
        if (P) s -= P[e];
        R[e] = s;
        v[0] += s * s;
    }
    block_sum<1>(v, red);
    if (threadIdx.x == 0 && partR) partR[blockIdx.x] = v[0];
}

__global__ void k_sub_p_sumsq(double *R, const double *P, int64_t n, double *partR,
                              const DevState *st)
{
    __shared__ double red[32];
    if (st && st->stop) return;
    int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    int64_t beg = (int64_t)blockIdx.x * chunk, end = beg + chunk < n ? beg + chunk : n;
    double v[1] = {0.0};
    for (int64_t e = beg + threadIdx.x; e < end; e += blockDim.x) {
        double s = R[e] - P[e];
        R[e] = s;
        v[0] += s * s;
    }
    block_sum<1>(v, red);
    if (threadIdx.x == 0) partR[blockIdx.x] = v[0];
}

// FISTA residual of the extrapolated point: R(Y) = R_k + beta (R_k - R_{k-1}) (linear in Theta)
__global__ void k_fista_rcomb(double *RY, const double *Rk, const double *Rkm1, const double *beta,
                              int64_t n, const DevState *st)
{
    if (st && st->stop) return;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double b = beta[st->it];
    if (i < n) RY[i] = Rk[i] + b * (Rk[i] - Rkm1[i]);
}

// ------------------------------------------------------------------------------ S3-S6 bwd
// One CTA per work unit (a Fock tile, or one probe-range split of a heavy tile):
//   GEMM   G[T x N] = F_tile^T[T x W] R_win[W x N]  (thread (rg,cg): TR rows x TC columns)
//   epi 1  G += gamma L Y   (stencil, eq. regul; free ends at k = 0, M-1, reading R8)
//   epi 2  one SEG-lane segment per Fock row, the row held in registers:
//          KKT partial (df = 2G), regulariser pair (k, k+1),
//          X = Y - t_k G, Michelot threshold, Theta_next = max(X - tau, 0).
template <int TC, int MODE, bool FISTA, int VMAX>
__global__ void __launch_bounds__(256) k_bwd(BwdArgs a)
{
    extern __shared__ __align__(16) double smem[];
    __shared__ double red[32 * NSC_TILE];
    __shared__ int s_last;
    __shared__ int32_t s_lo[WCAP_MAX], s_len[WCAP_MAX];
    __shared__ int64_t s_off[WCAP_MAX];
    const DevState *st = a.state;
    if (st && st->stop) return;
    const int64_t it = st ? st->it : 0;
    if (MODE == BWD_EVAL && FISTA && (it % a.kkt_every) != 0) return;
    const double beta = (FISTA && MODE == BWD_STEP) ? a.beta[it] : 0.0;

    const int N = a.N, CG = a.CG, RG = a.RG, KC = a.KC;
    const int T = RG * TR;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
    const int rg = tid / CG, cg = tid - (tid / CG) * CG;
    const bool gth = tid < RG * CG;
    const bool vec = (N & 1) == 0;
    const BwdUnit u = a.units[blockIdx.x];
    const int k0 = u.k0, Tt = u.k1 - u.k0;
    const int thsz = (T + 2) * N;
    const int rsz = (KC * N + CG * TC + 1) & ~1;
    double *Th = smem;                                 // (T+2) x N : rows k0-1 .. k1 of Theta_k
    double *Tp = Th + thsz;                            // FISTA: Theta_{k-1}
    double *Gs = FISTA ? Tp + thsz : Tp;               // T x N
    double *Fc = Gs + T * N;                           // 2 x KC x T
    double *Rc = Fc + 2 * KC * T;                      // 2 x rsz
    const bool need_theta = (MODE != BWD_GRAD) || a.gamma != 0.0;

    auto load_theta = [&]() {
        const int tot = (Tt + 2) * N;
        const int64_t kg0 = a.kb + k0 - 1;               // global row of smem row 0
        const int v0 = kg0 < 0 ? N : 0;
        const int v1 = (kg0 + Tt + 1 >= a.M) ? (int)(a.M - kg0) * N : tot;
        const int64_t base = (int64_t)(k0 - 1) * N;
        stage_run(Th, a.theta + base, tot, v0, v1, a.theta, vec);
        if (FISTA) stage_run(Tp, a.theta_prev + base, tot, v0, v1, a.theta, vec);
    };
    if (u.nsplit == 1 && need_theta) load_theta();
    cp_async_commit();
    for (int j = tid; j < u.p1 - u.p0; j += nthr) {   // band tables of the unit's probes
        s_lo[j] = a.band.lo[u.p0 + j];
        s_len[j] = a.band.len[u.p0 + j];
        s_off[j] = a.band.off[u.p0 + j];
    }
    __syncthreads();

    auto stage = [&](int buf, int c) {
        const int pbeg = u.p0 + c * KC;
        double *F = Fc + buf * KC * T;
        const int64_t kg0 = a.kb + k0;
        for (int j = warp; j < KC; j += nw) {      // one warp per probe of the chunk
            const int d = pbeg + j;
            int ra = 0, rb = 0;
            const double *src = a.band.val;
            if (d < u.p1) {
                const int64_t lo = s_lo[d - u.p0], len = s_len[d - u.p0];
                ra = (int)max((int64_t)0, lo - kg0);
                rb = (int)min((int64_t)Tt, lo + len - kg0);
                src = a.band.val + s_off[d - u.p0] + (kg0 - lo);
            }
            for (int r = lane; r < T; r += 32) {
                const bool ok = r >= ra && r < rb;
                cp_async8(&F[j * T + r], ok ? src + r : a.band.val, ok);
            }
        }
        const int kc = min(KC, u.p1 - pbeg);
        stage_run(Rc + buf * rsz, a.R + (int64_t)pbeg * N, KC * N, 0, kc * N, a.R, vec);
    };

    double acc[TR][TC];
#pragma unroll
    for (int i = 0; i < TR; i++)
#pragma unroll
        for (int c = 0; c < TC; c++) acc[i][c] = 0.0;

    const int nch = (u.p1 - u.p0 + KC - 1) / KC;
    if (nch > 0) stage(0, 0);
    cp_async_commit();
    for (int c = 0; c < nch; c++) {
        if (c + 1 < nch) stage((c + 1) & 1, c + 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        if (gth) {
            const double *F = Fc + (c & 1) * KC * T + rg * TR;
            const double *Rr = Rc + (c & 1) * rsz + cg;
            const int kc = min(KC, u.p1 - (u.p0 + c * KC));
            for (int j = 0; j < kc; j++) {
                const double2 f01 = *reinterpret_cast<const double2 *>(F + j * T);
                const double2 f23 = *reinterpret_cast<const double2 *>(F + j * T + 2);
                const double fv[TR] = {f01.x, f01.y, f23.x, f23.y};
                double rv[TC];
#pragma unroll
                for (int cc = 0; cc < TC; cc++) rv[cc] = Rr[j * N + cc * CG];
#pragma unroll
                for (int i = 0; i < TR; i++)
#pragma unroll
                    for (int cc = 0; cc < TC; cc++) acc[i][cc] = fma(fv[i], rv[cc], acc[i][cc]);
            }
        }
        __syncthreads();
    }

    if (u.nsplit > 1) {
        // split-K fix-up: publish the partial G, the last unit of the tile sums all slots in
        // slot order (deterministic, independent of which unit finishes last).
        const int64_t tsz = (int64_t)T * N;
        double *slot = a.scratch + (u.slot_base + u.slot) * tsz;
        if (gth)
#pragma unroll
            for (int i = 0; i < TR; i++) {
                int row = rg * TR + i;
#pragma unroll
                for (int cc = 0; cc < TC; cc++) {
                    int n = cg + cc * CG;
                    if (row < Tt && n < N) __stcg(&slot[row * N + n], acc[i][cc]);
                }
            }
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = (atomicAdd(&a.counters[u.tile], 1) == u.nsplit - 1);
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        if (need_theta) load_theta();
        cp_async_commit();
        if (gth)
#pragma unroll
            for (int i = 0; i < TR; i++) {
                int row = rg * TR + i;
#pragma unroll
                for (int cc = 0; cc < TC; cc++) {
                    int n = cg + cc * CG;
                    double s = 0.0;
                    if (row < Tt && n < N)
                        for (int sl = 0; sl < u.nsplit; sl++)
                            s += __ldcg(&a.scratch[(u.slot_base + sl) * tsz + row * N + n]);
                    acc[i][cc] = s;
                }
            }
        if (tid == 0) a.counters[u.tile] = 0;
    }
    cp_async_wait<0>();
    __syncthreads();

    // ---- epilogue 1: park the GEMM result in shared memory (row pass below adds the stencil)
    if (gth) {
#pragma unroll
        for (int i = 0; i < TR; i++) {
            const int row = rg * TR + i;
#pragma unroll
            for (int cc = 0; cc < TC; cc++) {
                const int n = cg + cc * CG;
                if (row < Tt && n < N) Gs[row * N + n] = acc[i][cc];
            }
        }
    }
    __syncthreads();

    // ---- epilogue 2: one SEG-lane segment per Fock row, row values in registers:
    //      G = acc + gamma L Y (eq. regul, free ends at global k = 0, M-1: reading R8),
    //      regulariser pair (k, k+1), KKT partial (df = 2G, reading R7),
    //      X = Y - t_k G, Michelot threshold (reading R4), Theta_next = max(X - tau, 0).
    double sc[NSC_TILE] = {0.0, 0.0, 0.0, 0.0};
    const bool do_kkt = ((MODE == BWD_EVAL) || !FISTA) && (it % a.kkt_every) == 0;
    const double gamma = a.gamma;
    if constexpr (VMAX > 0) {
        const int SEG = a.SEG;
        // rows per pass: as many segments as fill the tile in the fewest passes; warps beyond
        // them skip the row pass (idle warps cost no issue slots)
        const int maxseg = nthr / SEG;
        const int passes = (Tt + maxseg - 1) / maxseg;
        const int nseg = passes ? (Tt + passes - 1) / passes : 1;
        const int seg = tid / SEG, sl = tid & (SEG - 1);
        bool colok[VMAX];
#pragma unroll
        for (int v = 0; v < VMAX; v++) colok[v] = sl + SEG * v < N;
        if ((warp * 32) / SEG >= nseg) goto rowpass_done;   // warp-uniform
        for (int rb = 0; rb < Tt; rb += nseg) {
            const int row = rb + seg;
            const bool act = row < Tt && seg < nseg && row < rb + nseg;
            const int kl = k0 + row;
            const int64_t kg = a.kb + kl;
            const bool has_prev = kg > 0, has_next = kg + 1 < a.M;
            const double *thr = Th + (row + 1) * N + sl;
            double th[VMAX], g[VMAX];
#pragma unroll
            for (int v = 0; v < VMAX; v++) {
                const bool ok = act && colok[v];
                const double t0 = ok ? thr[SEG * v] : 0.0;
                const double tn = (ok && has_next) ? thr[SEG * v + N] : t0;
                double gg = ok ? Gs[row * N + sl + SEG * v] : 0.0;
                if (has_next) {
                    const double dd = t0 - tn;
                    sc[SC_REG] += dd * dd;
                }
                if (gamma != 0.0) {
                    const double tp = (ok && has_prev) ? thr[SEG * v - N] : t0;
                    double lap;
                    if (FISTA) {
                        const double *tq = Tp + (row + 1) * N + sl + SEG * v;
                        const double y0 = t0 + beta * (t0 - (ok ? tq[0] : 0.0));
                        const double yp = has_prev ? tp + beta * (tp - (ok ? tq[-N] : 0.0)) : y0;
                        const double yn = has_next ? tn + beta * (tn - (ok ? tq[N] : 0.0)) : y0;
                        lap = (y0 - yp) + (y0 - yn);
                    } else {
                        lap = (t0 - tp) + (t0 - tn);
                    }
                    gg = fma(gamma, lap, gg);
                }
                th[v] = t0;
                g[v] = gg;
            }
            if (MODE == BWD_GRAD) {
                if (act) {
                    double *o = a.out + (int64_t)kl * N + sl;
#pragma unroll
                    for (int v = 0; v < VMAX; v++)
                        if (colok[v]) o[SEG * v] = g[v];
                }
                continue;
            }
            if (do_kkt) {
                double mn = INFINITY;
#pragma unroll
                for (int v = 0; v < VMAX; v++)
                    if (colok[v]) mn = dmin(mn, g[v]);
                mn = 2.0 * seg_min(mn, SEG);
                const double lam = act ? -mn : 0.0, lamp = fmax(lam, 0.0);
#pragma unroll
                for (int v = 0; v < VMAX; v++) {
                    const double df = 2.0 * g[v];
                    const double x1 = th[v] * (df + lam), x2 = th[v] * (df + lamp);
                    sc[SC_KKT] += x1 * x1;
                    sc[SC_KKTP] += x2 * x2;
                }
            }
            if (MODE == BWD_STEP) {
                const double t = act ? a.tstep[kl] : 0.0;
                double s = 0.0, xm = -INFINITY;
#pragma unroll
                for (int v = 0; v < VMAX; v++) {
                    const bool ok = act && colok[v] && (seg < nseg);
                    double y = th[v];
                    if (FISTA && ok) y = y + beta * (y - Tp[(row + 1) * N + sl + SEG * v]);
                    const double xv = y - t * g[v];
                    g[v] = ok ? xv : -INFINITY;
                    s += ok ? xv : 0.0;
                    xm = dmax(xm, g[v]);
                }
                s = seg_sum(s, SEG);
                xm = seg_max(xm, SEG);
                // start from the larger of two lower bounds of the threshold: the mean bound
                // (sum x - 1)/N and max x - 1 (the largest coordinate projects to <= 1); from a
                // lower bound the Michelot/Newton updates increase monotonically to tau*.
                int cnt = N + 1;
                double tau = fmax((s - 1.0) / (double)N, xm - 1.0);
                bool done = !act || seg >= nseg;
                for (int round = 0; round <= N; round++) {
                    if (__all_sync(0xffffffffu, done)) break;
                    double ps = 0.0;
                    int pc = 0;
#pragma unroll
                    for (int v = 0; v < VMAX; v++) {
                        const bool in = g[v] > tau;
                        ps += in ? g[v] : 0.0;
                        pc += in;
                    }
                    ps = seg_sum(ps, SEG);
                    pc = seg_sum_i(pc, SEG);
                    if (!done) {
                        if (pc >= cnt) {
                            done = true;
                        } else {
                            cnt = pc;
                            tau = (ps - 1.0) / (double)pc;
                        }
                    }
                }
                if (act && seg < nseg) {
                    double *o = a.out + (int64_t)kl * N + sl;
#pragma unroll
                    for (int v = 0; v < VMAX; v++)
                        if (colok[v]) o[SEG * v] = fmax(g[v] - tau, 0.0);
                }
            }
        }
    rowpass_done:;
    } else {
        // wide rows (N > 512): one warp per row, values streamed from shared memory
        for (int row = warp; row < Tt; row += nw) {
            const int kl = k0 + row;
            const int64_t kg = a.kb + kl;
            double *g = Gs + row * N;
            const double *th = Th + (row + 1) * N;
            if (gamma != 0.0)
                for (int n = lane; n < N; n += 32) {
                    auto Y = [&](int r) {
                        double t = Th[r * N + n];
                        if (FISTA) t = t + beta * (t - Tp[r * N + n]);
                        return t;
                    };
                    const double yc = Y(row + 1);
                    double lap = 0.0;
                    if (kg > 0) lap += yc - Y(row);
                    if (kg < a.M - 1) lap += yc - Y(row + 2);
                    g[n] = fma(gamma, lap, g[n]);
                }
            if (MODE == BWD_GRAD) {
                for (int n = lane; n < N; n += 32) a.out[(int64_t)kl * N + n] = g[n];
                continue;
            }
            if (kg + 1 < a.M)
                for (int n = lane; n < N; n += 32) {
                    const double dd = th[n] - th[n + N];
                    sc[SC_REG] += dd * dd;
                }
            if (do_kkt) {
                double mn = INFINITY;
                for (int n = lane; n < N; n += 32) mn = fmin(mn, 2.0 * g[n]);
                mn = warp_min(mn);
                const double lam = -mn, lamp = fmax(lam, 0.0);
                for (int n = lane; n < N; n += 32) {
                    const double df = 2.0 * g[n];
                    const double x1 = th[n] * (df + lam), x2 = th[n] * (df + lamp);
                    sc[SC_KKT] += x1 * x1;
                    sc[SC_KKTP] += x2 * x2;
                }
            }
            if (MODE == BWD_STEP) {
                const double t = a.tstep[kl];
                double s = 0.0;
                for (int n = lane; n < N; n += 32) {
                    double y = th[n];
                    if (FISTA) y = y + beta * (y - Tp[(row + 1) * N + n]);
                    const double x = y - t * g[n];
                    g[n] = x;
                    s += x;
                }
                __syncwarp();
                s = warp_sum(s);
                const double tau = michelot_tau(g, N, s);
                double *o = a.out + (int64_t)kl * N;
                for (int n = lane; n < N; n += 32) o[n] = fmax(g[n] - tau, 0.0);
            }
            __syncwarp();
        }
    }
    if (MODE == BWD_GRAD) return;
    block_sum<NSC_TILE>(sc, red);
    if (tid == 0) {
        double *p = a.part + (int64_t)u.tile * NSC_TILE;
        if (do_kkt) {
            p[SC_KKT] = sc[SC_KKT];
            p[SC_KKTP] = sc[SC_KKTP];
        }
        p[SC_REG] = sc[SC_REG];
        if (MODE == BWD_STEP || !FISTA) p[SC_DTH] = sc[SC_DTH];
    }
}

// standalone row projection (test hook): warp per row
__global__ void k_project_rows(const double *X, int64_t M, int N, double *Y)
{
    const int lane = threadIdx.x & 31;
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (row >= M) return;
    const double *x = X + row * N;
    double s = 0.0;
    for (int n = lane; n < N; n += 32) s += x[n];
    s = warp_sum(s);
    const double tau = michelot_tau(x, N, s);
    for (int n = lane; n < N; n += 32) Y[row * N + n] = fmax(x[n] - tau, 0.0);
}

// ------------------------------------------------------------------------------ S6 scalars
__global__ void k_scalars_local(const double *partR, int nblkR, const double *partT, int ntiles,
                                int include_r2, double *vec, const DevState *st)
{
    __shared__ double red[32 * NV];
    if (st && st->stop) return;
    double v[NV] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (include_r2)
        for (int b = threadIdx.x; b < nblkR; b += blockDim.x) v[V_R2] += partR[b];
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
        const double *p = partT + (int64_t)t * NSC_TILE;
        v[V_KKT] += p[SC_KKT];
        v[V_KKTP] += p[SC_KKTP];
        v[V_REG] += p[SC_REG];
        v[V_DTH] += p[SC_DTH];
    }
    block_sum<NV>(v, red);
    if (threadIdx.x == 0)
        for (int i = 0; i < NV; i++) vec[i] = v[i];
}

__global__ void k_finalize(const double *vec, int64_t N, int64_t M, double gamma, double tol,
                           int final_eval, int kkt_every, double *trace, double *kkt,
                           double *kktp, int64_t trace_len, DevState *st)
{
    if (threadIdx.x != 0) return;
    if (st->stop) return;
    const int64_t k = st->it;
    const double f = vec[V_R2] + gamma * vec[V_REG];
    const bool kv = final_eval || (k % kkt_every) == 0;
    const double nm = (double)N * (double)M;
    const double r = kv ? sqrt(vec[V_KKT] / nm) : NAN;
    const double rp = kv ? sqrt(vec[V_KKTP] / nm) : NAN;
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
static inline int cdiv64(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

cudaError_t launch_probe_edges(const double *alpha2, int64_t D, int64_t M, double c_sigma,
                               int margin, int32_t *lo, int32_t *hi, cudaStream_t s)
{
    k_probe_edges<<<cdiv64(D, 256), 256, 0, s>>>(alpha2, D, M, c_sigma, margin, lo, hi);
    return cudaGetLastError();
}
cudaError_t launch_probe_values(const double *alpha2, int64_t D, Band b, cudaStream_t s)
{
    k_probe_values<<<(unsigned)D, 128, 0, s>>>(alpha2, b, const_cast<double *>(b.val));
    return cudaGetLastError();
}
cudaError_t launch_probe_rowsum(int64_t D, Band b, double *s_out, cudaStream_t s)
{
    k_probe_rowsum<<<(unsigned)D, 128, 0, s>>>(b, s_out);
    return cudaGetLastError();
}
cudaError_t launch_sqs_weights(int ntiles, int T, const int32_t *tile_dA, const int32_t *tile_dB,
                               int Ml, int64_t kb, Band b, const double *s, double gamma,
                               double *w, double *tstep, cudaStream_t st)
{
    (void)ntiles;
    k_sqs_weights<<<cdiv64(Ml, 128), 128, 0, st>>>(T, tile_dA, tile_dB, Ml, kb, b, s, gamma, w,
                                                   tstep);
    return cudaGetLastError();
}
cudaError_t launch_pow_fwd(int64_t D, Band b, const double *v, int64_t kb, double *q,
                           cudaStream_t s)
{
    k_pow_fwd<<<(unsigned)D, 128, 0, s>>>(b, v, kb, q);
    return cudaGetLastError();
}
cudaError_t launch_pow_bwd(int ntiles, int T, const int32_t *tile_dA, const int32_t *tile_dB,
                           int Ml, int64_t kb, Band b, const double *q, double *u,
                           cudaStream_t s)
{
    (void)ntiles;
    k_pow_bwd<<<cdiv64(Ml, 128), 128, 0, s>>>(T, tile_dA, tile_dB, Ml, kb, b, q, u);
    return cudaGetLastError();
}
cudaError_t launch_sumsq(const double *x, int64_t n, double *part, int nblk, cudaStream_t s)
{
    k_sumsq<<<nblk, 256, 0, s>>>(x, n, part);
    return cudaGetLastError();
}
cudaError_t launch_reduce_vec(const double *part, int nblk, int stride, int nvals, double *out,
                              cudaStream_t s)
{
    k_reduce_vec<<<1, 256, 0, s>>>(part, nblk, stride, nvals, out);
    return cudaGetLastError();
}
cudaError_t launch_scale(double *v, const double *u, const double *nrm2, int64_t n,
                         cudaStream_t s)
{
    k_scale<<<cdiv64(n, 256), 256, 0, s>>>(v, u, nrm2, n);
    return cudaGetLastError();
}
cudaError_t launch_fill(double *x, int64_t n, double v, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    k_fill<<<cdiv64(n, 256), 256, 0, s>>>(x, n, v);
    return cudaGetLastError();
}

// thread-shape selection: TC columns per thread, CG column groups, RG row groups
static int pick_shape(int N, int *CG, int *RG, int *TC)
{
    int tc = (N <= 32) ? 1 : (N <= 64) ? 2 : (N <= 100) ? 5 : (N <= 128) ? 4 : 8;
    int cg = (N + tc - 1) / tc;
    int rg = 256 / cg;
    if (rg > 8) rg = 8;
    if (rg < 1) rg = 1;
    *CG = cg;
    *RG = rg;
    *TC = tc;
    return ((cg * rg + 31) / 32) * 32;
}
int fwd_threads(int N, int *CG, int *RG, int *TC) { return pick_shape(N, CG, RG, TC); }
int bwd_threads(int N, int *CG, int *RG, int *TC) { return pick_shape(N, CG, RG, TC); }

size_t bwd_smem_bytes(int N, int RG, int KC, bool fista)
{
    int CG, RGx, TC;
    pick_shape(N, &CG, &RGx, &TC);
    const size_t T = (size_t)RG * TR;
    size_t el = (T + 2) * N * (fista ? 2 : 1) + T * N + 2 * (size_t)KC * T +
                2 * (((size_t)KC * N + (size_t)CG * TC + 1) & ~(size_t)1);
    return el * sizeof(double);
}
size_t fwd_smem_bytes(int N, int RG, int KR)
{
    int CG, RGx, TC;
    pick_shape(N, &CG, &RGx, &TC);
    const size_t KP = (size_t)RG * TR;
    size_t el = 2 * (((size_t)KR * N + (size_t)CG * TC + 1) & ~(size_t)1) + 2 * (size_t)KR * (KP + 2);
    return el * sizeof(double);
}

template <int TC>
static cudaError_t fwd_tc(const FwdArgs &a, int nunits, int nthr, size_t smem, cudaStream_t s)
{
    k_fwd<TC><<<nunits, nthr, smem, s>>>(a);
    return cudaGetLastError();
}

// opt every kernel with dynamic smem into the large carve-out (once, before any graph capture)
template <int TC, int VM>
static cudaError_t prep_bwd()
{
    const int big = 200 * 1024;
    cudaError_t e = cudaFuncSetAttribute(k_bwd<TC, BWD_STEP, false, VM>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_bwd<TC, BWD_STEP, true, VM>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_bwd<TC, BWD_GRAD, false, VM>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_bwd<TC, BWD_EVAL, false, VM>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_bwd<TC, BWD_EVAL, true, VM>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    return e;
}
template <int TC>
static cudaError_t prep_tc()
{
    const int big = 200 * 1024;
    cudaError_t e = cudaFuncSetAttribute(k_fwd<TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess) e = prep_bwd<TC, 4>();
    if (e == cudaSuccess) e = prep_bwd<TC, 8>();
    if (e == cudaSuccess) e = prep_bwd<TC, 13>();
    if (e == cudaSuccess) e = prep_bwd<TC, 16>();
    if (e == cudaSuccess) e = prep_bwd<TC, 0>();
    return e;
}
int device_sm_count()
{
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
    return cache[dev] > 0 ? cache[dev] : 148;
}

cudaError_t prepare_kernels()
{
    // the shared-memory attribute is per device: prepare each device ordinal once
    static uint64_t done_mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0;
    if (done_mask & bit) return cudaSuccess;
    bool done = false;
    cudaError_t e = prep_tc<1>();
    if (e == cudaSuccess) e = prep_tc<2>();
    if (e == cudaSuccess) e = prep_tc<4>();
    if (e == cudaSuccess) e = prep_tc<5>();
    if (e == cudaSuccess) e = prep_tc<8>();
    done = e == cudaSuccess;
    if (done) done_mask |= bit;
    return e;
}

cudaError_t launch_fwd(const FwdArgs &a, int nunits, int TC, cudaStream_t s, size_t *smem_out)
{
    if (nunits <= 0) return cudaSuccess;
    const int nthr = ((a.CG * a.RG + 31) / 32) * 32;
    const size_t smem = fwd_smem_bytes(a.N, a.RG, a.KR);
    if (smem_out) *smem_out = smem;
    switch (TC) {
        case 1: return fwd_tc<1>(a, nunits, nthr, smem, s);
        case 2: return fwd_tc<2>(a, nunits, nthr, smem, s);
        case 4: return fwd_tc<4>(a, nunits, nthr, smem, s);
        case 5: return fwd_tc<5>(a, nunits, nthr, smem, s);
        case 8: return fwd_tc<8>(a, nunits, nthr, smem, s);
    }
    return cudaErrorInvalidValue;
}

template <int TC, int MODE, bool FISTA>
static cudaError_t bwd_tcm(const BwdArgs &a, int nunits, int nthr, size_t smem, cudaStream_t s)
{
    const int vpl = (a.N + a.SEG - 1) / a.SEG;
    if (vpl <= 4)
        k_bwd<TC, MODE, FISTA, 4><<<nunits, nthr, smem, s>>>(a);
    else if (vpl <= 8)
        k_bwd<TC, MODE, FISTA, 8><<<nunits, nthr, smem, s>>>(a);
    else if (vpl <= 13)
        k_bwd<TC, MODE, FISTA, 13><<<nunits, nthr, smem, s>>>(a);
    else if (vpl <= 16)
        k_bwd<TC, MODE, FISTA, 16><<<nunits, nthr, smem, s>>>(a);
    else
        k_bwd<TC, MODE, FISTA, 0><<<nunits, nthr, smem, s>>>(a);
    return cudaGetLastError();
}

template <int TC>
static cudaError_t bwd_tc(const BwdArgs &a, int nunits, int mode, int nthr, size_t smem,
                          cudaStream_t s)
{
    const bool fista = a.beta != nullptr;
    switch (mode) {
        case BWD_STEP:
            return fista ? bwd_tcm<TC, BWD_STEP, true>(a, nunits, nthr, smem, s)
                         : bwd_tcm<TC, BWD_STEP, false>(a, nunits, nthr, smem, s);
        case BWD_GRAD: return bwd_tcm<TC, BWD_GRAD, false>(a, nunits, nthr, smem, s);
        case BWD_EVAL:
            return fista ? bwd_tcm<TC, BWD_EVAL, true>(a, nunits, nthr, smem, s)
                         : bwd_tcm<TC, BWD_EVAL, false>(a, nunits, nthr, smem, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_bwd(const BwdArgs &a, int nunits, int TC, int mode, cudaStream_t s)
{
    if (nunits <= 0) return cudaSuccess;
    const int nthr = ((a.CG * a.RG + 31) / 32) * 32;
    // EVAL in FISTA mode uses the FISTA smem layout only for the kkt_every gate; Theta_{k-1}
    // is not read there (beta = 0), so the plain layout suffices.
    const bool fista_layout = a.beta != nullptr && mode == BWD_STEP;
    const size_t smem = bwd_smem_bytes(a.N, a.RG, a.KC, fista_layout || a.beta != nullptr);
    switch (TC) {
        case 1: return bwd_tc<1>(a, nunits, mode, nthr, smem, s);
        case 2: return bwd_tc<2>(a, nunits, mode, nthr, smem, s);
        case 4: return bwd_tc<4>(a, nunits, mode, nthr, smem, s);
        case 5: return bwd_tc<5>(a, nunits, mode, nthr, smem, s);
        case 8: return bwd_tc<8>(a, nunits, mode, nthr, smem, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_reduce_R(const double *rpart, const int64_t *red_beg, const int64_t *red_rows,
                            const double *P, double *R, int64_t D, int N, double *partR,
                            int nblk, const DevState *st, cudaStream_t s)
{
    k_reduce_R<<<nblk, 256, 0, s>>>(rpart, red_beg, red_rows, P, R, D, N, partR, st);
    return cudaGetLastError();
}
// ---- in-process collective (virtual ranks, SURVEY 4 "virtual shard"): out = sum of the ranks'
// buffers in rank order (every rank computes the same sum in the same order: replicated results
// are bitwise identical, as after an allreduce)
__global__ void k_vsum(VPtrs v, int n_ranks, int64_t n, double *out)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        double s = v.p[0][e];
        for (int r = 1; r < n_ranks; r++) s += v.p[r][e];
        out[e] = s;
    }
}
cudaError_t launch_vsum(const VPtrs &v, int n_ranks, int64_t n, double *out, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 4 * 148);
    k_vsum<<<grid, 256, 0, s>>>(v, n_ranks, n, out);
    return cudaGetLastError();
}

// ---- band-aware residual exchange: rank g touches the probes
// [bx.dlo[g], bx.dhi[g]) (contiguous: band edges are monotone); probe d is summed over the ranks
// S(d) = {q : dlo[q] <= d < dhi[q]} (contiguous) in rank order, its own partial from R and a
// peer's from src[q] (rows from bx.start[q]); then P is subtracted.  ||R||^2 partials count each
// probe once, on its owner min S(d).  Warp per probe; block partial to partR[blockIdx.x].
__global__ void __launch_bounds__(256) k_band_combine(BandX bx, int rank, int nranks, const double *P, double *R,
                                                      int N, double *partR, const DevState *st)
{
    __shared__ double red[8];
    if (st && st->stop) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double ss = 0.0;
    for (int64_t d = bx.dlo[rank] + (int64_t)blockIdx.x * 8 + warp; d < bx.dhi[rank]; d += (int64_t)gridDim.x * 8) {
        int qa = rank, qb = rank;
        while (qa > 0 && d >= bx.dlo[qa - 1] && d < bx.dhi[qa - 1]) qa--;
        while (qb + 1 < nranks && d >= bx.dlo[qb + 1] && d < bx.dhi[qb + 1]) qb++;
        const bool own = qa == rank;
        for (int n = lane; n < N; n += 32) {
            double v = 0.0;
            for (int q = qa; q <= qb; q++)
                v += (q == rank) ? R[d * N + n] : bx.src[q][(d - bx.start[q]) * N + n];
            v -= P[d * N + n];
            R[d * N + n] = v;
            if (own) ss = fma(v, v, ss);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < 8; w++) v += red[w];
        partR[blockIdx.x] = v;
    }
}
cudaError_t launch_band_combine(const BandX &bx, int rank, int nranks, const double *P, double *R, int N,
                                double *partR, int nblk, const DevState *st, cudaStream_t s)
{
    k_band_combine<<<nblk, 256, 0, s>>>(bx, rank, nranks, P, R, N, partR, st);
    return cudaGetLastError();
}

cudaError_t launch_sub_p_sumsq(double *R, const double *P, int64_t n, double *partR, int nblk,
                               const DevState *st, cudaStream_t s)
{
    k_sub_p_sumsq<<<nblk, 256, 0, s>>>(R, P, n, partR, st);
    return cudaGetLastError();
}
cudaError_t launch_scalars_local(const double *partR, int nblkR, const double *partT,
                                 int ntiles, int include_r2, double *vec, const DevState *st,
                                 cudaStream_t s)
{
    k_scalars_local<<<1, 256, 0, s>>>(partR, nblkR, partT, ntiles, include_r2, vec, st);
    return cudaGetLastError();
}
cudaError_t launch_finalize(const double *vec, int64_t N, int64_t M, double gamma, double tol,
                            int final_eval, int kkt_every, double *trace, double *kkt,
                            double *kktp, int64_t trace_len, DevState *st, cudaStream_t s)
{
    k_finalize<<<1, 32, 0, s>>>(vec, N, M, gamma, tol, final_eval, kkt_every, trace, kkt, kktp,
                                trace_len, st);
    return cudaGetLastError();
}
cudaError_t launch_project_rows(const double *X, int64_t M, int N, double *Y, cudaStream_t s)
{
    k_project_rows<<<cdiv64(M * 32, 256), 256, 0, s>>>(X, M, N, Y);
    return cudaGetLastError();
}
cudaError_t launch_fista_rcomb(double *RY, const double *Rk, const double *Rkm1,
                               const double *beta, int64_t n, const DevState *st,
                               cudaStream_t s)
{
    k_fista_rcomb<<<cdiv64(n, 256), 256, 0, s>>>(RY, Rk, Rkm1, beta, n, st);
    return cudaGetLastError();
}

}  // namespace qdt
