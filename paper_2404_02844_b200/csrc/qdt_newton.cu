// qdt_newton.cu -- element and row kernels of the two-stage two-metric projected truncated
// Newton solve (reading R16).  The Hessian
// products H d = 2 (F^T F d + gamma L d) reuse the forward (k_fwd_mma / k_fwd) and gradient
// (k_bwd, BWD_GRAD) kernels; these kernels add the metric, the CG vector updates, the arc
// derivatives, the line-search arcs and the fixed-order reductions (no atomics in any sum:
// fixed grid, fixed per-thread order, fixed tree, then one block over the block partials).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "qdt_internal.h"

namespace qdt {

constexpr int NT_THR = 256;

__device__ __forceinline__ double nt_wsum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double nt_wmin(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// block-wide fixed-order sum of K values per thread -> part[blockIdx.x * K + j]
template <int K>
__device__ __forceinline__ void nt_block_store(double (&v)[K], double *part)
{
    __shared__ double red[K][NT_THR / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < K; j++) {
        const double w = nt_wsum(v[j]);
        if (lane == 0) red[j][warp] = w;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double s = 0.0;
        for (int w = 0; w < NT_THR / 32; w++) s += red[threadIdx.x][w];
        part[(int64_t)blockIdx.x * K + threadIdx.x] = s;
    }
}

// sum of K-vectors of block partials (one warp, fixed order) -> out[0..K)
__global__ void k_nt_final(const double *part, int nblk, int K, double *out)
{
    const int lane = threadIdx.x;
    for (int j = 0; j < K; j++) {
        double s = 0.0;
        for (int b = lane; b < nblk; b += 32) s += part[(int64_t)b * K + j];
        s = nt_wsum(s);
        if (lane == 0) out[j] = s;
    }
}

// PCG set-up (stage 1: m == nullptr; stage 2: row maxima m, fixed entries n = m(i)):
// gr = df (stage 2: df_in - df_{i,m(i)}), act = theta <= eps && gr > 0, b = -gr,
// x = b / hd on act, r = b on the free set, z = r / hd, d = z  (hd = h_i, stage 2: 2 h_i)
__global__ void k_nt_pcg_init(const double *g, const double *theta, const double *h, const int32_t *m,
                              int N, int64_t n, double eps, double *gr, uint8_t *act, double *x, double *r,
                              double *z, double *d, double *part)
{
    double v[1] = {0.0};   // ||r||^2 partial
    for (int64_t i = (int64_t)blockIdx.x * NT_THR + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT_THR) {
        const int64_t k = i / N;
        const int c = (int)(i - k * N);
        const double hd = m ? 2.0 * h[k] : h[k];
        const bool fixed = m && c == m[k];
        const double gi = fixed ? 0.0 : (m ? g[i] - g[k * N + m[k]] : g[i]);
        const bool a = !fixed && theta[i] <= eps && gi > 0.0;
        const double b = fixed ? 0.0 : -gi;
        gr[i] = gi;
        act[i] = a ? 1 : 0;
        x[i] = (a && hd > 0.0) ? b / hd : 0.0;
        const double ri = (!fixed && !a) ? b : 0.0;
        r[i] = ri;
        const double zi = hd > 0.0 ? ri / hd : 0.0;
        z[i] = zi;
        d[i] = zi;
        v[0] += ri * ri;
    }
    nt_block_store<1>(v, part);
}

// dots: mode 0: a.b; mode 1: a.b skipping act; mode 2 (stage-2 arc slope): sum gr p' with
// p' = 0 where theta <= 0 and p < 0
__global__ void k_nt_dot(const double *a, const double *b, const uint8_t *act, const double *theta, int mode,
                         int64_t n, double *part)
{
    double v[1] = {0.0};
    for (int64_t i = (int64_t)blockIdx.x * NT_THR + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT_THR) {
        double bi = b[i];
        if (mode == 1 && act[i]) bi = 0.0;
        if (mode == 2 && theta[i] <= 0.0 && bi < 0.0) bi = 0.0;
        v[0] += a[i] * bi;
    }
    nt_block_store<1>(v, part);
}

// sum_i g_i (T_i - Theta_i) over the variables (stage 2: n != m(i))
__global__ void k_nt_dotdiff(const double *g, const double *T, const double *theta, const int32_t *m, int N,
                             int64_t n, double *part)
{
    double v[1] = {0.0};
    for (int64_t i = (int64_t)blockIdx.x * NT_THR + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT_THR) {
        const int64_t k = i / N;
        if (m && (int)(i - k * N) == m[k]) continue;
        v[0] += g[i] * (T[i] - theta[i]);
    }
    nt_block_store<1>(v, part);
}

__global__ void k_nt_scale_mask(double *x, const uint8_t *act, double s, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * NT_THR + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT_THR)
        x[i] = (act && act[i]) ? 0.0 : s * x[i];
}

// x += a d, r -= a Hd, z = r / hd; partials ||r||^2, r.z
__global__ void k_nt_cg_update(double *x, double *r, double *z, const double *d, const double *Hd, double a,
                               const double *h, const int32_t *m, int N, int64_t n, double *part)
{
    double v[2] = {0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * NT_THR + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT_THR) {
        const int64_t k = i / N;
        const double hd = m ? 2.0 * h[k] : h[k];
        x[i] += a * d[i];
        const double ri = r[i] - a * Hd[i];
        r[i] = ri;
        const double zi = hd > 0.0 ? ri / hd : 0.0;
        z[i] = zi;
        v[0] += ri * ri;
        v[1] += ri * zi;
    }
    nt_block_store<2>(v, part);
}

__global__ void k_nt_cg_dir(double *d, const double *z, double beta, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * NT_THR + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT_THR)
        d[i] = z[i] + beta * d[i];
}

// stage 2 expansion u = Z v: u_in = v_in (n != m), u_im = -sum_{n != m} v_in  (warp per row)
__global__ void k_nt_zexp(const double *v, const int32_t *m, int64_t M, int N, double *u)
{
    const int lane = threadIdx.x & 31;
    const int64_t k = (int64_t)blockIdx.x * (NT_THR / 32) + (threadIdx.x >> 5);
    if (k >= M) return;
    const int mk = m[k];
    double s = 0.0;
    for (int c = lane; c < N; c += 32)
        if (c != mk) {
            const double x = v[k * N + c];
            u[k * N + c] = x;
            s += x;
        }
    s = nt_wsum(s);
    if (lane == 0) u[k * N + mk] = -s;
}

// stage 2 reduction Z^T w: out_in = w_in - w_im (n != m), out_im = 0; then 0 on act
__global__ void k_nt_zred(double *w, const int32_t *m, const uint8_t *act, int64_t M, int N)
{
    const int lane = threadIdx.x & 31;
    const int64_t k = (int64_t)blockIdx.x * (NT_THR / 32) + (threadIdx.x >> 5);
    if (k >= M) return;
    const int mk = m[k];
    const double wm = w[k * N + mk];
    __syncwarp();
    for (int c = lane; c < N; c += 32) {
        const int64_t i = k * N + c;
        w[i] = (c == mk || act[i]) ? 0.0 : w[i] - wm;
    }
}

// stage 1 arc derivative: d0 = projection of p onto the simplex tangent cone at theta (row):
// d0_j = p_j - mu on the support, max(p_j - mu, 0) on the zeros; mu by Michelot rounds from the
// lower bound sf / nf (h(mu) = sf - nf mu + sum_zeros max(p - mu, 0) is >= 0 there)
__global__ void k_nt_tangent(const double *theta, const double *p, int64_t M, int N, double *d0)
{
    const int lane = threadIdx.x & 31;
    const int64_t k = (int64_t)blockIdx.x * (NT_THR / 32) + (threadIdx.x >> 5);
    if (k >= M) return;
    const double *th = theta + k * N, *pr = p + k * N;
    double sf = 0.0;
    int nf = 0;
    for (int c = lane; c < N; c += 32)
        if (th[c] > 0.0) {
            sf += pr[c];
            nf++;
        }
    sf = nt_wsum(sf);
    for (int o = 16; o > 0; o >>= 1) nf += __shfl_xor_sync(0xffffffffu, nf, o);
    double mu;
    if (nf == 0) {
        mu = -INFINITY;
    } else {
        mu = sf / (double)nf;
        int cnt = -1;
        for (int round = 0; round <= N; round++) {
            double s = 0.0;
            int a = 0;
            for (int c = lane; c < N; c += 32)
                if (!(th[c] > 0.0) && pr[c] > mu) {
                    s += pr[c];
                    a++;
                }
            s = nt_wsum(s);
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (a == cnt) break;
            cnt = a;
            mu = (sf + s) / (double)(nf + a);
        }
    }
    for (int c = lane; c < N; c += 32) {
        const double v = pr[c] - mu;
        d0[k * N + c] = (th[c] > 0.0) ? v : (v > 0.0 ? v : 0.0);
    }
}

// X = theta + a p
__global__ void k_nt_axpy(const double *theta, const double *p, double a, int64_t n, double *X)
{
    for (int64_t i = (int64_t)blockIdx.x * NT_THR + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT_THR)
        X[i] = theta[i] + a * p[i];
}

// stage 2 arc: T_in = max(theta_in + a p_in, 0) (n != m), T_im = 1 - sum; *neg = 1 if any T_im < 0
__global__ void k_nt_clamp_arc(const double *theta, const double *p, double a, const int32_t *m, int64_t M,
                               int N, double *T, int *neg)
{
    const int lane = threadIdx.x & 31;
    const int64_t k = (int64_t)blockIdx.x * (NT_THR / 32) + (threadIdx.x >> 5);
    if (k >= M) return;
    const int mk = m[k];
    double s = 0.0;
    for (int c = lane; c < N; c += 32)
        if (c != mk) {
            double v = theta[k * N + c] + a * p[k * N + c];
            v = v > 0.0 ? v : 0.0;
            T[k * N + c] = v;
            s += v;
        }
    s = nt_wsum(s);
    if (lane == 0) {
        const double tm = 1.0 - s;
        T[k * N + mk] = tm;
        if (tm < 0.0) *neg = 1;
    }
}

// transformation step (Alg. 1): m(i) = first argmax of row i; theta_{i,m} = 1 - sum_{n != m}
__global__ void k_nt_transform(double *theta, int64_t M, int N, int32_t *m)
{
    const int lane = threadIdx.x & 31;
    const int64_t k = (int64_t)blockIdx.x * (NT_THR / 32) + (threadIdx.x >> 5);
    if (k >= M) return;
    double *th = theta + k * N;
    double bv = -INFINITY;
    int bi = N;
    for (int c = lane; c < N; c += 32)
        if (th[c] > bv) {
            bv = th[c];
            bi = c;
        }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    double s = 0.0;
    for (int c = lane; c < N; c += 32)
        if (c != bi) s += th[c];
    s = nt_wsum(s);
    __syncwarp();
    if (lane == 0) {
        th[bi] = 1.0 - s;
        m[k] = bi;
    }
}

// f parts: sum R^2 (D x N), sum of regulariser pairs (rows k, k+1 < M); KKT sums (R7 and the
// paper's clamped multiplier) from df = g (warp per Fock row)
__global__ void k_nt_sumsq(const double *R, int64_t n, double *part)
{
    double v[1] = {0.0};
    for (int64_t i = (int64_t)blockIdx.x * NT_THR + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT_THR)
        v[0] += R[i] * R[i];
    nt_block_store<1>(v, part);
}

__global__ void k_nt_rowstats(const double *theta, const double *g, int64_t M, int N, double *part)
{
    const int lane = threadIdx.x & 31;
    double v[3] = {0.0, 0.0, 0.0};   // regulariser pairs, KKT (unclamped), KKT (clamped)
    for (int64_t k = (int64_t)blockIdx.x * (NT_THR / 32) + (threadIdx.x >> 5); k < M;
         k += (int64_t)gridDim.x * (NT_THR / 32)) {
        double mn = INFINITY;
        if (g)
            for (int c = lane; c < N; c += 32) mn = fmin(mn, g[k * N + c]);
        mn = nt_wmin(mn);
        const double lam = -mn, lamp = lam > 0.0 ? lam : 0.0;
        for (int c = lane; c < N; c += 32) {
            const double t = theta[k * N + c];
            if (k + 1 < M) {
                const double dd = t - theta[(k + 1) * N + c];
                v[0] += dd * dd;
            }
            if (g) {
                const double df = g[k * N + c];
                const double a = t * (df + lam), b = t * (df + lamp);
                v[1] += a * a;
                v[2] += b * b;
            }
        }
    }
    nt_block_store<3>(v, part);
}

// Hessian diagonal per Fock row, h_k = 2 (sum_d F_{d,k}^2 + gamma L_kk) (Table 1),
// from the tiled F (64 rows x 4 probe slices per tile, slices combined in a fixed order)
__global__ void __launch_bounds__(256) k_nt_hdiag(int Ml, int64_t kb, int64_t M, const int32_t *tile_dA,
                                                  const int32_t *tile_dB, const int64_t *fb_off, const double *Fb,
                                                  double gamma, double *h)
{
    __shared__ double part[4][ST];
    const int t = blockIdx.x, r = threadIdx.x & (ST - 1), q = threadIdx.x >> 6;
    const int dA = tile_dA[t], W = tile_dB[t] - dA;
    const double *f = Fb + fb_off[t] + r;
    double acc = 0.0;
    for (int j = q; j < W; j += 4) {
        const double v = f[(int64_t)j * STP];
        acc += v * v;
    }
    part[q][r] = acc;
    __syncthreads();
    const int k = t * ST + r;
    if (q || k >= Ml) return;
    const int64_t kg = kb + k;
    const double lkk = M > 1 ? (double)((kg > 0) + (kg < M - 1)) : 0.0;
    h[k] = 2.0 * (((part[0][r] + part[1][r]) + (part[2][r] + part[3][r])) + gamma * lkk);
}

// ---------------------------------------------------------------------------- launchers
cudaError_t nt_hdiag(int ntiles, int Ml, int64_t kb, int64_t M, const int32_t *tile_dA, const int32_t *tile_dB,
                     const int64_t *fb_off, const double *Fb, double gamma, double *h, cudaStream_t s)
{
    if (ntiles <= 0) return cudaSuccess;
    k_nt_hdiag<<<ntiles, 4 * ST, 0, s>>>(Ml, kb, M, tile_dA, tile_dB, fb_off, Fb, gamma, h);
    return cudaGetLastError();
}

static inline int nt_grid(int64_t n) { return (int)std::min<int64_t>(NT_BLK, (n + NT_THR - 1) / NT_THR); }
static inline int nt_rows(int64_t M) { return (int)((M + NT_THR / 32 - 1) / (NT_THR / 32)); }

cudaError_t nt_pcg_init(const double *g, const double *theta, const double *h, const int32_t *m, int N,
                        int64_t n, double eps, double *gr, uint8_t *act, double *x, double *r, double *z, double *d,
                        double *part, double *out, cudaStream_t s)
{
    const int G = nt_grid(n);
    k_nt_pcg_init<<<G, NT_THR, 0, s>>>(g, theta, h, m, N, n, eps, gr, act, x, r, z, d, part);
    k_nt_final<<<1, 32, 0, s>>>(part, G, 1, out);
    return cudaGetLastError();
}

cudaError_t nt_dot(const double *a, const double *b, const uint8_t *act, const double *theta, int mode, int64_t n,
                   double *part, double *out, cudaStream_t s)
{
    const int G = nt_grid(n);
    k_nt_dot<<<G, NT_THR, 0, s>>>(a, b, act, theta, mode, n, part);
    k_nt_final<<<1, 32, 0, s>>>(part, G, 1, out);
    return cudaGetLastError();
}

cudaError_t nt_dotdiff(const double *g, const double *T, const double *theta, const int32_t *m, int N, int64_t n,
                       double *part, double *out, cudaStream_t s)
{
    const int G = nt_grid(n);
    k_nt_dotdiff<<<G, NT_THR, 0, s>>>(g, T, theta, m, N, n, part);
    k_nt_final<<<1, 32, 0, s>>>(part, G, 1, out);
    return cudaGetLastError();
}

cudaError_t nt_scale_mask(double *x, const uint8_t *act, double sc, int64_t n, cudaStream_t s)
{
    k_nt_scale_mask<<<nt_grid(n), NT_THR, 0, s>>>(x, act, sc, n);
    return cudaGetLastError();
}

cudaError_t nt_cg_update(double *x, double *r, double *z, const double *d, const double *Hd, double a,
                         const double *h, const int32_t *m, int N, int64_t n, double *part, double *out,
                         cudaStream_t s)
{
    const int G = nt_grid(n);
    k_nt_cg_update<<<G, NT_THR, 0, s>>>(x, r, z, d, Hd, a, h, m, N, n, part);
    k_nt_final<<<1, 32, 0, s>>>(part, G, 2, out);
    return cudaGetLastError();
}

cudaError_t nt_cg_dir(double *d, const double *z, double beta, int64_t n, cudaStream_t s)
{
    k_nt_cg_dir<<<nt_grid(n), NT_THR, 0, s>>>(d, z, beta, n);
    return cudaGetLastError();
}

cudaError_t nt_zexp(const double *v, const int32_t *m, int64_t M, int N, double *u, cudaStream_t s)
{
    k_nt_zexp<<<nt_rows(M), NT_THR, 0, s>>>(v, m, M, N, u);
    return cudaGetLastError();
}

cudaError_t nt_zred(double *w, const int32_t *m, const uint8_t *act, int64_t M, int N, cudaStream_t s)
{
    k_nt_zred<<<nt_rows(M), NT_THR, 0, s>>>(w, m, act, M, N);
    return cudaGetLastError();
}

cudaError_t nt_tangent(const double *theta, const double *p, int64_t M, int N, double *d0, cudaStream_t s)
{
    k_nt_tangent<<<nt_rows(M), NT_THR, 0, s>>>(theta, p, M, N, d0);
    return cudaGetLastError();
}

cudaError_t nt_axpy(const double *theta, const double *p, double a, int64_t n, double *X, cudaStream_t s)
{
    k_nt_axpy<<<nt_grid(n), NT_THR, 0, s>>>(theta, p, a, n, X);
    return cudaGetLastError();
}

cudaError_t nt_clamp_arc(const double *theta, const double *p, double a, const int32_t *m, int64_t M, int N,
                         double *T, int *neg, cudaStream_t s)
{
    k_nt_clamp_arc<<<nt_rows(M), NT_THR, 0, s>>>(theta, p, a, m, M, N, T, neg);
    return cudaGetLastError();
}

cudaError_t nt_transform(double *theta, int64_t M, int N, int32_t *m, cudaStream_t s)
{
    k_nt_transform<<<nt_rows(M), NT_THR, 0, s>>>(theta, M, N, m);
    return cudaGetLastError();
}

cudaError_t nt_fparts(const double *R, int64_t nR, const double *theta, const double *g, int64_t M, int N,
                      double *part, double *out, cudaStream_t s)
{
    const int G1 = nt_grid(nR);
    k_nt_sumsq<<<G1, NT_THR, 0, s>>>(R, nR, part);
    k_nt_final<<<1, 32, 0, s>>>(part, G1, 1, out);
    if (theta) {
        const int G2 = (int)std::min<int64_t>(NT_BLK, nt_rows(M));
        k_nt_rowstats<<<G2, NT_THR, 0, s>>>(theta, g, M, N, part + NT_BLK);
        k_nt_final<<<1, 32, 0, s>>>(part + NT_BLK, G2, 3, out + 1);
    }
    return cudaGetLastError();
}

}  // namespace qdt
