/*
 * qdt_oracle.c -- CPU ORACLE for the phase-insensitive detector-tomography hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2404_02844_b200/) never imports, links or calls anything in oracle/, and this
 * file shares no code, header, table or helper with it.
 *
 * Plain, slow, obviously-correct fp64 C: one thread, straight loops, no blocking,
 * no fusion, built with -O2 -ffp-contract=off.  Every function cites the passage of
 * /root/reference/PAPER.md (PAPER.md:<line>, section / equation) it follows, or the
 * reading in DESIGN.md ("Readings") where the paper is silent.
 *
 * Notation: Theta = Pi (M x N, row-major, row k = Fock level,
 * column n = outcome); F (D x M) coherent-probe matrix, eq. Fmatrix PAPER.md:107-109;
 * P (D x N) outcome probabilities, eq. Matrix PAPER.md:48-50.
 *
 * Parity status of every function is listed in DESIGN.md section "Oracle pins".
 *
 * Scalar reductions over whole matrices (||R||_F^2, the regulariser sum, the KKT sums,
 * power-iteration norms) accumulate in x87 extended precision: a plain double running sum
 * of 10^7 - 10^8 nonnegative terms carries a biased rounding error (measured 5e-10 relative
 * on the Large config) that would exceed the objective gate of reading R5.
 *
 * Threads (oracle-MT): the file builds with OpenMP.  Work is split only where
 * the split leaves every floating-point operation and its order unchanged -- a probe row of
 * F Theta, a block of Fock rows of F^T R (each element still sums over probes d in increasing
 * order), elementwise and per-row work -- and every scalar reduction is summed in a FIXED chunk
 * order (OR_CHUNK elements / OR_RCHUNK rows per chunk, chunk partials in extended precision,
 * then added in chunk order) that does not depend on the thread count.  So the result is
 * bit-identical for any number of threads (tests/test_oracle_mt.py); or_set_threads(1) is the
 * single-thread parity reference.
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_CHUNK 8192   /* elements per partial sum of a flat reduction */
#define OR_RCHUNK 64    /* rows per partial sum of a row-structured reduction */
#define OR_RB 256       /* Fock rows per block of the backward product */

void or_set_threads(int n)
{
#ifdef _OPENMP
    omp_set_num_threads(n > 0 ? n : omp_get_num_procs());
#else
    (void)n;
#endif
}

int or_get_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* sum_i x_i^2 in fixed chunks (chunk partials in extended precision, added in chunk order) */
static double sumsq(const double *x, int64_t n)
{
    const int64_t nc = (n + OR_CHUNK - 1) / OR_CHUNK;
    long double *part = (long double *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(long double));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nc; c++) {
        long double s = 0.0L;
        const int64_t e = (c + 1) * OR_CHUNK < n ? (c + 1) * OR_CHUNK : n;
        for (int64_t i = c * OR_CHUNK; i < e; i++) s += (long double)(x[i] * x[i]);
        part[c] = s;
    }
    long double t = 0.0L;
    for (int64_t c = 0; c < nc; c++) t += part[c];
    free(part);
    return (double)t;
}

/* sum_i (a_i - b_i)^2, same chunking */
static double sumsq_diff(const double *a, const double *b, int64_t n)
{
    const int64_t nc = (n + OR_CHUNK - 1) / OR_CHUNK;
    long double *part = (long double *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(long double));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nc; c++) {
        long double s = 0.0L;
        const int64_t e = (c + 1) * OR_CHUNK < n ? (c + 1) * OR_CHUNK : n;
        for (int64_t i = c * OR_CHUNK; i < e; i++) {
            const double d = a[i] - b[i];
            s += (long double)(d * d);
        }
        part[c] = s;
    }
    long double t = 0.0L;
    for (int64_t c = 0; c < nc; c++) t += part[c];
    free(part);
    return (double)t;
}

/* sum_i a_i b_i in extended precision, same chunking */
static double dotl(const double *a, const double *b, int64_t n)
{
    const int64_t nc = (n + OR_CHUNK - 1) / OR_CHUNK;
    long double *part = (long double *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(long double));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nc; c++) {
        long double s = 0.0L;
        const int64_t e = (c + 1) * OR_CHUNK < n ? (c + 1) * OR_CHUNK : n;
        for (int64_t i = c * OR_CHUNK; i < e; i++) s += (long double)a[i] * (long double)b[i];
        part[c] = s;
    }
    long double t = 0.0L;
    for (int64_t c = 0; c < nc; c++) t += part[c];
    free(part);
    return (double)t;
}

#define OR_OK 0
#define OR_EINVAL 1

/* ------------------------------------------------------------------------------------
 * Band of a probe row (reading R1; "Only the relevant non-zero
 * blocks of F are stored", "a sparse storage of F").
 *   s = sqrt(mu);  lo = max(0, floor(mu - c*s));  hi = min(M-1, ceil(mu + c*s) + margin)
 *   mu == 0 (vacuum probe): the single entry k = 0.
 * Every operation is one IEEE round-to-nearest operation (no FMA contraction: this file
 * is compiled with -ffp-contract=off).
 * ---------------------------------------------------------------------------------- */
void or_band(double mu, int64_t M, double c_sigma, int64_t margin, int64_t *lo, int64_t *hi)
{
    if (mu == 0.0) {
        *lo = 0;
        *hi = 0;
        return;
    }
    double s = sqrt(mu);
    double cs = c_sigma * s;
    double a = mu - cs;
    double b = mu + cs;
    double l = floor(a);
    double h = ceil(b) + (double)margin;
    int64_t L = (l < 0.0) ? 0 : (int64_t)l;
    int64_t H = (h > (double)(M - 1)) ? (M - 1) : (int64_t)h;
    if (L > M - 1) L = M - 1; /* probe mean beyond the cutoff: keep the last row */
    if (H < L) H = L;
    *lo = L;
    *hi = H;
}

/* ------------------------------------------------------------------------------------
 * F_{d,i} = |alpha_d|^{2i} e^{-|alpha_d|^2} / i!     (eq. Fmatrix)
 * The definition written out in log space, ln F = i ln mu - mu - ln Gamma(i+1), evaluated
 * in IEEE binary128 (libquadmath, 113-bit significand) so that the final rounding to
 * double dominates the error; the exponential of the (small, |ln F| < ~40) binary128
 * logarithm is taken in x87 extended precision.
 * ---------------------------------------------------------------------------------- */
static double pmf_from_log(__float128 l) { return (double)expl((long double)l); }

double or_poisson_pmf(int64_t i, double mu)
{
    if (mu == 0.0) return (i == 0) ? 1.0 : 0.0;
    __float128 l = (__float128)i * logq((__float128)mu) - (__float128)mu
                   - lgammaq((__float128)i + 1);
    return pmf_from_log(l);
}

/* Banded F construction: row d stored as (lo[d], len[d], values at off[d] .. off[d]+len-1)
 * (probe-major; PAPER.md:257 + DESIGN.md R1).  Two-phase: call with val == NULL to get the
 * band tables and nnz = off[D]; then call again with val of size nnz.  ln Gamma(i+1) is
 * tabulated once per call (binary128) for the rows that bands touch. */
int or_build_probes(const double *alpha2, int64_t D, int64_t M, double c_sigma, int64_t margin,
                    int64_t *lo, int64_t *len, int64_t *off, double *val)
{
    if (D < 1 || M < 1) return OR_EINVAL;
    off[0] = 0;
    int64_t kmax = 0;
    for (int64_t d = 0; d < D; d++) {
        int64_t l, h;
        or_band(alpha2[d], M, c_sigma, margin, &l, &h);
        lo[d] = l;
        len[d] = h - l + 1;
        off[d + 1] = off[d] + len[d];
        if (h > kmax) kmax = h;
    }
    if (val) {
        __float128 *lg = (__float128 *)malloc((size_t)(kmax + 1) * sizeof(__float128));
        char *have = (char *)calloc((size_t)(kmax + 1), 1);
        for (int64_t d = 0; d < D; d++)
            for (int64_t j = 0; j < len[d]; j++)
                if (!have[lo[d] + j]) {
                    lg[lo[d] + j] = lgammaq((__float128)(lo[d] + j) + 1);
                    have[lo[d] + j] = 1;
                }
        for (int64_t d = 0; d < D; d++) {
            double mu = alpha2[d];
            if (mu == 0.0) {
                for (int64_t j = 0; j < len[d]; j++) val[off[d] + j] = (lo[d] + j == 0) ? 1.0 : 0.0;
                continue;
            }
            __float128 lm = logq((__float128)mu);
            for (int64_t j = 0; j < len[d]; j++) {
                int64_t i = lo[d] + j;
                val[off[d] + j] = pmf_from_log((__float128)i * lm - (__float128)mu - lg[i]);
            }
        }
        free(lg);
        free(have);
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------------------
 * Euclidean projection onto the probability simplex S = {y : y >= 0, sum y = 1}
 * ("the point closest to x that is on S").  The paper uses Condat's
 * algorithm; the oracle uses the textbook sort-based method, which gives
 * the same projection (reading R4):
 *   u = x sorted descending;  rho = max{ j : u_j > (sum_{i<=j} u_i - 1)/j };
 *   tau = (sum_{i<=rho} u_i - 1)/rho;   y = max(x - tau, 0).
 * ---------------------------------------------------------------------------------- */
static int cmp_desc(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return (x < y) - (x > y);
}

double or_project_simplex(const double *x, int64_t n, double *y, double *work)
{
    memcpy(work, x, (size_t)n * sizeof(double));
    qsort(work, (size_t)n, sizeof(double), cmp_desc);
    double cum = 0.0, tau = 0.0;
    for (int64_t j = 0; j < n; j++) {
        cum += work[j];
        double t = (cum - 1.0) / (double)(j + 1);
        if (work[j] > t) tau = t;
    }
    for (int64_t j = 0; j < n; j++) {
        double v = x[j] - tau;
        y[j] = (v > 0.0) ? v : 0.0;
    }
    return tau;
}

/* Row-wise generalisation P_{S^M} (eq. Mp1_proj). */
void or_project_rows(const double *X, int64_t M, int64_t N, double *Y)
{
#pragma omp parallel
    {
        double *work = (double *)malloc((size_t)N * sizeof(double));
#pragma omp for schedule(static)
        for (int64_t k = 0; k < M; k++) or_project_simplex(X + k * N, N, Y + k * N, work);
        free(work);
    }
}

/* ------------------------------------------------------------------------------------
 * Residual R = F Theta - P  (objective row of Table 1; the auxiliary
 * O = F Pi of PAPER.md:258).  For each probe d in order and each k in its band in
 * increasing order: R[d,:] += F[d,k] * Theta[k,:]; P is subtracted last.
 * ---------------------------------------------------------------------------------- */
void or_forward(const int64_t *lo, const int64_t *len, const int64_t *off, const double *val,
                int64_t D, const double *Theta, const double *P, int64_t N, double *R)
{
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t d = 0; d < D; d++) {   /* probe rows are independent */
        double *r = R + d * N;
        for (int64_t n = 0; n < N; n++) r[n] = 0.0;
        for (int64_t j = 0; j < len[d]; j++) {
            double f = val[off[d] + j];
            const double *th = Theta + (lo[d] + j) * N;
            for (int64_t n = 0; n < N; n++) r[n] += f * th[n];
        }
        if (P)
            for (int64_t n = 0; n < N; n++) r[n] -= P[d * N + n];
    }
}

/* (L Theta) for the nearest-neighbour regulariser g = gamma sum_n sum_{i=0}^{M-2}
 * (Pi_{i,n} - Pi_{i+1,n})^2 (eq. regul):  L = D^T D with D the
 * (M-1) x M forward difference, free ends (reading R8).  grad g = 2 gamma L Theta. */
void or_laplacian(const double *Theta, int64_t M, int64_t N, double *LT)
{
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < M; k++)
        for (int64_t n = 0; n < N; n++) {
            double v = 0.0;
            if (k > 0) v += Theta[k * N + n] - Theta[(k - 1) * N + n];
            if (k < M - 1) v += Theta[k * N + n] - Theta[(k + 1) * N + n];
            LT[k * N + n] = v;
        }
}

/* Half gradient G = F^T R + gamma L Theta  (gradient row of Table 1, PAPER.md:243;
 * grad f = 2G, reading R0).  For each d in order and each k in its band:
 * G[k,:] += F[d,k] R[d,:]; then gamma L Theta is added.  Threads take blocks of OR_RB Fock rows;
 * inside a block the probe loop runs in the same increasing order, so every element of G is the
 * same sequence of operations as in the single loop over d. */
void or_backward(const int64_t *lo, const int64_t *len, const int64_t *off, const double *val,
                 int64_t D, int64_t M, const double *R, const double *Theta, int64_t N,
                 double gamma, double *G)
{
    const int64_t nb = (M + OR_RB - 1) / OR_RB;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; b++) {
        const int64_t r0 = b * OR_RB, r1 = (r0 + OR_RB < M) ? r0 + OR_RB : M;
        memset(G + r0 * N, 0, (size_t)((r1 - r0) * N) * sizeof(double));
        for (int64_t d = 0; d < D; d++) {
            const int64_t a = lo[d] > r0 ? lo[d] : r0;
            const int64_t e = (lo[d] + len[d] < r1) ? lo[d] + len[d] : r1;
            for (int64_t k = a; k < e; k++) {
                double f = val[off[d] + (k - lo[d])];
                double *g = G + k * N;
                const double *r = R + d * N;
                for (int64_t n = 0; n < N; n++) g[n] += f * r[n];
            }
        }
    }
    if (gamma != 0.0 && M > 1) {
        double *LT = (double *)malloc((size_t)(M * N) * sizeof(double));
        or_laplacian(Theta, M, N, LT);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < M * N; i++) G[i] += gamma * LT[i];
        free(LT);
    }
}

/* sum_n sum_{i=0}^{M-2} (Theta_{i,n} - Theta_{i+1,n})^2   (eq. regul):
 * the pairs (i, i+1) with i < M-1, i.e. sum (a - b)^2 over the first (M-1) N entries against the
 * entries one row below (fixed chunks, see the header) */
double or_regul(const double *Theta, int64_t M, int64_t N)
{
    if (M < 2) return 0.0;
    return sumsq_diff(Theta, Theta + N, (M - 1) * N);
}

/* f(Theta) = ||P - F Theta||_2^2 + gamma * regul   (eq. min_obj2 PAPER.md:70 + eq. regul) */
double or_objective(const int64_t *lo, const int64_t *len, const int64_t *off, const double *val,
                    int64_t D, int64_t M, const double *P, const double *Theta, int64_t N,
                    double gamma)
{
    double *R = (double *)malloc((size_t)(D * N) * sizeof(double));
    or_forward(lo, len, off, val, D, Theta, P, N, R);
    double s = sumsq(R, D * N);
    free(R);
    return s + gamma * or_regul(Theta, M, N);
}

/* KKT measure:
 *   r = sqrt( 1/(NM) sum_{n,i} (Pi_{i,n} (df_{i,n} + lambda_i))^2 ),
 *   paper: lambda_i = max(0, -min_n df_{i,n});  reading R7: unclamped lambda_i = -min_n df.
 * df = 2G (reading R0).  Returns the unclamped value; *paper_out gets the clamped one. */
double or_kkt(const double *Theta, const double *G, int64_t M, int64_t N, double *paper_out)
{
    const int64_t nc = (M + OR_RCHUNK - 1) / OR_RCHUNK;
    long double *ps = (long double *)malloc((size_t)nc * 2 * sizeof(long double));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nc; c++) {
    long double s = 0.0L, sp = 0.0L;
    const int64_t k1 = ((c + 1) * OR_RCHUNK < M) ? (c + 1) * OR_RCHUNK : M;
    for (int64_t k = c * OR_RCHUNK; k < k1; k++) {
        double mn = INFINITY;
        for (int64_t n = 0; n < N; n++) {
            double df = 2.0 * G[k * N + n];
            if (df < mn) mn = df;
        }
        double lam = -mn;
        double lamp = (lam > 0.0) ? lam : 0.0;
        for (int64_t n = 0; n < N; n++) {
            double df = 2.0 * G[k * N + n];
            double a = Theta[k * N + n] * (df + lam);
            double b = Theta[k * N + n] * (df + lamp);
            s += (long double)(a * a);
            sp += (long double)(b * b);
        }
    }
    ps[2 * c] = s;
    ps[2 * c + 1] = sp;
    }
    long double s = 0.0L, sp = 0.0L;
    for (int64_t c = 0; c < nc; c++) {
        s += ps[2 * c];
        sp += ps[2 * c + 1];
    }
    free(ps);
    if (paper_out) *paper_out = sqrt((double)sp / ((double)N * (double)M));
    return sqrt((double)s / ((double)N * (double)M));
}

/* ------------------------------------------------------------------------------------
 * Step-size setup (reading R2; the paper's own metric is the diagonal
 * preconditioner of PAPER.md:231 / PAPER.md:456, Hessian diagonal Table 1).
 * SQS majorizer: w_k = sum_d F_{d,k} s_d + 4 gamma,  s_d = sum_j F_{d,j}.
 * ---------------------------------------------------------------------------------- */
void or_sqs_weights(const int64_t *lo, const int64_t *len, const int64_t *off, const double *val,
                    int64_t D, int64_t M, double gamma, double *w)
{
    double *sd = (double *)malloc((size_t)D * sizeof(double));
    for (int64_t d = 0; d < D; d++) {
        double s = 0.0;
        for (int64_t j = 0; j < len[d]; j++) s += val[off[d] + j];
        sd[d] = s;
    }
    const int64_t nb = (M + OR_RB - 1) / OR_RB;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; b++) {   /* w[k] sums over d in increasing order (as one loop) */
        const int64_t r0 = b * OR_RB, r1 = (r0 + OR_RB < M) ? r0 + OR_RB : M;
        for (int64_t k = r0; k < r1; k++) w[k] = 0.0;
        for (int64_t d = 0; d < D; d++) {
            const int64_t a = lo[d] > r0 ? lo[d] : r0;
            const int64_t e = (lo[d] + len[d] < r1) ? lo[d] + len[d] : r1;
            for (int64_t k = a; k < e; k++) w[k] += val[off[d] + (k - lo[d])] * sd[d];
        }
        for (int64_t k = r0; k < r1; k++) w[k] += 4.0 * gamma;
    }
    free(sd);
}

/* Power iteration for rho ~ lambda_max(F^T F): v0 = 1/sqrt(M); exactly K_pow iterations of
 * v <- F^T F v / ||F^T F v||; rho = ||F v||^2 (Rayleigh quotient, ||v|| = 1). */
double or_power_iteration(const int64_t *lo, const int64_t *len, const int64_t *off,
                          const double *val, int64_t D, int64_t M, int64_t K_pow)
{
    double *v = (double *)malloc((size_t)M * sizeof(double));
    double *u = (double *)malloc((size_t)M * sizeof(double));
    double *q = (double *)malloc((size_t)D * sizeof(double));
    for (int64_t k = 0; k < M; k++) v[k] = 1.0 / sqrt((double)M);
    for (int64_t it = 0; it < K_pow; it++) {
        or_forward(lo, len, off, val, D, v, NULL, 1, q);
        or_backward(lo, len, off, val, D, M, q, v, 1, 0.0, u);
        double nn = sqrt(sumsq(u, M));
        if (nn == 0.0) break;
        for (int64_t k = 0; k < M; k++) v[k] = u[k] / nn;
    }
    or_forward(lo, len, off, val, D, v, NULL, 1, q);
    double rho = sumsq(q, D);
    free(v);
    free(u);
    free(q);
    return rho;
}

/* ------------------------------------------------------------------------------------
 * Projected-gradient solve (north_star: "Each iteration evaluates the gradient
 * F^T(F Theta - P) + gamma L Theta, then projects every Fock-index row onto the
 * probability simplex"; projection stage of Alg. 2 PAPER.md:518-539 with the Newton
 * direction replaced by a fixed diagonal metric, reading R2).
 *
 *   Theta_0 = 1/N or theta0.
 *   step 0: SQS      t_k = 1/w_k  (0 if w_k == 0: row frozen, reading R9)
 *   step 1: LIPSCHITZ t = 1/(1.01 rho + 4 gamma), rho from 100 power iterations
 *   step 2: BB       Barzilai-Borwein scalar step (north_star "power-iteration Lipschitz bound
 *            or Barzilai-Borwein"; reading R14): t_0 = t_LIP; for k >= 1 with s = Theta_k -
 *            Theta_{k-1}: t_k = <s,s> / <s,Hs>, <s,Hs> = ||R_k - R_{k-1}||^2 + gamma ||D s||^2
 *            (H = F^T F + gamma L, the Hessian of f/2), clamped to [t_LIP, 1e6 t_LIP];
 *            t_LIP when <s,Hs> <= 0.  Plain projected gradient only (accel ignored).
 *   step 3: BB with the exact line search along the projected direction (SURVEY 8(f) row 3,
 *            reading R17): t_k as step 2, Z = P_{S^M}(Theta_k - t_k G), d = Z - Theta_k; f is
 *            quadratic along d, f(Theta + l d) = f + 2 l <G,d> + l^2 (||F d||^2 + gamma ||D d||^2),
 *            so l* = clip(-<G,d> / (||F d||^2 + gamma ||D d||^2), 0, 1) (1 when the curvature
 *            is 0) and Theta_{k+1} = Theta_k + l* d (a convex combination: feasible).  The
 *            projection gives -<G,d> >= ||d||^2 / t_k exactly; near convergence the computed
 *            <G,d> cancels to roundoff (row-constant multiplier part of G against rows of d that
 *            sum to 0), so the numerator is max(-<G,d>, ||d||^2 / t_k) (reading R17).
 *   accel 1: FISTA extrapolation Y_k = Theta_k + (tau_k - 1)/tau_{k+1} (Theta_k - Theta_{k-1}),
 *            tau_0 = 1, tau_{k+1} = (1 + sqrt(1 + 4 tau_k^2))/2 (Beck-Teboulle).  Resume state
 *            (SURVEY 8(b)): theta_prev = Theta_{-1} (NULL: Theta_0) and tau0 = tau_0 (< 1: 1);
 *            theta_prev_out / tau_out (may be NULL) receive Theta_{k-1} and tau_k of the returned
 *            iterate k.
 *   iteration k (reading R3):
 *     R = F Y - P;  G = F^T R + gamma L Y;  Theta_{k+1} = P_{S^M}(Y - t o G);
 *     trace[k] = f(Theta_k);  kkt[k] = r(Theta_k) (G at Theta_k; for FISTA an extra pass);
 *     if r(Theta_k) <= tol (checked when k % kkt_every == 0): stop, return Theta_k.
 *   after iters iterations: trace[iters] = f(Theta_iters), kkt[iters] = r(Theta_iters).
 * Returns the number of iterations done.
 * ---------------------------------------------------------------------------------- */
int64_t or_solve(const int64_t *lo, const int64_t *len, const int64_t *off, const double *val,
                 int64_t D, int64_t M, const double *P, int64_t N, double gamma, double tol,
                 int64_t iters, int step_mode, int accel, int64_t kkt_every, const double *theta0,
                 double *Theta, double *trace, double *kkt_trace, double *kkt_paper_trace,
                 double *step_out, const double *theta_prev, double tau0, double *theta_prev_out,
                 double *tau_out)
{
    size_t MN = (size_t)(M * N);
    double *Tprev = (double *)malloc(MN * sizeof(double));
    double *Y = (double *)malloc(MN * sizeof(double));
    double *X = (double *)malloc(MN * sizeof(double));
    double *G = (double *)malloc(MN * sizeof(double));
    double *Gk = (double *)malloc(MN * sizeof(double));
    double *R = (double *)malloc((size_t)(D * N) * sizeof(double));
    double *t = (double *)malloc((size_t)M * sizeof(double));
    if (kkt_every < 1) kkt_every = 1;

    double t_lip = 0.0;
    double *Rprev = NULL;
    const int bb_ls = step_mode == 3;
    if (bb_ls) step_mode = 2;
    if (step_mode == 2) {
        accel = 0;
        double rho = or_power_iteration(lo, len, off, val, D, M, 100);
        t_lip = 1.0 / (1.01 * rho + 4.0 * gamma);
        for (int64_t k = 0; k < M; k++) t[k] = t_lip;
        if (step_out) *step_out = t_lip;
        Rprev = (double *)malloc((size_t)(D * N) * sizeof(double));
    } else if (step_mode == 0) {
        or_sqs_weights(lo, len, off, val, D, M, gamma, t);
        for (int64_t k = 0; k < M; k++) t[k] = (t[k] > 0.0) ? 1.0 / t[k] : 0.0;
        if (step_out) *step_out = 0.0;
    } else {
        double rho = or_power_iteration(lo, len, off, val, D, M, 100);
        double ts = 1.0 / (1.01 * rho + 4.0 * gamma);
        for (int64_t k = 0; k < M; k++) t[k] = ts;
        if (step_out) *step_out = ts;
    }

    for (size_t i = 0; i < MN; i++) Theta[i] = theta0 ? theta0[i] : 1.0 / (double)N;
    if (accel && theta_prev)
        memcpy(Tprev, theta_prev, MN * sizeof(double));
    else
        memcpy(Tprev, Theta, MN * sizeof(double));
    double tau = (accel && tau0 >= 1.0) ? tau0 : 1.0;
    int64_t k;
    for (k = 0; k < iters; k++) {
        double beta = 0.0, tau_next = tau;
        if (accel) {
            tau_next = (1.0 + sqrt(1.0 + 4.0 * tau * tau)) / 2.0;
            beta = (tau - 1.0) / tau_next;
        }
#pragma omp parallel for schedule(static)
        for (size_t i = 0; i < MN; i++) Y[i] = Theta[i] + beta * (Theta[i] - Tprev[i]);
        /* gradient at Y */
        or_forward(lo, len, off, val, D, Y, P, N, R);
        if (step_mode == 2 && k >= 1) {
            /* BB: s = Theta_k - Theta_{k-1} (Tprev), <s,Hs> = ||R_k - R_{k-1}||^2 + gamma ||D s||^2 */
            /* s = Theta_k - Theta_{k-1} (X as scratch); ||D s||^2 = regulariser sum of s */
#pragma omp parallel for schedule(static)
            for (size_t i = 0; i < MN; i++) X[i] = Theta[i] - Tprev[i];
            const double ss = sumsq(X, (int64_t)MN);
            const double sh = sumsq_diff(R, Rprev, D * N);
            const double sd = or_regul(X, M, N);
            double shs = sh + gamma * sd;
            double tb = t_lip;
            if (shs > 0.0) {
                tb = ss / shs;
                if (tb < t_lip) tb = t_lip;
                if (tb > 1e6 * t_lip) tb = 1e6 * t_lip;
            }
            for (int64_t r = 0; r < M; r++) t[r] = tb;
        }
        if (step_mode == 2) memcpy(Rprev, R, (size_t)(D * N) * sizeof(double));
        or_backward(lo, len, off, val, D, M, R, Y, N, gamma, G);
        /* f(Theta_k) and r(Theta_k) */
        double fk, rk = NAN, rpk = NAN;
        const double *Gt = G;
        if (beta != 0.0) {
            or_forward(lo, len, off, val, D, Theta, P, N, R);
            if (k % kkt_every == 0) {
                or_backward(lo, len, off, val, D, M, R, Theta, N, gamma, Gk);
                Gt = Gk;
            } else {
                Gt = NULL;
            }
        }
        fk = sumsq(R, D * N) + gamma * or_regul(Theta, M, N);
        if (Gt && (k % kkt_every == 0)) rk = or_kkt(Theta, Gt, M, N, &rpk);
        if (trace) trace[k] = fk;
        if (kkt_trace) kkt_trace[k] = rk;
        if (kkt_paper_trace) kkt_paper_trace[k] = rpk;
        if (k % kkt_every == 0 && rk <= tol) break; /* NaN compares false */
        /* step + projection */
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < M; r++)
            for (int64_t n = 0; n < N; n++) X[r * N + n] = Y[r * N + n] - t[r] * G[r * N + n];
        memcpy(Tprev, Theta, MN * sizeof(double));
        or_project_rows(X, M, N, Theta);
        if (bb_ls) {
            /* exact line search along d = Z - Theta_k (Z in Theta, Theta_k in Tprev; X, R scratch) */
#pragma omp parallel for schedule(static)
            for (size_t i = 0; i < MN; i++) X[i] = Theta[i] - Tprev[i];
            double *Fd = (double *)malloc((size_t)(D * N) * sizeof(double));
            or_forward(lo, len, off, val, D, X, NULL, N, Fd);
            const double fdd = sumsq(Fd, D * N);
            const double ddd = or_regul(X, M, N);
            const double gd = dotl(G, X, (int64_t)MN);   /* G at Theta_k (plain PG: Y = Theta_k) */
            const double dd = sumsq(X, (int64_t)MN);
            free(Fd);
            const double den = fdd + gamma * ddd;
            const double num = fmax(-gd, dd / t[0]);     /* scalar BB step: t[r] = t_k for every row */
            double lam = 1.0;
            if (den > 0.0) {
                lam = num / den;
                lam = lam < 0.0 ? 0.0 : (lam > 1.0 ? 1.0 : lam);
            }
#pragma omp parallel for schedule(static)
            for (size_t i = 0; i < MN; i++) Theta[i] = Tprev[i] + lam * X[i];
        }
        tau = tau_next;
    }
    if (k == iters) {
        or_forward(lo, len, off, val, D, Theta, P, N, R);
        or_backward(lo, len, off, val, D, M, R, Theta, N, gamma, G);
        double s = sumsq(R, D * N);
        double rp;
        double r = or_kkt(Theta, G, M, N, &rp);
        if (trace) trace[iters] = s + gamma * or_regul(Theta, M, N);
        if (kkt_trace) kkt_trace[iters] = r;
        if (kkt_paper_trace) kkt_paper_trace[iters] = rp;
    }
    if (theta_prev_out) memcpy(theta_prev_out, Tprev, MN * sizeof(double));
    if (tau_out) *tau_out = tau;
    free(Tprev);
    free(Y);
    free(X);
    free(G);
    free(Gk);
    free(R);
    free(t);
    free(Rprev);
    return k;
}

/* ------------------------------------------------------------------------------------
 * Long-range smoothing (eq. smoothing):
 *   Pi~_{i,n} = 1/(2 Ns(i) + 1) sum_{j = i - Ns(i)}^{i + Ns(i)} Pi_{j,n},   Ns(i) = floor(i / div)
 * (the paper's N_smooth = i/50), rows i < exclude unchanged (the lowest ~100 photon numbers are
 * excluded).  DESIGN.md reading R13: the window is clipped to the rows that exist,
 * [max(0, i - Ns), min(M - 1, i + Ns)], and the average is over the rows in it, so every smoothed
 * row is a convex combination of rows of Pi.
 * ---------------------------------------------------------------------------------- */
void or_smooth(const double *Theta, int64_t M, int64_t N, int64_t exclude, int64_t div, double *out)
{
    for (int64_t i = 0; i < M; i++) {
        if (i < exclude || div <= 0) {
            for (int64_t n = 0; n < N; n++) out[i * N + n] = Theta[i * N + n];
            continue;
        }
        int64_t ns = i / div;
        int64_t lo = i - ns < 0 ? 0 : i - ns;
        int64_t hi = i + ns > M - 1 ? M - 1 : i + ns;
        for (int64_t n = 0; n < N; n++) {
            double s = 0.0;
            for (int64_t j = lo; j <= hi; j++) s += Theta[j * N + n];
            out[i * N + n] = s / (double)(hi - lo + 1);
        }
    }
}

/* ------------------------------------------------------------------------------------
 * Two-stage, two-metric projected truncated Newton (Alg. 3 of PAPER.md:536-544: stage 1 =
 * Alg. 2, stage 2 = Alg. 1), SURVEY 8(f) row 1.
 * Readings (R16): f is the paper's objective incl. gamma * regul; df = 2G (R0);
 * H d = 2 (F^T F d + gamma L d) acts on each column of d independently (Table 1 "Hessian
 * products"); its diagonal h_i = 2 (sum_d F_{d,i}^2 + gamma L_ii) (Table 1,
 * PAPER.md:245).  The metric D of eq. 2metric D / I: entries in the active
 * set I = {x <= eps, df > 0} keep only their diagonal, the others the Hessian restricted to
 * the free set; D p = -df is solved by diagonally preconditioned CG from p = 0,
 * truncated at cg_max iterations or ||r|| <= min(0.5, sqrt||b||) ||b|| (Nocedal-Wright's
 * forcing sequence; the paper only says "truncated").  Line search alpha = beta^m, beta = 3/4,
 * c = 1/10.  armijo = 0 (default): the paper's printed condition
 *   f(P[x + beta^m p]) <= f(x) + c beta^m d/dalpha f(P[x + alpha p])|_{alpha=0},
 * the derivative being the one-sided arc slope at 0 (stage 1: df . Pi_T(p); stage 2: the reduced
 * gradient . p with p_j -> 0 where x_j = 0 and p_j < 0); a direction whose slope is >= 0 admits no
 * step length (the condition cannot certify descent: DESIGN.md reading R16).  armijo = 1:
 * Bertsekas' secant form along the projection arc f(x(alpha)) <= f(x) + c df . (x(alpha) - x).
 * Stage switch when the
 * one-sided derivative of the stage-1 arc at alpha = 0, df . d0 with d0 the projection of p
 * onto the simplex tangent cone at Theta, satisfies |df . d0| <= switch_tol.  Stop when the
 * KKT measure (R7, unclamped multiplier) <= eps_kkt, or when no step length is accepted in
 * stage 2; a stage-1 iteration that admits none switches to stage 2 (stage 1 carries no
 * convergence proof).
 * ---------------------------------------------------------------------------------- */
typedef struct {
    const int64_t *lo, *len, *off;
    const double *val;
    int64_t D, M, N;
    const double *P;
    double gamma;
} or_prob;

/* H v = 2 (F^T (F v) + gamma L v) */
static void nt_hess(const or_prob *q, const double *v, double *out, double *Rw)
{
    or_forward(q->lo, q->len, q->off, q->val, q->D, v, NULL, q->N, Rw);
    or_backward(q->lo, q->len, q->off, q->val, q->D, q->M, Rw, v, q->N, q->gamma, out);
    for (int64_t i = 0; i < q->M * q->N; i++) out[i] *= 2.0;
}

/* df = 2 G(Theta) */
static void nt_grad(const or_prob *q, const double *Th, double *g, double *Rw)
{
    or_forward(q->lo, q->len, q->off, q->val, q->D, Th, q->P, q->N, Rw);
    or_backward(q->lo, q->len, q->off, q->val, q->D, q->M, Rw, Th, q->N, q->gamma, g);
    for (int64_t i = 0; i < q->M * q->N; i++) g[i] *= 2.0;
}

static double nt_f(const or_prob *q, const double *Th)
{
    return or_objective(q->lo, q->len, q->off, q->val, q->D, q->M, q->P, Th, q->N, q->gamma);
}


/* Hessian diagonal per Fock row: h_i = 2 (sum_d F_{d,i}^2 + gamma L_ii) */
void or_hess_diag(const int64_t *lo, const int64_t *len, const int64_t *off, const double *val,
                  int64_t D, int64_t M, double gamma, double *h)
{
    for (int64_t i = 0; i < M; i++) h[i] = 0.0;
    for (int64_t d = 0; d < D; d++)
        for (int64_t j = 0; j < len[d]; j++) {
            double f = val[off[d] + j];
            h[lo[d] + j] += f * f;
        }
    for (int64_t i = 0; i < M; i++) {
        double lii = (M > 1) ? ((i > 0) + (i < M - 1)) : 0.0;
        h[i] = 2.0 * (h[i] + gamma * lii);
    }
}

/* Tangent-cone projection of p at a point Theta of the simplex (one row):
 * d = argmin ||d - p|| s.t. sum d = 0, d_j >= 0 where Theta_j = 0.  d_j = p_j - mu on the
 * support, max(p_j - mu, 0) on the zeros; mu solves sum d(mu) = 0 (sort of the breakpoints). */
static void nt_tangent_row(const double *th, const double *p, int64_t N, double *d, double *work)
{
    int64_t nf = 0, nz = 0;
    double sf = 0.0;
    for (int64_t j = 0; j < N; j++) {
        if (th[j] > 0.0) { sf += p[j]; nf++; } else work[nz++] = p[j];
    }
    qsort(work, (size_t)nz, sizeof(double), cmp_desc);
    /* h(mu) = sf - nf mu + sum_{zeros} max(p_j - mu, 0), decreasing; find the root */
    double mu;
    if (nf == 0 && nz == 0) return;
    double cum = 0.0;
    int64_t k = 0;       /* number of zero-entries above mu */
    mu = (nf > 0) ? sf / (double)nf : work[0];
    if (nf > 0) {
        /* candidate with the k largest zero entries active: mu = (sf + cum_k) / (nf + k) */
        for (k = 0; k <= nz; k++) {
            if (k > 0) cum += work[k - 1];
            double m = (sf + cum) / (double)(nf + k);
            double upper = (k > 0) ? work[k - 1] : INFINITY;   /* active ones must exceed mu */
            double lower = (k < nz) ? work[k] : -INFINITY;     /* inactive ones must not */
            if (m < upper && m >= lower) { mu = m; break; }
        }
    } else {
        for (k = 1; k <= nz; k++) {
            cum += work[k - 1];
            double m = cum / (double)k;
            double lower = (k < nz) ? work[k] : -INFINITY;
            if (m >= lower) { mu = m; break; }
        }
    }
    for (int64_t j = 0; j < N; j++) {
        double v = p[j] - mu;
        d[j] = (th[j] > 0.0) ? v : (v > 0.0 ? v : 0.0);
    }
}

/* CG stopping rule override for the pins: rtol >= 0 replaces the forcing term (-1: default) */
static double nt_cg_rtol = -1.0;
void or_newton_set_cg_rtol(double rtol) { nt_cg_rtol = rtol; }

/* Truncated PCG for the masked system: free entries (mask 0) solve H_FF x_F = b_F, active
 * entries (mask 1) x = b / hdiag.  Stage 2 (m != NULL) works in the reduced variables of the
 * transformation Theta_{i,m(i)} = 1 - sum_{n != m(i)} x_{i,n} (entries n = m(i) are held at 0)
 * with H~ = Z^T H Z and diagonal 2 h_i.  Returns the CG iteration count. */
static int64_t nt_pcg(const or_prob *q, const int64_t *m, const unsigned char *act, const double *hrow,
                      const double *b, int64_t cg_max, double *x, double *ws)
{
    const int64_t M = q->M, N = q->N, n = M * N;
    double *r = ws, *z = ws + n, *d = ws + 2 * n, *Hd = ws + 3 * n, *u = ws + 4 * n, *Rw = ws + 5 * n;
    int64_t it = 0;
    for (int64_t i = 0; i < n; i++) {
        const int64_t k = i / N, c = i % N;
        const double hd = m ? 2.0 * hrow[k] : hrow[k];
        const int fixed = m && c == m[k];
        x[i] = 0.0;
        r[i] = 0.0;
        if (fixed) continue;
        if (act[i]) x[i] = hd > 0.0 ? b[i] / hd : 0.0;
        else r[i] = b[i];
    }
    const double bn = sqrt(dotl(r, r, n));
    const double tol = (nt_cg_rtol >= 0.0 ? nt_cg_rtol : fmin(0.5, sqrt(bn))) * bn;
    for (int64_t i = 0; i < n; i++) {
        const double hd = m ? 2.0 * hrow[i / N] : hrow[i / N];
        z[i] = hd > 0.0 ? r[i] / hd : 0.0;
        d[i] = z[i];
    }
    double rz = dotl(r, z, n);
    for (it = 0; it < cg_max && bn > 0.0; it++) {
        if (rz <= 0.0) break;
        /* Hd = mask_F (H~ d) */
        if (m) {
            for (int64_t k = 0; k < M; k++) {
                double s = 0.0;
                for (int64_t c = 0; c < N; c++)
                    if (c != m[k]) { u[k * N + c] = d[k * N + c]; s += d[k * N + c]; }
                u[k * N + m[k]] = -s;
            }
            nt_hess(q, u, Hd, Rw);
            for (int64_t k = 0; k < M; k++) {
                const double hm = Hd[k * N + m[k]];
                for (int64_t c = 0; c < N; c++) Hd[k * N + c] -= hm;
                Hd[k * N + m[k]] = 0.0;
            }
        } else {
            nt_hess(q, d, Hd, Rw);
        }
        for (int64_t i = 0; i < n; i++)
            if (act[i]) Hd[i] = 0.0;
        const double dHd = dotl(d, Hd, n);
        if (dHd <= 0.0) break;
        const double a = rz / dHd;
        for (int64_t i = 0; i < n; i++) {
            x[i] += a * d[i];
            r[i] -= a * Hd[i];
        }
        if (sqrt(dotl(r, r, n)) <= tol) { it++; break; }
        for (int64_t i = 0; i < n; i++) {
            const double hd = m ? 2.0 * hrow[i / N] : hrow[i / N];
            z[i] = hd > 0.0 ? r[i] / hd : 0.0;
        }
        const double rz2 = dotl(r, z, n);
        const double beta = rz2 / rz;
        rz = rz2;
        for (int64_t i = 0; i < n; i++) d[i] = z[i] + beta * d[i];
    }
    return it;
}

/* One Newton direction (exposed for the pins): stage 1 (m == NULL) or stage 2 (row maxima m).
 * g: df at Theta (stage 2: at the transformed Theta~); out p (M x N; stage 2: 0 at n = m(i));
 * returns the CG iteration count; *slope = df . d0 (stage 1: d0 = tangent-cone projection of
 * p; stage 2: d0 = p with p_j -> 0 where x_j = 0 and p_j < 0, in reduced variables). */
int64_t or_newton_direction(const int64_t *lo, const int64_t *len, const int64_t *off,
                            const double *val, int64_t D, int64_t M, const double *P, int64_t N,
                            double gamma, const double *Theta, const int64_t *m, double eps_active,
                            int64_t cg_max, double *p, double *slope)
{
    or_prob q = {lo, len, off, val, D, M, N, P, gamma};
    const int64_t n = M * N;
    double *g = malloc(sizeof(double) * n), *gr = malloc(sizeof(double) * n), *b = malloc(sizeof(double) * n);
    double *h = malloc(sizeof(double) * M), *ws = malloc(sizeof(double) * (5 * n + D * N + N));
    unsigned char *act = malloc((size_t)n);
    or_hess_diag(lo, len, off, val, D, M, gamma, h);
    nt_grad(&q, Theta, g, ws);
    for (int64_t i = 0; i < n; i++) {
        const int64_t k = i / N, c = i % N;
        gr[i] = m ? (c == m[k] ? 0.0 : g[i] - g[k * N + m[k]]) : g[i];
        act[i] = (!m || c != m[k]) && Theta[i] <= eps_active && gr[i] > 0.0;
        b[i] = -gr[i];
    }
    const int64_t it = nt_pcg(&q, m, act, h, b, cg_max, p, ws);
    if (slope) {
        double s = 0.0;
        if (!m) {
            double *d0 = ws, *work = ws + n;
            for (int64_t k = 0; k < M; k++) nt_tangent_row(Theta + k * N, p + k * N, N, d0 + k * N, work);
            s = dotl(g, d0, n);
        } else {
            long double t = 0.0L;
            for (int64_t i = 0; i < n; i++) {
                const double pj = (Theta[i] <= 0.0 && p[i] < 0.0) ? 0.0 : p[i];
                t += (long double)gr[i] * pj;
            }
            s = (double)t;
        }
        *slope = s;
    }
    free(g); free(gr); free(b); free(h); free(ws); free(act);
    return it;
}

/* Row maxima m(i) = argmax_n Theta_{i,n}, first index on ties (Table 1 "row-maxima"). */
void or_row_argmax(const double *Theta, int64_t M, int64_t N, int64_t *m)
{
    for (int64_t k = 0; k < M; k++) {
        int64_t a = 0;
        for (int64_t c = 1; c < N; c++)
            if (Theta[k * N + c] > Theta[k * N + a]) a = c;
        m[k] = a;
    }
}

/* The two-stage solve.  Theta (M x N) in: start (rows on the simplex), out: result.
 * Logs (length max_iter + 1): trace f_k, kkt r_KKT(Theta_k) (R7), stage of step k (1/2),
 * CG iterations of step k, accepted alpha of step k.  Returns the iterations done (k of the
 * returned Theta); *switch_out = first stage-2 iteration (-1 if none). */
int64_t or_newton(const int64_t *lo, const int64_t *len, const int64_t *off, const double *val,
                  int64_t D, int64_t M, const double *P, int64_t N, double gamma, double *Theta,
                  int64_t max_iter, double eps_kkt, double eps_active, int64_t cg_max,
                  double switch_tol, int64_t max_ls, int armijo, double *trace, double *kkt, int64_t *stage_log,
                  int64_t *cg_log, double *alpha_log, int64_t *switch_out)
{
    or_prob q = {lo, len, off, val, D, M, N, P, gamma};
    const int64_t n = M * N;
    const double beta = 0.75, c_arm = 0.1;
    double *g = malloc(sizeof(double) * n), *G2 = malloc(sizeof(double) * n), *p = malloc(sizeof(double) * n);
    double *T1 = malloc(sizeof(double) * n), *X = malloc(sizeof(double) * n), *Rw = malloc(sizeof(double) * D * N);
    int64_t *mrow = malloc(sizeof(int64_t) * M);
    int stage = 1;
    int64_t k = 0;
    if (switch_out) *switch_out = -1;
    for (k = 0;; k++) {
        nt_grad(&q, Theta, g, Rw);
        for (int64_t i = 0; i < n; i++) G2[i] = 0.5 * g[i];
        const double f = nt_f(&q, Theta);
        double kp;
        const double r = or_kkt(Theta, G2, M, N, &kp);
        trace[k] = f;
        kkt[k] = r;
        if (r <= eps_kkt || k >= max_iter) break;
        double slope = 0.0;
        int64_t it = 0;
        if (stage == 1) {
            it = or_newton_direction(lo, len, off, val, D, M, P, N, gamma, Theta, NULL, eps_active, cg_max,
                                     p, &slope);
            if (fabs(slope) <= switch_tol) {
                stage = 2;
                if (switch_out) *switch_out = k;
            }
        }
        int64_t used_stage = stage;
        if (stage == 2) {
            or_row_argmax(Theta, M, N, mrow);
            for (int64_t i = 0; i < M; i++) {   /* transformation step (Alg. 1) */
                double s = 0.0;
                for (int64_t c = 0; c < N; c++)
                    if (c != mrow[i]) s += Theta[i * N + c];
                Theta[i * N + mrow[i]] = 1.0 - s;
            }
            it = or_newton_direction(lo, len, off, val, D, M, P, N, gamma, Theta, mrow, eps_active, cg_max,
                                     p, &slope);
            nt_grad(&q, Theta, g, Rw);   /* df at Theta~ (reduced gradient for the Armijo term) */
        }
        const double f0 = (stage == 2) ? nt_f(&q, Theta) : f;
        double alpha = 0.0;
        int accepted = 0;
        for (int64_t l = 0; l < max_ls && !accepted; l++) {
            const double a = pow(beta, (double)l);
            if (used_stage == 1) {
                for (int64_t i = 0; i < n; i++) X[i] = Theta[i] + a * p[i];
                or_project_rows(X, M, N, T1);
            } else {
                for (int64_t i = 0; i < M; i++) {
                    double s = 0.0;
                    for (int64_t c = 0; c < N; c++) {
                        if (c == mrow[i]) continue;
                        double v = Theta[i * N + c] + a * p[i * N + c];
                        v = v > 0.0 ? v : 0.0;   /* P_{0,inf} */
                        T1[i * N + c] = v;
                        s += v;
                    }
                    T1[i * N + mrow[i]] = 1.0 - s;
                }
                int ok = 1;
                for (int64_t i = 0; i < M; i++)
                    if (T1[i * N + mrow[i]] < 0.0) ok = 0;
                if (!ok) continue;
            }
            if (armijo == 0) {
                /* the paper's condition: f(P[Theta + a p]) <= f0 + c a slope,
                 * slope = one-sided arc derivative at alpha = 0 (this iteration's stage) */
                if (!(slope < 0.0)) break;   /* no descent certified: no admissible step length */
                const double f1 = nt_f(&q, T1);
                if (f1 <= f0 + c_arm * a * slope) {
                    accepted = 1;
                    alpha = a;
                }
                continue;
            }
            /* secant form along the arc: f(T1) <= f0 + c df . (T1 - Theta) (stage 2: reduced df) */
            long double dd = 0.0L;
            for (int64_t i = 0; i < n; i++) {
                const int64_t rr = i / N, cc = i % N;
                double gi = g[i];
                if (used_stage == 2) {
                    if (cc == mrow[rr]) continue;
                    gi = g[i] - g[rr * N + mrow[rr]];
                }
                dd += (long double)gi * (long double)(T1[i] - Theta[i]);
            }
            const double f1 = nt_f(&q, T1);
            if (f1 <= f0 + c_arm * (double)dd) {
                accepted = 1;
                alpha = a;
            }
        }
        if (!accepted && used_stage == 1) {
            /* stage 1 has no convergence guarantee: when its arc admits no
             * step length, switch to the globally convergent stage 2 and redo iteration k */
            stage = 2;
            if (switch_out) *switch_out = k;
            k--;
            continue;
        }
        stage_log[k] = used_stage;
        cg_log[k] = it;
        alpha_log[k] = alpha;
        if (!accepted) break;   /* no admissible step length: stalled */
        memcpy(Theta, T1, sizeof(double) * n);
    }
    free(g); free(G2); free(p); free(T1); free(X); free(Rw); free(mrow);
    return k;
}
