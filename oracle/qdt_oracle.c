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
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

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
    double *work = (double *)malloc((size_t)N * sizeof(double));
    for (int64_t k = 0; k < M; k++) or_project_simplex(X + k * N, N, Y + k * N, work);
    free(work);
}

/* ------------------------------------------------------------------------------------
 * Residual R = F Theta - P  (objective row of Table 1; the auxiliary
 * O = F Pi of PAPER.md:258).  For each probe d in order and each k in its band in
 * increasing order: R[d,:] += F[d,k] * Theta[k,:]; P is subtracted last.
 * ---------------------------------------------------------------------------------- */
void or_forward(const int64_t *lo, const int64_t *len, const int64_t *off, const double *val,
                int64_t D, const double *Theta, const double *P, int64_t N, double *R)
{
    for (int64_t d = 0; d < D; d++) {
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
 * G[k,:] += F[d,k] R[d,:]; then gamma L Theta is added. */
void or_backward(const int64_t *lo, const int64_t *len, const int64_t *off, const double *val,
                 int64_t D, int64_t M, const double *R, const double *Theta, int64_t N,
                 double gamma, double *G)
{
    memset(G, 0, (size_t)(M * N) * sizeof(double));
    for (int64_t d = 0; d < D; d++)
        for (int64_t j = 0; j < len[d]; j++) {
            double f = val[off[d] + j];
            double *g = G + (lo[d] + j) * N;
            const double *r = R + d * N;
            for (int64_t n = 0; n < N; n++) g[n] += f * r[n];
        }
    if (gamma != 0.0 && M > 1) {
        double *LT = (double *)malloc((size_t)(M * N) * sizeof(double));
        or_laplacian(Theta, M, N, LT);
        for (int64_t i = 0; i < M * N; i++) G[i] += gamma * LT[i];
        free(LT);
    }
}

/* sum_n sum_{i=0}^{M-2} (Theta_{i,n} - Theta_{i+1,n})^2   (eq. regul) */
double or_regul(const double *Theta, int64_t M, int64_t N)
{
    long double s = 0.0L; /* long scalar sums accumulate in extended precision (see header) */
    for (int64_t k = 0; k + 1 < M; k++)
        for (int64_t n = 0; n < N; n++) {
            double d = Theta[k * N + n] - Theta[(k + 1) * N + n];
            s += (long double)(d * d);
        }
    return (double)s;
}

/* ||R||_F^2 over D x N entries, extended-precision accumulator */
static double sumsq(const double *R, int64_t n)
{
    long double s = 0.0L;
    for (int64_t i = 0; i < n; i++) s += (long double)(R[i] * R[i]);
    return (double)s;
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
    long double s = 0.0L, sp = 0.0L;
    for (int64_t k = 0; k < M; k++) {
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
    for (int64_t k = 0; k < M; k++) w[k] = 0.0;
    for (int64_t d = 0; d < D; d++) {
        double s = 0.0;
        for (int64_t j = 0; j < len[d]; j++) s += val[off[d] + j];
        for (int64_t j = 0; j < len[d]; j++) w[lo[d] + j] += val[off[d] + j] * s;
    }
    for (int64_t k = 0; k < M; k++) w[k] += 4.0 * gamma;
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
 *   accel 1: FISTA extrapolation Y_k = Theta_k + (tau_k - 1)/tau_{k+1} (Theta_k - Theta_{k-1}),
 *            tau_0 = 1, tau_{k+1} = (1 + sqrt(1 + 4 tau_k^2))/2.
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
                 double *step_out)
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
    memcpy(Tprev, Theta, MN * sizeof(double));
    double tau = 1.0;
    int64_t k;
    for (k = 0; k < iters; k++) {
        double beta = 0.0, tau_next = tau;
        if (accel) {
            tau_next = (1.0 + sqrt(1.0 + 4.0 * tau * tau)) / 2.0;
            beta = (tau - 1.0) / tau_next;
        }
        for (size_t i = 0; i < MN; i++) Y[i] = Theta[i] + beta * (Theta[i] - Tprev[i]);
        /* gradient at Y */
        or_forward(lo, len, off, val, D, Y, P, N, R);
        if (step_mode == 2 && k >= 1) {
            /* BB: s = Theta_k - Theta_{k-1} (Tprev), <s,Hs> = ||R_k - R_{k-1}||^2 + gamma ||D s||^2 */
            long double ss = 0.0L, sh = 0.0L, sd = 0.0L;
            for (size_t i = 0; i < MN; i++) {
                double d = Theta[i] - Tprev[i];
                ss += (long double)(d * d);
            }
            for (int64_t i = 0; i < D * N; i++) {
                double d = R[i] - Rprev[i];
                sh += (long double)(d * d);
            }
            for (int64_t r = 0; r + 1 < M; r++)
                for (int64_t n = 0; n < N; n++) {
                    double a = Theta[r * N + n] - Tprev[r * N + n];
                    double b = Theta[(r + 1) * N + n] - Tprev[(r + 1) * N + n];
                    sd += (long double)((a - b) * (a - b));
                }
            double shs = (double)sh + gamma * (double)sd;
            double tb = t_lip;
            if (shs > 0.0) {
                tb = (double)ss / shs;
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
        for (int64_t r = 0; r < M; r++)
            for (int64_t n = 0; n < N; n++) X[r * N + n] = Y[r * N + n] - t[r] * G[r * N + n];
        memcpy(Tprev, Theta, MN * sizeof(double));
        or_project_rows(X, M, N, Theta);
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
