/*
 * qdt.h -- C ABI of the B200-native phase-insensitive detector-tomography solver
 *          (hot path of arXiv:2404.02844, "Scalable quantum detector tomography by
 *          high-performance computing").
 *
 * Problem (eq. min; regulariser eq. regul):
 *     min_Theta  f(Theta) = ||P - F Theta||_F^2 + gamma * sum_n sum_{k=0}^{M-2} (Theta_{k,n} - Theta_{k+1,n})^2
 *     s.t.       Theta_{k,n} >= 0,  sum_n Theta_{k,n} = 1   for every Fock row k.
 *   Theta (= Pi of the paper) : M x N, row-major, row k = Fock level, column n = outcome.
 *   F                          : D x M, F_{d,k} = mu_d^k e^{-mu_d} / k!,  mu_d = |alpha_d|^2
 *                                (eq. Fmatrix), stored banded.
 *   P                          : D x N, row-major outcome probabilities (eq. Matrix).
 *
 * Method (DESIGN.md "Readings" R0-R12): projected gradient.  One iteration k maps
 *   Theta_k -> Theta_{k+1} = P_{S^M}( Y_k - t o G(Y_k) ),   G = F^T (F Y - P) + gamma L Y = grad f / 2,
 * with the row-wise simplex projection P_{S^M} of eq. Mp1_proj, Y_k = Theta_k
 * (plain) or the FISTA extrapolation, and t a fixed diagonal metric: SQS row weights
 * t_k = 1/w_k, w = F^T F 1 + 4 gamma, or one Lipschitz scalar 1/(1.01 rho + 4 gamma) with rho
 * from 100 power iterations.  Convergence measure: the KKT residual of PAPER.md:563-567.
 *
 * Conventions (all functions):
 *   - Every call returns qdt_status; QDT_OK == 0.  No C++ exception crosses the ABI.  On a
 *     non-OK status, qdt_last_error(ctx) returns a message naming the offending argument.
 *   - Ownership: the caller owns every input and output buffer (caller-allocated, sizes as
 *     stated).  Handles are created by qdt_init / qdt_build_probes / qdt_probes_from_banded
 *     and released by qdt_finalize / qdt_probes_free.  No caller pointer is kept after a
 *     call returns.
 *   - Pointers are HOST pointers unless `mem_device` (solve/objective options) is 1; then P,
 *     Theta and theta0 are device pointers on ctx's device, ordered on ctx's stream.
 *   - A ctx is not thread-safe: one ctx per (process, GPU).
 *   - Multi-GPU is SPMD over the Fock axis: with nranks > 1 every rank calls every function
 *     with identical replicated inputs; qdt_build_probes, qdt_solve and qdt_objective are
 *     collective (NCCL over NVLink).  Rank g owns Fock rows [k_begin, k_end) (cost balanced).
 *   - There is no CPU fallback: without a CUDA device every call returns QDT_ERR_CUDA.
 */
#ifndef QDT_H
#define QDT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    QDT_OK = 0,
    QDT_ERR_INVALID_ARG = 1, /* a size/scalar/option out of range, or a NULL required pointer */
    QDT_ERR_UNSORTED = 2,    /* alpha2 not nondecreasing */
    QDT_ERR_NONFINITE = 3,   /* NaN/Inf in alpha2, P, theta0, or a non-finite objective */
    QDT_ERR_OOM = 4,         /* device allocation failed / memory plan exceeds free HBM */
    QDT_ERR_CUDA = 5,        /* CUDA runtime error (no device, launch failure, ...) */
    QDT_ERR_NCCL = 6,        /* NCCL unavailable or a collective failed */
    QDT_ERR_TRUNCATED = 7,   /* strict_mass: a probe row loses mass at the cutoff M */
    QDT_ERR_STATE = 8        /* handle/ctx mismatch (e.g. probes built on another ctx) */
} qdt_status;

typedef enum {
    QDT_STEP_SQS = 0,       /* row-constant diagonal majorizer, t_k = 1 / (F^T F 1 + 4 gamma)_k */
    QDT_STEP_LIPSCHITZ = 1, /* scalar t = 1 / (1.01 rho + 4 gamma), rho: 100 power iterations   */
    QDT_STEP_BB = 2,        /* Barzilai-Borwein scalar step <s,s>/<s,Hs> clamped to [t_LIP, 1e6 t_LIP]
                               (reading R14); plain PG (accel = 0)                       */
    QDT_STEP_BB_LS = 3      /* BB + exact line search along d = P(Theta - t G) - Theta:
                               Theta_{k+1} = Theta + l* d, l* = argmin over [0, 1] of the quadratic
                               f(Theta + l d) (reading R17); monotone; plain PG, allreduce exchange */
} qdt_step_mode;

typedef struct qdt_ctx qdt_ctx;       /* device, stream, NCCL comm, workspace, last error  */
typedef struct qdt_probes qdt_probes; /* banded F of this rank's Fock slice + tile plans     */

typedef enum {
    QDT_COMM_NCCL = 0,   /* one process per GPU, NCCL over NVLink (the production path)            */
    QDT_COMM_INPROC = 1  /* virtual ranks: one host thread per rank inside one process, device
                            buffers shared directly (all ranks on one device, or peer-accessible
                            devices); the same planner, kernels, halo and reductions as NCCL, with
                            sums in rank order.  Runs the multi-rank library path on one GPU
                            (tests); solves run iteration by iteration (no graph). */
} qdt_comm_kind;

typedef struct {
    int32_t device;             /* CUDA device ordinal                                       */
    int32_t rank, nranks;       /* SPMD rank / world size (1 = single GPU)                   */
    const void *nccl_unique_id; /* 128-byte ncclUniqueId (same on every rank); NULL if nranks==1 */
    void *cuda_stream;          /* cudaStream_t to run on; NULL -> ctx-owned stream           */
    int32_t comm;               /* qdt_comm_kind (nranks > 1), default QDT_COMM_NCCL            */
    int64_t group_key;          /* QDT_COMM_INPROC: ranks calling qdt_init with the same key (and
                                   nranks) form one group; each rank calls from its own thread  */
} qdt_init_opts;

typedef struct {
    double c_sigma;      /* band half-width in units of sqrt(mu) (reading R1), default 6     */
    int32_t margin;      /* extra rows above the band, default 16                            */
    int32_t strict_mass; /* 1: a band clipped at M-1 is an error (QDT_ERR_TRUNCATED)        */
} qdt_probe_opts;

typedef struct {
    int32_t step;          /* qdt_step_mode, default QDT_STEP_SQS                              */
    int32_t accel;         /* 0 = plain projected gradient, 1 = FISTA extrapolation            */
    const double *theta0;  /* initial Theta (M x N, or local rows if !gather); NULL -> 1/N     */
    int32_t check_every;   /* host polls the device stop flag every this many iterations (16)  */
    int32_t kkt_every;     /* FISTA: evaluate r_KKT(Theta_k) every this many iterations (1)    */
    int32_t mem_device;    /* 1: P / theta0 / theta_out are device pointers                    */
    int32_t gather_theta;  /* nranks>1: 1 -> theta_out is the full M x N on every rank         */
    int32_t use_graph;     /* 1 (default): replay the iteration as a CUDA graph                */
    /* FISTA resume state (accel = 1; the paper restarts its second stage from a given
     * Pi): a solve stopped at Theta_k continues bit for bit as the uninterrupted one
     * when called with theta0 = Theta_k, theta_prev = Theta_{k-1} and fista_t = tau_k.          */
    const double *theta_prev; /* Theta_{k-1}, same layout as theta0; NULL -> Theta_{-1} = Theta_0  */
    double fista_t;        /* tau_k of the Beck-Teboulle sequence at the resume point (>= 1); 0 -> 1 */
    double *theta_prev_out;/* receives Theta_{k-1} of the returned Theta_k (layout of theta_out);
                              may be NULL; FISTA only                                            */
    int32_t exchange;      /* nranks > 1, residual exchange: 0 (default) allreduce of the D x N
                              partial residual; 1 band-aware: each rank sums only the probes whose
                              bands touch its slice, with the peers whose slices they also touch
                              (the paper's neighbour exchange); not with BB  */
} qdt_solve_opts;

typedef struct {
    int64_t iters_done;    /* k at which the solve stopped (== iters if the cap was hit)       */
    int32_t converged;     /* 1 if r_KKT(Theta_k) <= tol stopped the solve                     */
    double kkt0;           /* r_KKT(Theta_0)                                                   */
    double kkt;            /* r_KKT(Theta_iters_done), unclamped multiplier (reading R7)       */
    double kkt_paper;      /* same with the paper's clamped lambda = max(0, -min df)           */
    double f_final;        /* f(Theta_iters_done)                                               */
    double step_scalar;    /* LIPSCHITZ step t (0 for SQS)                                     */
    int64_t k_begin, k_end;/* this rank's Fock rows                                            */
    int64_t nnz;           /* stored entries of F on this rank                                  */
    double min_row_mass;   /* min_d sum_k F_{d,k} over stored bands (truncation diagnostic)    */
    int64_t uncovered_rows;/* Fock rows (this rank) touched by no probe band (reading R9)      */
    double loop_ms;        /* CUDA-event time of the iteration loop on ctx's stream            */
    double fista_t;        /* FISTA: tau of the returned iterate (resume state), 0 otherwise    */
} qdt_solve_info;

/* ------------------------------------------------------------------------------ context */
/* Write a fresh 128-byte NCCL unique id (rank 0 of a multi-GPU job calls this and
 * broadcasts it).  Errors: NCCL unavailable -> QDT_ERR_NCCL. */
qdt_status qdt_nccl_unique_id(void *out128);
/* Host-only Fock-axis shard planner (used by qdt_build_probes; exported for tests): given
 * band edges lo[D], hi[D] (inclusive, global rows), cut [0, M) into nranks contiguous
 * slices at equal prefix sums of the per-row cost 16 + 0.7 cov(k).  cuts: int64[nranks+1]. */
qdt_status qdt_shard_cuts(const int64_t *lo, const int64_t *hi, int64_t D, int64_t M,
                          int32_t nranks, int64_t *cuts);
/* Create a context on opts->device.  nranks > 1 initialises an NCCL communicator from
 * opts->nccl_unique_id (collective over all ranks).  opts == NULL -> device 0, 1 rank. */
qdt_status qdt_init(qdt_ctx **ctx, const qdt_init_opts *opts);
qdt_status qdt_finalize(qdt_ctx *ctx);
/* Thread-local message for the last non-OK status of ctx (never NULL). */
const char *qdt_last_error(const qdt_ctx *ctx);

/* ------------------------------------------------------------------------------ probes */
/* S0: build the banded probe matrix F from host alpha2[D] (mu_d = |alpha_d|^2,
 * finite, >= 0, nondecreasing) for Fock cutoff M (eq. Fmatrix; band:
 * reading R1).  Band edges and values are computed on the device (log-space Poisson pmf,
 * Loader's saddle-point form).  opts == NULL -> defaults.  Collective when nranks > 1: rank
 * g stores only entries with k in its Fock slice.
 * Errors: D < 1, M < 1 -> INVALID_ARG; non-finite or negative mu -> INVALID_ARG;
 * decreasing mu -> UNSORTED; strict_mass and a clipped band -> TRUNCATED. */
qdt_status qdt_build_probes(qdt_ctx *ctx, const double *alpha2, int64_t D, int64_t M,
                            const qdt_probe_opts *opts, qdt_probes **out);
/* Test hook: a probe handle from an arbitrary banded F instead of the Poisson
 * generator.  Probe d stores rows [lo[d], lo[d] + len[d]) (global Fock indices) with values
 * vals[off_d + j], off_d = sum_{e<d} len_e (probe-major, host pointers, copied: the caller keeps
 * ownership).  Requirements: len[d] >= 1, 0 <= lo[d], lo[d] + len[d] <= M, and both band edges
 * nondecreasing in d (the structure the S0 bands of sorted probes have; the tile planner relies
 * on contiguous probe windows).  Collective when nranks > 1 (every rank passes the full bands).
 * Errors: bad sizes / edges -> INVALID_ARG; decreasing edges -> UNSORTED; non-finite values ->
 * NONFINITE. */
qdt_status qdt_probes_from_banded(qdt_ctx *ctx, int64_t D, int64_t M, const int64_t *lo,
                                  const int64_t *len, const double *vals, qdt_probes **out);
qdt_status qdt_probes_free(qdt_probes *probes);
/* Band tables and sizes of this rank: any output pointer may be NULL.  lo/len: host
 * int64[D] (global first row and length of the locally stored band), val: host double[nnz]
 * (probe-major, the band of probe d at [off_d, off_d + len_d), off_d = sum_{e<d} len_e). */
qdt_status qdt_probes_export(qdt_ctx *ctx, const qdt_probes *probes, int64_t *nnz,
                             int64_t *k_begin, int64_t *k_end, int64_t *lo, int64_t *len,
                             double *val);

/* ------------------------------------------------------------------------------ solve */
/* Projected-gradient solve.  P: D x N (host, or device if
 * opts->mem_device).  1 <= N <= 10 240 (N > 1024: sweep kernels only), gamma >= 0 finite, tol >= 0,
 * iters >= 0.
 * theta_out: M x N (or the local (k_end-k_begin) x N rows when nranks > 1 and
 * !gather_theta) receiving Theta_{iters_done}; NULL: no copy of the result (trace / info only,
 * e.g. when Theta fills the device and the caller times the iterations).  trace_out (may be NULL): host double[iters+1],
 * trace_out[k] = f(Theta_k) for k <= iters_done (reading R3); kkt_out (may be NULL): host
 * double[iters+1] with r_KKT(Theta_k) (NaN where not evaluated).  Early stop at the first
 * k with r_KKT(Theta_k) <= tol returns Theta_k.  info may be NULL.  Collective. */
qdt_status qdt_solve(qdt_ctx *ctx, const qdt_probes *F, const double *P, int64_t N, double gamma,
                     double tol, int64_t iters, const qdt_solve_opts *opts, double *theta_out,
                     double *trace_out, double *kkt_out, qdt_solve_info *info);

/* f(Theta) = ||P - F Theta||^2 + gamma * regul (eq. min_obj2 + eq. regul) and, if kkt_out
 * != NULL, r_KKT(Theta) (unclamped, reading R7).  Theta: M x N (all ranks pass the full
 * matrix).  mem_device as in qdt_solve_opts.  Collective. */
qdt_status qdt_objective(qdt_ctx *ctx, const qdt_probes *F, const double *P, const double *theta,
                         int64_t N, double gamma, int32_t mem_device, double *f_out,
                         double *kkt_out);

/* Long-range smoothing (eq. smoothing; reading R13):
 *   out_{i,n} = mean of theta_{j,n} over j in [i - Ns(i), i + Ns(i)] clipped to [0, M - 1],
 *   Ns(i) = floor(i / div) (the paper's N_smooth = i/50: div = 50), rows i < exclude copied (the
 *   paper excludes the lowest ~100 photon numbers: exclude = 100); div <= 0 copies everything.
 * theta, out: M x N row-major, HOST pointers unless mem_device (then device pointers on ctx's
 * device, ordered on ctx's stream; out may not alias theta).  Every output row is a convex
 * combination of input rows (stays on the simplex).  The smoothed matrix is the warm start of a
 * second solve (opts->theta0).  Single rank only (nranks > 1 -> QDT_ERR_INVALID_ARG).
 * Errors: M, N < 1, exclude < 0, NULL pointers -> INVALID_ARG; non-finite host theta -> NONFINITE. */
qdt_status qdt_smooth(qdt_ctx *ctx, const double *theta, int64_t M, int64_t N, int64_t exclude,
                      int64_t div, int32_t mem_device, double *out);

/* Two-stage, two-metric projected truncated Newton (the paper's optimiser: Alg. 2 = stage 1,
 * Alg. 1 = stage 2, Alg. 3 = the two stages; reading R16).
 * Per outer iteration: df = 2 (F^T (F Theta - P) + gamma L Theta); the metric D of eq. 2metric
 * (active set I = {theta <= eps_active, df > 0} keeps only the Hessian diagonal
 * h_i = 2 (sum_d F_{d,i}^2 + gamma L_ii)); D p = -df by diagonally preconditioned CG from 0
 * (H d = 2 (F^T F d + gamma L d), <= cg_max iterations, ||r|| <= min(1/2, sqrt||b||) ||b||);
 * Armijo along the projection arc (beta = 3/4, c = 1/10, <= max_ls step lengths; the test is
 * opts->armijo's); stage 1
 * arcs P_{S^M}[Theta + alpha p], stage 2 (row maxima m(i) eliminated by the sum constraint)
 * arcs max(x + alpha p, 0); switch to stage 2 when |df . Pi_T(p)| <= switch_tol or when a
 * stage-1 iteration admits no step length.  Stops when r_KKT (reading R7) <= eps_kkt, after
 * max_iter iterations, or when stage 2 admits no step length.  Single rank only.
 *   P, theta0: host (mem_device = 0) or device pointers, D x N / M x N row-major; theta0 NULL:
 *   Theta_0 = 1/N.  theta_out: M x N (same memory kind).  trace_out / kkt_out: host arrays of
 *   max_iter + 1 (NaN past the last iteration); stage_out / cg_out / alpha_out: host arrays of
 *   max_iter (per accepted step), any may be NULL.  Errors: QDT_ERR_INVALID_ARG (shapes,
 *   options, nranks > 1), QDT_ERR_NONFINITE, QDT_ERR_OOM, QDT_ERR_CUDA. */
typedef struct {
    int32_t max_iter;          /* outer iterations */
    int32_t cg_max;            /* CG iterations per direction (default 50) */
    int32_t max_ls;            /* step lengths tried per line search (default 60) */
    int32_t mem_device;        /* 1: P / theta0 / theta_out are device pointers */
    double eps_active;         /* active-set threshold (default 1e-8) */
    double switch_tol;         /* stage switch |df . Pi_T(p)| (default 1e-4) */
    const double *theta0;      /* optional start (rows on the simplex) */
    int32_t armijo;            /* line-search test.  0 (default): the paper's printed condition
                                  f(P[Pi + beta^m p]) <= f(Pi) + c beta^m d/dalpha f(P[Pi + alpha p])|_0
                                  (the one-sided arc derivative at alpha = 0, the
                                  same slope as the stage switch; a direction with slope >= 0 admits
                                  no step length); 1: Bertsekas' secant form
                                  f(Pi(alpha)) <= f(Pi) + c df . (Pi(alpha) - Pi)                 */
} qdt_newton_opts;

typedef struct {
    int64_t iters_done;        /* k of the returned Theta */
    int64_t switch_iter;       /* first stage-2 iteration (-1: none) */
    int64_t cg_total;          /* CG iterations (Hessian products) over the solve */
    double f_final, kkt;       /* f and r_KKT of the returned Theta */
    double loop_ms;            /* device time of the iterations (CUDA events) */
} qdt_newton_info;

qdt_status qdt_solve_newton(qdt_ctx *ctx, const qdt_probes *F, const double *P, int64_t N, double gamma,
                            double eps_kkt, const qdt_newton_opts *opts, double *theta_out,
                            double *trace_out, double *kkt_out, int32_t *stage_out, int32_t *cg_out,
                            double *alpha_out, qdt_newton_info *info);

/* ------------------------------------------------------------------------------ kernel hooks
 * The individual steps of one iteration, for per-kernel parity tests.  They run the same
 * kernels as qdt_solve.  All arrays are HOST pointers, full (global) sizes, nranks == 1. */
/* R = F Theta - P (P may be NULL: R = F Theta).  Theta M x N, R D x N. */
qdt_status qdt_residual(qdt_ctx *ctx, const qdt_probes *F, const double *theta, const double *P,
                        int64_t N, double *R_out);
/* G = F^T R + gamma L Theta (half gradient, reading R0).  R D x N, Theta M x N, G M x N. */
qdt_status qdt_gradient(qdt_ctx *ctx, const qdt_probes *F, const double *R, const double *theta,
                        int64_t N, double gamma, double *G_out);
/* One iteration of the given step/accel=0 map on Theta: Theta_next = P_{S^M}(Theta - t o G). */
qdt_status qdt_step(qdt_ctx *ctx, const qdt_probes *F, const double *P, const double *theta,
                    int64_t N, double gamma, int32_t step_mode, double *theta_next);
/* Row-wise simplex projection Y = P_{S^M}(X) of an M x N matrix (warp Michelot). */
qdt_status qdt_project_rows(qdt_ctx *ctx, const double *X, int64_t M, int64_t N, double *Y_out);
/* Step setup: SQS weights w[M] = F^T F 1 + 4 gamma (w_out may be NULL) and the power-
 * iteration estimate rho of lambda_max(F^T F) after k_pow iterations (rho_out may be NULL). */
qdt_status qdt_step_setup(qdt_ctx *ctx, const qdt_probes *F, double gamma, int32_t k_pow,
                          double *w_out, double *rho_out);

/* ------------------------------------------------------------------------------ profiling */
/* When enabled, qdt_solve runs without a graph and brackets every kernel launch with CUDA
 * events on ctx's stream; qdt_profile_get returns per-kernel (count, total ms) for the kernel
 * names "probe_edges", "probe_values", "fwd_partial", "reduce_R", "bwd_step", "scalars",
 * "allreduce_R", "halo". */
qdt_status qdt_profile_enable(qdt_ctx *ctx, int32_t enable);
qdt_status qdt_profile_get(qdt_ctx *ctx, const char *kernel, int64_t *count, double *total_ms);
/* Number of kernels this library launched on ctx since qdt_init (graph nodes counted per
 * replay). */
qdt_status qdt_launch_count(qdt_ctx *ctx, int64_t *count);

#ifdef __cplusplus
}
#endif
#endif /* QDT_H */
