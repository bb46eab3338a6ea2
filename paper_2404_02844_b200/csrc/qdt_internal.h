// qdt_internal.h -- declarations shared by the host runtime (qdt_api.cu) and the sm_100a
// kernels (qdt_kernels.cu).  Not part of the public ABI (include/qdt.h is).
#pragma once
#include <cuda.h>   // CUtensorMap (type only; the encoder is fetched through the runtime)
#include <cuda_runtime.h>
#include <stdint.h>

namespace qdt {

// Bwd work unit: rows [k0, k1) (local) of bwd tile `tile`, probe range [p0, p1) of its window.
// A tile whose window is wider than the split cap is cut into nsplit units along the probe
// axis (split-K); each writes a partial G into scratch slot slot_base + slot and the last one
// to finish sums the slots in slot order (deterministic) and runs the epilogue.
struct BwdUnit {
    int32_t k0, k1;
    int32_t p0, p1;
    int32_t tile;
    int32_t slot;
    int32_t nsplit;
    int32_t pad;
    int64_t slot_base;
};

// Fwd work unit: Rpart rows [poff, poff + p1 - p0) receive sum_{k in [k0,k1)} F[d,k] Theta[k,:]
// for d in [p0, p1).  [k0, k1) is already tightened to the union of the group's bands.
struct FwdUnit {
    int32_t k0, k1;
    int32_t p0, p1;
    int64_t poff;
};

// Band tables of the local Fock slice: probe d stores rows [lo[d], lo[d] + len[d]) (GLOBAL row
// indices) at val[off[d] ...]; len[d] == 0 when the band misses the slice.
struct Band {
    const int32_t *lo;
    const int32_t *len;
    const int64_t *off;
    const double *val;
};

enum BwdMode { BWD_STEP = 0, BWD_GRAD = 1, BWD_EVAL = 2 };

// per-tile scalar partials written by the bwd kernel
enum { SC_KKT = 0, SC_KKTP = 1, SC_REG = 2, SC_DTH = 3, NSC_TILE = 4 };
// reduced scalar vector (after the cross-rank allreduce)
enum { V_R2 = 0, V_KKT = 1, V_KKTP = 2, V_REG = 3, V_DTH = 4, NV = 5 };

// device-side solve state (stop flag and iteration counter; graph-replay safe)
struct DevState {
    int32_t stop;
    int32_t converged;
    int64_t it;
    int64_t iters_done;
    int32_t nonfinite;
    int32_t pad;
};

struct BwdArgs {
    int N, CG, RG, KC;
    int SEG;                   // lanes per Fock row in the row epilogue (power of two <= 32)
    const BwdUnit *units;
    Band band;
    const double *R;
    const double *theta;       // local row 0; rows -1 and Ml readable (halo)
    const double *theta_prev;  // FISTA: Theta_{k-1} (same layout) or nullptr
    const double *beta;        // FISTA: beta_k indexed by state->it (nullptr -> plain)
    int kkt_every;             // MODE_EVAL runs only when state->it % kkt_every == 0
    int64_t kb, M;
    int Ml;
    const double *tstep;       // per local row
    double gamma;
    double *out;               // Theta_next (local row 0) or G
    double *scratch;
    int *counters;
    double *part;              // [ntiles x NSC_TILE]
    const DevState *state;
};

struct FwdArgs {
    int N, CG, RG, KR;
    const FwdUnit *units;
    Band band;
    const double *theta;       // local row 0
    int64_t kb;
    double *rpart;
    const DevState *state;
};

// ---- sweep path (qdt_sweep.cu): fp64 tensor-core (DMMA) kernels for N <= 128
constexpr int ST = 64;          // Fock rows per sweep tile (8 DMMA m-blocks)
constexpr int STP = ST + 4;     // pitch of a tiled-F row: conflict-free A fragments
constexpr int SKC = 16;         // probes per staged bwd chunk (4 DMMA k-steps)
constexpr int SWCAP = 128;      // bwd split cap (probes per unit)
constexpr int FWCAP = 48;       // fwd unit union-window cap (probes): 2 CTAs/SM of k_fwd_mma at N = 100
constexpr int FWNB = FWCAP / 8; // fwd DMMA probe n-blocks per unit
constexpr int FW_MAXT = 16;     // fwd unit length cap (tiles)
constexpr int SC2_BLOCKS = 64;  // first-level blocks of the scalar reduction
constexpr int SW_NBMAX = 16;    // sweep path: N <= 8 * SW_NBMAX outcomes (every kernel variant)
constexpr int SW_NBX = 20;      // plain steps up to N = 8 * SW_NBX (even) on k_bwd_mma alone

struct SwUnit {                 // bwd unit: tile, probe range [p0, p1) of its window, split-K info
    int32_t tile, p0, p1, slot, nsplit, pad;
    int64_t slot_base;
};
struct FwUnit {                 // fwd unit: tiles [t0, t1), union window [u0, u1), partial rows
    int32_t t0, t1, u0, u1;
    int64_t poff;
};
struct SweepArgs {
    int N, Ml;
    int Nv;                     // outcomes (< N when the row pitch N carries a zero pad column; 0: N)
    int64_t kb, M;
    const SwUnit *units;
    const int64_t *fb_off;
    const int32_t *tile_dA;
    const double *Fb;
    const double *R;
    const double *theta;        // local row 0; rows -1 and Ml readable
    double *out;
    const double *tstep;
    const double *tscal;        // BB: one device scalar step for every row (nullptr: tstep)
    double gamma;
    double *scratch;
    int *counters;
    double *part;
    int kkt_every;
    int nunits;                 // set by launch_bwd_mma (persistent grid)
    int eval;                   // 1: evaluation pass (G, KKT both multipliers, regulariser; no step)
    int eval_gate;              // evaluation pass runs only when state->it % kkt_every == 0
    const double *theta_prev;   // FISTA step: Theta_{k-1} (same layout as theta)
    const double *beta;         // FISTA step: beta_k indexed by state->it (nullptr: plain PG)
    const DevState *state;
    int tm_on;                  // set by launch_bwd_mma: the Theta tile arrives by 2-D tensor copy
    alignas(64) CUtensorMap tm_theta;   // box (tp_pitch(NB) x 66) over rows -1 .. Ml of theta
    alignas(64) CUtensorMap tm_prev;    // same over theta_prev (FISTA)
};
struct SweepFwdArgs {
    int N, Ml;
    const FwUnit *units;
    const int64_t *fb_off;
    const int32_t *tile_dA, *tile_dB;
    const double *Fb;
    const double *theta;
    double *rpart;
    int ncc;                    // column chunks of 8 NB outcomes (set by launch_fwd_mma)
    const DevState *state;
};
struct WideArgs {               // wide-N sweep (N > 128): k_grad_wide + k_proj_wide
    const double *tscal = nullptr;   // one device scalar step (BB) instead of tstep per row
    int N, Ml, ncc;             // ncc: 128-column chunks (set by launch_grad_wide)
    int Nv;                     // outcomes (< N when the row pitch N carries a zero pad column)
    int64_t kb, M;
    const SwUnit *units;
    const int64_t *fb_off;
    const int32_t *tile_dA;
    const double *Fb;
    const double *R;
    const double *theta;        // local row 0; rows -1 and Ml readable
    double *G;                  // Ml x N gradient (half), written by k_grad_wide
    double *out;                // Theta_{k+1} (k_proj_wide, not in eval)
    const double *tstep;
    double gamma;
    double *scratch;
    int *counters;              // per (tile, chunk)
    double *part;               // grad: slot tile * ncc + cc; proj: slot part_b + block
    int64_t part_b;
    int kkt_every;
    int eval;
    int eval_gate;              // FISTA evaluation pass: only when state->it % kkt_every == 0
    const double *theta_prev;   // FISTA step: Theta_{k-1}
    const double *beta;         // FISTA step: beta_k by state->it (nullptr: plain)
    const DevState *state;
    const int32_t *row_da = nullptr, *row_db = nullptr;   // probes covering local row k: [row_da, row_db)
                                                          // (k_grad_wide skips k-steps outside a warp's rows)
};
// ---- single-CTA persistent solve (qdt_small.cu): the whole problem in shared memory
struct SmallArgs {
    int D, M, N, nnz;
    const int32_t *lo, *len;
    const int64_t *off;
    const double *val;
    const int32_t *row_da, *row_db;   // probes covering Fock row k: [row_da[k], row_db[k])
    const double *theta0, *theta_prev, *P, *tstep, *beta;
    double gamma, tol;
    int64_t iters;
    int kkt_every, fista;
    double *trace, *kkt, *kktp;
    int64_t trace_len;
    double *theta_out, *prev_out;
    DevState *state;
};
// ---- grid-persistent cooperative solve (qdt_coop.cu): latency-bound sizes (Medium)
struct CoopArgs {
    int D, M, N, Nv;
    const int32_t *lo, *len;
    const int64_t *off;
    const double *val;
    const int32_t *row_da, *row_db;   // probes covering Fock row k: [row_da[k], row_db[k])
    const int64_t *toff;              // transposed band: F[d][k] at FT[toff[k] + d - row_da[k]]
    const double *FT;
    double *theta[3];                 // Theta_k in theta[k % nbuf] (local row 0)
    double *R[2];                     // R_k (FISTA: R_k / R_{k-1} alternate by k & 1)
    double *RY;                       // FISTA: R(Y_k)
    const double *P, *tstep, *beta;
    double gamma, tol;
    int64_t iters;
    int kkt_every, fista, resume;     // resume: R[1] holds R_{-1} = F Theta_{-1} - P
    double *trace, *kkt, *kktp;
    int64_t trace_len;
    double *part;                     // 2 x grid x 4 per-CTA partials
    unsigned *bar;                    // grid barrier: arrival counter, generation (zeroed)
    DevState *state;
};
bool coop_supported(int N);
int coop_max_grid();
cudaError_t launch_coop_solve(const CoopArgs &a, cudaStream_t s);
cudaError_t launch_build_FT(Band b, int D, const int32_t *row_da, const int64_t *toff, double *FT, cudaStream_t s);
size_t small_solve_smem(int64_t D, int64_t M, int N, int64_t nnz, int fista);
constexpr int SD_NR = 16;       // dense small solve: widest row held in registers
size_t small_dense_smem(int64_t D, int64_t M, int N, int fista);   // SIZE_MAX when N > SD_NR
cudaError_t launch_small_solve(const SmallArgs &a, cudaStream_t s);
constexpr size_t SMALL_SMEM_MAX = 200 * 1024;

// ---- fused wide-row step (qdt_wide.cu): N > 160, one cluster of C CTAs per 32-row tile
constexpr int WT = 16;          // Fock rows per wide tile (a quarter of a 64-row sweep tile)
constexpr int WKC = 8;          // probes per staged chunk
constexpr int WSTAGES = 4;      // chunk ring depth
constexpr int WFP = 20;         // staged F row pitch (16 rows + 4: conflict-free A fragments)
constexpr int W_NBW_MAX = 5;    // n-blocks per warp: <= 640 columns per CTA
constexpr int W_NG = 16;        // n-group warps per CTA
constexpr unsigned W_LANES = (1u << WT) - 1;   // lanes of warp 0 that own the tile's rows
constexpr int W_THREADS = 512;
constexpr int W_CMAX = 16;      // CTAs per cluster (non-portable above 8)
constexpr int GEN_NMAX = 1024;  // widest row of the general CUDA-core kernels (hooks, Newton)
constexpr int QDT_NMAX = W_CMAX * 8 * W_NG * W_NBW_MAX;   // widest row of the fused wide step (10 240)
struct WStepArgs {
    int N, Nv, Ml;
    int C, Wc;                  // CTAs per cluster, columns per CTA (multiple of 8)
    int64_t kb, M;
    const int32_t *tlist;       // tile indices, cluster c owns tlist[toff[c] .. toff[c + 1]) (Fock order)
    const int32_t *toff;
    const int64_t *fb_off;
    const int32_t *tile_dA, *tile_dB;   // 64-row sweep tiles (wide tile tt uses sweep tile tt >> 2)
    const double *Fb;
    const double *R;
    const double *theta;        // local row 0; rows -1 and Ml readable
    const double *theta_prev;   // FISTA step: Theta_{k-1}
    const double *beta;         // FISTA step: beta_k by state->it (nullptr: plain)
    double *out;
    const double *tstep;
    const double *tscal;        // one device scalar step (nullptr: tstep per row)
    double gamma;
    double *tau_prev;           // per local row: the last step's threshold (warm start), or nullptr
    double *part;               // [grid x NSC_TILE] scalar partials
    int kkt_every;
    int eval, eval_gate;
    const DevState *state;
};
size_t wide_step_smem(int Wc);
int wide_nbw(int Wc);
int wide_max_clusters(int C, int Wc);
cudaError_t prepare_wide_kernels();
cudaError_t launch_wide_step(const WStepArgs &a, int nclusters, cudaStream_t s);
cudaError_t launch_grad_wide(const WideArgs &a, int nunits, cudaStream_t s);
cudaError_t launch_proj_wide(const WideArgs &a, cudaStream_t s);
int wide_nb(int N);                                  // balanced column-chunk width / 8 (N > 128)
int wide_fwd_nb(int N);                              // same for the forward (<= 13 n-blocks: 2 CTAs / SM)
constexpr int PW_BLOCKS = 148 * 8;                   // k_proj_wide grid cap (contiguous row ranges)
int wide_proj_blocks(int Ml);
cudaError_t prepare_sweep_kernels();
constexpr int BB_NBLK = 296;
cudaError_t launch_bb_stats(const double *th, const double *tp, int64_t Ml, int64_t kb, int64_t M, int N,
                            const double *R, const double *Rp, int64_t nR, double *part, double *vec3,
                            const DevState *st, cudaStream_t s);
cudaError_t launch_bb_step(const double *vec3, double gamma, double tlip, double *tout,
                           const DevState *st, cudaStream_t s);
cudaError_t launch_bbls_stats(const double *th, const double *zt, int64_t Ml, int64_t kb, int64_t M, int N,
                              const double *Rk, const double *Rz, int64_t nR, double *part, double *vec,
                              const DevState *st, cudaStream_t s);
cudaError_t launch_bbls_dir(const double *th, const double *zt, double *dd, int64_t n, const DevState *st,
                            cudaStream_t s);
cudaError_t launch_bbls_step(const double *vec, double gamma, const double *tbb, double *lam, const double *th,
                             double *zt, int64_t n, const DevState *st, cudaStream_t s);
cudaError_t launch_smooth(const double *X, int64_t M, int N, int64_t exclude, int64_t div, double *S,
                          double *T, double *Tx, double *Y, cudaStream_t s);
cudaError_t launch_sqs_weights_tiled(int ntiles, int Ml, const int32_t *tile_dA,
                                     const int32_t *tile_dB, const int64_t *fb_off, const double *Fb,
                                     const double *s, double gamma, double *w, double *tstep,
                                     cudaStream_t st);
int sweep_nb(int N);            // DMMA n-blocks instantiated for N (0: N too wide, general path)
size_t sweep_bwd_smem(int N, int NB, bool fista, bool tp = false);
size_t sweep_fwd_smem(int N, int NB);
cudaError_t launch_tile_F(Band b, int64_t kb, int Ml, int ntiles, const int32_t *tile_dA,
                          const int32_t *tile_dB, const int64_t *fb_off, double *Fb,
                          cudaStream_t s);
cudaError_t launch_bwd_mma(const SweepArgs &a, int nunits, int NB, cudaStream_t s);
cudaError_t launch_bwd_split(const SweepArgs &a, int nunits, int NB, cudaStream_t s);
int sweep_split_mode();
cudaError_t launch_fwd_mma(const SweepFwdArgs &a, int nunits, int NB, cudaStream_t s);
cudaError_t launch_reduce_R2(const double *rpart, const int64_t *red_beg, const int64_t *red_rows,
                             const double *P, double *R, int D, int N, double *partR,
                             const DevState *st, cudaStream_t s);
cudaError_t launch_scalars2(const double *partR, int nR, const double *partT, int ntiles,
                            int include_r2, double *stage, int *arrive, double *vec, int64_t N,
                            int64_t M, double gamma, double tol, int final_eval, int kkt_every,
                            double *trace, double *kkt, double *kktp, int64_t trace_len,
                            DevState *st, int finalize, cudaStream_t s);

// launchers (qdt_kernels.cu); return cudaGetLastError()
cudaError_t launch_probe_edges(const double *alpha2, int64_t D, int64_t M, double c_sigma,
                               int margin, int32_t *lo, int32_t *hi, cudaStream_t s);
cudaError_t launch_probe_values(const double *alpha2, int64_t D, Band b, cudaStream_t s);
cudaError_t launch_probe_rowsum(int64_t D, Band b, double *s_out, cudaStream_t s);
cudaError_t launch_sqs_weights(int ntiles, int T, const int32_t *tile_dA, const int32_t *tile_dB,
                               int Ml, int64_t kb, Band b, const double *s, double gamma,
                               double *w, double *tstep, cudaStream_t st);
cudaError_t launch_pow_fwd(int64_t D, Band b, const double *v, int64_t kb, double *q,
                           cudaStream_t s);
cudaError_t launch_pow_bwd(int ntiles, int T, const int32_t *tile_dA, const int32_t *tile_dB,
                           int Ml, int64_t kb, Band b, const double *q, double *u,
                           cudaStream_t s);
cudaError_t launch_sumsq(const double *x, int64_t n, double *part, int nblk, cudaStream_t s);
cudaError_t launch_reduce_vec(const double *part, int nblk, int stride, int nvals, double *out,
                              cudaStream_t s);
cudaError_t launch_scale(double *v, const double *u, const double *nrm2, int64_t n,
                         cudaStream_t s);
cudaError_t launch_fill(double *x, int64_t n, double v, cudaStream_t s);

cudaError_t prepare_kernels();
int device_sm_count();            // SM count of the current device (cached per ordinal)
int fwd_threads(int N, int *CG, int *RG, int *TC);
int bwd_threads(int N, int *CG, int *RG, int *TC);
constexpr int TR = 4;  // rows (bwd) / probes (fwd) per thread
constexpr int WCAP_MAX = 128;  // max probes per work unit (split cap / fwd group)

cudaError_t launch_fwd(const FwdArgs &a, int nunits, int TC, cudaStream_t s, size_t *smem_out);
cudaError_t launch_bwd(const BwdArgs &a, int nunits, int TC, int mode, cudaStream_t s);
size_t bwd_smem_bytes(int N, int RG, int KC, bool fista);
size_t fwd_smem_bytes(int N, int RG, int KR);
cudaError_t launch_reduce_R(const double *rpart, const int64_t *red_beg, const int64_t *red_rows,
                            const double *P, double *R, int64_t D, int N, double *partR,
                            int nblk, const DevState *st, cudaStream_t s);
constexpr int VMAX = 16;        // ranks of an in-process (virtual) group
struct VPtrs {
    const double *p[VMAX];
};
cudaError_t launch_vsum(const VPtrs &v, int n_ranks, int64_t n, double *out, cudaStream_t s);
struct BandX {                  // band-aware residual exchange tables (per rank of the group)
    int64_t dlo[VMAX], dhi[VMAX];   // probes touching rank q's slice: [dlo[q], dhi[q])
    const double *src[VMAX];        // peer q's partial rows (received copy), row start[q]
    int64_t start[VMAX];
};
cudaError_t launch_band_combine(const BandX &bx, int rank, int nranks, const double *P, double *R, int N,
                                double *partR, int nblk, const DevState *st, cudaStream_t s);
cudaError_t launch_sub_p_sumsq(double *R, const double *P, int64_t n, double *partR, int nblk,
                               const DevState *st, cudaStream_t s);
cudaError_t launch_scalars_local(const double *partR, int nblkR, const double *partT,
                                 int ntiles, int include_r2, double *vec, const DevState *st,
                                 cudaStream_t s);
cudaError_t launch_finalize(const double *vec, int64_t N, int64_t M, double gamma, double tol,
                            int final_eval, int kkt_every, double *trace, double *kkt,
                            double *kktp, int64_t trace_len, DevState *st, cudaStream_t s);
cudaError_t launch_project_rows(const double *X, int64_t M, int N, double *Y, cudaStream_t s);
cudaError_t launch_fista_rcomb(double *RY, const double *Rk, const double *Rkm1,
                               const double *beta, int64_t n, const DevState *st,
                               cudaStream_t s);


// ---- two-stage two-metric projected truncated Newton (qdt_newton.cu; reading R16)
constexpr int NT_BLK = 296;    // reduction grid (block partials, then one warp)
cudaError_t nt_pcg_init(const double *g, const double *theta, const double *h, const int32_t *m, int N,
                        int64_t n, double eps, double *gr, uint8_t *act, double *x, double *r, double *z, double *d,
                        double *part, double *out, cudaStream_t s);
cudaError_t nt_dot(const double *a, const double *b, const uint8_t *act, const double *theta, int mode, int64_t n,
                   double *part, double *out, cudaStream_t s);
cudaError_t nt_dotdiff(const double *g, const double *T, const double *theta, const int32_t *m, int N, int64_t n,
                       double *part, double *out, cudaStream_t s);
cudaError_t nt_scale_mask(double *x, const uint8_t *act, double sc, int64_t n, cudaStream_t s);
cudaError_t nt_cg_update(double *x, double *r, double *z, const double *d, const double *Hd, double a,
                         const double *h, const int32_t *m, int N, int64_t n, double *part, double *out,
                         cudaStream_t s);
cudaError_t nt_cg_dir(double *d, const double *z, double beta, int64_t n, cudaStream_t s);
cudaError_t nt_zexp(const double *v, const int32_t *m, int64_t M, int N, double *u, cudaStream_t s);
cudaError_t nt_zred(double *w, const int32_t *m, const uint8_t *act, int64_t M, int N, cudaStream_t s);
cudaError_t nt_tangent(const double *theta, const double *p, int64_t M, int N, double *d0, cudaStream_t s);
cudaError_t nt_axpy(const double *theta, const double *p, double a, int64_t n, double *X, cudaStream_t s);
cudaError_t nt_clamp_arc(const double *theta, const double *p, double a, const int32_t *m, int64_t M, int N,
                         double *T, int *neg, cudaStream_t s);
cudaError_t nt_transform(double *theta, int64_t M, int N, int32_t *m, cudaStream_t s);
cudaError_t nt_hdiag(int ntiles, int Ml, int64_t kb, int64_t M, const int32_t *tile_dA, const int32_t *tile_dB,
                     const int64_t *fb_off, const double *Fb, double gamma, double *h, cudaStream_t s);
cudaError_t nt_fparts(const double *R, int64_t nR, const double *theta, const double *g, int64_t M, int N,
                      double *part, double *out, cudaStream_t s);
}  // namespace qdt
