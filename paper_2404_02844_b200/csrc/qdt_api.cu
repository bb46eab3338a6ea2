// qdt_api.cu -- host runtime behind include/qdt.h: context, probe handle, Fock-axis shard
// and tile planner, memory plan, CUDA-graph iteration loop, NCCL exchange (multi-GPU).
//
// Every numerical step runs in the kernels of qdt_kernels.cu; this file only validates,
// plans, allocates, launches and copies.  There is no CPU compute path.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <map>
#include <mutex>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: phase ranges for nsys / ncu (no-ops without a tool)

#include "../../include/qdt.h"
#include "qdt_internal.h"

using namespace qdt;

// ------------------------------------------------------------------------------ NCCL (dlopen)
// NCCL is loaded at run time (libnccl.so.2, the copy torch already mapped when present) so
// that single-GPU use needs no NCCL at all.  Only the few entry points used are declared.
namespace {
typedef void *nccl_comm_t;
typedef struct { char internal[128]; } nccl_uid_t;
typedef int nccl_result_t;
enum { NCCL_FLOAT64 = 8, NCCL_SUM = 0 };
struct NcclApi {
    void *h = nullptr;
    nccl_result_t (*commInitRank)(nccl_comm_t *, int, nccl_uid_t, int) = nullptr;
    nccl_result_t (*commDestroy)(nccl_comm_t) = nullptr;
    nccl_result_t (*allReduce)(const void *, void *, size_t, int, int, nccl_comm_t,
                               cudaStream_t) = nullptr;
    nccl_result_t (*send)(const void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*recv)(void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*groupStart)() = nullptr;
    nccl_result_t (*getUniqueId)(nccl_uid_t *) = nullptr;
    nccl_result_t (*groupEnd)() = nullptr;
    const char *(*getErrorString)(nccl_result_t) = nullptr;
    nccl_result_t (*commGetAsyncError)(nccl_comm_t, nccl_result_t *) = nullptr;   // optional
    bool load(std::string &err)
    {
        if (h) return true;
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *n : names)
            if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) {
            err = "NCCL not found (dlopen libnccl.so.2 failed)";
            return false;
        }
#define QDT_SYM(f, s)                                              \
    *(void **)(&f) = dlsym(h, s);                                  \
    if (!f) {                                                      \
        err = std::string("NCCL symbol missing: ") + s;            \
        return false;                                              \
    }
        QDT_SYM(commInitRank, "ncclCommInitRank");
        QDT_SYM(commDestroy, "ncclCommDestroy");
        QDT_SYM(allReduce, "ncclAllReduce");
        QDT_SYM(send, "ncclSend");
        QDT_SYM(recv, "ncclRecv");
        QDT_SYM(groupStart, "ncclGroupStart");
        QDT_SYM(groupEnd, "ncclGroupEnd");
        QDT_SYM(getErrorString, "ncclGetErrorString");
        QDT_SYM(getUniqueId, "ncclGetUniqueId");
#undef QDT_SYM
        *(void **)(&commGetAsyncError) = dlsym(h, "ncclCommGetAsyncError");
        return true;
    }
};
NcclApi g_nccl;
}  // namespace

// ------------------------------------------------------------------------------ structures
// In-process group of virtual ranks (qdt_init_opts.comm = QDT_COMM_INPROC): one host thread per
// rank, every rank's device memory visible to the others (same device).  A barrier posts, per
// rank, one pointer / integer and an event recorded on that rank's stream at arrival; posting
// slots and events alternate by barrier parity, so a rank one barrier ahead never overwrites
// what a slower rank is still reading.
struct VGroup {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0, joined = 0;
    uint64_t gen = 0;
    const void *ptr[2][VMAX] = {};
    int64_t ival[2][VMAX] = {};
    cudaEvent_t ev[2][VMAX] = {};
};
static std::mutex g_vg_mu;
static std::map<int64_t, std::shared_ptr<VGroup>> g_vgroups;

struct DevBuf {
    void *p = nullptr;
    size_t n = 0;
};

struct qdt_ctx {
    int device = 0, rank = 0, nranks = 1;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    nccl_comm_t ncomm = nullptr;
    std::string err;
    bool profiling = false;
    std::map<std::string, std::pair<int64_t, double>> prof;
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    int64_t launches = 0;
    std::map<std::string, DevBuf> ws;  // grow-only workspace
    int nblkR = 148 * 4;
    int comm = 0;                      // QDT_COMM_NCCL / QDT_COMM_INPROC
    std::shared_ptr<VGroup> vg;        // in-process group
    cudaEvent_t vev[2] = {nullptr, nullptr};
    uint64_t vpar = 0;                 // barriers passed (parity selects slots / events)
    // the last instantiated solve-loop graph and the key it was captured under (configuration
    // + every device pointer it bakes in): a repeated qdt_solve with the same key replays it
    cudaGraphExec_t gexec = nullptr;
    std::vector<uint64_t> gkey;
    int64_t glaunches = 0;
};

static std::atomic<uint64_t> g_serial{1};   // unique ids of probe handles / plans (graph keys)

struct Plan {
    uint64_t serial = g_serial++;
    int N = 0, T = 0, CG = 0, RG = 0, TC = 0, KC = 0, KR = 0, TF = 0, nthr = 0, SEG = 32;
    int ntiles = 0;
    int32_t *d_tile_dA = nullptr, *d_tile_dB = nullptr;
    int nbunits = 0;
    BwdUnit *d_bunits = nullptr;
    int64_t nslots = 0;
    int nfunits = 0;
    FwdUnit *d_funits = nullptr;
    int64_t nrpart = 0;
    int64_t *d_red_beg = nullptr, *d_red_rows = nullptr;
    // sweep path (DMMA kernels, N <= 128): NB n-blocks; bwd/fwd units; reduce lists
    int NB = 0;
    int NW = 0;                       // wide-N sweep (N > 128, even, <= 1024): 128-column chunks
    // fused wide step (N > 128, even pitch): clusters of wx_C CTAs x wx_Wc columns per 32-row tile
    int NX = 0;
    int wx_C = 1, wx_Wc = 0, wx_ncl = 0;
    int32_t *d_wx_tlist = nullptr, *d_wx_toff = nullptr;
    bool gen = true;                  // general (CUDA-core) plan built (N <= 1024)
    int nR = 0;                       // partR entries written by the residual reduction
    int sw_nbunits = 0;
    SwUnit *d_swunits = nullptr;
    int64_t sw_nslots = 0;
    int sw_nfunits = 0;
    FwUnit *d_fwunits = nullptr;
    int64_t sw_nrpart = 0;
    int64_t *d_sw_red_beg = nullptr, *d_sw_red_rows = nullptr;
    ~Plan()
    {
        cudaFree(d_wx_tlist);
        cudaFree(d_wx_toff);
        cudaFree(d_swunits);
        cudaFree(d_fwunits);
        cudaFree(d_sw_red_beg);
        cudaFree(d_sw_red_rows);
        cudaFree(d_tile_dA);
        cudaFree(d_tile_dB);
        cudaFree(d_bunits);
        cudaFree(d_funits);
        cudaFree(d_red_beg);
        cudaFree(d_red_rows);
    }
};

struct qdt_probes {
    uint64_t serial = g_serial++;
    qdt_ctx *ctx = nullptr;
    int64_t D = 0, M = 0, kb = 0, ke = 0, Ml = 0;
    double c_sigma = 6.0;
    int margin = 16;
    double *d_alpha2 = nullptr;
    int32_t *d_lo = nullptr, *d_len = nullptr;
    int64_t *d_off = nullptr;
    double *d_val = nullptr;
    int64_t nnz = 0;
    std::vector<int32_t> lo_g, hi_g, lo_l, len_l;
    std::vector<int64_t> off;
    std::vector<int64_t> cuts;   // Fock-axis shard cuts of every rank (nranks + 1)
    std::vector<int64_t> dlo_r, dhi_r;   // per rank: probes [dlo_r[q], dhi_r[q]) touch rank q's slice
    double min_row_mass = 1.0;
    int64_t uncovered = 0;
    std::map<int, std::unique_ptr<Plan>> plans;
    // sweep tiling (independent of N): ST-row tiles, probe windows, tiled F blocks
    int sw_ntiles = 0;
    std::vector<int32_t> sw_dA, sw_dB;
    std::vector<int64_t> sw_fboff;
    int32_t *d_sw_dA = nullptr, *d_sw_dB = nullptr;
    int64_t *d_fb_off = nullptr;
    double *d_Fb = nullptr;
    int32_t *d_row_da = nullptr, *d_row_db = nullptr;   // probes covering each local row (small / coop solve)
    int64_t *d_toff = nullptr;                         // coop solve: transposed band offsets (Ml + 1)
    double *d_FT = nullptr;                            // coop solve: transposed band values (nnz)
    // step-setup cache (per probe handle): the step t_k per local row of the last (mode, gamma); F
    // is immutable, so a repeated solve reuses the SQS weights / the 100-step power iteration
    double *d_tcache = nullptr;
    int tc_mode = -1;
    double tc_gamma = NAN, tc_scalar = 0.0;
    Band band() const { return Band{d_lo, d_len, d_off, d_val}; }
    ~qdt_probes()
    {
        cudaFree(d_row_da);
        cudaFree(d_row_db);
        cudaFree(d_toff);
        cudaFree(d_FT);
        cudaFree(d_tcache);
        cudaFree(d_sw_dA);
        cudaFree(d_sw_dB);
        cudaFree(d_fb_off);
        cudaFree(d_Fb);
        cudaFree(d_alpha2);
        cudaFree(d_lo);
        cudaFree(d_len);
        cudaFree(d_off);
        cudaFree(d_val);
    }
};

// two CUDA events destroyed with their owner (every early return of a solve releases them)
struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaError_t create()
    {
        cudaError_t e = cudaEventCreate(&a);
        return e == cudaSuccess ? cudaEventCreate(&b) : e;
    }
    ~EventPair()
    {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

// NVTX range for the duration of a scope (solve phases: probes, setup, loop, evaluation, outputs)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// ------------------------------------------------------------------------------ errors
static thread_local std::string tl_err;

static qdt_status fail(qdt_ctx *ctx, qdt_status st, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    tl_err = buf;
    if (ctx) ctx->err = buf;
    return st;
}

#define CK(call)                                                                                \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? QDT_ERR_OOM : QDT_ERR_CUDA,      \
                        "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);   \
    } while (0)

#define CKN(call)                                                                               \
    do {                                                                                        \
        nccl_result_t r_ = (call);                                                              \
        if (r_ != 0)                                                                            \
            return fail(ctx, QDT_ERR_NCCL, "%s: %s", #call, g_nccl.getErrorString(r_));         \
    } while (0)

#define CKS(call)                            \
    do {                                     \
        qdt_status s_ = (call);              \
        if (s_ != QDT_OK) return s_;         \
    } while (0)

template <class T>
static qdt_status ws_get(qdt_ctx *ctx, const char *name, size_t count, T **out)
{
    DevBuf &b = ctx->ws[name];
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (b.n < bytes) {
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
        b.n = 0;
        cudaError_t e = cudaMalloc(&b.p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, QDT_ERR_OOM, "workspace '%s': cudaMalloc(%zu) failed: %s", name, bytes,
                        cudaGetErrorString(e));
        }
        b.n = bytes;
    }
    *out = (T *)b.p;
    return QDT_OK;
}

// kernel launch bookkeeping: counts launches; in profiling mode brackets with events
template <class F>
static cudaError_t run_k(qdt_ctx *ctx, const char *name, int nlaunch, F &&f)
{
    cudaEvent_t a = nullptr, b = nullptr;
    if (ctx->profiling) {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, ctx->stream);
    }
    cudaError_t e = f();
    ctx->launches += nlaunch;
    if (ctx->profiling) {
        cudaEventRecord(b, ctx->stream);
        ctx->pending.push_back({name, {a, b}});
    }
    return e;
}

static void flush_profile(qdt_ctx *ctx)
{
    if (ctx->pending.empty()) return;
    cudaStreamSynchronize(ctx->stream);
    for (auto &p : ctx->pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.second.first, p.second.second);
        auto &slot = ctx->prof[p.first];
        slot.first += 1;
        slot.second += ms;
        cudaEventDestroy(p.second.first);
        cudaEventDestroy(p.second.second);
    }
    ctx->pending.clear();
}

// ------------------------------------------------------------------------------ context
extern "C" qdt_status qdt_nccl_unique_id(void *out128)
{
    if (!out128) return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_nccl_unique_id: NULL");
    std::string err;
    if (!g_nccl.load(err)) return fail(nullptr, QDT_ERR_NCCL, "%s", err.c_str());
    nccl_uid_t uid;
    nccl_result_t r = g_nccl.getUniqueId(&uid);
    if (r != 0) return fail(nullptr, QDT_ERR_NCCL, "ncclGetUniqueId: %s", g_nccl.getErrorString(r));
    memcpy(out128, &uid, sizeof uid);
    return QDT_OK;
}

extern "C" qdt_status qdt_init(qdt_ctx **out, const qdt_init_opts *o)
{
    qdt_ctx *ctx = nullptr;
    if (!out) return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_init: ctx out-pointer is NULL");
    *out = nullptr;
    int dev = o ? o->device : 0;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, QDT_ERR_CUDA, "qdt_init: no CUDA device (%s)", cudaGetErrorString(e));
    }
    if (dev < 0 || dev >= ndev)
        return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_init: device %d out of range [0,%d)", dev,
                    ndev);
    std::unique_ptr<qdt_ctx> c(new qdt_ctx());
    ctx = c.get();
    c->device = dev;
    c->rank = o ? o->rank : 0;
    c->nranks = o ? std::max(1, o->nranks) : 1;
    if (c->rank < 0 || c->rank >= c->nranks)
        return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_init: rank %d not in [0,%d)", c->rank,
                    c->nranks);
    CK(cudaSetDevice(dev));
    if (o && o->cuda_stream) {
        c->stream = (cudaStream_t)o->cuda_stream;
    } else {
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    c->nblkR = nsm * 4;
    CK(prepare_kernels());
    CK(prepare_sweep_kernels());
    CK(prepare_wide_kernels());
    c->comm = (o && c->nranks > 1) ? o->comm : QDT_COMM_NCCL;
    if (c->nranks > 1 && c->comm == QDT_COMM_INPROC) {
        if (c->nranks > VMAX)
            return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_init: in-process groups have <= %d ranks", VMAX);
        CK(cudaEventCreateWithFlags(&c->vev[0], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->vev[1], cudaEventDisableTiming));
        {
            std::lock_guard<std::mutex> lk(g_vg_mu);
            auto &g = g_vgroups[o->group_key];
            if (!g) {
                g = std::make_shared<VGroup>();
                g->n = c->nranks;
            }
            if (g->n != c->nranks)
                return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_init: group %lld has %d ranks, not %d",
                            (long long)o->group_key, g->n, c->nranks);
            c->vg = g;
            if (++g->joined == g->n) g_vgroups.erase(o->group_key);   // complete: a later group may reuse the key
        }
        *out = c.release();
        return QDT_OK;
    }
    if (c->nranks > 1) {
        if (!o->nccl_unique_id)
            return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_init: nranks > 1 needs nccl_unique_id");
        std::string err;
        if (!g_nccl.load(err)) return fail(nullptr, QDT_ERR_NCCL, "qdt_init: %s", err.c_str());
        nccl_uid_t uid;
        memcpy(&uid, o->nccl_unique_id, sizeof uid);
        nccl_result_t r = g_nccl.commInitRank(&c->ncomm, c->nranks, uid, c->rank);
        if (r != 0)
            return fail(nullptr, QDT_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.getErrorString(r));
    }
    *out = c.release();
    return QDT_OK;
}

extern "C" qdt_status qdt_finalize(qdt_ctx *ctx)
{
    if (!ctx) return QDT_OK;
    cudaSetDevice(ctx->device);
    flush_profile(ctx);
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    for (auto &kv : ctx->ws) cudaFree(kv.second.p);
    if (ctx->ncomm) g_nccl.commDestroy(ctx->ncomm);
    if (ctx->vev[0]) cudaEventDestroy(ctx->vev[0]);
    if (ctx->vev[1]) cudaEventDestroy(ctx->vev[1]);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return QDT_OK;
}

extern "C" const char *qdt_last_error(const qdt_ctx *ctx)
{
    if (ctx && !ctx->err.empty()) return ctx->err.c_str();
    return tl_err.c_str();
}

extern "C" qdt_status qdt_profile_enable(qdt_ctx *ctx, int32_t enable)
{
    if (!ctx) return fail(nullptr, QDT_ERR_INVALID_ARG, "ctx is NULL");
    flush_profile(ctx);
    ctx->profiling = enable != 0;
    if (enable) ctx->prof.clear();
    return QDT_OK;
}

extern "C" qdt_status qdt_profile_get(qdt_ctx *ctx, const char *kernel, int64_t *count,
                                      double *total_ms)
{
    if (!ctx || !kernel) return fail(ctx, QDT_ERR_INVALID_ARG, "ctx/kernel is NULL");
    flush_profile(ctx);
    auto it = ctx->prof.find(kernel);
    if (count) *count = it == ctx->prof.end() ? 0 : it->second.first;
    if (total_ms) *total_ms = it == ctx->prof.end() ? 0.0 : it->second.second;
    return QDT_OK;
}

extern "C" qdt_status qdt_launch_count(qdt_ctx *ctx, int64_t *count)
{
    if (!ctx || !count) return fail(ctx, QDT_ERR_INVALID_ARG, "ctx/count is NULL");
    *count = ctx->launches;
    return QDT_OK;
}

// ------------------------------------------------------------------------------ collectives
// In-process barrier: post (p, iv) and an event of this rank's stream, wait for every rank; out
// gets every rank's posting, and this rank's stream then waits for every rank's event.
struct VPost {
    const void *p[VMAX];
    int64_t iv[VMAX];
};
static qdt_status vg_barrier(qdt_ctx *ctx, const void *p, int64_t iv, VPost *out)
{
    VGroup &g = *ctx->vg;
    const int par = (int)(ctx->vpar & 1);
    CK(cudaEventRecord(ctx->vev[par], ctx->stream));
    {
        std::unique_lock<std::mutex> lk(g.mu);
        g.ptr[par][ctx->rank] = p;
        g.ival[par][ctx->rank] = iv;
        g.ev[par][ctx->rank] = ctx->vev[par];
        const uint64_t my = g.gen;
        if (++g.arrived == g.n) {
            g.arrived = 0;
            g.gen++;
            g.cv.notify_all();
        } else {
            g.cv.wait(lk, [&] { return g.gen != my; });
        }
        for (int q = 0; q < g.n; q++) {
            if (out) {
                out->p[q] = g.ptr[par][q];
                out->iv[q] = g.ival[par][q];
            }
            if (q != ctx->rank) CK(cudaStreamWaitEvent(ctx->stream, g.ev[par][q], 0));
        }
    }
    ctx->vpar++;
    return QDT_OK;
}

static qdt_status allreduce(qdt_ctx *ctx, double *buf, size_t n, const char *name)
{
    if (ctx->nranks == 1 || n == 0) return QDT_OK;
    if (ctx->vg) {   // in-process: every rank sums all buffers in rank order, then copies back
        VPost post;
        CKS(vg_barrier(ctx, buf, (int64_t)n, &post));
        double *tmp;
        CKS(ws_get(ctx, "vsum_tmp", n, &tmp));
        VPtrs v;
        for (int q = 0; q < ctx->nranks; q++) v.p[q] = (const double *)post.p[q];
        CK(run_k(ctx, name, 1, [&]() { return launch_vsum(v, ctx->nranks, (int64_t)n, tmp, ctx->stream); }));
        CKS(vg_barrier(ctx, nullptr, 0, nullptr));   // every rank has read every buffer
        CK(cudaMemcpyAsync(buf, tmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        return QDT_OK;
    }
    nccl_result_t r = 0;
    cudaError_t e = run_k(ctx, name, 1, [&]() {
        r = g_nccl.allReduce(buf, buf, n, NCCL_FLOAT64, NCCL_SUM, ctx->ncomm, ctx->stream);
        return cudaSuccess;
    });
    (void)e;
    if (r != 0) return fail(ctx, QDT_ERR_NCCL, "ncclAllReduce(%s): %s", name, g_nccl.getErrorString(r));
    return QDT_OK;
}

// All-gather of the row slices: full (M x N, pitch N) receives every rank's slice rows
// [cuts[g], cuts[g+1]) at its place; src: this rank's local rows.  NCCL: grouped send/recv of
// the slices (no zero-padded allreduce of the whole matrix).
static qdt_status gather_rows(qdt_ctx *ctx, const qdt_probes *p, const double *src, int64_t N, double *full)
{
    CK(cudaMemcpyAsync(full + p->kb * N, src, sizeof(double) * p->Ml * N, cudaMemcpyDeviceToDevice, ctx->stream));
    if (ctx->nranks == 1) return QDT_OK;
    if (ctx->vg) {
        VPost post;
        CKS(vg_barrier(ctx, src, 0, &post));
        for (int q = 0; q < ctx->nranks; q++)
            if (q != ctx->rank)
                CK(cudaMemcpyAsync(full + p->cuts[q] * N, post.p[q], sizeof(double) * (p->cuts[q + 1] - p->cuts[q]) * N,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
        CKS(vg_barrier(ctx, nullptr, 0, nullptr));
        return QDT_OK;
    }
    nccl_result_t e = 0;
    run_k(ctx, "gather", 1, [&]() {
        g_nccl.groupStart();
        for (int q = 0; q < ctx->nranks; q++) {
            if (q == ctx->rank) continue;
            const int64_t qb = p->cuts[q], qe = p->cuts[q + 1];
            e |= g_nccl.send(src, (size_t)(p->Ml * N), NCCL_FLOAT64, q, ctx->ncomm, ctx->stream);
            e |= g_nccl.recv(full + qb * N, (size_t)((qe - qb) * N), NCCL_FLOAT64, q, ctx->ncomm, ctx->stream);
        }
        e |= g_nccl.groupEnd();
        return cudaSuccess;
    });
    if (e != 0) return fail(ctx, QDT_ERR_NCCL, "row gather failed");
    return QDT_OK;
}

// NCCL communicator health (polled with the stop flag): an asynchronous error (a peer died, a
// network failure) fails the solve instead of hanging it
static qdt_status nccl_health(qdt_ctx *ctx)
{
    if (!ctx->ncomm || !g_nccl.commGetAsyncError) return QDT_OK;
    nccl_result_t ae = 0;
    const nccl_result_t r = g_nccl.commGetAsyncError(ctx->ncomm, &ae);
    if (r != 0 || ae != 0)
        return fail(ctx, QDT_ERR_NCCL, "NCCL asynchronous error: %s", g_nccl.getErrorString(r ? r : ae));
    return QDT_OK;
}

// ------------------------------------------------------------------------------ planner
// Fock-axis shard cut (multi-GPU): contiguous [k_g, k_{g+1}) at equal prefix sums of the
// per-row cost c(k) = 16 + 0.7 cov(k) (bytes-equivalent per column).
static void shard_bounds(const std::vector<int32_t> &lo, const std::vector<int32_t> &hi, int64_t M,
                         int nranks, std::vector<int64_t> &cuts)
{
    std::vector<int64_t> diff(M + 1, 0);
    for (size_t d = 0; d < lo.size(); d++) {
        diff[lo[d]] += 1;
        diff[(int64_t)hi[d] + 1] -= 1;
    }
    std::vector<double> pre(M + 1, 0.0);
    int64_t cov = 0;
    for (int64_t k = 0; k < M; k++) {
        cov += diff[k];
        pre[k + 1] = pre[k] + 16.0 + 0.7 * (double)cov;
    }
    cuts.assign(nranks + 1, 0);
    cuts[nranks] = M;
    for (int g = 1; g < nranks; g++) {
        double target = pre[M] * g / nranks;
        int64_t k = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
        cuts[g] = std::min<int64_t>(std::max<int64_t>(k, cuts[g - 1] + 1), M);
    }
    for (int g = 1; g <= nranks; g++) cuts[g] = std::max(cuts[g], cuts[g - 1]);
}

extern "C" qdt_status qdt_shard_cuts(const int64_t *lo, const int64_t *hi, int64_t D, int64_t M,
                                     int32_t nranks, int64_t *cuts)
{
    if (!lo || !hi || !cuts || D < 1 || M < 1 || nranks < 1)
        return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_shard_cuts: bad arguments");
    std::vector<int32_t> l(D), h(D);
    for (int64_t d = 0; d < D; d++) {
        if (lo[d] < 0 || hi[d] < lo[d] || hi[d] >= M)
            return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_shard_cuts: band %lld invalid", (long long)d);
        l[d] = (int32_t)lo[d];
        h[d] = (int32_t)hi[d];
    }
    std::vector<int64_t> c;
    shard_bounds(l, h, M, nranks, c);
    for (int g = 0; g <= nranks; g++) cuts[g] = c[g];
    return QDT_OK;
}

// Sweep tiling of the local slice (once per probe handle): ST-row tiles, their contiguous probe
// windows [dA, dB) and the tiled F blocks (W_t x STP doubles, zero outside each band).
static qdt_status build_sweep_tiling(qdt_ctx *ctx, qdt_probes *p)
{
    if (p->d_Fb) return QDT_OK;
    const int64_t Ml = p->Ml, kb = p->kb, D = p->D;
    const int nt = (int)((Ml + ST - 1) / ST);
    p->sw_ntiles = nt;
    p->sw_dA.assign(nt, INT32_MAX);
    p->sw_dB.assign(nt, 0);
    for (int64_t d = 0; d < D; d++) {
        if (p->len_l[d] == 0) continue;
        const int64_t a = (p->lo_l[d] - kb) / ST, b = (p->lo_l[d] + p->len_l[d] - 1 - kb) / ST;
        for (int64_t t = a; t <= b; t++) {
            p->sw_dA[t] = std::min<int32_t>(p->sw_dA[t], (int32_t)d);
            p->sw_dB[t] = std::max<int32_t>(p->sw_dB[t], (int32_t)d + 1);
        }
    }
    for (int t = 0; t < nt; t++)
        if (p->sw_dA[t] == INT32_MAX) p->sw_dA[t] = p->sw_dB[t] = (t > 0 ? p->sw_dB[t - 1] : 0);
    p->sw_fboff.assign(nt + 1, 0);
    for (int t = 0; t < nt; t++) p->sw_fboff[t + 1] = p->sw_fboff[t] + (int64_t)(p->sw_dB[t] - p->sw_dA[t]) * STP;
    cudaStream_t s = ctx->stream;
    CK(cudaMalloc(&p->d_sw_dA, sizeof(int32_t) * nt));
    CK(cudaMalloc(&p->d_sw_dB, sizeof(int32_t) * nt));
    CK(cudaMalloc(&p->d_fb_off, sizeof(int64_t) * (nt + 1)));
    CK(cudaMalloc(&p->d_Fb, sizeof(double) * std::max<int64_t>(2, p->sw_fboff[nt] + 2)));
    CK(cudaMemcpyAsync(p->d_sw_dA, p->sw_dA.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(p->d_sw_dB, p->sw_dB.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(p->d_fb_off, p->sw_fboff.data(), sizeof(int64_t) * (nt + 1), cudaMemcpyHostToDevice, s));
    CK(run_k(ctx, "tile_F", 1, [&]() {
        return launch_tile_F(p->band(), kb, (int)Ml, nt, p->d_sw_dA, p->d_sw_dB, p->d_fb_off, p->d_Fb, s);
    }));
    CK(cudaStreamSynchronize(s));
    return QDT_OK;
}

static bool sweep_enabled()
{
    const char *e = getenv("QDT_SWEEP");
    return !(e && e[0] == '0');
}

// Forward units over tiles [t0, t1), emitted in ascending Fock order (so that every probe's
// partial rows are listed in ascending Fock order):
//  - narrow windows: runs of consecutive tiles whose union window is <= FWCAP probes (<= FW_MAXT
//    tiles): one partial row per (run, probe);
//  - runs of wide windows (> FWCAP probes, low Fock rows / wide N): probe-major, groups of FWCAP
//    consecutive probes over the tiles their bands touch (<= FW_MAXT tiles per unit), so that a
//    probe gets one partial row per group unit instead of one per tile.
template <class Emit>
static void plan_fwd_units(const qdt_probes *p, int t0, int t1, Emit &&emit, int maxt = FW_MAXT)
{
    const int FW_MAXT = maxt;   // tiles per unit (fewer on small problems: more units for the SMs)
    const std::vector<int32_t> &dA = p->sw_dA, &dB = p->sw_dB;
    int t = t0;
    while (t < t1) {
        if (dB[t] <= dA[t]) {
            t++;
            continue;
        }
        if (dB[t] - dA[t] <= FWCAP) {
            const int g0 = t, u0 = dA[t];
            int u1 = dB[t];
            t++;
            while (t < t1 && dB[t] > dA[t] && dB[t] - dA[t] <= FWCAP && std::max(u1, (int)dB[t]) - u0 <= FWCAP &&
                   t - g0 < FW_MAXT) {
                u1 = std::max(u1, (int)dB[t]);
                t++;
            }
            emit(g0, t, u0, u1);
            continue;
        }
        const int r0 = t;
        while (t < t1 && dB[t] - dA[t] > FWCAP) t++;
        const int r1 = t;                       // wide run [r0, r1)
        const int P0 = dA[r0], P1 = dB[r1 - 1];
        int ta = r0;
        for (int g0 = P0; g0 < P1; g0 += FWCAP) {
            const int g1 = std::min(P1, g0 + FWCAP);
            while (ta < r1 && dB[ta] <= g0) ta++;          // first tile meeting the group
            int tb = ta;
            while (tb < r1 && dA[tb] < g1) tb++;           // one past the last
            for (int c0 = ta; c0 < tb; c0 += FW_MAXT) emit(c0, std::min(tb, c0 + FW_MAXT), g0, g1);
        }
    }
}


// split cap of the k_grad_wide units (N > 128, plans without k_bwd_mma): every split unit writes
// and re-reads a 64 x 128 fragment-ordered partial per column chunk (64 KB), which at the SWCAP of
// k_bwd_mma (128) was ~0.6 GB of scratch traffic per Large gradient (ncu DRAM 1.02 GB against
// 0.35 GB algorithmic).  Measured at Large (profiles/r02_v7): cap 128 0.551 ms, 256 0.419, 512
// 0.373, 1024 0.361, 2048 0.361, 4096 0.409, unsplit 1.21 (the 12 746-probe tile 0 serialises).
// QDT_WIDE_SWCAP overrides (A/B).
constexpr int WIDE_SWCAP = 2048;
static int wide_swcap()
{
    static const int cap = [] {
        const char *e = getenv("QDT_WIDE_SWCAP");
        const int v = e ? atoi(e) : 0;
        return v >= SKC ? (v / SKC) * SKC : WIDE_SWCAP;
    }();
    return cap;
}

// Sweep units for N: bwd units (tile, probe sub-range <= SWCAP, split-K slots), fwd units (runs
// of <= FW_MAXT tiles whose union window is <= FWCAP probes; wider windows split by FWCAP), and
// per-probe lists of partial rows in ascending Fock order.
static qdt_status build_sweep_plan(qdt_ctx *ctx, qdt_probes *p, Plan *pl)
{
    CKS(build_sweep_tiling(ctx, p));
    const int nt = p->sw_ntiles;
    const int64_t D = p->D;
    const int nsm = device_sm_count();
    // split cap of the bwd units (a smaller cap for small problems measured slower: the split-K
    // fix-up sums more slots, profiles/r02_v3)
    const int cap = (pl->NW && !pl->NB) ? wide_swcap() : SWCAP;   // k_bwd_mma (NB) keeps SWCAP
    std::vector<SwUnit> bu;
    int64_t slot = 0;
    for (int t = 0; t < nt; t++) {
        const int dA = p->sw_dA[t], W = p->sw_dB[t] - dA;
        const int ns = std::max(1, (W + cap - 1) / cap);
        int chunk = ns > 1 ? (W + ns - 1) / ns : W;
        if (ns > 1) chunk = ((chunk + SKC - 1) / SKC) * SKC;
        for (int s = 0; s < ns; s++) {
            SwUnit u;
            u.tile = t;
            u.p0 = std::min(dA + s * chunk, dA + W);
            u.p1 = std::min(dA + W, u.p0 + chunk);
            u.slot = s;
            u.nsplit = ns;
            u.pad = 0;
            u.slot_base = ns > 1 ? slot : 0;
            bu.push_back(u);
        }
        if (ns > 1) slot += ns;
    }
    pl->sw_nslots = slot;
    std::stable_sort(bu.begin(), bu.end(),
                     [](const SwUnit &x, const SwUnit &y) { return (x.p1 - x.p0) > (y.p1 - y.p0); });
    pl->sw_nbunits = (int)bu.size();

    std::vector<FwUnit> fu;
    std::vector<std::vector<int64_t>> lists(D);
    int64_t poff = 0;
    auto emit = [&](int t0, int t1, int u0, int u1) {
        if (u1 <= u0) return;
        FwUnit u;
        u.t0 = t0;
        u.t1 = t1;
        u.u0 = u0;
        u.u1 = u1;
        u.poff = poff;
        fu.push_back(u);
        for (int d = u0; d < u1; d++) lists[d].push_back(poff + (d - u0));
        poff += u1 - u0;
    };
    // tiles per fwd unit: FW_MAXT, halved while the plan gives fewer than 2 units per SM
    int maxt = FW_MAXT;
    for (;;) {
        int64_t nu = 0;
        plan_fwd_units(p, 0, nt, [&](int, int, int u0, int u1) { nu += u1 > u0; }, maxt);
        if (nu >= 2 * nsm || maxt <= 1) break;
        maxt /= 2;
    }
    plan_fwd_units(p, 0, nt, emit, maxt);
    pl->sw_nrpart = poff;
    std::vector<int64_t> red_beg(D + 1, 0), red_rows;
    for (int64_t d = 0; d < D; d++) red_beg[d + 1] = red_beg[d] + (int64_t)lists[d].size();
    red_rows.reserve(red_beg[D]);
    for (int64_t d = 0; d < D; d++) red_rows.insert(red_rows.end(), lists[d].begin(), lists[d].end());
    std::stable_sort(fu.begin(), fu.end(), [](const FwUnit &x, const FwUnit &y) {
        return (int64_t)(x.u1 - x.u0) * (x.t1 - x.t0) > (int64_t)(y.u1 - y.u0) * (y.t1 - y.t0);
    });
    pl->sw_nfunits = (int)fu.size();
    cudaStream_t s = ctx->stream;
    CK(cudaMalloc(&pl->d_swunits, sizeof(SwUnit) * std::max<size_t>(1, bu.size())));
    CK(cudaMalloc(&pl->d_fwunits, sizeof(FwUnit) * std::max<size_t>(1, fu.size())));
    CK(cudaMalloc(&pl->d_sw_red_beg, sizeof(int64_t) * (D + 1)));
    CK(cudaMalloc(&pl->d_sw_red_rows, sizeof(int64_t) * std::max<size_t>(1, red_rows.size())));
    if (!bu.empty()) CK(cudaMemcpyAsync(pl->d_swunits, bu.data(), sizeof(SwUnit) * bu.size(), cudaMemcpyHostToDevice, s));
    if (!fu.empty()) CK(cudaMemcpyAsync(pl->d_fwunits, fu.data(), sizeof(FwUnit) * fu.size(), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(pl->d_sw_red_beg, red_beg.data(), sizeof(int64_t) * (D + 1), cudaMemcpyHostToDevice, s));
    if (!red_rows.empty())
        CK(cudaMemcpyAsync(pl->d_sw_red_rows, red_rows.data(), sizeof(int64_t) * red_rows.size(),
                           cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    return QDT_OK;
}

// QDT_SMALL=0 keeps small problems on the multi-kernel loop (A/B)
static bool small_enabled()
{
    const char *e = getenv("QDT_SMALL");
    return !(e && e[0] == '0');
}

// QDT_COOP=0 keeps latency-bound problems on the multi-kernel loop (A/B)
static bool coop_enabled()
{
    const char *e = getenv("QDT_COOP");
    return !(e && e[0] == '0');
}
constexpr int64_t COOP_MAX_ROWS = 16384;   // grid-persistent solve: Fock rows of a latency-bound problem

// QDT_WIDE=new selects the fused cluster step at every N > 128 (A/B, tests); N > 1024 always takes it
static bool wide_new_forced()
{
    const char *e = getenv("QDT_WIDE");   // read at every plan build (plans are cached per probe handle and N)
    return e && !strcmp(e, "new");
}

// Fused wide step (qdt_wide.cu): C CTAs per cluster, Wc columns each (multiple of 8, <= 640), the
// 16-row tiles of the slice list-scheduled over the co-resident clusters: tiles in Fock order, each
// to the cluster whose work so far is least (cost = window probes + a fixed epilogue share), so
// that every cluster's list is in Fock order and the clusters sweep the axis together (the R rows
// of the moving window are shared in L2).  C: the fewest CTAs with Wc <= 640, raised while the
// slice has few tiles per cluster and the per-CTA chunk stays >= 128 columns.
static qdt_status build_wide_plan(qdt_ctx *ctx, qdt_probes *p, Plan *pl)
{
    const int N = pl->N;
    const int nbt = (N + 7) / 8;                                   // n-blocks of the row
    const int ntw = (int)((p->Ml + WT - 1) / WT);
    auto wc_of = [&](int C) { return 8 * ((nbt + C - 1) / C); };
    const int wmax = 8 * W_NG * W_NBW_MAX;                          // 640 columns per CTA
    int C = (N + wmax - 1) / wmax;
    if (C > W_CMAX) return fail(ctx, QDT_ERR_INVALID_ARG, "N = %d exceeds the fused wide step (max %d)", N, W_CMAX * wmax);
    const int nsm = device_sm_count();
    while (C < W_CMAX && wc_of(C + 1) >= 128 && (int64_t)ntw < 6LL * (nsm / C)) C++;
    while (C > 1 && (int64_t)(C - 1) * wc_of(C) >= N) C--;           // every CTA owns >= 1 column pair
    const int Wc = wc_of(C);
    int ncl = wide_max_clusters(C, Wc);
    if (ncl <= 0) return fail(ctx, QDT_ERR_CUDA, "fused wide step: no co-resident cluster of %d CTAs", C);
    ncl = std::min(ncl, std::max(1, ntw));
    // list scheduling in Fock order (min-heap of (work, cluster))
    const int64_t E = 48;   // epilogue share of a tile, in window probes (measured order of magnitude)
    std::vector<std::vector<int32_t>> lists(ncl);
    std::vector<std::pair<int64_t, int>> heap;
    for (int c = 0; c < ncl; c++) heap.push_back({0, c});
    auto cmp = [](const std::pair<int64_t, int> &x, const std::pair<int64_t, int> &y) { return x > y; };
    std::make_heap(heap.begin(), heap.end(), cmp);
    for (int tt = 0; tt < ntw; tt++) {
        const int t64 = tt >> 2;
        std::pop_heap(heap.begin(), heap.end(), cmp);
        auto &h = heap.back();
        lists[h.second].push_back(tt);
        h.first += (p->sw_dB[t64] - p->sw_dA[t64]) + E;
        std::push_heap(heap.begin(), heap.end(), cmp);
    }
    std::vector<int32_t> tl, off(ncl + 1, 0);
    tl.reserve(ntw);
    for (int c = 0; c < ncl; c++) {
        tl.insert(tl.end(), lists[c].begin(), lists[c].end());
        off[c + 1] = (int32_t)tl.size();
    }
    pl->wx_C = C;
    pl->wx_Wc = Wc;
    pl->wx_ncl = ncl;
    CK(cudaMalloc(&pl->d_wx_tlist, sizeof(int32_t) * std::max<size_t>(1, tl.size())));
    CK(cudaMalloc(&pl->d_wx_toff, sizeof(int32_t) * (ncl + 1)));
    if (!tl.empty()) CK(cudaMemcpy(pl->d_wx_tlist, tl.data(), sizeof(int32_t) * tl.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(pl->d_wx_toff, off.data(), sizeof(int32_t) * (ncl + 1), cudaMemcpyHostToDevice));
    return QDT_OK;
}

// N > GEN_NMAX: only the DMMA forward + fused wide step exist
static qdt_status build_wide_only_plan(qdt_ctx *ctx, qdt_probes *p, int N, std::unique_ptr<Plan> pl, Plan **out)
{
    if (!sweep_enabled() || N % 2) return fail(ctx, QDT_ERR_INVALID_ARG, "N = %d needs the sweep kernels (even pitch)", N);
    pl->NX = 1;
    CKS(build_sweep_plan(ctx, p, pl.get()));
    CKS(build_wide_plan(ctx, p, pl.get()));
    pl->nR = ctx->nranks == 1 ? (int)((p->D + 7) / 8) : ctx->nblkR;
    *out = pl.get();
    p->plans[N] = std::move(pl);
    return QDT_OK;
}

static qdt_status build_plan(qdt_ctx *ctx, qdt_probes *p, int N, Plan **out)
{
    auto it = p->plans.find(N);
    if (it != p->plans.end()) {
        *out = it->second.get();
        return QDT_OK;
    }
    std::unique_ptr<Plan> pl(new Plan());
    pl->N = N;
    pl->gen = N <= GEN_NMAX;   // the CUDA-core kernels (hooks, Newton) stop at 1024 outcomes
    if (!pl->gen) return build_wide_only_plan(ctx, p, N, std::move(pl), out);
    pl->nthr = bwd_threads(N, &pl->CG, &pl->RG, &pl->TC);
    if (pl->CG * pl->RG > 1024)
        return fail(ctx, QDT_ERR_INVALID_ARG, "N = %d too large for the general kernels", N);
    pl->T = pl->RG * TR;
    // row-epilogue segment: smallest power of two with ceil(N/SEG) <= 16 values per lane
    pl->SEG = 1;
    while (pl->SEG < 32 && (N + pl->SEG - 1) / pl->SEG > 16) pl->SEG <<= 1;
    pl->KC = std::min(32, std::max(2, 800 / N));
    pl->KR = std::min(32, std::max(4, 2048 / N));
    pl->TF = 256;
    const int64_t Ml = p->Ml, kb = p->kb, D = p->D;
    const int T = pl->T, TF = pl->TF, KP = pl->RG * TR;

    // ---- bwd tiles and windows
    const int ntiles = (int)((Ml + T - 1) / T);
    pl->ntiles = ntiles;
    std::vector<int32_t> dA(ntiles, INT32_MAX), dB(ntiles, 0);
    for (int64_t d = 0; d < D; d++) {
        if (p->len_l[d] == 0) continue;
        int64_t a = (p->lo_l[d] - kb) / T, b = (p->lo_l[d] + p->len_l[d] - 1 - kb) / T;
        for (int64_t t = a; t <= b; t++) {
            dA[t] = std::min<int32_t>(dA[t], (int32_t)d);
            dB[t] = std::max<int32_t>(dB[t], (int32_t)d + 1);
        }
    }
    for (int t = 0; t < ntiles; t++)
        if (dA[t] == INT32_MAX) dA[t] = dB[t] = 0;
    // split cap: windows wider than Wcap probes are split along the probe axis
    const int Wcap = std::min(WCAP_MAX, std::max(64, 4 * pl->KC));
    std::vector<BwdUnit> bu;
    bu.reserve(ntiles + 64);
    int64_t slot = 0;
    for (int t = 0; t < ntiles; t++) {
        int W = dB[t] - dA[t];
        int ns = std::max(1, (W + Wcap - 1) / Wcap);
        int chunk = ns > 1 ? (W + ns - 1) / ns : W;
        for (int s = 0; s < ns; s++) {
            BwdUnit u;
            u.k0 = t * T;
            u.k1 = (int32_t)std::min<int64_t>(Ml, (int64_t)(t + 1) * T);
            u.p0 = dA[t] + s * chunk;
            u.p1 = std::min(dB[t], u.p0 + chunk);
            if (u.p1 < u.p0) u.p1 = u.p0;
            u.tile = t;
            u.slot = s;
            u.nsplit = ns;
            u.pad = 0;
            u.slot_base = ns > 1 ? slot : 0;
            bu.push_back(u);
        }
        if (ns > 1) slot += ns;
    }
    pl->nslots = slot;
    // heavy (widest probe range) units first
    std::stable_sort(bu.begin(), bu.end(),
                     [](const BwdUnit &x, const BwdUnit &y) { return (x.p1 - x.p0) > (y.p1 - y.p0); });
    pl->nbunits = (int)bu.size();

    // ---- fwd tiles, probe groups, per-probe partial-row lists
    const int nft = (int)((Ml + TF - 1) / TF);
    std::vector<int32_t> fA(nft, INT32_MAX), fB(nft, 0);
    for (int64_t d = 0; d < D; d++) {
        if (p->len_l[d] == 0) continue;
        int64_t a = (p->lo_l[d] - kb) / TF, b = (p->lo_l[d] + p->len_l[d] - 1 - kb) / TF;
        for (int64_t t = a; t <= b; t++) {
            fA[t] = std::min<int32_t>(fA[t], (int32_t)d);
            fB[t] = std::max<int32_t>(fB[t], (int32_t)d + 1);
        }
    }
    std::vector<FwdUnit> fu;
    std::vector<std::vector<int64_t>> lists(D);
    int64_t poff = 0;
    for (int t = 0; t < nft; t++) {
        if (fA[t] == INT32_MAX) continue;
        const int64_t r0 = (int64_t)t * TF, r1 = std::min<int64_t>(Ml, r0 + TF);
        for (int g0 = fA[t]; g0 < fB[t]; g0 += KP) {
            const int g1 = std::min(fB[t], g0 + KP);
            int64_t k0 = INT64_MAX, k1 = -1;
            for (int d = g0; d < g1; d++) {
                if (p->len_l[d] == 0) continue;
                int64_t a = std::max<int64_t>(r0, p->lo_l[d] - kb);
                int64_t b = std::min<int64_t>(r1, p->lo_l[d] + p->len_l[d] - kb);
                if (a >= b) continue;
                k0 = std::min(k0, a);
                k1 = std::max(k1, b);
                lists[d].push_back(poff + (d - g0));
            }
            if (k1 < 0) continue;
            FwdUnit u;
            u.k0 = (int32_t)k0;
            u.k1 = (int32_t)k1;
            u.p0 = g0;
            u.p1 = g1;
            u.poff = poff;
            fu.push_back(u);
            poff += g1 - g0;
        }
    }
    pl->nrpart = poff;
    std::stable_sort(fu.begin(), fu.end(), [](const FwdUnit &x, const FwdUnit &y) {
        return (int64_t)(x.p1 - x.p0) * (x.k1 - x.k0) > (int64_t)(y.p1 - y.p0) * (y.k1 - y.k0);
    });
    pl->nfunits = (int)fu.size();
    std::vector<int64_t> red_beg(D + 1, 0), red_rows;
    for (int64_t d = 0; d < D; d++) red_beg[d + 1] = red_beg[d] + (int64_t)lists[d].size();
    red_rows.reserve(red_beg[D]);
    for (int64_t d = 0; d < D; d++) red_rows.insert(red_rows.end(), lists[d].begin(), lists[d].end());

    // ---- upload
    CK(cudaMalloc(&pl->d_tile_dA, sizeof(int32_t) * std::max(1, ntiles)));
    CK(cudaMalloc(&pl->d_tile_dB, sizeof(int32_t) * std::max(1, ntiles)));
    CK(cudaMalloc(&pl->d_bunits, sizeof(BwdUnit) * std::max<size_t>(1, bu.size())));
    CK(cudaMalloc(&pl->d_funits, sizeof(FwdUnit) * std::max<size_t>(1, fu.size())));
    CK(cudaMalloc(&pl->d_red_beg, sizeof(int64_t) * (D + 1)));
    CK(cudaMalloc(&pl->d_red_rows, sizeof(int64_t) * std::max<size_t>(1, red_rows.size())));
    cudaStream_t s = ctx->stream;
    CK(cudaMemcpyAsync(pl->d_tile_dA, dA.data(), sizeof(int32_t) * ntiles, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(pl->d_tile_dB, dB.data(), sizeof(int32_t) * ntiles, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(pl->d_bunits, bu.data(), sizeof(BwdUnit) * bu.size(), cudaMemcpyHostToDevice, s));
    if (!fu.empty())
        CK(cudaMemcpyAsync(pl->d_funits, fu.data(), sizeof(FwdUnit) * fu.size(), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(pl->d_red_beg, red_beg.data(), sizeof(int64_t) * (D + 1), cudaMemcpyHostToDevice, s));
    if (!red_rows.empty())
        CK(cudaMemcpyAsync(pl->d_red_rows, red_rows.data(), sizeof(int64_t) * red_rows.size(),
                           cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    pl->NB = sweep_enabled() ? sweep_nb(N) : 0;
    // wide kernels for N > 128 (even): the whole path, or (N <= 160) beside the NB > 16 plain step
    const bool wide = sweep_enabled() && (!pl->NB || pl->NB > SW_NBMAX) && N % 2 == 0;
    // N <= 1024: the fused step where the axis gives many tiles and the rows are wide (stress_cut,
    // M = 10^5 x N = 10^3: 1.87 against 2.02 ms per iteration), the two-kernel wide sweep otherwise
    // (Large, M = 10^4: heavy low-k windows with few tiles favour its split-K units)
    pl->NX = (wide && (wide_new_forced() || (N > 512 && p->Ml >= 32768))) ? 1 : 0;
    pl->NW = (wide && !pl->NX && N <= 1024) ? 1 : 0;
    if (pl->NB || pl->NW || pl->NX) CKS(build_sweep_plan(ctx, p, pl.get()));
    if (pl->NX) CKS(build_wide_plan(ctx, p, pl.get()));
    pl->nR = ctx->nranks == 1 ? (int)((D + 7) / 8) : ctx->nblkR;
    *out = pl.get();
    p->plans[N] = std::move(pl);
    return QDT_OK;
}

// Shard, local band tables and values of a probe handle whose global edges lo_g / hi_g are set:
// values from the S0 kernel (vals == nullptr: p->d_alpha2 holds mu) or copied from host vals
// (global probe-major bands, qdt_probes_from_banded).
static qdt_status finish_probes(qdt_ctx *ctx, qdt_probes *p, const double *vals)
{
    cudaStream_t s = ctx->stream;
    const int64_t D = p->D, M = p->M;
    // shard the Fock axis
    std::vector<int64_t> &cuts = p->cuts;
    shard_bounds(p->lo_g, p->hi_g, M, ctx->nranks, cuts);
    p->kb = cuts[ctx->rank];
    p->ke = cuts[ctx->rank + 1];
    p->dlo_r.assign(ctx->nranks, 0);
    p->dhi_r.assign(ctx->nranks, 0);
    for (int q = 0; q < ctx->nranks; q++) {   // band edges are monotone: contiguous probe ranges
        int64_t a = D, b = 0;
        for (int64_t d = 0; d < D; d++)
            if (p->lo_g[d] < cuts[q + 1] && p->hi_g[d] >= cuts[q]) {
                a = std::min(a, d);
                b = std::max(b, d + 1);
            }
        p->dlo_r[q] = a < b ? a : 0;
        p->dhi_r[q] = a < b ? b : 0;
    }
    p->Ml = p->ke - p->kb;
    if (p->Ml < 1) return fail(ctx, QDT_ERR_INVALID_ARG, "rank %d owns no Fock rows (M too small)", ctx->rank);
    p->lo_l.resize(D);
    p->len_l.resize(D);
    p->off.resize(D + 1);
    p->off[0] = 0;
    for (int64_t d = 0; d < D; d++) {
        int64_t a = std::max<int64_t>(p->lo_g[d], p->kb), b = std::min<int64_t>(p->hi_g[d], p->ke - 1);
        p->lo_l[d] = (int32_t)a;
        p->len_l[d] = b >= a ? (int32_t)(b - a + 1) : 0;
        p->off[d + 1] = p->off[d] + p->len_l[d];
    }
    p->nnz = p->off[D];
    {   // uncovered rows of this slice (reading R9)
        std::vector<int32_t> diff(p->Ml + 1, 0);
        for (int64_t d = 0; d < D; d++)
            if (p->len_l[d]) {
                diff[p->lo_l[d] - p->kb] += 1;
                diff[p->lo_l[d] - p->kb + p->len_l[d]] -= 1;
            }
        int64_t c = 0, unc = 0;
        for (int64_t k = 0; k < p->Ml; k++) {
            c += diff[k];
            unc += (c == 0);
        }
        p->uncovered = unc;
    }
    CK(cudaMemcpyAsync(p->d_lo, p->lo_l.data(), sizeof(int32_t) * D, cudaMemcpyHostToDevice, s));
    CK(cudaMalloc(&p->d_len, sizeof(int32_t) * D));
    CK(cudaMemcpyAsync(p->d_len, p->len_l.data(), sizeof(int32_t) * D, cudaMemcpyHostToDevice, s));
    CK(cudaMalloc(&p->d_off, sizeof(int64_t) * (D + 1)));
    CK(cudaMemcpyAsync(p->d_off, p->off.data(), sizeof(int64_t) * (D + 1), cudaMemcpyHostToDevice, s));
    CK(cudaMalloc(&p->d_val, sizeof(double) * std::max<int64_t>(1, p->nnz)));
    if (vals) {   // host values of the global bands: keep this slice's part of each band
        std::vector<double> hv(std::max<int64_t>(1, p->nnz));
        int64_t go = 0;
        for (int64_t d = 0; d < D; d++) {
            if (p->len_l[d]) memcpy(hv.data() + p->off[d], vals + go + (p->lo_l[d] - p->lo_g[d]), sizeof(double) * p->len_l[d]);
            go += (int64_t)p->hi_g[d] - p->lo_g[d] + 1;
        }
        CK(cudaMemcpyAsync(p->d_val, hv.data(), sizeof(double) * p->nnz, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    } else {   // S0 (b): values on the device
        CK(run_k(ctx, "probe_values", 1, [&]() { return launch_probe_values(p->d_alpha2, D, p->band(), s); }));
    }
    // stored mass per probe (diagnostic; summed over ranks)
    double *d_s = nullptr;
    CKS(ws_get(ctx, "probe_s", D, &d_s));
    CK(run_k(ctx, "probe_rowsum", 1, [&]() { return launch_probe_rowsum(D, p->band(), d_s, s); }));
    CKS(allreduce(ctx, d_s, D, "allreduce_s"));
    std::vector<double> hs(D);
    CK(cudaMemcpyAsync(hs.data(), d_s, sizeof(double) * D, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    p->min_row_mass = *std::min_element(hs.begin(), hs.end());
    return QDT_OK;
}


// ------------------------------------------------------------------------------ probes
extern "C" qdt_status qdt_build_probes(qdt_ctx *ctx, const double *alpha2, int64_t D, int64_t M,
                                       const qdt_probe_opts *o, qdt_probes **out)
{
    if (!ctx) return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_build_probes: ctx is NULL");
    if (!out || !alpha2) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_build_probes: NULL pointer");
    *out = nullptr;
    if (D < 1) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_build_probes: D = %lld < 1", (long long)D);
    if (M < 1 || M > INT32_MAX - 64)
        return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_build_probes: M = %lld out of range", (long long)M);
    if (D > INT32_MAX) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_build_probes: D too large");
    for (int64_t d = 0; d < D; d++) {
        if (!isfinite(alpha2[d]) || alpha2[d] < 0.0)
            return fail(ctx, QDT_ERR_INVALID_ARG, "alpha2[%lld] = %g is not finite and >= 0",
                        (long long)d, alpha2[d]);
        if (d > 0 && alpha2[d] < alpha2[d - 1])
            return fail(ctx, QDT_ERR_UNSORTED, "alpha2 not nondecreasing at d = %lld", (long long)d);
    }
    double c_sigma = o ? o->c_sigma : 6.0;
    int margin = o ? o->margin : 16;
    if (!(c_sigma > 0.0) || !isfinite(c_sigma) || margin < 0)
        return fail(ctx, QDT_ERR_INVALID_ARG, "probe opts: c_sigma must be > 0, margin >= 0");
    CK(cudaSetDevice(ctx->device));
    NvtxRange nv("qdt_build_probes");
    cudaStream_t s = ctx->stream;
    std::unique_ptr<qdt_probes> p(new qdt_probes());
    p->ctx = ctx;
    p->D = D;
    p->M = M;
    p->c_sigma = c_sigma;
    p->margin = margin;
    // S0 (a): band edges on the device
    CK(cudaMalloc(&p->d_alpha2, sizeof(double) * D));
    CK(cudaMemcpyAsync(p->d_alpha2, alpha2, sizeof(double) * D, cudaMemcpyHostToDevice, s));
    int32_t *d_hi = nullptr;
    CK(cudaMalloc(&p->d_lo, sizeof(int32_t) * D));
    CK(cudaMalloc(&d_hi, sizeof(int32_t) * D));
    CK(run_k(ctx, "probe_edges", 1,
             [&]() { return launch_probe_edges(p->d_alpha2, D, M, c_sigma, margin, p->d_lo, d_hi, s); }));
    p->lo_g.resize(D);
    p->hi_g.resize(D);
    CK(cudaMemcpyAsync(p->lo_g.data(), p->d_lo, sizeof(int32_t) * D, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(p->hi_g.data(), d_hi, sizeof(int32_t) * D, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(d_hi);
    if (o && o->strict_mass) {
        for (int64_t d = 0; d < D; d++) {
            double mu = alpha2[d];
            if (mu > 0.0 && p->hi_g[d] == M - 1 && mu + c_sigma * sqrt(mu) > (double)(M - 1))
                return fail(ctx, QDT_ERR_TRUNCATED,
                            "probe %lld (|alpha|^2 = %g) is clipped by the cutoff M = %lld",
                            (long long)d, mu, (long long)M);
        }
    }
    CKS(finish_probes(ctx, p.get(), nullptr));
    *out = p.release();
    return QDT_OK;
}

// Test hook: a banded F given directly.  lo[d], len[d] (global rows, len >= 1,
// lo + len <= M, both edges nondecreasing in d like the Poisson bands of S0), vals probe-major
// (band of probe d at off_d = sum_{e<d} len_e).  Values are copied (host pointers).
extern "C" qdt_status qdt_probes_from_banded(qdt_ctx *ctx, int64_t D, int64_t M, const int64_t *lo,
                                             const int64_t *len, const double *vals, qdt_probes **out)
{
    if (!ctx) return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_probes_from_banded: ctx is NULL");
    if (!out || !lo || !len || !vals) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_probes_from_banded: NULL pointer");
    *out = nullptr;
    if (D < 1 || D > INT32_MAX) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_probes_from_banded: D = %lld", (long long)D);
    if (M < 1 || M > INT32_MAX - 64)
        return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_probes_from_banded: M = %lld out of range", (long long)M);
    int64_t nnz = 0;
    for (int64_t d = 0; d < D; d++) {
        if (len[d] < 1 || lo[d] < 0 || lo[d] + len[d] > M)
            return fail(ctx, QDT_ERR_INVALID_ARG, "band %lld = [%lld, +%lld) outside [0, M)", (long long)d,
                        (long long)lo[d], (long long)len[d]);
        if (d > 0 && (lo[d] < lo[d - 1] || lo[d] + len[d] < lo[d - 1] + len[d - 1]))
            return fail(ctx, QDT_ERR_UNSORTED, "band edges not nondecreasing at d = %lld", (long long)d);
        nnz += len[d];
    }
    for (int64_t i = 0; i < nnz; i++)
        if (!isfinite(vals[i])) return fail(ctx, QDT_ERR_NONFINITE, "vals[%lld] is not finite", (long long)i);
    CK(cudaSetDevice(ctx->device));
    std::unique_ptr<qdt_probes> p(new qdt_probes());
    p->ctx = ctx;
    p->D = D;
    p->M = M;
    p->lo_g.resize(D);
    p->hi_g.resize(D);
    for (int64_t d = 0; d < D; d++) {
        p->lo_g[d] = (int32_t)lo[d];
        p->hi_g[d] = (int32_t)(lo[d] + len[d] - 1);
    }
    CK(cudaMalloc(&p->d_lo, sizeof(int32_t) * D));
    CKS(finish_probes(ctx, p.get(), vals));
    *out = p.release();
    return QDT_OK;
}

extern "C" qdt_status qdt_probes_free(qdt_probes *p)
{
    if (!p) return QDT_OK;
    cudaSetDevice(p->ctx->device);
    delete p;
    return QDT_OK;
}

extern "C" qdt_status qdt_probes_export(qdt_ctx *ctx, const qdt_probes *p, int64_t *nnz,
                                        int64_t *k_begin, int64_t *k_end, int64_t *lo,
                                        int64_t *len, double *val)
{
    if (!ctx || !p) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_probes_export: NULL handle");
    if (p->ctx != ctx) return fail(ctx, QDT_ERR_STATE, "probes were built on another ctx");
    if (nnz) *nnz = p->nnz;
    if (k_begin) *k_begin = p->kb;
    if (k_end) *k_end = p->ke;
    for (int64_t d = 0; d < p->D; d++) {
        if (lo) lo[d] = p->lo_l[d];
        if (len) len[d] = p->len_l[d];
    }
    if (val && p->nnz) {
        CK(cudaMemcpyAsync(val, p->d_val, sizeof(double) * p->nnz, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return QDT_OK;
}

// ------------------------------------------------------------------------------ step setup
// SQS weights (t_k = 1/w_k) or the power-iteration Lipschitz scalar (reading R2).
static qdt_status step_setup(qdt_ctx *ctx, qdt_probes *p, Plan *pl, int mode, double gamma,
                             int k_pow, double *d_tstep, double *d_w, double *rho_out,
                             double *tscalar_out)
{
    cudaStream_t s = ctx->stream;
    const int64_t D = p->D, Ml = p->Ml;
    if (mode == QDT_STEP_SQS || d_w) {
        double *d_s;
        CKS(ws_get(ctx, "setup_s", D, &d_s));
        CK(run_k(ctx, "probe_rowsum", 1, [&]() { return launch_probe_rowsum(D, p->band(), d_s, s); }));
        CKS(allreduce(ctx, d_s, D, "allreduce_s"));
        CK(run_k(ctx, "sqs_weights", 1, [&]() {
            if (p->d_Fb)   // tiled F of the sweep path: coalesced, one block per Fock tile
                return launch_sqs_weights_tiled(p->sw_ntiles, (int)Ml, p->d_sw_dA, p->d_sw_dB, p->d_fb_off,
                                                p->d_Fb, d_s, gamma, d_w,
                                                mode == QDT_STEP_SQS ? d_tstep : nullptr, s);
            return launch_sqs_weights(pl->ntiles, pl->T, pl->d_tile_dA, pl->d_tile_dB, (int)Ml, p->kb,
                                      p->band(), d_s, gamma, d_w,
                                      mode == QDT_STEP_SQS ? d_tstep : nullptr, s);
        }));
    }
    if (mode == QDT_STEP_LIPSCHITZ || rho_out) {
        // v0 = 1/sqrt(M); K_pow iterations of v <- F^T F v / ||F^T F v||; rho = ||F v||^2.  The
        // products act on single columns: the general tiles of the N = 1 plan serve every N
        if (!pl->gen) CKS(build_plan(ctx, p, 1, &pl));
        double *v, *u, *q, *part, *nrm;
        const int nb = ctx->nblkR;
        CKS(ws_get(ctx, "pow_v", Ml, &v));
        CKS(ws_get(ctx, "pow_u", Ml, &u));
        CKS(ws_get(ctx, "pow_q", D, &q));
        CKS(ws_get(ctx, "pow_part", nb, &part));
        CKS(ws_get(ctx, "pow_nrm", 2, &nrm));
        CK(launch_fill(v, Ml, 1.0 / sqrt((double)p->M), s));
        ctx->launches++;
        for (int i = 0; i < k_pow; i++) {
            CK(run_k(ctx, "pow_fwd", 1, [&]() { return launch_pow_fwd(D, p->band(), v, p->kb, q, s); }));
            CKS(allreduce(ctx, q, D, "allreduce_pow"));
            CK(run_k(ctx, "pow_bwd", 1, [&]() {
                return launch_pow_bwd(pl->ntiles, pl->T, pl->d_tile_dA, pl->d_tile_dB, (int)Ml, p->kb,
                                      p->band(), q, u, s);
            }));
            CK(run_k(ctx, "pow_norm", 3, [&]() {
                cudaError_t e = launch_sumsq(u, Ml, part, nb, s);
                if (e == cudaSuccess) e = launch_reduce_vec(part, nb, 1, 1, nrm, s);
                return e;
            }));
            CKS(allreduce(ctx, nrm, 1, "allreduce_pow"));
            CK(run_k(ctx, "pow_scale", 1, [&]() { return launch_scale(v, u, nrm, Ml, s); }));
        }
        CK(run_k(ctx, "pow_fwd", 1, [&]() { return launch_pow_fwd(D, p->band(), v, p->kb, q, s); }));
        CKS(allreduce(ctx, q, D, "allreduce_pow"));
        CK(run_k(ctx, "pow_norm", 2, [&]() {
            cudaError_t e = launch_sumsq(q, D, part, nb, s);
            if (e == cudaSuccess) e = launch_reduce_vec(part, nb, 1, 1, nrm, s);
            return e;
        }));
        double rho = 0.0;
        CK(cudaMemcpyAsync(&rho, nrm, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (rho_out) *rho_out = rho;
        if (mode == QDT_STEP_LIPSCHITZ) {
            const double t = 1.0 / (1.01 * rho + 4.0 * gamma);
            if (tscalar_out) *tscalar_out = t;
            CK(launch_fill(d_tstep, Ml, t, s));
            ctx->launches++;
        }
    }
    return QDT_OK;
}

extern "C" qdt_status qdt_step_setup(qdt_ctx *ctx, const qdt_probes *F, double gamma, int32_t k_pow,
                                     double *w_out, double *rho_out)
{
    if (!ctx || !F) return fail(ctx, QDT_ERR_INVALID_ARG, "NULL handle");
    if (!(gamma >= 0.0) || !isfinite(gamma) || k_pow < 0)
        return fail(ctx, QDT_ERR_INVALID_ARG, "gamma must be finite >= 0, k_pow >= 0");
    qdt_probes *p = const_cast<qdt_probes *>(F);
    Plan *pl;
    CKS(build_plan(ctx, p, 1, &pl));
    double *d_w = nullptr, *d_t;
    CKS(ws_get(ctx, "setup_t", p->Ml, &d_t));
    if (w_out) CKS(ws_get(ctx, "setup_w", p->Ml, &d_w));
    double rho = 0.0;
    CKS(step_setup(ctx, p, pl, w_out ? QDT_STEP_SQS : QDT_STEP_LIPSCHITZ, gamma, k_pow, d_t, d_w,
                   rho_out ? &rho : nullptr, nullptr));
    if (w_out) {
        CK(cudaMemcpyAsync(w_out, d_w, sizeof(double) * p->Ml, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    if (rho_out) *rho_out = rho;
    return QDT_OK;
}

// ------------------------------------------------------------------------------ iteration
struct SolveBufs {
    double *theta[3] = {nullptr, nullptr, nullptr};  // (Ml + 2) x N, pointer to local row 0
    double *R[2] = {nullptr, nullptr};
    double *RY = nullptr;
    double *rpart = nullptr, *partR = nullptr, *partT = nullptr, *vec = nullptr;
    double *tstep = nullptr, *scratch = nullptr, *P = nullptr;
    double *trace = nullptr, *kkt = nullptr, *kktp = nullptr, *beta = nullptr;
    int *counters = nullptr;
    DevState *state = nullptr;
    double *sc2_stage = nullptr;
    int *sc2_arrive = nullptr;
    double *bb_part = nullptr, *bb_vec = nullptr, *tbb = nullptr;  // BB step statistics / scalar
    double *Gw = nullptr;      // wide-N sweep: Ml x N gradient
    double *tau_prev = nullptr;  // fused wide step: per-row threshold of the last step (warm start)
};

struct IterCfg {
    qdt_probes *p;
    Plan *pl;
    int N;
    double gamma, tol;
    int fista;
    int kkt_every;
    int64_t trace_len;
    int bb = 0;                // Barzilai-Borwein step (reading R14): 1 plain, 2 with the line search (R17)
    double tlip = 0.0;         // its safeguard / first step
    int Nv = 0;                // outcomes when N is a padded pitch (pad_cols), else 0
    int bx = 0;                // band-aware residual exchange (nranks > 1)
};

static inline int nvalid(const IterCfg &c) { return c.Nv ? c.Nv : c.N; }

// Band-aware residual exchange: R holds this rank's partial rows
// (zero for probes that miss the slice).  With every peer q whose slice shares probes with ours,
// the shared probe rows [max(dlo), min(dhi)) are exchanged (NCCL send/recv, or copies inside an
// in-process group); k_band_combine sums each touched probe over its ranks in rank order,
// subtracts P and accumulates ||R||^2 on the probe's lowest rank.
static qdt_status band_exchange(qdt_ctx *ctx, const IterCfg &c, SolveBufs &b, double *R, bool withP)
{
    qdt_probes *p = c.p;
    const int G = ctx->nranks, g = ctx->rank, N = c.N;
    const int64_t a0 = p->dlo_r[g], a1 = p->dhi_r[g];
    BandX bx;
    memset(&bx, 0, sizeof bx);
    int64_t tot = 0;
    std::vector<int64_t> ov0(G, 0), ov1(G, 0), off(G, 0);
    for (int q = 0; q < G; q++) {
        bx.dlo[q] = p->dlo_r[q];
        bx.dhi[q] = p->dhi_r[q];
        if (q == g) continue;
        ov0[q] = std::max(a0, p->dlo_r[q]);
        ov1[q] = std::min(a1, p->dhi_r[q]);
        if (ov1[q] < ov0[q]) ov1[q] = ov0[q];
        off[q] = tot;
        tot += (ov1[q] - ov0[q]) * N;
    }
    double *recv = nullptr;
    CKS(ws_get(ctx, "bx_recv", std::max<int64_t>(1, tot), &recv));
    for (int q = 0; q < G; q++) {
        bx.src[q] = recv + off[q];
        bx.start[q] = ov0[q];
    }
    if (ctx->vg) {
        VPost post;
        CKS(vg_barrier(ctx, R, 0, &post));
        for (int q = 0; q < G; q++)
            if (q != g && ov1[q] > ov0[q])
                CK(cudaMemcpyAsync(recv + off[q], (const double *)post.p[q] + ov0[q] * N,
                                   sizeof(double) * (ov1[q] - ov0[q]) * N, cudaMemcpyDeviceToDevice, ctx->stream));
        CKS(vg_barrier(ctx, nullptr, 0, nullptr));
    } else {
        nccl_result_t e = 0;
        run_k(ctx, "band_exchange", 1, [&]() {
            g_nccl.groupStart();
            for (int q = 0; q < G; q++) {
                if (q == g || ov1[q] <= ov0[q]) continue;
                const size_t n = (size_t)((ov1[q] - ov0[q]) * N);
                e |= g_nccl.send(R + ov0[q] * N, n, NCCL_FLOAT64, q, ctx->ncomm, ctx->stream);
                e |= g_nccl.recv(recv + off[q], n, NCCL_FLOAT64, q, ctx->ncomm, ctx->stream);
            }
            e |= g_nccl.groupEnd();
            return cudaSuccess;
        });
        if (e != 0) return fail(ctx, QDT_ERR_NCCL, "band-aware exchange failed");
    }
    static const double zero = 0.0;
    (void)zero;
    double *Pz = b.P;
    if (!withP) {   // no data term: subtract zeros
        CKS(ws_get(ctx, "bx_zero", (size_t)p->D * N, &Pz));
        CK(cudaMemsetAsync(Pz, 0, sizeof(double) * p->D * N, ctx->stream));
    }
    CK(run_k(ctx, "reduce_R", 1, [&]() {
        return launch_band_combine(bx, g, G, Pz, R, N, b.partR, c.pl->nR, b.state, ctx->stream);
    }));
    return QDT_OK;
}

static qdt_status fwd_reduce(qdt_ctx *ctx, const IterCfg &c, SolveBufs &b, const double *theta,
                             double *R, bool withP, double *partR_alt = nullptr)
{
    if (partR_alt) {   // a side product (e.g. F d of the line search): keep ||R_k||^2's partials
        SolveBufs b2 = b;
        b2.partR = partR_alt;
        return fwd_reduce(ctx, c, b2, theta, R, withP, nullptr);
    }
    cudaStream_t s = ctx->stream;
    Plan *pl = c.pl;
    qdt_probes *p = c.p;
    const bool multi = ctx->nranks > 1;
    if (pl->NB || pl->NW || pl->NX) {
        const int fnb = (pl->NW || pl->NX) ? wide_fwd_nb(c.N) : pl->NB;   // wide N: balanced column chunks
        SweepFwdArgs fa;
        fa.N = c.N;
        fa.Ml = (int)p->Ml;
        fa.units = pl->d_fwunits;
        fa.fb_off = p->d_fb_off;
        fa.tile_dA = p->d_sw_dA;
        fa.tile_dB = p->d_sw_dB;
        fa.Fb = p->d_Fb;
        fa.theta = theta;
        fa.rpart = b.rpart;
        fa.state = b.state;
        CK(run_k(ctx, "fwd_partial", 1, [&]() { return launch_fwd_mma(fa, pl->sw_nfunits, fnb, s); }));
        if (!multi) {
            CK(run_k(ctx, "reduce_R", 1, [&]() {
                return launch_reduce_R2(b.rpart, pl->d_sw_red_beg, pl->d_sw_red_rows, withP ? b.P : nullptr,
                                        R, (int)p->D, c.N, b.partR, b.state, s);
            }));
            return QDT_OK;
        }
        CK(run_k(ctx, "reduce_R", 1, [&]() {
            return launch_reduce_R2(b.rpart, pl->d_sw_red_beg, pl->d_sw_red_rows, nullptr, R, (int)p->D,
                                    c.N, nullptr, b.state, s);
        }));
        if (c.bx) return band_exchange(ctx, c, b, R, withP);
        CKS(allreduce(ctx, R, (size_t)p->D * c.N, "allreduce_R"));
        if (withP)
            CK(run_k(ctx, "reduce_R", 1, [&]() {
                return launch_sub_p_sumsq(R, b.P, p->D * (int64_t)c.N, b.partR, pl->nR, b.state, s);
            }));
        return QDT_OK;
    }
    FwdArgs fa;
    fa.N = c.N;
    fa.CG = pl->CG;
    fa.RG = pl->RG;
    fa.KR = pl->KR;
    fa.units = pl->d_funits;
    fa.band = p->band();
    fa.theta = theta;
    fa.kb = p->kb;
    fa.rpart = b.rpart;
    fa.state = b.state;
    CK(run_k(ctx, "fwd_partial", 1, [&]() { return launch_fwd(fa, pl->nfunits, pl->TC, s, nullptr); }));
    CK(run_k(ctx, "reduce_R", 1, [&]() {   // warp per probe, fixed list order (any N)
        return launch_reduce_R2(b.rpart, pl->d_red_beg, pl->d_red_rows, (withP && !multi) ? b.P : nullptr,
                                R, (int)p->D, c.N, multi ? nullptr : b.partR, b.state, s);
    }));
    if (multi) {
        if (c.bx) return band_exchange(ctx, c, b, R, withP);
        CKS(allreduce(ctx, R, (size_t)p->D * c.N, "allreduce_R"));
        if (withP)
            CK(run_k(ctx, "reduce_R", 1, [&]() {
                return launch_sub_p_sumsq(R, b.P, p->D * (int64_t)c.N, b.partR, pl->nR, b.state, s);
            }));
    }
    return QDT_OK;
}

static BwdArgs bwd_args(qdt_ctx *ctx, const IterCfg &c, SolveBufs &b, const double *R,
                        const double *theta, const double *theta_prev, double *out, bool fista)
{
    (void)ctx;
    BwdArgs a;
    Plan *pl = c.pl;
    a.N = c.N;
    a.CG = pl->CG;
    a.RG = pl->RG;
    a.KC = pl->KC;
    a.SEG = pl->SEG;
    a.units = pl->d_bunits;
    a.band = c.p->band();
    a.R = R;
    a.theta = theta;
    a.theta_prev = fista ? theta_prev : nullptr;
    a.beta = fista ? b.beta : nullptr;
    a.kkt_every = c.kkt_every;
    a.kb = c.p->kb;
    a.M = c.p->M;
    a.Ml = (int)c.p->Ml;
    a.tstep = b.tstep;
    a.gamma = c.gamma;
    a.out = out;
    a.scratch = b.scratch;
    a.counters = b.counters;
    a.part = b.partT;
    a.state = b.state;
    return a;
}

static qdt_status halo_exchange(qdt_ctx *ctx, const IterCfg &c, double *theta)
{
    if (ctx->nranks == 1) return QDT_OK;
    const int N = c.N, r = ctx->rank;
    const int64_t Ml = c.p->Ml;
    if (ctx->vg) {   // copy the neighbours' edge rows into the halo rows
        VPost post;
        CKS(vg_barrier(ctx, theta, Ml, &post));
        if (r > 0)
            CK(cudaMemcpyAsync(theta - N, (const double *)post.p[r - 1] + (post.iv[r - 1] - 1) * N, sizeof(double) * N,
                               cudaMemcpyDeviceToDevice, ctx->stream));
        if (r + 1 < ctx->nranks)
            CK(cudaMemcpyAsync(theta + Ml * N, post.p[r + 1], sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
        CKS(vg_barrier(ctx, nullptr, 0, nullptr));
        ctx->launches += 0;
        return QDT_OK;
    }
    nccl_result_t e = 0;
    run_k(ctx, "halo", 1, [&]() {
        g_nccl.groupStart();
        if (r > 0) {
            e |= g_nccl.send(theta, N, NCCL_FLOAT64, r - 1, ctx->ncomm, ctx->stream);
            e |= g_nccl.recv(theta - N, N, NCCL_FLOAT64, r - 1, ctx->ncomm, ctx->stream);
        }
        if (r + 1 < ctx->nranks) {
            e |= g_nccl.send(theta + (Ml - 1) * N, N, NCCL_FLOAT64, r + 1, ctx->ncomm, ctx->stream);
            e |= g_nccl.recv(theta + Ml * N, N, NCCL_FLOAT64, r + 1, ctx->ncomm, ctx->stream);
        }
        e |= g_nccl.groupEnd();
        return cudaSuccess;
    });
    if (e != 0) return fail(ctx, QDT_ERR_NCCL, "halo exchange failed");
    return QDT_OK;
}

// S6: tile partials (ntiles of them, from whichever bwd kernel ran) + ||R||^2 partials -> trace,
// KKT, stop flag.  Single GPU: one k_scalars2 launch; multi-GPU: k_scalars2 (local sums),
// allreduce of the 5-vector, k_finalize.
static qdt_status scalars(qdt_ctx *ctx, const IterCfg &c, SolveBufs &b, int final_eval, int ntiles,
                          const double *part = nullptr)
{
    const double *partT = part ? part : b.partT;
    cudaStream_t s = ctx->stream;
    const bool multi = ctx->nranks > 1;
    const int ke = final_eval ? 1 : c.kkt_every;
    CK(run_k(ctx, "scalars", 1, [&]() {
        return launch_scalars2(b.partR, c.pl->nR, partT, ntiles, (ctx->rank == 0 || c.bx), b.sc2_stage, b.sc2_arrive,
                               b.vec, nvalid(c), c.p->M, c.gamma, c.tol, final_eval, ke, b.trace, b.kkt, b.kktp,
                               c.trace_len, b.state, multi ? 0 : 1, s);
    }));
    if (!multi) return QDT_OK;
    CKS(allreduce(ctx, b.vec, NV, "allreduce_scalars"));
    CK(run_k(ctx, "scalars", 1, [&]() {
        return launch_finalize(b.vec, nvalid(c), c.p->M, c.gamma, c.tol, final_eval, ke, b.trace, b.kkt, b.kktp,
                               c.trace_len, b.state, s);
    }));
    return QDT_OK;
}

// sweep bwd launcher: the N-split 512-thread kernel for FISTA steps (its two staged tiles leave
// one CTA per SM: 16 warps instead of 8), the 256-thread kernel otherwise (QDT_SPLITN overrides:
// 0 never, 1 always; measured in profiles/r01_v5)
static cudaError_t launch_bwd_any(const SweepArgs &a, int nunits, int NB, cudaStream_t s)
{
    const int m = sweep_split_mode();
    const bool fis = a.beta != nullptr && !a.eval;
    const bool split = NB <= SW_NBMAX && (m == 1 || (m == 2 && fis));
    return split ? launch_bwd_split(a, nunits, NB, s) : launch_bwd_mma(a, nunits, NB, s);
}

static SweepArgs sweep_args(const IterCfg &c, SolveBufs &b, const double *R, const double *theta,
                            double *out)
{
    SweepArgs a;
    a.N = c.N;
    a.Nv = nvalid(c);
    a.Ml = (int)c.p->Ml;
    a.kb = c.p->kb;
    a.M = c.p->M;
    a.units = c.pl->d_swunits;
    a.fb_off = c.p->d_fb_off;
    a.tile_dA = c.p->d_sw_dA;
    a.Fb = c.p->d_Fb;
    a.R = R;
    a.theta = theta;
    a.out = out;
    a.tstep = b.tstep;
    a.tscal = nullptr;
    a.gamma = c.gamma;
    a.scratch = b.scratch;
    a.counters = b.counters;
    a.part = b.partT;
    a.kkt_every = c.kkt_every;
    a.nunits = 0;
    a.eval = 0;
    a.eval_gate = 0;
    a.theta_prev = nullptr;
    a.beta = nullptr;
    a.state = b.state;
    return a;
}

static WideArgs wide_args(const IterCfg &c, SolveBufs &b, const double *R, const double *theta,
                          double *out)
{
    WideArgs w;
    w.N = c.N;
    w.Nv = nvalid(c);
    w.Ml = (int)c.p->Ml;
    w.ncc = (c.N + 127) / 128;
    w.kb = c.p->kb;
    w.M = c.p->M;
    w.units = c.pl->d_swunits;
    w.fb_off = c.p->d_fb_off;
    w.tile_dA = c.p->d_sw_dA;
    w.Fb = c.p->d_Fb;
    w.R = R;
    w.theta = theta;
    w.G = b.Gw;
    w.out = out;
    w.tstep = b.tstep;
    w.gamma = c.gamma;
    w.scratch = b.scratch;
    w.counters = b.counters;
    w.part = b.partT;
    w.part_b = (int64_t)c.p->sw_ntiles * w.ncc;
    w.kkt_every = c.kkt_every;
    w.eval = 0;
    w.eval_gate = 0;
    w.theta_prev = nullptr;
    w.beta = nullptr;
    w.state = b.state;
    w.row_da = c.p->d_row_da;
    w.row_db = c.p->d_row_db;
    return w;
}

static WStepArgs wstep_args(const IterCfg &c, SolveBufs &b, const double *R, const double *theta, double *out)
{
    WStepArgs w;
    w.N = c.N;
    w.Nv = nvalid(c);
    w.Ml = (int)c.p->Ml;
    w.C = c.pl->wx_C;
    w.Wc = c.pl->wx_Wc;
    w.kb = c.p->kb;
    w.M = c.p->M;
    w.tlist = c.pl->d_wx_tlist;
    w.toff = c.pl->d_wx_toff;
    w.fb_off = c.p->d_fb_off;
    w.tile_dA = c.p->d_sw_dA;
    w.tile_dB = c.p->d_sw_dB;
    w.Fb = c.p->d_Fb;
    w.R = R;
    w.theta = theta;
    w.theta_prev = nullptr;
    w.beta = nullptr;
    w.out = out;
    w.tstep = b.tstep;
    w.tscal = nullptr;
    w.gamma = c.gamma;
    w.tau_prev = b.tau_prev;
    w.part = b.partT;
    w.kkt_every = c.kkt_every;
    w.eval = 0;
    w.eval_gate = 0;
    w.state = b.state;
    return w;
}

static int wstep_nparts(const IterCfg &c) { return c.pl->wx_ncl * c.pl->wx_C; }

static int wide_nparts(const IterCfg &c)
{
    return c.p->sw_ntiles * ((c.N + 127) / 128) + wide_proj_blocks((int)c.p->Ml);
}

// QDT_WIDE_PLAIN=1: plain steps at 128 < N <= 160 on the two wide kernels instead of k_bwd_mma
// (A/B measurement)
static bool wide_plain_forced()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("QDT_WIDE_PLAIN");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// one iteration with phase index j (buffer rotation)
static qdt_status iteration(qdt_ctx *ctx, const IterCfg &c, SolveBufs &b, int64_t j)
{
    cudaStream_t s = ctx->stream;
    Plan *pl = c.pl;
    int ntiles = pl->ntiles;
    if (c.bb) {
        // BB: R_k, the step statistics of s = Theta_k - Theta_{k-1} and R_k - R_{k-1}, t_k, the step
        double *cur = b.theta[j % 2], *prv = b.theta[(j + 1) % 2];
        double *Rk = b.R[j % 2], *Rkm1 = b.R[(j + 1) % 2];
        qdt_probes *p = c.p;
        CKS(fwd_reduce(ctx, c, b, cur, Rk, true));
        CK(run_k(ctx, "bb_step", 2, [&]() {
            return launch_bb_stats(cur, prv, p->Ml, p->kb, p->M, c.N, ctx->rank == 0 ? Rk : nullptr, Rkm1,
                                   p->D * (int64_t)c.N, b.bb_part, b.bb_vec, b.state, s);
        }));
        CKS(allreduce(ctx, b.bb_vec, 3, "allreduce_scalars"));
        CK(run_k(ctx, "bb_step", 1, [&]() { return launch_bb_step(b.bb_vec, c.gamma, c.tlip, b.tbb, b.state, s); }));
        double *nxt = b.theta[(j + 1) % 2];
        int nparts = c.p->sw_ntiles;
        if (pl->NB) {   // N <= 160 (even above 128): k_bwd_mma with the scalar step
            SweepArgs a = sweep_args(c, b, Rk, cur, nxt);
            a.tscal = b.tbb;
            CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_bwd_mma(a, pl->sw_nbunits, pl->NB, s); }));
        } else if (pl->NX) {
            WStepArgs w = wstep_args(c, b, Rk, cur, nxt);
            w.tscal = b.tbb;
            CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_wide_step(w, pl->wx_ncl, s); }));
            nparts = wstep_nparts(c);
        } else {
            WideArgs w = wide_args(c, b, Rk, cur, nxt);
            w.tscal = b.tbb;
            CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_grad_wide(w, pl->sw_nbunits, s); }));
            CK(run_k(ctx, "proj_step", 1, [&]() { return launch_proj_wide(w, s); }));
            nparts = wide_nparts(c);
        }
        CKS(halo_exchange(ctx, c, nxt));
        if (c.bb == 2) {
            // exact line search along d = Z - Theta_k (reading R17): F d by a forward pass of d, the
            // step statistics, lambda* on the device, Theta_{k+1} = Theta_k + lambda* d over Z
            CK(run_k(ctx, "bb_step", 1, [&]() {
                return launch_bbls_dir(cur - c.N, nxt - c.N, b.theta[2] - c.N, (p->Ml + 2) * (int64_t)c.N, b.state, s);
            }));
            double *pr_alt;
            CKS(ws_get(ctx, "partR_alt", std::max(ctx->nblkR, pl->nR), &pr_alt));
            CKS(fwd_reduce(ctx, c, b, b.theta[2], b.RY, false, pr_alt));
            CK(run_k(ctx, "bb_step", 2, [&]() {
                return launch_bbls_stats(cur, nxt, p->Ml, p->kb, p->M, c.N, ctx->rank == 0 ? Rk : nullptr, b.RY,
                                         p->D * (int64_t)c.N, b.bb_part, b.bb_vec, b.state, s);
            }));
            CKS(allreduce(ctx, b.bb_vec, 5, "allreduce_scalars"));
            CK(run_k(ctx, "bb_step", 2, [&]() {
                return launch_bbls_step(b.bb_vec, c.gamma, b.tbb, b.tbb + 1, cur - c.N, nxt - c.N,
                                        (p->Ml + 2) * (int64_t)c.N, b.state, s);
            }));
        }
        CKS(scalars(ctx, c, b, 0, nparts));
        return QDT_OK;
    }
    if (!c.fista && pl->NX && (!pl->NB || wide_plain_forced())) {
        double *cur = b.theta[j % 2], *nxt = b.theta[(j + 1) % 2];
        CKS(fwd_reduce(ctx, c, b, cur, b.R[0], true));
        WStepArgs w = wstep_args(c, b, b.R[0], cur, nxt);
        CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_wide_step(w, pl->wx_ncl, s); }));
        CKS(halo_exchange(ctx, c, nxt));
        CKS(scalars(ctx, c, b, 0, wstep_nparts(c)));
        return QDT_OK;
    }
    if (!c.fista && pl->NW && (!pl->NB || wide_plain_forced())) {
        double *cur = b.theta[j % 2], *nxt = b.theta[(j + 1) % 2];
        CKS(fwd_reduce(ctx, c, b, cur, b.R[0], true));
        WideArgs w = wide_args(c, b, b.R[0], cur, nxt);
        CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_grad_wide(w, pl->sw_nbunits, s); }));
        CK(run_k(ctx, "proj_step", 1, [&]() { return launch_proj_wide(w, s); }));
        CKS(halo_exchange(ctx, c, nxt));
        CKS(scalars(ctx, c, b, 0, wide_nparts(c)));
        return QDT_OK;
    }
    if (!c.fista && pl->NB) {
        double *cur = b.theta[j % 2], *nxt = b.theta[(j + 1) % 2];
        CKS(fwd_reduce(ctx, c, b, cur, b.R[0], true));
        SweepArgs a = sweep_args(c, b, b.R[0], cur, nxt);
        CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_bwd_any(a, pl->sw_nbunits, pl->NB, s); }));
        CKS(halo_exchange(ctx, c, nxt));
        ntiles = c.p->sw_ntiles;
    } else if (c.fista && pl->NX) {
        // FISTA, fused wide step: R_k, R(Y), gated KKT evaluation of Theta_k, then the step from Y
        double *cur = b.theta[j % 3], *prev = b.theta[(j + 2) % 3], *nxt = b.theta[(j + 1) % 3];
        double *Rk = b.R[j % 2], *Rkm1 = b.R[(j + 1) % 2];
        CKS(fwd_reduce(ctx, c, b, cur, Rk, true));
        CK(run_k(ctx, "fista_rcomb", 1, [&]() {
            return launch_fista_rcomb(b.RY, Rk, Rkm1, b.beta, c.p->D * (int64_t)c.N, b.state, s);
        }));
        WStepArgs ev = wstep_args(c, b, Rk, cur, nullptr);
        ev.eval = 1;
        ev.eval_gate = 1;
        CK(run_k(ctx, "bwd_eval", 1, [&]() { return launch_wide_step(ev, pl->wx_ncl, s); }));
        WStepArgs w = wstep_args(c, b, b.RY, cur, nxt);
        w.theta_prev = prev;
        w.beta = b.beta;
        CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_wide_step(w, pl->wx_ncl, s); }));
        CKS(halo_exchange(ctx, c, nxt));
        ntiles = wstep_nparts(c);
    } else if (c.fista && pl->NW) {
        // FISTA, wide N: R_k, R(Y), gated KKT evaluation of Theta_k, then the step from Y
        double *cur = b.theta[j % 3], *prev = b.theta[(j + 2) % 3], *nxt = b.theta[(j + 1) % 3];
        double *Rk = b.R[j % 2], *Rkm1 = b.R[(j + 1) % 2];
        CKS(fwd_reduce(ctx, c, b, cur, Rk, true));
        CK(run_k(ctx, "fista_rcomb", 1, [&]() {
            return launch_fista_rcomb(b.RY, Rk, Rkm1, b.beta, c.p->D * (int64_t)c.N, b.state, s);
        }));
        WideArgs ev = wide_args(c, b, Rk, cur, nullptr);
        ev.eval = 1;
        ev.eval_gate = 1;
        CK(run_k(ctx, "bwd_eval", 1, [&]() { return launch_grad_wide(ev, pl->sw_nbunits, s); }));
        CK(run_k(ctx, "proj_eval", 1, [&]() { return launch_proj_wide(ev, s); }));
        WideArgs w = wide_args(c, b, b.RY, cur, nxt);
        w.theta_prev = prev;
        w.beta = b.beta;
        CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_grad_wide(w, pl->sw_nbunits, s); }));
        CK(run_k(ctx, "proj_step", 1, [&]() { return launch_proj_wide(w, s); }));
        CKS(halo_exchange(ctx, c, nxt));
        ntiles = wide_nparts(c);
    } else if (c.fista && pl->NB) {
        // FISTA on the sweep kernels: R_k, R(Y) = R_k + beta (R_k - R_{k-1}) (linear), the KKT of
        // Theta_k on the recorded iterations (evaluation pass gated on the device), then the
        // step from Y = Theta_k + beta (Theta_k - Theta_{k-1}) formed in the epilogue
        double *cur = b.theta[j % 3], *prev = b.theta[(j + 2) % 3], *nxt = b.theta[(j + 1) % 3];
        double *Rk = b.R[j % 2], *Rkm1 = b.R[(j + 1) % 2];
        CKS(fwd_reduce(ctx, c, b, cur, Rk, true));
        CK(run_k(ctx, "fista_rcomb", 1, [&]() {
            return launch_fista_rcomb(b.RY, Rk, Rkm1, b.beta, c.p->D * (int64_t)c.N, b.state, s);
        }));
        SweepArgs ev = sweep_args(c, b, Rk, cur, nullptr);
        ev.eval = 1;
        ev.eval_gate = 1;
        CK(run_k(ctx, "bwd_eval", 1, [&]() { return launch_bwd_any(ev, pl->sw_nbunits, pl->NB, s); }));
        SweepArgs a = sweep_args(c, b, b.RY, cur, nxt);
        a.theta_prev = prev;
        a.beta = b.beta;
        CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_bwd_any(a, pl->sw_nbunits, pl->NB, s); }));
        CKS(halo_exchange(ctx, c, nxt));
        ntiles = c.p->sw_ntiles;
    } else if (!c.fista) {
        double *cur = b.theta[j % 2], *nxt = b.theta[(j + 1) % 2];
        CKS(fwd_reduce(ctx, c, b, cur, b.R[0], true));
        BwdArgs a = bwd_args(ctx, c, b, b.R[0], cur, nullptr, nxt, false);
        CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_bwd(a, pl->nbunits, pl->TC, BWD_STEP, s); }));
        CKS(halo_exchange(ctx, c, nxt));
    } else {
        double *cur = b.theta[j % 3], *prev = b.theta[(j + 2) % 3], *nxt = b.theta[(j + 1) % 3];
        double *Rk = b.R[j % 2], *Rkm1 = b.R[(j + 1) % 2];
        CKS(fwd_reduce(ctx, c, b, cur, Rk, true));
        CK(run_k(ctx, "fista_rcomb", 1, [&]() {
            return launch_fista_rcomb(b.RY, Rk, Rkm1, b.beta, c.p->D * (int64_t)c.N, b.state, s);
        }));
        BwdArgs ev = bwd_args(ctx, c, b, Rk, cur, prev, nxt, true);
        CK(run_k(ctx, "bwd_eval", 1, [&]() { return launch_bwd(ev, pl->nbunits, pl->TC, BWD_EVAL, s); }));
        BwdArgs a = bwd_args(ctx, c, b, b.RY, cur, prev, nxt, true);
        CK(run_k(ctx, "bwd_step", 1, [&]() { return launch_bwd(a, pl->nbunits, pl->TC, BWD_STEP, s); }));
        CKS(halo_exchange(ctx, c, nxt));
    }
    CKS(scalars(ctx, c, b, 0, ntiles));
    return QDT_OK;
}

// Workspace shared by solve / objective / hooks, sized for both the general and the sweep plan.
// Buffers read by bulk copies carry 2+ doubles of slack past their last element.
static qdt_status common_bufs(qdt_ctx *ctx, qdt_probes *p, Plan *pl, int64_t N, SolveBufs &b)
{
    cudaStream_t s = ctx->stream;
    const int64_t D = p->D;
    CKS(ws_get(ctx, "R0", D * N + 4, &b.R[0]));
    CKS(ws_get(ctx, "rpart", std::max<int64_t>(1, std::max(pl->nrpart, pl->sw_nrpart)) * N + 4,
               &b.rpart));
    CKS(ws_get(ctx, "partR", std::max(ctx->nblkR, pl->nR), &b.partR));
    const int ncc = (int)((N + 127) / 128);
    const int nt = std::max(1, std::max({pl->ntiles, p->sw_ntiles * (pl->NW ? ncc : 1) + (int)((p->Ml + 7) / 8),
                                         pl->wx_ncl * pl->wx_C}));
    if (pl->NW) CKS(ws_get(ctx, "Gw", p->Ml * N + 4, &b.Gw));
    if (pl->NX) {
        CKS(ws_get(ctx, "tau_prev", p->Ml, &b.tau_prev));
        CK(cudaMemsetAsync(b.tau_prev, 0xff, sizeof(double) * p->Ml, s));   // NaN: no warm start yet
    }
    CKS(ws_get(ctx, "partT", (size_t)nt * NSC_TILE, &b.partT));
    CK(cudaMemsetAsync(b.partT, 0, sizeof(double) * nt * NSC_TILE, s));
    CKS(ws_get(ctx, "vec", NV, &b.vec));
    CKS(ws_get(ctx, "tstep", p->Ml, &b.tstep));
    const int64_t scr = std::max<int64_t>(1, std::max({pl->nslots * pl->T * N, pl->sw_nslots * 1024 * ((pl->NB + 1) / 2 + 1),
                                                       pl->NW ? pl->sw_nslots * ncc * 8192 : (int64_t)0}));
    CKS(ws_get(ctx, "scratch", scr, &b.scratch));
    CKS(ws_get(ctx, "counters", nt, &b.counters));
    CK(cudaMemsetAsync(b.counters, 0, sizeof(int) * nt, s));
    CKS(ws_get(ctx, "state", 1, &b.state));
    CK(cudaMemsetAsync(b.state, 0, sizeof(DevState), s));  // it = 0, stop = 0 (hooks); solve re-inits
    CKS(ws_get(ctx, "sc2_stage", SC2_BLOCKS * NV, &b.sc2_stage));
    CKS(ws_get(ctx, "sc2_arrive", 1, &b.sc2_arrive));
    CK(cudaMemsetAsync(b.sc2_arrive, 0, sizeof(int), s));
    return QDT_OK;
}

// Evaluation of f, r_KKT (both multipliers) at theta: residual, then a G pass without a step
// (sweep kernels when the plan has them), then the final-eval scalars.
static qdt_status eval_pass(qdt_ctx *ctx, const IterCfg &c0, SolveBufs &b, double *theta)
{
    cudaStream_t s = ctx->stream;
    IterCfg c = c0;
    c.fista = 0;
    c.kkt_every = 1;
    Plan *pl = c.pl;
    CKS(fwd_reduce(ctx, c, b, theta, b.R[0], true));
    if (pl->NX && !(pl->NB && pl->NB <= SW_NBMAX)) {
        WStepArgs w = wstep_args(c, b, b.R[0], theta, nullptr);
        w.eval = 1;
        CK(run_k(ctx, "bwd_eval", 1, [&]() { return launch_wide_step(w, pl->wx_ncl, s); }));
        CKS(scalars(ctx, c, b, 1, wstep_nparts(c)));
    } else if (pl->NW) {
        WideArgs w = wide_args(c, b, b.R[0], theta, nullptr);
        w.eval = 1;
        CK(run_k(ctx, "bwd_eval", 1, [&]() { return launch_grad_wide(w, pl->sw_nbunits, s); }));
        CK(run_k(ctx, "proj_eval", 1, [&]() { return launch_proj_wide(w, s); }));
        CKS(scalars(ctx, c, b, 1, wide_nparts(c)));
    } else if (pl->NB) {
        SweepArgs a = sweep_args(c, b, b.R[0], theta, nullptr);
        a.eval = 1;
        CK(run_k(ctx, "bwd_eval", 1, [&]() { return launch_bwd_any(a, pl->sw_nbunits, pl->NB, s); }));
        CKS(scalars(ctx, c, b, 1, c.p->sw_ntiles));
    } else {
        BwdArgs a = bwd_args(ctx, c, b, b.R[0], theta, nullptr, nullptr, false);
        CK(run_k(ctx, "bwd_eval", 1, [&]() { return launch_bwd(a, pl->nbunits, pl->TC, BWD_EVAL, s); }));
        CKS(scalars(ctx, c, b, 1, pl->ntiles));
    }
    return QDT_OK;
}

static qdt_status upload_rows(qdt_ctx *ctx, double *dst, const double *src, int64_t rows, int N,
                              bool device_src)
{
    CK(cudaMemcpyAsync(dst, src, sizeof(double) * rows * N,
                       device_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream));
    return QDT_OK;
}

static qdt_status check_finite_host(qdt_ctx *ctx, const double *x, int64_t n, const char *what)
{
    for (int64_t i = 0; i < n; i++)
        if (!isfinite(x[i]))
            return fail(ctx, QDT_ERR_NONFINITE, "%s[%lld] is not finite", what, (long long)i);
    return QDT_OK;
}

// Odd N > 128 (the paper's N = 151): the wide kernels need an even row pitch, so solve
// and objective run on an internal pitch N + 1 whose pad column is zero in P and Theta (hence in
// R and G), and is excluded from the projection, the KKT sums and their M*N normalisation.
static int64_t pad_cols(int64_t N)
{
    return (sweep_enabled() && N > 8 * SW_NBMAX && (N & 1)) ? N + 1 : N;
}

// rows x ncols doubles between row pitches (in doubles)
static qdt_status copy_cols(qdt_ctx *ctx, double *dst, int64_t dp, const double *src, int64_t sp,
                            int64_t ncols, int64_t rows, cudaMemcpyKind k)
{
    if (rows <= 0) return QDT_OK;
    if (dp == ncols && sp == ncols)
        CK(cudaMemcpyAsync(dst, src, sizeof(double) * rows * ncols, k, ctx->stream));
    else
        CK(cudaMemcpy2DAsync(dst, sizeof(double) * dp, src, sizeof(double) * sp, sizeof(double) * ncols,
                             rows, k, ctx->stream));
    return QDT_OK;
}

extern "C" qdt_status qdt_solve(qdt_ctx *ctx, const qdt_probes *F, const double *P, int64_t Nu,
                                double gamma, double tol, int64_t iters, const qdt_solve_opts *o,
                                double *theta_out, double *trace_out, double *kkt_out,
                                qdt_solve_info *info)
{
    if (!ctx) return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_solve: ctx is NULL");
    if (!F || !P) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve: NULL pointer");
    if (F->ctx != ctx) return fail(ctx, QDT_ERR_STATE, "qdt_solve: probes built on another ctx");
    if (Nu < 1 || Nu > QDT_NMAX) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve: N = %lld not in [1, %d]", (long long)Nu, QDT_NMAX);
    const int64_t N = pad_cols(Nu);   // internal row pitch
    if (!(gamma >= 0.0) || !isfinite(gamma)) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve: gamma must be finite and >= 0");
    if (!(tol >= 0.0)) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve: tol must be >= 0");
    if (iters < 0) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve: iters < 0");
    qdt_solve_opts opt;
    memset(&opt, 0, sizeof opt);
    opt.step = QDT_STEP_SQS;
    opt.check_every = 16;
    opt.kkt_every = 1;
    opt.use_graph = 1;
    if (o) opt = *o;
    if (opt.fista_t != 0.0 && !(opt.fista_t >= 1.0 && isfinite(opt.fista_t)))
        return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve: fista_t must be 0 or a finite value >= 1");
    if (opt.step < QDT_STEP_SQS || opt.step > QDT_STEP_BB_LS)
        return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve: unknown step mode %d", opt.step);
    const bool bb = opt.step == QDT_STEP_BB || opt.step == QDT_STEP_BB_LS;
    if (bb && opt.accel)
        return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve: the BB step is plain projected gradient (accel = 0)");
    if (opt.exchange != 0 && opt.exchange != 1)
        return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve: exchange must be 0 (allreduce) or 1 (band-aware)");
    if (opt.exchange == 1 && bb)
        return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve: the BB step needs the full residual (exchange = 0)");
    if (opt.check_every < 1) opt.check_every = 16;
    if (opt.kkt_every < 1) opt.kkt_every = 1;
    const bool dev = opt.mem_device != 0;
    qdt_probes *p = const_cast<qdt_probes *>(F);
    const int64_t D = p->D, Ml = p->Ml, M = p->M;
    if (!dev) {
        CKS(check_finite_host(ctx, P, D * Nu, "P"));
        if (opt.theta0)
            CKS(check_finite_host(ctx, opt.theta0, (ctx->nranks > 1 && !opt.gather_theta ? Ml : M) * Nu,
                                  "theta0"));
        if (opt.theta_prev && opt.accel)
            CKS(check_finite_host(ctx, opt.theta_prev, (ctx->nranks > 1 && !opt.gather_theta ? Ml : M) * Nu,
                                  "theta_prev"));
    }
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    Plan *pl;
    NvtxRange nv_solve("qdt_solve");
    CKS(build_plan(ctx, p, (int)N, &pl));

    // memory plan (fails before allocating the big buffers)
    {
        const int nb = opt.accel ? 3 : 2;
        double need = 8.0 * ((double)nb * (Ml + 2) * N + (opt.accel ? 3.0 : 1.0) * D * N + D * N +
                             (double)std::max(pl->nrpart, pl->sw_nrpart) * N +
                             (double)std::max<int64_t>(pl->nslots * pl->T * N, pl->sw_nslots * 1024 * ((pl->NB + 1) / 2 + 1)) +
                             2.0 * Ml);
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        size_t have = fr;
        for (auto &kv : ctx->ws) have += kv.second.n;
        if (need > 0.97 * (double)have)
            return fail(ctx, QDT_ERR_OOM, "memory plan: need %.2f GB, %.2f GB available", need / 1e9,
                        have / 1e9);
    }
    const int fista = opt.accel ? 1 : 0;
    const int nbuf = fista ? 3 : 2;
    SolveBufs b;
    const size_t rowsz = (size_t)(Ml + 2) * N;
    const char *tn[3] = {"theta0", "theta1", "theta2"};
    for (int i = 0; i < nbuf; i++) {
        double *t;
        CKS(ws_get(ctx, tn[i], rowsz + 2, &t));
        b.theta[i] = t + N;
        CK(cudaMemsetAsync(t, 0, sizeof(double) * rowsz, s));
    }
    CKS(common_bufs(ctx, p, pl, N, b));
    if (bb) {
        CKS(ws_get(ctx, "R1", D * N + 4, &b.R[1]));
        CK(cudaMemsetAsync(b.R[1], 0, sizeof(double) * D * N, s));
        CKS(ws_get(ctx, "bb_part", 5 * BB_NBLK, &b.bb_part));
        CKS(ws_get(ctx, "bb_vec", 5, &b.bb_vec));
        CKS(ws_get(ctx, "tbb", 2, &b.tbb));   // [0] t_k, [1] lambda* (line search)
        if (opt.step == QDT_STEP_BB_LS) {
            CKS(ws_get(ctx, "RY", D * N + 4, &b.RY));
            double *t2;
            CKS(ws_get(ctx, "theta2", rowsz + 2, &t2));   // the direction d = Z - Theta_k
            b.theta[2] = t2 + N;
            CK(cudaMemsetAsync(t2, 0, sizeof(double) * rowsz, s));
        }
    }
    if (fista) {
        CKS(ws_get(ctx, "R1", D * N + 4, &b.R[1]));
        CKS(ws_get(ctx, "RY", D * N + 4, &b.RY));
        CK(cudaMemsetAsync(b.R[1], 0, sizeof(double) * D * N, s));
    }
    const int64_t tl = iters + 1;
    // trace buffers sized by capacity (>= 4096 entries), so that calls of different lengths keep
    // the same buffers and the captured loop graph stays valid (the host bounds the iterations)
    const int64_t tcap = std::max<int64_t>(4096, tl);
    CKS(ws_get(ctx, "trace", tcap, &b.trace));
    CKS(ws_get(ctx, "kkt", tcap, &b.kkt));
    CKS(ws_get(ctx, "kktp", tcap, &b.kktp));
    CK(launch_fill(b.trace, tl, NAN, s));
    CK(launch_fill(b.kkt, tl, NAN, s));
    CK(launch_fill(b.kktp, tl, NAN, s));
    ctx->launches += 3;
    if (dev && N == Nu) {
        b.P = const_cast<double *>(P);
    } else {
        CKS(ws_get(ctx, "P", D * N, &b.P));
        if (N != Nu) CK(cudaMemsetAsync(b.P, 0, sizeof(double) * D * N, s));
        CKS(copy_cols(ctx, b.P, N, P, Nu, Nu, D, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    }
    std::vector<double> betas, taus;
    if (fista) {
        // Beck-Teboulle momentum: tau_{k+1} = (1 + sqrt(1 + 4 tau_k^2)) / 2, beta_k = (tau_k - 1) / tau_{k+1},
        // from tau_0 = 1 or the resume state opts.fista_t
        CKS(ws_get(ctx, "beta", tcap, &b.beta));
        betas.resize(tl);
        taus.resize(tl + 1);
        double tau = opt.fista_t >= 1.0 ? opt.fista_t : 1.0;
        for (int64_t k = 0; k < tl; k++) {
            taus[k] = tau;
            double tn_ = (1.0 + sqrt(1.0 + 4.0 * tau * tau)) / 2.0;
            betas[k] = (tau - 1.0) / tn_;
            tau = tn_;
        }
        taus[tl] = tau;
        CK(cudaMemcpyAsync(b.beta, betas.data(), sizeof(double) * tl, cudaMemcpyHostToDevice, s));
    }
    // Theta_0 = 1/N or theta0 (full M x N; local rows when nranks > 1 and
    // !gather_theta)
    if (opt.theta0) {
        const double *src = opt.theta0;
        if (ctx->nranks == 1 || opt.gather_theta) src += p->kb * Nu;
        CKS(copy_cols(ctx, b.theta[0], N, src, Nu, Nu, Ml, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    } else {
        CK(launch_fill(b.theta[0], Ml * N, 1.0 / (double)Nu, s));
        ctx->launches++;
        if (N != Nu) CK(cudaMemset2DAsync(b.theta[0] + Nu, sizeof(double) * N, 0, sizeof(double), Ml, s));
    }
    IterCfg c{p, pl, (int)N, gamma, tol, fista, opt.kkt_every, tcap};
    c.Nv = (int)Nu;
    c.bx = (ctx->nranks > 1 && opt.exchange == 1) ? 1 : 0;
    CKS(halo_exchange(ctx, c, b.theta[0]));
    if (fista && opt.theta_prev) {
        // resume: Theta_{k-1} given (same layout as theta0); R_{k-1} = F Theta_{k-1} - P for the
        // first extrapolated residual R(Y) = (1 + beta) R_k - beta R_{k-1}
        const double *src = opt.theta_prev;
        if (ctx->nranks == 1 || opt.gather_theta) src += p->kb * Nu;
        CKS(copy_cols(ctx, b.theta[2], N, src, Nu, Nu, Ml, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
        CKS(halo_exchange(ctx, c, b.theta[2]));
        CKS(fwd_reduce(ctx, c, b, b.theta[2], b.R[1], true));
    } else if (fista) {
        CK(cudaMemcpyAsync(b.theta[2] - N, b.theta[0] - N, sizeof(double) * rowsz, cudaMemcpyDeviceToDevice, s));
    }
    double tscalar = 0.0;
    {
        NvtxRange nv("qdt_solve:step_setup");
        const int smode = bb ? QDT_STEP_LIPSCHITZ : opt.step;
        if (p->d_tcache && p->tc_mode == smode && p->tc_gamma == gamma) {   // cached step (same F, mode, gamma)
            CK(cudaMemcpyAsync(b.tstep, p->d_tcache, sizeof(double) * Ml, cudaMemcpyDeviceToDevice, s));
            tscalar = p->tc_scalar;
        } else {
            CKS(step_setup(ctx, p, pl, smode, gamma, 100, b.tstep, nullptr, nullptr, &tscalar));
            if (!p->d_tcache) CK(cudaMalloc(&p->d_tcache, sizeof(double) * std::max<int64_t>(1, Ml)));
            CK(cudaMemcpyAsync(p->d_tcache, b.tstep, sizeof(double) * Ml, cudaMemcpyDeviceToDevice, s));
            p->tc_mode = smode;
            p->tc_gamma = gamma;
            p->tc_scalar = tscalar;
        }
    }
    c.bb = bb ? (opt.step == QDT_STEP_BB_LS ? 2 : 1) : 0;
    c.tlip = tscalar;
    DevState st0;
    memset(&st0, 0, sizeof st0);
    st0.iters_done = -1;
    CK(cudaMemcpyAsync(b.state, &st0, sizeof st0, cudaMemcpyHostToDevice, s));

    // ---- small problems: the whole solve in one persistent CTA (qdt_small.cu)
    const bool small = ctx->nranks == 1 && !bb && small_enabled() &&
                       (small_solve_smem(D, Ml, (int)N, p->nnz, fista) <= SMALL_SMEM_MAX ||
                        small_dense_smem(D, Ml, (int)N, fista) <= SMALL_SMEM_MAX) && D * N < (1LL << 30);
    // ---- latency-bound sizes (Medium): the whole solve in one grid-persistent kernel (qdt_coop.cu)
    const bool coop = !small && ctx->nranks == 1 && !bb && coop_enabled() && coop_supported((int)N) &&
                      Ml <= COOP_MAX_ROWS && Ml >= 1 && D * N < (1LL << 30);
    if ((small || coop || pl->NW) && !p->d_row_da) {
        std::vector<int32_t> da(Ml, 0), db(Ml, 0);
        int64_t a0 = 0;
        for (int64_t k = 0; k < Ml; k++) {   // band edges are monotone: contiguous covering probes
            while (a0 < D && (p->len_l[a0] == 0 || p->lo_l[a0] + p->len_l[a0] - 1 - p->kb < k)) a0++;
            int64_t b0 = a0;
            while (b0 < D && p->lo_l[b0] - p->kb <= k && p->len_l[b0] > 0) b0++;
            da[k] = (int32_t)a0;
            db[k] = (int32_t)b0;
        }
        CK(cudaMalloc(&p->d_row_da, sizeof(int32_t) * Ml));
        CK(cudaMalloc(&p->d_row_db, sizeof(int32_t) * Ml));
        CK(cudaMemcpy(p->d_row_da, da.data(), sizeof(int32_t) * Ml, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(p->d_row_db, db.data(), sizeof(int32_t) * Ml, cudaMemcpyHostToDevice));
    }
    if (coop && !p->d_FT) {   // transposed band (once per probe handle)
        std::vector<int32_t> da(Ml), db(Ml);
        CK(cudaMemcpy(da.data(), p->d_row_da, sizeof(int32_t) * Ml, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(db.data(), p->d_row_db, sizeof(int32_t) * Ml, cudaMemcpyDeviceToHost));
        std::vector<int64_t> toff(Ml + 1, 0);
        for (int64_t k = 0; k < Ml; k++) toff[k + 1] = toff[k] + (db[k] - da[k]);
        CK(cudaMalloc(&p->d_toff, sizeof(int64_t) * (Ml + 1)));
        CK(cudaMalloc(&p->d_FT, sizeof(double) * std::max<int64_t>(1, toff[Ml])));
        CK(cudaMemcpy(p->d_toff, toff.data(), sizeof(int64_t) * (Ml + 1), cudaMemcpyHostToDevice));
        CK(run_k(ctx, "build_FT", 1, [&]() { return launch_build_FT(p->band(), (int)D, p->d_row_da, p->d_toff, p->d_FT, s); }));
    }

    // ---- the hot loop: graph of `period` iterations replayed
    const int period = fista ? 12 : 16;   // multiple of the buffer rotation (3 / 2)
    const bool use_graph = opt.use_graph && !ctx->profiling && iters >= period && !ctx->vg && !small && !coop;
    DevState hst;
    int64_t done = 0;
    bool stopped = false;
    cudaGraphExec_t gexec = nullptr;
    int64_t graph_launches = 0;
    if (use_graph) {
        std::vector<uint64_t> key;
        auto put = [&](const void *x, size_t n) {
            const size_t k0 = key.size();
            key.resize(k0 + (n + 7) / 8, 0);
            memcpy(key.data() + k0, x, n);
        };
        put(&c.p->serial, sizeof c.p->serial);   // ids, not addresses: a freed handle's address may
        put(&c.pl->serial, sizeof c.pl->serial); // be reused by a different one
        put(&c.N, sizeof c.N);
        put(&c.gamma, sizeof c.gamma);
        put(&c.tol, sizeof c.tol);
        put(&c.fista, sizeof c.fista);
        put(&c.kkt_every, sizeof c.kkt_every);
        put(&c.trace_len, sizeof c.trace_len);
        put(&c.bb, sizeof c.bb);
        put(&c.tlip, sizeof c.tlip);
        put(&c.Nv, sizeof c.Nv);
        put(&c.bx, sizeof c.bx);
        put(&b, sizeof b);   // every device pointer the loop reads or writes (pointer-only struct)
        put(&period, sizeof period);
        put(&ctx->stream, sizeof ctx->stream);
        if (ctx->gexec && key == ctx->gkey) {
            gexec = ctx->gexec;
            graph_launches = ctx->glaunches;
        } else {
            if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
            ctx->gexec = nullptr;
            ctx->gkey.clear();
            cudaGraph_t g;
            int64_t l0 = ctx->launches;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            qdt_status cs = QDT_OK;
            for (int j = 0; j < period && cs == QDT_OK; j++) cs = iteration(ctx, c, b, j);
            cudaError_t ee = cudaStreamEndCapture(s, &g);
            if (cs != QDT_OK) return cs;
            CK(ee);
            graph_launches = ctx->launches - l0;
            ctx->launches = l0;
            CK(cudaGraphInstantiate(&gexec, g, 0));
            cudaGraphDestroy(g);
            ctx->gexec = gexec;
            ctx->gkey = key;
            ctx->glaunches = graph_launches;
        }
    }
    EventPair evp;
    CK(evp.create());
    cudaEvent_t ev0 = evp.a, ev1 = evp.b;
    NvtxRange nv_loop("qdt_solve:iterations");
    CK(cudaEventRecord(ev0, s));
    const int64_t check = tol > 0.0 ? std::max<int64_t>(period, (opt.check_every / period) * period) : INT64_MAX;
    int64_t since = 0;
    if (small) {
        SmallArgs sa;
        sa.D = (int)D;
        sa.M = (int)Ml;
        sa.N = (int)N;
        sa.nnz = (int)p->nnz;
        sa.lo = p->d_lo;
        sa.len = p->d_len;
        sa.off = p->d_off;
        sa.val = p->d_val;
        sa.row_da = p->d_row_da;
        sa.row_db = p->d_row_db;
        sa.theta0 = b.theta[0];
        sa.theta_prev = (fista && opt.theta_prev) ? b.theta[2] : nullptr;
        sa.P = b.P;
        sa.tstep = b.tstep;
        sa.beta = b.beta;
        sa.gamma = gamma;
        sa.tol = tol;
        sa.iters = iters;
        sa.kkt_every = opt.kkt_every;
        sa.fista = fista;
        sa.trace = b.trace;
        sa.kkt = b.kkt;
        sa.kktp = b.kktp;
        sa.trace_len = tcap;
        sa.theta_out = b.theta[1];
        sa.prev_out = fista ? b.theta[2] : nullptr;
        sa.state = b.state;
        CK(run_k(ctx, "small_solve", 1, [&]() { return launch_small_solve(sa, s); }));
        done = iters;
    } else if (coop) {
        CoopArgs ca;
        ca.D = (int)D;
        ca.M = (int)Ml;
        ca.N = (int)N;
        ca.Nv = (int)Nu;
        ca.lo = p->d_lo;
        ca.len = p->d_len;
        ca.off = p->d_off;
        ca.val = p->d_val;
        ca.row_da = p->d_row_da;
        ca.row_db = p->d_row_db;
        ca.toff = p->d_toff;
        ca.FT = p->d_FT;
        for (int i = 0; i < 3; i++) ca.theta[i] = b.theta[i < nbuf ? i : 0];
        ca.R[0] = b.R[0];
        ca.R[1] = fista ? b.R[1] : b.R[0];
        ca.RY = fista ? b.RY : nullptr;
        ca.P = b.P;
        ca.tstep = b.tstep;
        ca.beta = b.beta;
        ca.gamma = gamma;
        ca.tol = tol;
        ca.iters = iters;
        ca.kkt_every = opt.kkt_every;
        ca.fista = fista;
        ca.resume = (fista && opt.theta_prev) ? 1 : 0;
        ca.trace = b.trace;
        ca.kkt = b.kkt;
        ca.kktp = b.kktp;
        ca.trace_len = tcap;
        double *cpart, *cbar;
        CKS(ws_get(ctx, "coop_part", (int64_t)2 * coop_max_grid() * 4, &cpart));
        CKS(ws_get(ctx, "coop_bar", 1, &cbar));
        CK(cudaMemsetAsync(cbar, 0, sizeof(double), s));
        ca.part = cpart;
        ca.bar = reinterpret_cast<unsigned *>(cbar);
        ca.state = b.state;
        CK(run_k(ctx, "coop_solve", 1, [&]() { return launch_coop_solve(ca, s); }));
        done = iters;
    }
    while (done < iters) {
        if (use_graph && iters - done >= period) {
            CK(cudaGraphLaunch(gexec, s));
            ctx->launches += graph_launches;
            done += period;
            since += period;
        } else {
            CKS(iteration(ctx, c, b, done));
            done += 1;
            since += 1;
        }
        if (since >= check) {
            since = 0;
            CK(cudaMemcpyAsync(&hst, b.state, sizeof hst, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            CKS(nccl_health(ctx));
            if (hst.stop) {
                stopped = true;
                break;
            }
        }
    }
    CK(cudaEventRecord(ev1, s));
    if (pl->NX && getenv("QDT_WDEBUG")) {   // diagnostic: fused wide step geometry and exchanges
        const int ng = pl->wx_ncl * pl->wx_C;
        std::vector<double> hp((size_t)ng * NSC_TILE);
        CK(cudaMemcpyAsync(hp.data(), b.partT, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double ex = 0, mx = 0;
        for (int i = 0; i < ng; i++) {
            ex += hp[(size_t)i * NSC_TILE + SC_DTH];
            mx = std::max(mx, hp[(size_t)i * NSC_TILE + SC_DTH]);
        }
        fprintf(stderr, "[qdt wide] N=%d C=%d Wc=%d clusters=%d tiles=%lld exchanges/CTA mean %.1f max %.0f (last step)\n",
                pl->N, pl->wx_C, pl->wx_Wc, pl->wx_ncl, (long long)((p->Ml + WT - 1) / WT), ex / ng, mx);
    }
    // ---- final evaluation at Theta_iters (if no early stop)
    CK(cudaMemcpyAsync(&hst, b.state, sizeof hst, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    stopped = hst.stop != 0;
    if (!small && !coop && stopped && hst.converged && !hst.nonfinite && (pl->NB || pl->NW || pl->NX) && !fista) {
        // the sweep loop evaluates the unclamped KKT only; re-evaluate Theta_kd once with the
        // general kernels so that trace/kkt/kkt_paper at kd come from one consistent pass
        DevState sr = hst;
        sr.stop = 0;
        sr.it = hst.iters_done;
        CK(cudaMemcpyAsync(b.state, &sr, sizeof sr, cudaMemcpyHostToDevice, s));
        CKS(eval_pass(ctx, c, b, b.theta[hst.iters_done % nbuf]));
        CK(cudaMemcpyAsync(b.state, &hst, sizeof hst, cudaMemcpyHostToDevice, s));
    }
    if (!small && !coop && !stopped) {
        CKS(eval_pass(ctx, c, b, b.theta[iters % nbuf]));
        CK(cudaMemcpyAsync(&hst, b.state, sizeof hst, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    if (hst.nonfinite)
        return fail(ctx, QDT_ERR_NONFINITE, "non-finite objective at iteration %lld", (long long)hst.iters_done);
    const int64_t kd = hst.iters_done;
    const double *res = small ? b.theta[1] : b.theta[kd % nbuf];
    // ---- outputs
    const bool gather = ctx->nranks > 1 && opt.gather_theta;
    if (!theta_out) {
        // result not requested (trace / info only)
    } else if (gather) {
        // assemble the full M x N on every rank: each rank's slice broadcast into place
        double *full;
        CKS(ws_get(ctx, "gather", M * N, &full));
        CKS(gather_rows(ctx, p, res, N, full));
        CKS(copy_cols(ctx, theta_out, Nu, full, N, Nu, M, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
    } else {
        CKS(copy_cols(ctx, theta_out, Nu, res, N, Nu, Ml, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
    }
    if (fista && opt.theta_prev_out) {   // resume state: Theta_{kd-1} (the initial Theta_{-1} when kd = 0)
        const double *prv = small ? b.theta[2] : b.theta[(kd + 2) % 3];
        if (gather) {
            double *full;
            CKS(ws_get(ctx, "gather", M * N, &full));
            CKS(gather_rows(ctx, p, prv, N, full));
            CKS(copy_cols(ctx, opt.theta_prev_out, Nu, full, N, Nu, M, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
        } else {
            CKS(copy_cols(ctx, opt.theta_prev_out, Nu, prv, N, Nu, Ml, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
        }
    }
    std::vector<double> hk(tl);
    if (trace_out) CK(cudaMemcpyAsync(trace_out, b.trace, sizeof(double) * tl, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hk.data(), b.kkt, sizeof(double) * tl, cudaMemcpyDeviceToHost, s));
    double kp_last = NAN;
    CK(cudaMemcpyAsync(&kp_last, b.kktp + kd, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (kkt_out) memcpy(kkt_out, hk.data(), sizeof(double) * tl);
    flush_profile(ctx);
    if (info) {
        info->iters_done = kd;
        info->converged = hst.converged;
        info->kkt0 = hk[0];
        info->kkt = hk[kd];
        info->kkt_paper = kp_last;
        double fl = NAN;
        CK(cudaMemcpyAsync(&fl, b.trace + kd, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        info->f_final = fl;
        info->step_scalar = tscalar;
        info->fista_t = fista ? taus[kd] : 0.0;
        info->k_begin = p->kb;
        info->k_end = p->ke;
        info->nnz = p->nnz;
        info->min_row_mass = p->min_row_mass;
        info->uncovered_rows = p->uncovered;
        float lm = 0.f;
        cudaEventElapsedTime(&lm, ev0, ev1);
        info->loop_ms = lm;
    }
    (void)stopped;
    return QDT_OK;
}

// ------------------------------------------------------------------------------ objective
extern "C" qdt_status qdt_objective(qdt_ctx *ctx, const qdt_probes *F, const double *P,
                                    const double *theta, int64_t Nu, double gamma,
                                    int32_t mem_device, double *f_out, double *kkt_out)
{
    if (!ctx) return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_objective: ctx is NULL");
    if (!F || !P || !theta || !f_out) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_objective: NULL pointer");
    if (F->ctx != ctx) return fail(ctx, QDT_ERR_STATE, "probes built on another ctx");
    if (Nu < 1 || Nu > QDT_NMAX) return fail(ctx, QDT_ERR_INVALID_ARG, "N out of range");
    const int64_t N = pad_cols(Nu);   // internal row pitch (qdt_solve)
    if (!(gamma >= 0.0) || !isfinite(gamma)) return fail(ctx, QDT_ERR_INVALID_ARG, "gamma must be finite >= 0");
    qdt_probes *p = const_cast<qdt_probes *>(F);
    const int64_t D = p->D, Ml = p->Ml;
    const bool dev = mem_device != 0;
    if (!dev) {
        CKS(check_finite_host(ctx, P, D * Nu, "P"));
        CKS(check_finite_host(ctx, theta, p->M * Nu, "theta"));
    }
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    Plan *pl;
    CKS(build_plan(ctx, p, (int)N, &pl));
    SolveBufs b;
    double *t;
    const size_t rowsz = (size_t)(Ml + 2) * N;
    CKS(ws_get(ctx, "theta0", rowsz + 2, &t));
    b.theta[0] = t + N;
    CK(cudaMemsetAsync(t, 0, sizeof(double) * rowsz, s));
    CKS(copy_cols(ctx, b.theta[0] - (p->kb > 0 ? N : 0), N, theta + (p->kb > 0 ? (p->kb - 1) * Nu : 0), Nu, Nu,
                  Ml + (p->kb > 0) + (p->ke < p->M), dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    CKS(common_bufs(ctx, p, pl, N, b));
    CKS(ws_get(ctx, "trace", 1, &b.trace));
    CKS(ws_get(ctx, "kkt", 1, &b.kkt));
    CKS(ws_get(ctx, "kktp", 1, &b.kktp));
    if (dev && N == Nu) {
        b.P = const_cast<double *>(P);
    } else {
        CKS(ws_get(ctx, "P", D * N, &b.P));
        if (N != Nu) CK(cudaMemsetAsync(b.P, 0, sizeof(double) * D * N, s));
        CKS(copy_cols(ctx, b.P, N, P, Nu, Nu, D, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    }
    DevState st0;
    memset(&st0, 0, sizeof st0);
    CK(cudaMemcpyAsync(b.state, &st0, sizeof st0, cudaMemcpyHostToDevice, s));
    IterCfg c{p, pl, (int)N, gamma, 0.0, 0, 1, 1};
    c.Nv = (int)Nu;
    CKS(eval_pass(ctx, c, b, b.theta[0]));
    double f = 0, r = 0;
    CK(cudaMemcpyAsync(&f, b.trace, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&r, b.kkt, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *f_out = f;
    if (kkt_out) *kkt_out = r;
    return QDT_OK;
}

// ------------------------------------------------------------------------------ kernel hooks
static qdt_status hook_common(qdt_ctx *ctx, const qdt_probes *F, int64_t N, Plan **pl)
{
    if (!ctx) return fail(nullptr, QDT_ERR_INVALID_ARG, "ctx is NULL");
    if (!F) return fail(ctx, QDT_ERR_INVALID_ARG, "probes is NULL");
    if (F->ctx != ctx) return fail(ctx, QDT_ERR_STATE, "probes built on another ctx");
    if (ctx->nranks != 1) return fail(ctx, QDT_ERR_INVALID_ARG, "kernel hooks are single-rank only");
    if (N < 1 || N > QDT_NMAX) return fail(ctx, QDT_ERR_INVALID_ARG, "N out of range");
    CK(cudaSetDevice(ctx->device));
    return build_plan(ctx, const_cast<qdt_probes *>(F), (int)N, pl);
}

extern "C" qdt_status qdt_residual(qdt_ctx *ctx, const qdt_probes *F, const double *theta,
                                   const double *P, int64_t N, double *R_out)
{
    Plan *pl;
    CKS(hook_common(ctx, F, N, &pl));
    if (!theta || !R_out) return fail(ctx, QDT_ERR_INVALID_ARG, "NULL pointer");
    qdt_probes *p = const_cast<qdt_probes *>(F);
    cudaStream_t s = ctx->stream;
    SolveBufs b;
    double *t;
    CKS(ws_get(ctx, "theta0", (size_t)(p->Ml + 2) * N + 2, &t));
    b.theta[0] = t + N;
    CK(cudaMemcpyAsync(b.theta[0], theta, sizeof(double) * p->Ml * N, cudaMemcpyHostToDevice, s));
    CKS(common_bufs(ctx, p, pl, N, b));
    if (P) {
        CKS(ws_get(ctx, "P", p->D * N, &b.P));
        CK(cudaMemcpyAsync(b.P, P, sizeof(double) * p->D * N, cudaMemcpyHostToDevice, s));
    }
    IterCfg c{p, pl, (int)N, 0.0, 0.0, 0, 1, 1};
    CKS(fwd_reduce(ctx, c, b, b.theta[0], b.R[0], P != nullptr));
    CK(cudaMemcpyAsync(R_out, b.R[0], sizeof(double) * p->D * N, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return QDT_OK;
}

extern "C" qdt_status qdt_gradient(qdt_ctx *ctx, const qdt_probes *F, const double *R,
                                   const double *theta, int64_t N, double gamma, double *G_out)
{
    Plan *pl;
    CKS(hook_common(ctx, F, N, &pl));
    if (!theta || !R || !G_out) return fail(ctx, QDT_ERR_INVALID_ARG, "NULL pointer");
    if (!(gamma >= 0.0) || !isfinite(gamma)) return fail(ctx, QDT_ERR_INVALID_ARG, "gamma must be finite >= 0");
    if (!pl->gen) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_gradient: N = %lld > %d (general kernels)", (long long)N, GEN_NMAX);
    qdt_probes *p = const_cast<qdt_probes *>(F);
    cudaStream_t s = ctx->stream;
    SolveBufs b;
    double *t, *G;
    CKS(ws_get(ctx, "theta0", (size_t)(p->Ml + 2) * N + 2, &t));
    b.theta[0] = t + N;
    CK(cudaMemcpyAsync(b.theta[0], theta, sizeof(double) * p->Ml * N, cudaMemcpyHostToDevice, s));
    CKS(common_bufs(ctx, p, pl, N, b));
    CK(cudaMemcpyAsync(b.R[0], R, sizeof(double) * p->D * N, cudaMemcpyHostToDevice, s));
    CKS(ws_get(ctx, "theta1", (size_t)(p->Ml + 2) * N + 2, &G));
    IterCfg c{p, pl, (int)N, gamma, 0.0, 0, 1, 1};
    BwdArgs a = bwd_args(ctx, c, b, b.R[0], b.theta[0], nullptr, G, false);
    a.state = nullptr;
    CK(run_k(ctx, "bwd_grad", 1, [&]() { return launch_bwd(a, pl->nbunits, pl->TC, BWD_GRAD, s); }));
    CK(cudaMemcpyAsync(G_out, G, sizeof(double) * p->Ml * N, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return QDT_OK;
}

extern "C" qdt_status qdt_step(qdt_ctx *ctx, const qdt_probes *F, const double *P,
                               const double *theta, int64_t N, double gamma, int32_t step_mode,
                               double *theta_next)
{
    if (!theta_next) return fail(ctx, QDT_ERR_INVALID_ARG, "NULL pointer");
    qdt_solve_opts o = {step_mode, 0, theta, 16, 1, 0, 0, 0};
    return qdt_solve(ctx, F, P, N, gamma, 0.0, 1, &o, theta_next, nullptr, nullptr, nullptr);
}

extern "C" qdt_status qdt_project_rows(qdt_ctx *ctx, const double *X, int64_t M, int64_t N,
                                       double *Y_out)
{
    if (!ctx) return fail(nullptr, QDT_ERR_INVALID_ARG, "ctx is NULL");
    if (!X || !Y_out) return fail(ctx, QDT_ERR_INVALID_ARG, "NULL pointer");
    if (M < 1 || N < 1 || N > INT32_MAX) return fail(ctx, QDT_ERR_INVALID_ARG, "bad shape");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    double *dx, *dy;
    CKS(ws_get(ctx, "projX", M * N, &dx));
    CKS(ws_get(ctx, "projY", M * N, &dy));
    CK(cudaMemcpyAsync(dx, X, sizeof(double) * M * N, cudaMemcpyHostToDevice, s));
    CK(run_k(ctx, "project_rows", 1, [&]() { return launch_project_rows(dx, M, (int)N, dy, s); }));
    CK(cudaMemcpyAsync(Y_out, dy, sizeof(double) * M * N, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return QDT_OK;
}

// ------------------------------------------------------------------------------ smoothing
extern "C" qdt_status qdt_smooth(qdt_ctx *ctx, const double *theta, int64_t M, int64_t N, int64_t exclude,
                                 int64_t div, int32_t mem_device, double *out)
{
    if (!ctx) return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_smooth: ctx is NULL");
    if (!theta || !out) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_smooth: NULL pointer");
    if (M < 1 || N < 1 || N > INT32_MAX || exclude < 0)
        return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_smooth: bad shape / exclude");
    if (ctx->nranks != 1) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_smooth: single rank only");
    const bool dev = mem_device != 0;
    if (!dev) CKS(check_finite_host(ctx, theta, M * N, "theta"));
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int64_t nch = (M + 255) / 256;
    double *X, *Y, *S, *T, *Tx;
    CKS(ws_get(ctx, "sm_S", M * N, &S));
    CKS(ws_get(ctx, "sm_T", nch * N, &T));
    CKS(ws_get(ctx, "sm_Tx", (nch + 1) * N, &Tx));
    if (dev) {
        X = const_cast<double *>(theta);
        Y = out;
    } else {
        CKS(ws_get(ctx, "sm_X", M * N, &X));
        CKS(ws_get(ctx, "sm_Y", M * N, &Y));
        CK(cudaMemcpyAsync(X, theta, sizeof(double) * M * N, cudaMemcpyHostToDevice, s));
    }
    CK(run_k(ctx, "smooth", 3, [&]() { return launch_smooth(X, M, (int)N, exclude, div, S, T, Tx, Y, s); }));
    if (!dev) CK(cudaMemcpyAsync(out, Y, sizeof(double) * M * N, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return QDT_OK;
}

// ------------------------------------------------------------------------------ Newton solve
// Host orchestration of the two-stage two-metric projected truncated Newton (include/qdt.h;
// reading R16), step for step as the oracle's or_newton: every vector operation, Hessian
// product, projection and reduction runs in kernels; the host holds the scalars of CG and the
// line search (one device->host copy per scalar decision).
namespace {
struct NtBufs {
    double *theta, *T1, *X, *g, *gr, *x, *r, *z, *d, *Hd, *u, *Rd, *h, *part, *scal, *d0;
    uint8_t *act;
    int32_t *m;
    int *neg;
};
}  // namespace

extern "C" qdt_status qdt_solve_newton(qdt_ctx *ctx, const qdt_probes *F, const double *P, int64_t N,
                                       double gamma, double eps_kkt, const qdt_newton_opts *o,
                                       double *theta_out, double *trace_out, double *kkt_out,
                                       int32_t *stage_out, int32_t *cg_out, double *alpha_out,
                                       qdt_newton_info *info)
{
    if (!ctx) return fail(nullptr, QDT_ERR_INVALID_ARG, "qdt_solve_newton: ctx is NULL");
    if (!F || !P || !theta_out || !o) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve_newton: NULL pointer");
    if (F->ctx != ctx) return fail(ctx, QDT_ERR_STATE, "qdt_solve_newton: probes built on another ctx");
    if (ctx->nranks != 1) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve_newton: single rank only");
    if (N < 1 || N > GEN_NMAX) return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve_newton: N out of range (max %d)", GEN_NMAX);
    if (!(gamma >= 0.0) || !isfinite(gamma)) return fail(ctx, QDT_ERR_INVALID_ARG, "gamma must be finite >= 0");
    if (o->max_iter < 0 || o->cg_max < 1 || o->max_ls < 1 || !(eps_kkt >= 0.0))
        return fail(ctx, QDT_ERR_INVALID_ARG, "qdt_solve_newton: bad options");
    qdt_probes *p = const_cast<qdt_probes *>(F);
    const int64_t D = p->D, M = p->Ml, n = M * N;
    const bool dev = o->mem_device != 0;
    if (!dev) {
        CKS(check_finite_host(ctx, P, D * N, "P"));
        if (o->theta0) CKS(check_finite_host(ctx, o->theta0, n, "theta0"));
    }
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    Plan *pl;
    CKS(build_plan(ctx, p, (int)N, &pl));
    {
        const double need = 8.0 * (14.0 * (M + 2) * N + 3.0 * D * N) + (double)n;
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        size_t have = fr;
        for (auto &kv : ctx->ws) have += kv.second.n;
        if (need > 0.97 * (double)have)
            return fail(ctx, QDT_ERR_OOM, "newton memory plan: need %.2f GB, %.2f GB available", need / 1e9,
                        have / 1e9);
    }
    SolveBufs b;
    NtBufs v;
    const size_t hz = (size_t)(M + 2) * N + 2;   // halo rows -1 and M (zero) + bulk-copy slack
    auto halo = [&](const char *name, double **out) -> qdt_status {
        double *t;
        CKS(ws_get(ctx, name, hz, &t));
        CK(cudaMemsetAsync(t, 0, sizeof(double) * hz, s));
        *out = t + N;
        return QDT_OK;
    };
    CKS(halo("theta0", &v.theta));
    b.theta[0] = v.theta;
    CKS(halo("nt_T1", &v.T1));
    CKS(halo("nt_d", &v.d));
    CKS(halo("nt_u", &v.u));
    CKS(halo("nt_X", &v.X));
    CKS(ws_get(ctx, "nt_g", n + 2, &v.g));
    CKS(ws_get(ctx, "nt_gr", n + 2, &v.gr));
    CKS(ws_get(ctx, "nt_x", n + 2, &v.x));
    CKS(ws_get(ctx, "nt_r", n + 2, &v.r));
    CKS(ws_get(ctx, "nt_z", n + 2, &v.z));
    CKS(ws_get(ctx, "nt_Hd", n + 2, &v.Hd));
    CKS(ws_get(ctx, "nt_d0", n + 2, &v.d0));
    CKS(ws_get(ctx, "nt_Rd", D * N + 4, &v.Rd));
    CKS(ws_get(ctx, "nt_h", M + 2, &v.h));
    CKS(ws_get(ctx, "nt_part", 4 * NT_BLK + 8, &v.part));
    CKS(ws_get(ctx, "nt_scal", 8, &v.scal));
    CKS(ws_get(ctx, "nt_act", n + 8, &v.act));
    CKS(ws_get(ctx, "nt_m", M + 2, &v.m));
    CKS(ws_get(ctx, "nt_neg", 2, &v.neg));
    CKS(common_bufs(ctx, p, pl, N, b));
    if (dev) {
        b.P = const_cast<double *>(P);
    } else {
        CKS(ws_get(ctx, "P", D * N, &b.P));
        CK(cudaMemcpyAsync(b.P, P, sizeof(double) * D * N, cudaMemcpyHostToDevice, s));
    }
    if (o->theta0)
        CK(cudaMemcpyAsync(v.theta, o->theta0, sizeof(double) * n,
                           dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    else
        CK(launch_fill(v.theta, n, 1.0 / (double)N, s));
    IterCfg c{p, pl, (int)N, gamma, 0.0, 0, 1, 1};
    // Hessian diagonal h_k = 2 (sum_d F_{d,k}^2 + gamma L_kk) from the tiled F (once)
    CKS(build_sweep_tiling(ctx, p));
    CK(run_k(ctx, "nt_setup", 1, [&]() {
        return nt_hdiag(p->sw_ntiles, (int)M, p->kb, p->M, p->d_sw_dA, p->d_sw_dB, p->d_fb_off, p->d_Fb, gamma,
                        v.h, s);
    }));
    double *hs = nullptr;
    CK(cudaMallocHost(&hs, sizeof(double) * 8));
    std::unique_ptr<double, decltype(&cudaFreeHost)> hs_guard(hs, &cudaFreeHost);   // freed on every return
    auto fetch = [&](int k) -> double {
        cudaMemcpyAsync(hs, v.scal, sizeof(double) * k, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        return hs[0];
    };
    auto hess = [&](const double *vin, double *out) -> qdt_status {
        CKS(fwd_reduce(ctx, c, b, vin, v.Rd, false));
        BwdArgs a = bwd_args(ctx, c, b, v.Rd, vin, nullptr, out, false);
        a.state = nullptr;
        CK(run_k(ctx, "nt_hess", 1, [&]() { return launch_bwd(a, pl->nbunits, pl->TC, BWD_GRAD, s); }));
        return QDT_OK;
    };
    auto grad = [&](const double *th) -> qdt_status {   // g = 2 G(th); R[0] = F th - P
        CKS(fwd_reduce(ctx, c, b, th, b.R[0], true));
        BwdArgs a = bwd_args(ctx, c, b, b.R[0], th, nullptr, v.g, false);
        a.state = nullptr;
        CK(run_k(ctx, "nt_grad", 1, [&]() { return launch_bwd(a, pl->nbunits, pl->TC, BWD_GRAD, s); }));
        CK(nt_scale_mask(v.g, nullptr, 2.0, n, s));
        return QDT_OK;
    };
    auto fval = [&](const double *th, const double *R, const double *g, double *kk) -> double {
        nt_fparts(R, D * N, th, g, M, (int)N, v.part, v.scal, s);
        cudaMemcpyAsync(hs, v.scal, sizeof(double) * 4, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (kk) *kk = sqrt(hs[2] / ((double)N * (double)M));
        return hs[0] + gamma * hs[1];
    };
    // direction: PCG on the metric (stage 2 when mrow != nullptr); x = p, returns CG iterations
    auto direction = [&](const int32_t *mrow, const double *th, int64_t *it_out) -> qdt_status {
        CK(nt_pcg_init(v.g, th, v.h, mrow, (int)N, n, o->eps_active, v.gr, v.act, v.x, v.r, v.z, v.d, v.part,
                       v.scal, s));
        const double bn = sqrt(fetch(1));
        const double tol = fmin(0.5, sqrt(bn)) * bn;
        CK(nt_dot(v.r, v.z, nullptr, nullptr, 0, n, v.part, v.scal, s));
        double rz = fetch(1);
        int64_t it = 0;
        for (it = 0; it < o->cg_max && bn > 0.0; it++) {
            if (rz <= 0.0) break;
            if (mrow) {
                CK(nt_zexp(v.d, mrow, M, (int)N, v.u, s));
                CKS(hess(v.u, v.Hd));
                CK(nt_scale_mask(v.Hd, nullptr, 2.0, n, s));
                CK(nt_zred(v.Hd, mrow, v.act, M, (int)N, s));
            } else {
                CKS(hess(v.d, v.Hd));
                CK(nt_scale_mask(v.Hd, v.act, 2.0, n, s));
            }
            CK(nt_dot(v.d, v.Hd, nullptr, nullptr, 0, n, v.part, v.scal, s));
            const double dHd = fetch(1);
            if (dHd <= 0.0) break;
            const double a = rz / dHd;
            CK(nt_cg_update(v.x, v.r, v.z, v.d, v.Hd, a, v.h, mrow, (int)N, n, v.part, v.scal, s));
            cudaMemcpyAsync(hs, v.scal, sizeof(double) * 2, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            if (sqrt(hs[0]) <= tol) {
                it++;
                break;
            }
            const double rz2 = hs[1];
            const double beta = rz2 / rz;
            rz = rz2;
            CK(nt_cg_dir(v.d, v.z, beta, n, s));
        }
        *it_out = it;
        return QDT_OK;
    };
    const int64_t K = o->max_iter;
    std::vector<double> tr(K + 1, NAN), kt(K + 1, NAN), al(K, NAN);
    std::vector<int32_t> stg(K, 0), cgl(K, 0);
    int stage = 1;
    int64_t k = 0, sw = -1, cg_total = 0;
    double f_last = NAN, kkt_last = NAN;
    EventPair ev;
    CK(ev.create());
    cudaEvent_t e0 = ev.a, e1 = ev.b;
    CK(cudaEventRecord(e0, s));
    for (k = 0;; k++) {
        CKS(grad(v.theta));
        double r;
        const double f = fval(v.theta, b.R[0], v.g, &r);
        tr[k] = f;
        kt[k] = r;
        f_last = f;
        kkt_last = r;
        if (!isfinite(f)) return fail(ctx, QDT_ERR_NONFINITE, "newton: non-finite objective at %lld", (long long)k);
        if (r <= eps_kkt || k >= K) break;
        int64_t it = 0;
        double f0 = f;
        double slope = 0.0;   // one-sided arc derivative at alpha = 0 of the stage that steps
        if (stage == 1) {
            CKS(direction(nullptr, v.theta, &it));
            CK(nt_tangent(v.theta, v.x, M, (int)N, v.d0, s));
            CK(nt_dot(v.g, v.d0, nullptr, nullptr, 0, n, v.part, v.scal, s));
            slope = fetch(1);
            if (fabs(slope) <= o->switch_tol) {
                stage = 2;
                sw = k;
            }
        }
        const int us = stage;   // the stage this iteration steps with
        if (us == 2) {
            CK(nt_transform(v.theta, M, (int)N, v.m, s));
            CKS(grad(v.theta));
            CKS(direction(v.m, v.theta, &it));
            // stage-2 arc slope: reduced gradient . p with p_j -> 0 where theta_j <= 0 and p_j < 0
            CK(nt_dot(v.gr, v.x, nullptr, v.theta, 2, n, v.part, v.scal, s));
            slope = fetch(1);
            f0 = fval(v.theta, b.R[0], nullptr, nullptr);
        }
        const bool paper_armijo = o->armijo == 0;
        double alpha = 0.0;
        bool accepted = false;
        for (int64_t l = 0; l < o->max_ls && !accepted; l++) {
            const double a = pow(0.75, (double)l);
            if (us == 1) {
                CK(nt_axpy(v.theta, v.x, a, n, v.X, s));
                CK(launch_project_rows(v.X, M, (int)N, v.T1, s));
            } else {
                CK(cudaMemsetAsync(v.neg, 0, sizeof(int), s));
                CK(nt_clamp_arc(v.theta, v.x, a, v.m, M, (int)N, v.T1, v.neg, s));
                int hneg = 0;
                CK(cudaMemcpyAsync(&hneg, v.neg, sizeof(int), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                if (hneg) continue;
            }
            if (paper_armijo) {
                // f(P[Theta + a p]) <= f(Theta) + c a slope; no descent certified
                // (slope >= 0): no admissible step length
                if (!(slope < 0.0)) break;
                CKS(fwd_reduce(ctx, c, b, v.T1, v.Rd, true));
                const double f1 = fval(v.T1, v.Rd, nullptr, nullptr);
                if (f1 <= f0 + 0.1 * a * slope) {
                    accepted = true;
                    alpha = a;
                }
                continue;
            }
            CK(nt_dotdiff(us == 2 ? v.gr : v.g, v.T1, v.theta, us == 2 ? v.m : nullptr, (int)N, n, v.part,
                          v.scal, s));
            const double dd = fetch(1);
            CKS(fwd_reduce(ctx, c, b, v.T1, v.Rd, true));
            const double f1 = fval(v.T1, v.Rd, nullptr, nullptr);
            if (f1 <= f0 + 0.1 * dd) {
                accepted = true;
                alpha = a;
            }
        }
        if (!accepted && us == 1) {   // stage 1 carries no convergence proof: switch, redo k
            stage = 2;
            sw = k;
            k--;
            continue;
        }
        if (k < K) {
            stg[k] = us;
            cgl[k] = (int32_t)it;
            al[k] = alpha;
        }
        cg_total += it;
        if (!accepted) break;
        CK(cudaMemcpyAsync(v.theta, v.T1, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    }
    CK(cudaEventRecord(e1, s));
    CK(cudaMemcpyAsync(theta_out, v.theta, sizeof(double) * n,
                       dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (trace_out) memcpy(trace_out, tr.data(), sizeof(double) * (K + 1));
    if (kkt_out) memcpy(kkt_out, kt.data(), sizeof(double) * (K + 1));
    if (stage_out && K) memcpy(stage_out, stg.data(), sizeof(int32_t) * K);
    if (cg_out && K) memcpy(cg_out, cgl.data(), sizeof(int32_t) * K);
    if (alpha_out && K) memcpy(alpha_out, al.data(), sizeof(double) * K);
    if (info) {
        info->iters_done = k;
        info->switch_iter = sw;
        info->cg_total = cg_total;
        info->f_final = f_last;
        info->kkt = kkt_last;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        info->loop_ms = ms;
    }
    return QDT_OK;
}
