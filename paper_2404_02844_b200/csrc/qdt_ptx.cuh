// qdt_ptx.cuh -- inline PTX / warp helpers shared by the sm_100a kernel files (mbarrier,
// bulk and tensor TMA copies, fp64 DMMA, quad / warp reductions).  Internal, not the ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace qdt {
// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// bulk global -> shared copy (16-byte aligned addresses, size a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 2-D tensor copy (TMA): box at coordinates (x, y) of the tensor map into shared memory;
// out-of-bounds elements (columns >= N of the padded box, rows past the array) arrive as zeros
__device__ __forceinline__ void tma_2d(void *dst, const CUtensorMap *tm, int x, int y, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
// bulk prefetch of a global range into L2 (no shared memory, no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// D(8x8) += A(8x4) B(4x8), fp64 tensor core.  Fragments (lane = 4 g + t):
//   a = A[g][t], b = B[t][g], (c0, c1) = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// fp64 min / max as compare + select (DSETP + two FSEL): sm_100a has no fp64 min/max instruction
// and fmin/fmax lower to a NaN-quieting sequence about twice as long.  For non-NaN operands the
// value is that of fmin / fmax; a NaN x is skipped (as by fmin / fmax), a NaN m propagates (the
// solve's non-finite check reports it).
__device__ __forceinline__ double dmin(double m, double x) { return x < m ? x : m; }
__device__ __forceinline__ double dmax(double m, double x) { return x > m ? x : m; }

// Order-preserving 32-bit key of a double's high word (sign-magnitude -> two's complement): x <= y
// implies dkey(x) <= dkey(y).  The key drops the low 32 mantissa bits, so a key minimum / maximum
// bounds the fp64 one from below through dkey_floor (the least double of the key's bucket).  Used
// where the row epilogues need a BOUND only (the Michelot start max X - 1, the "every entry stays
// active" and "min of the active set > tau" early exits): integer-pipe min / max and one 32-bit
// shuffle per exchange instead of DSETP + two FSEL on the half-rate fp64 pipe and two shuffles.
__device__ __forceinline__ int dkey(double x)
{
    const int h = __double2hiint(x);
    return h ^ ((h >> 31) & 0x7fffffff);
}
// identities of the key max / min: the keys of -inf and +inf (an empty reduction floors to -inf / +inf)
constexpr int DKEY_NINF = (int)0x800fffffu, DKEY_PINF = 0x7ff00000;
__device__ __forceinline__ double dkey_floor(int k)
{
    const int h = k ^ ((k >> 31) & 0x7fffffff);
    const bool top = (h & 0x7ff00000) == 0x7ff00000;   // the +-inf bucket: the infinity itself
    // negative: the largest magnitude of the bucket
    return __hiloint2double(top ? (h & (int)0xfff00000u) : h, (h < 0 && !top) ? -1 : 0);
}
__device__ __forceinline__ int quad_max_i(int v)
{
    v = max(v, __shfl_xor_sync(0xffffffffu, v, 1));
    v = max(v, __shfl_xor_sync(0xffffffffu, v, 2));
    return v;
}
__device__ __forceinline__ int quad_min_i(int v)
{
    v = min(v, __shfl_xor_sync(0xffffffffu, v, 1));
    v = min(v, __shfl_xor_sync(0xffffffffu, v, 2));
    return v;
}
// max(x, 0) by the sign bit (three integer-pipe operations, no fp64 compare); -0.0 gives +0.0
__device__ __forceinline__ double dclamp0(double x)
{
    const int h = __double2hiint(x), m = ~(h >> 31);
    return __hiloint2double(h & m, __double2loint(x) & m);
}

__device__ __forceinline__ double quad_sum(double v)
{
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    return v;
}
__device__ __forceinline__ int quad_sum_i(int v)
{
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    return v;
}
__device__ __forceinline__ double quad_max(double v)
{
    v = dmax(v, __shfl_xor_sync(0xffffffffu, v, 1));
    v = dmax(v, __shfl_xor_sync(0xffffffffu, v, 2));
    return v;
}
__device__ __forceinline__ double quad_min(double v)
{
    v = dmin(v, __shfl_xor_sync(0xffffffffu, v, 1));
    v = dmin(v, __shfl_xor_sync(0xffffffffu, v, 2));
    return v;
}
__device__ __forceinline__ double wmin(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double wmax(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int wsum_i(int v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double wsum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---- thread-block clusters (distributed shared memory)
__device__ __forceinline__ uint32_t cluster_ctarank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// every thread of every CTA of the cluster arrives; shared-memory writes before the barrier are
// visible to the cluster's loads after it (release / acquire)
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// load a double from the shared memory of CTA `rank` of the cluster at the address that `p` has
// in this CTA's shared window
__device__ __forceinline__ double ld_dsmem(const double *p, uint32_t rank)
{
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
    return v;
}
// store a double into the shared memory of CTA `rank` of the cluster at the address that `p` has
// in this CTA's shared window (ordered before the next barrier.cluster.arrive.release)
__device__ __forceinline__ void st_dsmem(double *p, uint32_t rank, double v)
{
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
}  // namespace qdt
