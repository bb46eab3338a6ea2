// Latency of a dependent chain of mma.sync m8n8k4 f64 (DMMA) and of dependent DFMA / DADD /
// shared-memory loads / 64-bit shuffles on one warp (clock64 deltas).  nvcc -arch sm_100a.
#include <cstdio>
__global__ void k(double *out, long long *cyc, int n)
{
    __shared__ double sm[1024];
    const int lane = threadIdx.x;
    for (int i = lane; i < 1024; i += 32) sm[i] = 1.0 + i * 1e-9;
    __syncwarp();
    double c0 = lane, c1 = 1.0, a = 1e-3, b = 2e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; i++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    long long t1 = clock64();
    double x = c0 + c1;
    for (int i = 0; i < n; i++) x = fma(x, 1.0000001, 1e-9);
    long long t2 = clock64();
    double y = x;
    for (int i = 0; i < n; i++) y = y + 1e-9;
    long long t3 = clock64();
    int idx = lane;
    for (int i = 0; i < n; i++) idx = (int)sm[(idx + 1) & 1023] & 1023;   // dependent LDS
    long long t4 = clock64();
    double z = y;
    for (int i = 0; i < n; i++) z = __shfl_xor_sync(0xffffffffu, z, 1) + 1e-9;
    long long t5 = clock64();
    // 4 independent DMMA chains
    double d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0, g0 = 0, g1 = 0;
    for (int i = 0; i < n; i++) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(g0), "+d"(g1) : "d"(a), "d"(b));
    }
    long long t6 = clock64();
    out[lane] = x + y + z + idx + d0 + d1 + e0 + e1 + f0 + f1 + g0 + g1;
    if (lane == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
    }
}
int main()
{
    double *o; long long *c, h[6];
    cudaMalloc(&o, 256); cudaMalloc(&c, 64);
    const int n = 1000;
    k<<<1, 32>>>(o, c, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, n); cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("{\"dmma_chain\": %.1f, \"dfma\": %.1f, \"dadd\": %.1f, \"lds_dep\": %.1f, \"shfl64_dadd\": %.1f, \"dmma_4chains_per_iter\": %.1f}\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
    return 0;
}
