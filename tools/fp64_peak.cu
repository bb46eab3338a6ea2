// fp64_peak.cu -- measure the B200 fp64 ceilings the roofline needs (MEASURED_PEAKS.json has
// no fp64 entry): DFMA (CUDA-core) and DMMA (mma.sync m8n8k4 f64 tensor core) throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, double a, double b)
{
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) s += x[i];
    if (s == 1.2345) out[0] = s;
}

__global__ void dmma_kernel(double *out, int iters)
{
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}

int main()
{
    double *out;
    cudaMalloc(&out, 8);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int blocksPerSM : {4, 8}) {
        int grid = nsm * blocksPerSM, block = 256;
        dfma_kernel<<<grid, block>>>(out, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        dfma_kernel<<<grid, block>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 16 * iters * (double)grid * block;
        printf("{\"kind\":\"dfma\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", blocksPerSM, ms,
               flops / ms / 1e9);
    }
    for (int blocksPerSM : {4, 8}) {
        int grid = nsm * blocksPerSM, block = 256;
        dmma_kernel<<<grid, block>>>(out, 100);
        cudaEventRecord(e0);
        dmma_kernel<<<grid, block>>>(out, iters / 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 8 * 4 * 8 * (double)(iters / 4) * grid * (block / 32);
        printf("{\"kind\":\"dmma\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", blocksPerSM, ms,
               flops / ms / 1e9);
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"err\":\"%s\"}\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
