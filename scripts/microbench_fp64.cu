// fp64 latency / throughput calibration on B200: dependent DFMA chain, independent
// DFMA throughput per SM, and the latency of the logistic loss-change / coef bodies (exp, expm1,
// log1p) as the step kernels use them.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb64 microbench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_chain(int iters, double *out, long long *cyc)
{
    double x = threadIdx.x * 1e-3, a = 1.0000001, b = 1e-9;
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) x = fma(x, a, b);
    const long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void dfma_tput(int iters, double *out, long long *cyc)
{
    double x[8];
    for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-3 + k;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = fma(x[k], 1.0000001, 1e-9);
    __syncthreads();
    const long long t1 = clock64();
    double s = 0;
    for (int k = 0; k < 8; k++) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void lr_chain(int iters, double *out, long long *cyc)
{
    double u = 0.3 + threadIdx.x * 1e-6, s = 0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        s += log1p(expm1(-u) * 0.4);
        u = u * 0.999 + s * 1e-9;
    }
    const long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void exp_chain(int iters, double *out, long long *cyc)
{
    double u = 0.3 + threadIdx.x * 1e-6, s = 0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        const double e = exp(-u);
        s += 1.0 / (1.0 + e);
        u = u * 0.999 + s * 1e-9;
    }
    const long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main()
{
    double *out;
    long long *cyc, h[1024];
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 8192);
    const int it = 4096;
    dfma_chain<<<1, 32>>>(it, out, cyc);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)h[0] / it);
    for (int nt : {128, 256, 512, 1024}) {
        dfma_tput<<<148, nt>>>(it, out, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA throughput, %4d threads/SM: %.1f DFMA/cycle/SM\n", nt, (double)it * 8 * nt / h[0]);
    }
    lr_chain<<<1, 32>>>(256, out, cyc);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("log1p(expm1(-u) * c) dependent latency: %.0f cycles\n", (double)h[0] / 256);
    exp_chain<<<1, 32>>>(256, out, cyc);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("exp + 1/(1+e) dependent latency: %.0f cycles\n", (double)h[0] / 256);
    return 0;
}
