// Latency calibration on B200 for the PCDN step design.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o microbench microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void chase_cg(const unsigned *p, int hops, unsigned *out, long long *cyc)
{
    unsigned x = 0;
    long long t0 = clock64();
    for (int h = 0; h < hops; h++) x = __ldcg(p + x);
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}
__global__ void chase_ca(const unsigned *p, int hops, unsigned *out, long long *cyc)
{
    unsigned x = 0;
    for (int h = 0; h < hops; h++) x = p[x];  // warm L1
    long long t0 = clock64();
    for (int h = 0; h < hops; h++) x = p[x];
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}
__global__ void chase_atomic(unsigned *p, int hops, unsigned *out, long long *cyc)
{
    unsigned x = 0;
    long long t0 = clock64();
    for (int h = 0; h < hops; h++) x = atomicAdd(p + (x & 1023), 0u) & 1023;
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}
__global__ void bar_cta(int iters, long long *cyc)
{
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void bar_cluster(int iters, long long *cyc)
{
    long long t0 = clock64();
    for (int i = 0; i < iters; i++)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__global__ void bar_grid(int iters, unsigned long long *ctr, long long *cyc)
{
    unsigned long long target = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        target += gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ctr, 1ULL);
            while (ld_acq(ctr) < target) {
            }
            __threadfence();
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
// dependent chain of (smem write, syncthreads, smem read): what a block-level reduction costs
__global__ void warp_shfl(int iters, long long *cyc, double *out)
{
    double v = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) v += __shfl_xor_sync(0xffffffffu, v, 1 + (i & 15));
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}


// DSMEM: dependent loads from a peer CTA's shared memory (cluster of 2), and returning atomics
__global__ void dsmem_chase(int hops, long long *cyc, unsigned *out)
{
    __shared__ unsigned buf[1024];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i * 389 + 7) & 1023;
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
        unsigned *peer = cl.map_shared_rank(buf, 1);
        unsigned x = 0;
        long long t0 = clock64();
        for (int h = 0; h < hops; h++) x = peer[x];
        long long t1 = clock64();
        out[0] = x;
        cyc[0] = t1 - t0;
        x = 0;
        t0 = clock64();
        for (int h = 0; h < hops; h++) x = atomicAdd(peer + (x & 1023), 0u) & 1023;
        t1 = clock64();
        out[1] = x;
        cyc[1] = t1 - t0;
        x = 0;
        t0 = clock64();
        for (int h = 0; h < hops; h++) x = buf[x];
        t1 = clock64();
        out[2] = x;
        cyc[2] = t1 - t0;
    }
    cl.sync();
}
// remote store then cluster barrier (the exchange pattern of a broadcast partial)
__global__ void dsmem_bcast_bar(int iters, long long *cyc)
{
    __shared__ double part[16][32];
    cg::cluster_group cl = cg::this_cluster();
    const int G = cl.num_blocks(), me = cl.block_rank();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (threadIdx.x < 32 * G) {
            const int dst = threadIdx.x >> 5, slot = threadIdx.x & 31;
            double *pp = cl.map_shared_rank(&part[me][slot], dst);
            *pp = (double)i;
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && me == 0) cyc[0] = t1 - t0;
}

int main()
{
    int dev = 0, clk = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    const int N = 1 << 18;  // 1 MiB of uint32: L2 resident
    std::vector<unsigned> h(N);
    // random cyclic permutation with stride to defeat prefetch
    std::vector<unsigned> perm(N);
    for (int i = 0; i < N; i++) perm[i] = i;
    unsigned long long r = 88172645463325252ULL;
    for (int i = N - 1; i > 0; i--) {
        r ^= r << 13; r ^= r >> 7; r ^= r << 17;
        int j = r % (i + 1);
        std::swap(perm[i], perm[j]);
    }
    for (int i = 0; i < N; i++) h[perm[i]] = perm[(i + 1) % N];
    unsigned *d, *out;
    long long *cyc;
    unsigned long long *ctr;
    CK(cudaMalloc(&d, N * 4));
    CK(cudaMalloc(&out, 64));
    CK(cudaMalloc(&cyc, 64));
    CK(cudaMalloc(&ctr, 64));
    double *dout;
    CK(cudaMalloc(&dout, 8 * 1024));
    CK(cudaMemcpy(d, h.data(), N * 4, cudaMemcpyHostToDevice));
    long long c;
    const int hops = 4096;
    chase_cg<<<1, 1>>>(d, hops, out, cyc);  // warm L2
    chase_cg<<<1, 1>>>(d, hops, out, cyc);
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("L2 hit latency (ld.cg chase): %.1f cycles\n", (double)c / hops);
    chase_ca<<<1, 1>>>(d, 2048, out, cyc);
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("ld.ca chase over 1 MiB (mostly L1 miss): %.1f cycles\n", (double)c / 2048);
    CK(cudaMemset(d, 0, 4096 * 4));
    chase_atomic<<<1, 1>>>(d, hops, out, cyc);
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("atomicAdd (returning) latency: %.1f cycles\n", (double)c / hops);
    for (int nt : {128, 512, 1024}) {
        bar_cta<<<1, nt>>>(10000, cyc);
        CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
        printf("__syncthreads %4d threads: %.1f cycles\n", nt, (double)c / 10000);
    }
    warp_shfl<<<1, 32>>>(10000, cyc, dout);
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("dependent shfl+dadd: %.1f cycles\n", (double)c / 10000);
    CK(cudaFuncSetAttribute(bar_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int cs : {1, 2, 4, 8, 16}) {
        for (int nt : {128, 512, 1024}) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(cs);
            cfg.blockDim = dim3(nt);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, bar_cluster, 10000, cyc));
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
            printf("cluster barrier %2d CTAs x %4d thr: %.1f cycles\n", cs, nt, (double)c / 10000);
        }
    }
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    for (int g : {16, 64, 148, 296}) {
        for (int nt : {512}) {
            CK(cudaMemset(ctr, 0, 8));
            int iters = 2000;
            void *args[] = {&iters, &ctr, &cyc};
            CK(cudaLaunchCooperativeKernel((void *)bar_grid, g, nt, args, 0, 0));
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
            printf("grid barrier %3d CTAs x %4d thr: %.1f cycles\n", g, nt, (double)c / iters);
        }
    }

    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(128);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, dsmem_chase, 4096, cyc, out));
        CK(cudaDeviceSynchronize());
        long long cc[3];
        CK(cudaMemcpy(cc, cyc, 24, cudaMemcpyDeviceToHost));
        printf("DSMEM load latency: %.1f cycles; DSMEM returning atomic: %.1f; local smem: %.1f\n",
               cc[0] / 4096.0, cc[1] / 4096.0, cc[2] / 4096.0);
    }
    CK(cudaFuncSetAttribute(dsmem_bcast_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int cs : {2, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(512);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, dsmem_bcast_bar, 10000, cyc));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
        printf("DSMEM broadcast + cluster barrier %2d CTAs x 512: %.1f cycles\n", cs, (double)c / 10000);
    }
    printf("SM clock attribute %d kHz, %d SMs\n", clk, nsm);
    return 0;
}
