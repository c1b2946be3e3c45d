// Dependent-load latency on B200 (pointer chase): one thread per CTA chases a random cycle through
// an array of `bytes` (stride = 32-B sectors), for `nctas` CTAs at once (1 = unloaded).  Prints
// cycles per load.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a microbench_lat.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void chase(const unsigned *__restrict__ next, long long steps, unsigned start, unsigned long long *out)
{
    unsigned p = start + blockIdx.x * 7919u;
    p = p % 1024u;
    const long long t0 = clock64();
    for (long long s = 0; s < steps; s++) p = __ldcg(&next[(size_t)p * 8]);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0) + (p == 0xffffffffu);
}

int main()
{
    const size_t sizes[] = {8ull << 20, 32ull << 20, 128ull << 20, 512ull << 20, 2048ull << 20, 6144ull << 20};
    for (size_t bytes : sizes) {
        const size_t nsec = bytes / 32;
        std::vector<unsigned> perm(nsec);
        for (size_t i = 0; i < nsec; i++) perm[i] = (unsigned)i;
        std::mt19937_64 rng(1);
        std::shuffle(perm.begin(), perm.end(), rng);
        std::vector<unsigned> h(nsec * 8, 0);
        for (size_t i = 0; i < nsec; i++) h[(size_t)perm[i] * 8] = perm[(i + 1) % nsec];
        unsigned *d;
        unsigned long long *o;
        cudaMalloc(&d, nsec * 32);
        cudaMalloc(&o, 1024 * 8);
        cudaMemcpy(d, h.data(), nsec * 32, cudaMemcpyHostToDevice);
        for (int nctas : {1, 148, 1184}) {
            const long long steps = 2000;
            chase<<<nctas, 32>>>(d, 100, 0, o);
            chase<<<nctas, 32>>>(d, steps, 12345, o);
            cudaDeviceSynchronize();
            std::vector<unsigned long long> ho(nctas);
            cudaMemcpy(ho.data(), o, 8 * nctas, cudaMemcpyDeviceToHost);
            double m = 0;
            for (auto v : ho) m += (double)v;
            printf("bytes %6zu MB  ctas %5d  cycles/load %.0f\n", bytes >> 20, nctas, m / nctas / steps);
        }
        cudaFree(d);
        cudaFree(o);
    }
    return 0;
}
