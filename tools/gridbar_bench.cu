// Microbenchmark: cost of a software grid barrier in a persistent kernel on
// B200 (flat counter vs two-level counter), used to size a per-step
// grid-synchronised front kernel.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// tools/gridbar_bench.cu -o /tmp/gridbar && /tmp/gridbar
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// flat: every CTA adds to one counter, spins on the generation word
__global__ void flat_bar(unsigned* cnt, unsigned* gen, int iters) {
    unsigned g = 0;
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            unsigned old = atomicAdd(cnt, 1u);
            if (old == gridDim.x - 1) {
                *cnt = 0;
                __threadfence();
                atomicAdd(gen, 1u);
            } else {
                while (ld_acquire(gen) == g) {}
            }
        }
        ++g;
        __syncthreads();
    }
}

// two-level: CTAs arrive at one of G group counters; the last of a group
// arrives at the root; the root's last arriver bumps the generation
__global__ void tree_bar(unsigned* cnt, unsigned* gen, int iters, int G) {
    unsigned g = 0;
    const int grp = blockIdx.x % G;
    const unsigned gsize = (gridDim.x - grp + G - 1) / G;
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            bool last = false;
            unsigned old = atomicAdd(cnt + 32 * (grp + 1), 1u);
            if (old == gsize - 1) {
                cnt[32 * (grp + 1)] = 0;
                unsigned o2 = atomicAdd(cnt, 1u);
                if (o2 == (unsigned)G - 1) {
                    cnt[0] = 0;
                    __threadfence();
                    atomicAdd(gen, 1u);
                    last = true;
                }
            }
            if (!last)
                while (ld_acquire(gen) == g) {}
        }
        ++g;
        __syncthreads();
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *cnt, *gen;
    cudaMalloc(&cnt, 64 * 1024);
    cudaMalloc(&gen, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000;
    for (int per = 1; per <= 2; ++per) {
        for (int threads : {256, 512}) {
            int grid = sms * per;
            for (int G : {0, 8, 16, 37}) {
                cudaMemset(cnt, 0, 64 * 1024);
                cudaMemset(gen, 0, 4);
                void* args0[] = {&cnt, &gen, (void*)&iters};
                void* args1[] = {&cnt, &gen, (void*)&iters, &G};
                for (int rep = 0; rep < 2; ++rep) {
                    cudaMemset(cnt, 0, 64 * 1024);
                    cudaMemset(gen, 0, 4);
                    cudaEventRecord(e0);
                    cudaError_t err;
                    if (G == 0)
                        err = cudaLaunchCooperativeKernel((void*)flat_bar, grid, threads, args0);
                    else
                        err = cudaLaunchCooperativeKernel((void*)tree_bar, grid, threads, args1);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    if (err != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(err)); return 1; }
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (rep == 1)
                        printf("grid %4d x %3d  %s G=%2d : %.3f us per barrier\n", grid, threads,
                               G ? "tree" : "flat", G, 1e3 * ms / iters);
                }
            }
        }
    }
    return 0;
}
