// Read-bandwidth probe for the dense activity scan's access pattern: 33.5 MB
// planes (16384^2 bits), 4 planes cycled so each read is L2-cold, 20
// launches per CUDA graph.  (1) grid-stride 16-byte loads, (2) one 4 KB bulk
// copy (cp.async.bulk) per warp-row into shared memory, 8 rows per CTA,
// (3) the same rows as 16-byte loads.  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o read_bw tools/read_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) rd_stride(const uint4* p, size_t n, uint32_t* out) {
    uint32_t a = 0;
    for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) {
        const uint4 v = __ldcs(p + i);
        a |= v.x | v.y | v.z | v.w;
    }
    if (a == 0x12345678u) out[0] = a;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int ROWS>
__global__ void __launch_bounds__(32 * ROWS) rd_bulk(const char* p, uint32_t* out) {
    __shared__ __align__(128) char buf[ROWS][4096];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (w == 0) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)),
                         "r"(ROWS * 4096) : "memory");
        __syncwarp();
        if (lane < ROWS)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                    sa(buf[lane])),
                "l"(p + ((size_t)blockIdx.x * ROWS + lane) * 4096), "r"(sa(&bar))
                : "memory");
    }
    asm volatile(
        "{\n .reg .pred q;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n @!q bra W_%=;\n}" ::"r"(
            sa(&bar))
        : "memory");
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint4 v = *reinterpret_cast<const uint4*>(&buf[w][lane * 128 + ((k + lane) & 7) * 16]);
        a |= v.x | v.y | v.z | v.w;
    }
    if (a == 0x12345678u) out[0] = a;
}

// the dense scan's strip pattern: CTA (bx, by) reads 8 region rows of 32
// tiles starting at tile column bx*W-1 and tile row by*R-1 (clipped)
template <int W, int R>
__global__ void __launch_bounds__(256) rd_strip(const char* p, uint32_t* out, int tiles) {
    __shared__ __align__(128) char buf[8][4096];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int x0 = blockIdx.x * W - (W < 32 ? 1 : 0), y0 = blockIdx.y * R - (R < 8 ? 1 : 0);
    const int c0 = max(x0, 0), c1 = min(x0 + 32, tiles), r0 = max(y0, 0), r1 = min(y0 + 8, tiles);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (w == 0) {
        const uint32_t rb = (c1 - c0) * 128;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)),
                         "r"(rb * (r1 - r0)) : "memory");
        __syncwarp();
        const int yy = y0 + lane;
        if (lane < 8 && yy >= r0 && yy < r1)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    sa(&buf[lane][(c0 - x0) * 128])),
                "l"(p + ((size_t)yy * tiles + c0) * 128), "r"(rb), "r"(sa(&bar))
                : "memory");
    }
    asm volatile(
        "{\n .reg .pred q;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n @!q bra W_%=;\n}" ::"r"(
            sa(&bar))
        : "memory");
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint4 v = *reinterpret_cast<const uint4*>(&buf[w][lane * 128 + ((k + lane) & 7) * 16]);
        a |= v.x | v.y | v.z | v.w;
    }
    if (a == 0x12345678u) out[0] = a;
}

template <int ROWS>
__global__ void __launch_bounds__(32 * ROWS) rd_rows(const uint4* p, uint32_t* out) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint4* r = p + ((size_t)blockIdx.x * ROWS + w) * 256;
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint4 v = __ldcs(r + k * 32 + lane);
        a |= v.x | v.y | v.z | v.w;
    }
    if (a == 0x12345678u) out[0] = a;
}

int main() {
    const size_t bytes = (size_t)16384 * 16384 / 8;
    char* pl[4];
    uint32_t* out;
    for (auto& q : pl) { cudaMalloc(&q, bytes); cudaMemset(q, 0, bytes); }
    cudaMalloc(&out, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaStream_t st;
    cudaStreamCreate(&st);
    auto timeit = [&](const char* name, auto launch) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 20; ++i) launch(pl[i % 4]);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / 100;
        printf("%-28s %7.2f us  %6.0f GB/s  err=%s\n", name, us, bytes / us / 1e3,
               cudaGetErrorString(cudaGetLastError()));
    };
    const size_t n4 = bytes / 16;
    for (int k : {2, 4, 8, 16})
        timeit(k == 2 ? "stride 2/SM" : k == 4 ? "stride 4/SM" : k == 8 ? "stride 8/SM" : "stride 16/SM",
               [&](char* p) { rd_stride<<<sms * k, 256, 0, st>>>((const uint4*)p, n4, out); });
    timeit("bulk 8 rows/CTA", [&](char* p) { rd_bulk<8><<<bytes / 4096 / 8, 256, 0, st>>>(p, out); });
    timeit("bulk 4 rows/CTA", [&](char* p) { rd_bulk<4><<<bytes / 4096 / 4, 128, 0, st>>>(p, out); });
    timeit("bulk 2 rows/CTA", [&](char* p) { rd_bulk<2><<<bytes / 4096 / 2, 64, 0, st>>>(p, out); });
    timeit("ldg 8 rows/CTA", [&](char* p) { rd_rows<8><<<bytes / 4096 / 8, 256, 0, st>>>((const uint4*)p, out); });
    timeit("ldg 4 rows/CTA", [&](char* p) { rd_rows<4><<<bytes / 4096 / 4, 128, 0, st>>>((const uint4*)p, out); });
    const int T = 512;
    timeit("strip 30x6 (scan)", [&](char* p) { rd_strip<30, 6><<<dim3(18, 86), 256, 0, st>>>(p, out, T); });
    timeit("strip 32x6", [&](char* p) { rd_strip<32, 6><<<dim3(16, 86), 256, 0, st>>>(p, out, T); });
    timeit("strip 30x8", [&](char* p) { rd_strip<30, 8><<<dim3(18, 64), 256, 0, st>>>(p, out, T); });
    timeit("strip 32x8", [&](char* p) { rd_strip<32, 8><<<dim3(16, 64), 256, 0, st>>>(p, out, T); });
    return 0;
}
