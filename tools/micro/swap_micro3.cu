// swap_micro3.cu — do L2 sector-promotion hints change the request size of SM-issued zero-copy reads?
// SM reads of mapped host memory go out as one PCIe read request per 128 B (swap_micro.cu: 51.3 GB/s, against
// 55.4 for the copy engine's larger requests).  Variants of the same warp-per-piece LDG.128 copy:
//   plain       ld.global.nc.L1::no_allocate.v4
//   L2::256B    ld.global.nc.L1::no_allocate.L2::256B.v4 (prefetch-size qualifier: 256-B L2 fills)
//   pf256       prefetch.global.L2 of the piece's lines, then plain loads
//   bulkpf      cp.async.bulk.prefetch.L2 of the whole piece (one request per piece), then plain loads
//   dma         cudaMemcpyAsync of the whole buffer (reference)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/swap_micro3 tools/micro/swap_micro3.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e = (x);                                                                  \
        if (e != cudaSuccess) {                                                               \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);          \
            exit(1);                                                                          \
        }                                                                                     \
    } while (0)

__device__ unsigned int g_ticket;

template <int MODE>
__device__ __forceinline__ uint4 ld(const uint4* p) {
    uint4 r;
    if (MODE == 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// MODE 0 plain, 1 L2::256B, 2 per-line prefetch first, 3 bulk L2 prefetch of the piece first
template <int MODE>
__global__ void __launch_bounds__(256) k_copy(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t bytes,
                                              uint32_t piece) {
    constexpr int U = 8;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t np = (uint32_t)((bytes + piece - 1) / piece);
    for (;;) {
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(&g_ticket, 1u);
        p = __shfl_sync(0xffffffffu, p, 0);
        if (p >= np) break;
        const uint64_t off = (uint64_t)p * piece;
        const uint32_t n16 = piece >> 4;
        const uint4* s = reinterpret_cast<const uint4*>(src + off);
        uint4* d = reinterpret_cast<uint4*>(dst + off);
        if (MODE == 2)
            for (uint32_t l = lane; l < piece / 256; l += 32)
                asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(src + off + 256ull * l));
        if (MODE == 3 && lane == 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + off), "r"(piece) : "memory");
        for (uint32_t i = lane; i < n16; i += U * 32) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = ld<MODE == 1 ? 1 : 0>(s + i + u * 32);
#pragma unroll
            for (int u = 0; u < U; ++u) d[i + u * 32] = v[u];
        }
    }
}

template <int MODE>
static float run(const uint8_t* src, uint8_t* dst, uint64_t bytes, uint32_t piece, int ctas, cudaStream_t s) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
        unsigned int z = 0;
        CK(cudaMemcpyToSymbolAsync(g_ticket, &z, 4, 0, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(a, s));
        k_copy<MODE><<<ctas, 256, 0, s>>>(src, dst, bytes, piece);
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (rep) best = ms < best ? ms : best;
    }
    return (float)(bytes / (best * 1e6));
}

int main() {
    const uint64_t bytes = 256ull << 20;
    uint8_t *h, *d;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    for (uint64_t i = 0; i < bytes; i += 4096) h[i] = (uint8_t)i;
    CK(cudaMalloc(&d, bytes));
    uint8_t* hd;
    CK(cudaHostGetDevicePointer(&hd, h, 0));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaEventRecord(a, s));
            CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
            CK(cudaEventRecord(b, s));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (rep) best = ms < best ? ms : best;
        }
        printf("dma (cudaMemcpyAsync 256 MiB)             %.1f GB/s\n", bytes / (best * 1e6));
    }
    for (int ctas : {32, 64, 148})
        for (uint32_t piece : {16384u, 65536u}) {
            printf("ctas %3d piece %5u KiB: plain %.1f  L2::256B %.1f  prefetch %.1f  bulk-prefetch %.1f GB/s\n", ctas, piece >> 10,
                   run<0>(hd, d, bytes, piece, ctas, s), run<1>(hd, d, bytes, piece, ctas, s), run<2>(hd, d, bytes, piece, ctas, s),
                   run<3>(hd, d, bytes, piece, ctas, s));
        }
    return 0;
}
