// swap_micro.cu — host(mapped, pinned) -> HBM copy variants on B200: which one saturates PCIe?
//   V0 copy-engine DMA (cudaMemcpyAsync)
//   V1 warp LDG.128 (U loads in flight per lane, warp claims pieces), release per piece
//   V2 TMA bulk: one thread per CTA streams cp.async.bulk global(host)->smem->global(HBM)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/swap_micro tools/micro/swap_micro.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ unsigned int g_ticket;
__device__ unsigned int g_ready[64];

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int U>
__global__ void __launch_bounds__(512) k_ldg(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t bytes,
                                             uint32_t piece, int fence) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t np = (uint32_t)((bytes + piece - 1) / piece);
    for (;;) {
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(&g_ticket, 1u);
        p = __shfl_sync(0xffffffffu, p, 0);
        if (p >= np) break;
        const uint64_t off = (uint64_t)p * piece;
        const uint32_t n16 = (uint32_t)(umin64(piece, bytes - off) >> 4);
        const uint4* s = reinterpret_cast<const uint4*>(src + off);
        uint4* d = reinterpret_cast<uint4*>(dst + off);
        uint32_t i = lane;
        for (; i + (U - 1) * 32 < n16; i += U * 32) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = ldnc(s + i + u * 32);
#pragma unroll
            for (int u = 0; u < U; ++u) d[i + u * 32] = v[u];
        }
        for (; i < n16; i += 32) d[i] = ldnc(s + i);
        if (fence) {
            __threadfence();
            __syncwarp();
            if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&g_ready[p & 63]), "r"(1u) : "memory");
        }
    }
}

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// One thread per CTA: ring of S buffers of CH bytes; CTA claims pieces of `piece` bytes.
__global__ void __launch_bounds__(32) k_tma(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t bytes,
                                            uint32_t piece, uint32_t CH, int S, int fence) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)S * CH);
    if (threadIdx.x != 0) return;
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t np = (uint32_t)((bytes + piece - 1) / piece);
    uint32_t phase_bits = 0;  // bit s = parity to wait for on bar[s]
    for (;;) {
        const uint32_t p = atomicAdd(&g_ticket, 1u);
        if (p >= np) break;
        const uint64_t off = (uint64_t)p * piece;
        const uint64_t pb = umin64(piece, bytes - off);
        const uint32_t nch = (uint32_t)((pb + CH - 1) / CH);
        auto issue_load = [&](uint32_t j) {
            const int s = j % S;
            const uint32_t nb = (uint32_t)umin64(CH, pb - (uint64_t)j * CH);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[s])), "r"(nb) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             s32(sm + (size_t)s * CH)),
                         "l"(src + off + (uint64_t)j * CH), "r"(nb), "r"(s32(&bar[s]))
                         : "memory");
        };
        for (uint32_t j = 0; j < nch && j < (uint32_t)S; ++j) issue_load(j);
        for (uint32_t j = 0; j < nch; ++j) {
            const int s = j % S;
            const uint32_t par = (phase_bits >> s) & 1u;
            uint32_t ok = 0;
            do {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(ok) : "r"(s32(&bar[s])), "r"(par) : "memory");
            } while (!ok);
            phase_bits ^= 1u << s;
            const uint32_t nb = (uint32_t)umin64(CH, pb - (uint64_t)j * CH);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off + (uint64_t)j * CH),
                         "r"(s32(sm + (size_t)s * CH)), "r"(nb) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (j + S < nch) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                issue_load(j + S);
            }
        }
        if (fence) {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&g_ready[p & 63]), "r"(1u) : "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    const uint64_t MAXB = 256ull << 20;
    uint8_t* h = nullptr;
    CK(cudaHostAlloc(&h, MAXB, cudaHostAllocPortable | cudaHostAllocMapped));
    for (uint64_t i = 0; i < MAXB / 8; ++i) reinterpret_cast<uint64_t*>(h)[i] = i * 0x9E3779B97F4A7C15ull;
    uint8_t* hd = nullptr;
    CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
    uint8_t* d = nullptr;
    CK(cudaMalloc(&d, MAXB));
    std::vector<uint8_t> back(MAXB);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    const unsigned zero = 0;

    auto check = [&](uint64_t bytes, const char* what) {
        CK(cudaMemcpy(back.data(), d, bytes, cudaMemcpyDeviceToHost));
        if (memcmp(back.data(), h, bytes) != 0) printf("  MISMATCH in %s\n", what);
        CK(cudaMemset(d, 0, bytes));
    };
    auto timeit = [&](auto launch, uint64_t bytes, const char* what, int reps = 7) {
        std::vector<float> ms;
        for (int r = 0; r < reps + 2; ++r) {
            CK(cudaMemcpyToSymbolAsync(g_ticket, &zero, 4, 0, cudaMemcpyHostToDevice, st));
            CK(cudaEventRecord(e0, st));
            launch();
            CK(cudaEventRecord(e1, st));
            CK(cudaStreamSynchronize(st));
            CK(cudaGetLastError());
            float t;
            CK(cudaEventElapsedTime(&t, e0, e1));
            if (r >= 2) ms.push_back(t);
        }
        std::sort(ms.begin(), ms.end());
        printf("%-48s %8.1f MB  med %8.3f ms  %6.2f GB/s  (best %6.2f)\n", what, bytes / 1e6, ms[ms.size() / 2],
               bytes / (ms[ms.size() / 2] * 1e6), bytes / (ms[0] * 1e6));
        check(bytes, what);
    };
    char name[128];
    for (uint64_t bytes : {8ull << 20, 51ull << 20, 219ull << 20}) {
        snprintf(name, sizeof name, "DMA cudaMemcpyAsync");
        timeit([&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st); }, bytes, name);
        for (int ctas : {32, 64, 148})
            for (uint32_t piece : {32u << 10, 64u << 10, 256u << 10}) {
                snprintf(name, sizeof name, "LDG U=8  ctas=%d thr=256 piece=%uK", ctas, piece >> 10);
                timeit([&] { k_ldg<8><<<ctas, 256, 0, st>>>(hd, d, bytes, piece, 1); }, bytes, name);
                snprintf(name, sizeof name, "LDG U=16 ctas=%d thr=256 piece=%uK", ctas, piece >> 10);
                timeit([&] { k_ldg<16><<<ctas, 256, 0, st>>>(hd, d, bytes, piece, 1); }, bytes, name);
            }
        for (int ctas : {16, 32, 64, 148})
            for (uint32_t CH : {8u << 10, 16u << 10, 32u << 10})
                for (uint32_t piece : {64u << 10, 256u << 10}) {
                    const int S = std::min<int>(12, (200 * 1024) / CH);
                    snprintf(name, sizeof name, "TMA ctas=%d CH=%uK S=%d piece=%uK", ctas, CH >> 10, S, piece >> 10);
                    timeit([&] { k_tma<<<ctas, 32, S * CH + 8 * S, st>>>(hd, d, bytes, piece, CH, S, 1); }, bytes, name);
                }
    }
    printf("done\n");
    return 0;
}
