// Microbenchmarks (tools only): cost of mbarrier try_wait / arrive and of tcgen05.mma chains.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ uint32_t mbar_try(uint64_t* b, uint32_t par) {
    uint32_t ok; asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory"); return ok; }
__device__ __forceinline__ uint32_t mbar_test(uint64_t* b, uint32_t par) {
    uint32_t ok; asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory"); return ok; }
__device__ __forceinline__ uint64_t desc(const void* p) { uint64_t a = smem_u32(p); return ((a >> 4) & 0x3FFF) | ((uint64_t)64 << 32) | (1ull << 46) | (2ull << 61); }
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)); }
__device__ __forceinline__ void commit(uint64_t* b) { asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)) : "memory"); }

__global__ void k_micro(long long* out, int N, int bn, int naccum) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bar = (uint64_t*)(sm + 65536);
    uint32_t* slot = (uint32_t*)(bar + 8);
    if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (threadIdx.x < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        // 1) try_wait on an already completed phase
        mbar_arrive(&bar[0]);
        while (!mbar_try(&bar[0], 0)) {}
        long long t0 = clock64();
        for (int i = 0; i < N; ++i) while (!mbar_try(&bar[0], 0)) {}
        long long t1 = clock64();
        out[0] = (t1 - t0) / N;
        // 2) test_wait on completed phase
        t0 = clock64();
        for (int i = 0; i < N; ++i) while (!mbar_test(&bar[0], 0)) {}
        t1 = clock64();
        out[1] = (t1 - t0) / N;
        // 3) arrive + wait round trip (same thread)
        uint32_t ph = 0;
        t0 = clock64();
        for (int i = 0; i < N; ++i) { mbar_arrive(&bar[1]); while (!mbar_try(&bar[1], ph)) {} ph ^= 1; }
        t1 = clock64();
        out[2] = (t1 - t0) / N;
        // 4) dependent MMA chain (same accumulator), N issues then commit+wait
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bn >> 3) << 17) | (8u << 24);
        uint64_t ad = desc(sm), bd = desc(sm + 16384);
        t0 = clock64();
        for (int i = 0; i < N; ++i) mma(tmem, ad, bd, idesc, 1);
        long long t_issue = clock64();
        commit(&bar[1]);
        while (!mbar_try(&bar[1], ph)) {} ph ^= 1;
        t1 = clock64();
        out[3] = (t_issue - t0) / N; out[4] = (t1 - t0) / N;
        // 5) independent accumulators (naccum round robin)
        t0 = clock64();
        for (int i = 0; i < N; ++i) mma(tmem + (uint32_t)((i % naccum) * bn), ad, bd, idesc, 1);
        t_issue = clock64();
        commit(&bar[1]);
        while (!mbar_try(&bar[1], ph)) {} ph ^= 1;
        t1 = clock64();
        out[5] = (t_issue - t0) / N; out[6] = (t1 - t0) / N;
        // 6) one MMA + commit + wait (latency of a single MMA)
        t0 = clock64();
        for (int i = 0; i < 16; ++i) { mma(tmem, ad, bd, idesc, 1); commit(&bar[1]); while (!mbar_try(&bar[1], ph)) {} ph ^= 1; }
        t1 = clock64();
        out[7] = (t1 - t0) / 16;
        // 7) globaltimer read cost
        t0 = clock64();
        unsigned long long g = 0;
        for (int i = 0; i < N; ++i) { unsigned long long x; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(x)); g += x; }
        t1 = clock64();
        out[8] = (t1 - t0) / N + (g == 1);
    }
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long* d; cudaMalloc(&d, 64 * 8);
    cudaFuncSetAttribute(k_micro, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    for (int bn : {16, 64, 128, 256}) for (int na : {1, 2, 4}) {
        if (na * bn > 512) continue;
        k_micro<<<1, 128, 80 * 1024>>>(d, 256, bn, na);
        long long h[16]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        printf("bn=%3d naccum=%d | try_wait(done) %lld cyc | test_wait %lld | arrive+wait %lld | dep MMA issue %lld, issue+complete %lld /mma | indep MMA issue %lld, +complete %lld /mma | single MMA+commit+wait %lld | globaltimer %lld  (%s)\n",
               bn, na, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
