// swap_micro2.cu — copy-engine variants for the swap engine (B200, PCIe Gen5 host link):
//   grouped DMA in one stream with cuStreamWriteValue32 progress words between groups (graph-captured
//   and plain), two DMA streams on halves, DMA + SM-TMA concurrently, write-combined host pages.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro/swap_micro2 tools/micro/swap_micro2.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <functional>
#include <vector>

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e = (x);                                                                  \
        if (e != cudaSuccess) {                                                               \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);          \
            exit(1);                                                                          \
        }                                                                                     \
    } while (0)

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ unsigned int g_ticket;
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32) k_tma(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t bytes,
                                            uint32_t piece, uint32_t CH, int S) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)S * CH);
    if (threadIdx.x != 0) return;
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t np = (uint32_t)((bytes + piece - 1) / piece);
    uint32_t phase_bits = 0;
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
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const uint64_t MAXB = 256ull << 20;
    uint8_t *h = nullptr, *hwc = nullptr, *d = nullptr;
    CK(cudaHostAlloc(&h, MAXB, cudaHostAllocPortable | cudaHostAllocMapped));
    CK(cudaHostAlloc(&hwc, MAXB, cudaHostAllocPortable | cudaHostAllocMapped | cudaHostAllocWriteCombined));
    for (uint64_t i = 0; i < MAXB / 8; ++i) reinterpret_cast<uint64_t*>(h)[i] = i * 0x9E3779B97F4A7C15ull;
    memcpy(hwc, h, MAXB);
    CK(cudaMalloc(&d, MAXB));
    uint32_t* prog = nullptr;
    CK(cudaMalloc(&prog, 4096));
    std::vector<uint8_t> back(MAXB);
    cudaStream_t st, st2;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, ef, ej;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreateWithFlags(&ef, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    const unsigned zero = 0;
    uint8_t* src = h;

    auto check = [&](uint64_t bytes, const char* what) {
        CK(cudaMemcpy(back.data(), d, bytes, cudaMemcpyDeviceToHost));
        if (memcmp(back.data(), h, bytes) != 0) printf("  MISMATCH in %s\n", what);
        CK(cudaMemset(d, 0, bytes));
    };
    auto timeit = [&](std::function<void()> launch, uint64_t bytes, const char* what, int reps = 7) {
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
        printf("%-56s %8.1f MB  med %8.3f ms  %6.2f GB/s  (best %6.2f)\n", what, bytes / 1e6, ms[ms.size() / 2],
               bytes / (ms[ms.size() / 2] * 1e6), bytes / (ms[0] * 1e6));
        check(bytes, what);
    };
    int wv_mode = 0;  // 0 default write-value (fenced), 1 no memory barrier, 2 no write-value
    auto grouped = [&](cudaStream_t s, uint64_t lo, uint64_t hi, uint64_t grp, uint32_t* word) {
        uint32_t k = 0;
        for (uint64_t o = lo; o < hi; o += grp) {
            const uint64_t nb = umin64(grp, hi - o);
            cudaMemcpyAsync(d + o, src + o, nb, cudaMemcpyHostToDevice, s);
            if (wv_mode == 0) cuStreamWriteValue32(s, (CUdeviceptr)word, (cuuint32_t)(++k), 0);
            if (wv_mode == 1) cuStreamWriteValue32(s, (CUdeviceptr)word, (cuuint32_t)(++k), CU_STREAM_WRITE_VALUE_NO_MEMORY_BARRIER);
        }
    };
    // copies serialised across two streams by events, each stream's fenced write-value overlapping
    // the other stream's next copy
    cudaEvent_t evc[64];
    for (int i = 0; i < 64; ++i) CK(cudaEventCreateWithFlags(&evc[i], cudaEventDisableTiming));
    auto chained = [&](uint64_t bytes, uint64_t grp) {
        cudaStream_t ss[2] = {st, st2};
        cudaEventRecord(ef, st);
        cudaStreamWaitEvent(st2, ef, 0);
        uint32_t k[2] = {0, 0};
        int i = 0;
        for (uint64_t o = 0; o < bytes; o += grp, ++i) {
            cudaStream_t s = ss[i & 1];
            if (i > 0) cudaStreamWaitEvent(s, evc[(i - 1) % 64], 0);
            cudaMemcpyAsync(d + o, src + o, umin64(grp, bytes - o), cudaMemcpyHostToDevice, s);
            cudaEventRecord(evc[i % 64], s);
            cuStreamWriteValue32(s, (CUdeviceptr)(prog + 32 * (i & 1)), (cuuint32_t)(++k[i & 1]), 0);
        }
        cudaEventRecord(ej, st2);
        cudaStreamWaitEvent(st, ej, 0);
    };
    // copies back to back on one stream; the fenced write-values on a second "flag" stream, each
    // after an event recorded behind its copy (the fence no longer stalls the copy stream)
    auto flagged = [&](uint64_t bytes, uint64_t grp) {
        cudaEventRecord(ef, st);
        cudaStreamWaitEvent(st2, ef, 0);
        uint32_t k = 0;
        int i = 0;
        for (uint64_t o = 0; o < bytes; o += grp, ++i) {
            cudaMemcpyAsync(d + o, src + o, umin64(grp, bytes - o), cudaMemcpyHostToDevice, st);
            cudaEventRecord(evc[i % 64], st);
            cudaStreamWaitEvent(st2, evc[i % 64], 0);
            cuStreamWriteValue32(st2, (CUdeviceptr)prog, (cuuint32_t)(++k), 0);
        }
        cudaEventRecord(ej, st2);
        cudaStreamWaitEvent(st, ej, 0);
    };
    char name[160];
    if (getenv("GAP_ONLY")) {
        for (uint64_t grp : {256ull << 10, 1ull << 20, 4ull << 20, 8ull << 20}) {
            snprintf(name, sizeof name, "DMA back-to-back + flags on a 2nd stream %lluK", (unsigned long long)(grp >> 10));
            timeit([&] { flagged(51ull << 20, grp); }, 51ull << 20, name);
        }
        for (uint64_t grp : {256ull << 10, 1ull << 20, 4ull << 20, 8ull << 20}) {
            snprintf(name, sizeof name, "DMA chained over 2 streams %lluK, fenced write-values", (unsigned long long)(grp >> 10));
            timeit([&] { chained(51ull << 20, grp); }, 51ull << 20, name);
        }
        for (uint64_t bytes : {51ull << 20}) {
            for (int mode = 0; mode < 3; ++mode) {
                wv_mode = mode;
                for (uint64_t grp : {256ull << 10, 1ull << 20, 4ull << 20}) {
                    snprintf(name, sizeof name, "DMA grouped %lluK, write-value mode %d (0 fenced, 1 no barrier, 2 none)",
                             (unsigned long long)(grp >> 10), mode);
                    timeit([&] { grouped(st, 0, bytes, grp, prog); }, bytes, name);
                }
            }
        }
        return 0;
    }
    for (uint64_t bytes : {51ull << 20, 219ull << 20}) {
        for (int wc = 0; wc < 2; ++wc) {
            src = wc ? hwc : h;
            snprintf(name, sizeof name, "DMA one copy%s", wc ? " [WC]" : "");
            timeit([&] { cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st); }, bytes, name);
            uint8_t* sd = nullptr;
            CK(cudaHostGetDevicePointer((void**)&sd, src, 0));
            snprintf(name, sizeof name, "TMA 32 ctas CH=16K S=12 piece=256K%s", wc ? " [WC]" : "");
            timeit([&] { k_tma<<<32, 32, 12 * (16 << 10) + 96, st>>>(sd, d, bytes, 256 << 10, 16 << 10, 12); }, bytes, name);
        }
        src = h;
        for (uint64_t grp : {256ull << 10, 1ull << 20, 2ull << 20, 4ull << 20, 8ull << 20}) {
            snprintf(name, sizeof name, "DMA grouped %lluK + writeValue (stream)", (unsigned long long)(grp >> 10));
            timeit([&] { grouped(st, 0, bytes, grp, prog); }, bytes, name);
            // graph-captured version
            cudaGraph_t g;
            cudaGraphExec_t ge;
            CK(cudaStreamBeginCapture(st2, cudaStreamCaptureModeThreadLocal));
            grouped(st2, 0, bytes, grp, prog);
            CK(cudaStreamEndCapture(st2, &g));
            CK(cudaGraphInstantiate(&ge, g, 0));
            snprintf(name, sizeof name, "DMA grouped %lluK + writeValue (graph)", (unsigned long long)(grp >> 10));
            timeit([&] { cudaGraphLaunch(ge, st); }, bytes, name);
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
            snprintf(name, sizeof name, "DMA grouped %lluK, 2 streams (halves)", (unsigned long long)(grp >> 10));
            timeit([&] {
                cudaEventRecord(ef, st);
                cudaStreamWaitEvent(st2, ef, 0);
                grouped(st, 0, bytes / 2, grp, prog);
                grouped(st2, bytes / 2, bytes, grp, prog + 32);
                cudaEventRecord(ej, st2);
                cudaStreamWaitEvent(st, ej, 0);
            }, bytes, name);
        }
        uint8_t* hd = nullptr;
        CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
        for (double f : {0.5, 0.8}) {
            const uint64_t cut = (uint64_t)(bytes * f) / 4096 * 4096;
            snprintf(name, sizeof name, "DMA %.0f%% (2M groups) || SM-TMA rest (16 ctas)", f * 100);
            timeit([&] {
                cudaEventRecord(ef, st);
                cudaStreamWaitEvent(st2, ef, 0);
                grouped(st, 0, cut, 2 << 20, prog);
                k_tma<<<16, 32, 12 * (16 << 10) + 96, st2>>>(hd + cut, d + cut, bytes - cut, 256 << 10, 16 << 10, 12);
                cudaEventRecord(ej, st2);
                cudaStreamWaitEvent(st, ej, 0);
            }, bytes, name);
        }
    }
    printf("done\n");
    return 0;
}
