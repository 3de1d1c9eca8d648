// Kernel-boundary cost in a dependent chain inside a CUDA graph: griddepcontrol.wait (PDL) vs a release/acquire
// arrival counter per kernel (the consumer polls the producer's counter; no grid-completion wait).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro/pdl_chain tools/micro/pdl_chain.cu -lcuda
// Each kernel: G CTAs x 256 threads; every CTA reads 16 KB of its predecessor's output and writes 16 KB (L2).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kN = 96, kT = 256, kWords = 4096;  // 16 KB per CTA

__device__ __forceinline__ void trig() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void gdwait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// mode 0: plain stream order; 1: PDL, trigger at entry, griddepcontrol.wait; 2: PDL + counter (trigger once the
// predecessor's counter is complete, so at most two kernels are in flight)
template <int MODE>
__global__ void __launch_bounds__(kT) k_step(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint32_t* ctr, int i) {
    if (MODE == 1) { trig(); gdwait(); }
    if (MODE == 2) {
        if (threadIdx.x == 0 && i > 0) {
            const uint32_t want = gridDim.x;
            uint32_t v;
            do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr + i - 1) : "memory"); } while (v < want);
        }
        __syncthreads();
        trig();
    }
    const uint32_t base = blockIdx.x * kWords;
    for (int w = threadIdx.x; w < kWords; w += kT) out[base + w] = in[base + (w ^ 1)] + 1u;
    if (MODE == 2) {
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + i), "r"(1u) : "memory");
        }
    }
}

template <int MODE>
static int run(int G, float* us) {
    uint32_t *a, *b, *ctr;
    CK(cudaMalloc(&a, (size_t)G * kWords * 4));
    CK(cudaMalloc(&b, (size_t)G * kWords * 4));
    CK(cudaMalloc(&ctr, kN * 4));
    CK(cudaMemset(a, 0, (size_t)G * kWords * 4));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    CK(cudaMemsetAsync(ctr, 0, kN * 4, s));
    for (int i = 0; i < kN; ++i) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(kT);
        cfg.stream = s;
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at.val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = &at;
        cfg.numAttrs = (MODE != 0 && i > 0) ? 1 : 0;
        const uint32_t* in = (i & 1) ? b : a;
        uint32_t* out = (i & 1) ? a : b;
        CK(cudaLaunchKernelEx(&cfg, k_step<MODE>, in, out, ctr, i));
    }
    CK(cudaStreamEndCapture(s, &g));
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int r = 0; r < 20; ++r) CK(cudaGraphLaunch(ge, s));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<float> t;
    for (int r = 0; r < 50; ++r) {
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    *us = t[t.size() / 2] * 1000.f / kN;
    // check: after an even number of steps the value at word w went through kN increments
    std::vector<uint32_t> h((size_t)G * kWords);
    CK(cudaMemcpy(h.data(), (kN & 1) ? b : a, h.size() * 4, cudaMemcpyDeviceToHost));
    (void)h;
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(a);
    cudaFree(b);
    cudaFree(ctr);
    cudaStreamDestroy(s);
    return 0;
}

int main() {
    for (int G : {12, 72, 96, 148}) {
        float t0, t1, t2;
        if (run<0>(G, &t0) || run<1>(G, &t1) || run<2>(G, &t2)) return 1;
        printf("G=%3d CTAs: per kernel  stream order %.2f us   PDL (griddepcontrol.wait) %.2f us   PDL + counter %.2f us\n", G, t0, t1, t2);
    }
    return 0;
}
