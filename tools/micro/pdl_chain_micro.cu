// Per-kernel floor of a back-to-back PDL chain (the resident invoke's structure): N launches of a
// kernel that waits on its predecessor (griddepcontrol.wait), reads one float per CTA of the
// predecessor's output, writes its own, and triggers its successor at entry or at exit.  Varies CTA
// count, threads, dynamic shared memory (co-residence of consecutive kernels) and the trigger point.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pdl tools/micro/pdl_chain_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_link(const float* in, float* out, int trigger_early, int work_iters) {
    extern __shared__ float sm[];
    if (trigger_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float v = in[blockIdx.x];
    for (int i = 0; i < work_iters; ++i) v = v * 1.0000001f + 1e-7f;
    if (threadIdx.x == 0) sm[0] = v;
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = sm[0] + 1.0f;
    if (!trigger_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    float *a, *b;
    cudaMalloc(&a, 1 << 20);
    cudaMalloc(&b, 1 << 20);
    cudaMemset(a, 0, 1 << 20);
    cudaFuncSetAttribute(k_link, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int N = 200;
    for (int pdl : {0, 1})
        for (int early : {0, 1})
            for (int ctas : {32, 72, 144})
                for (int threads : {128, 512})
                    for (int smem_kb : {0, 100, 200}) {
                        if (!pdl && early) continue;
                        cudaLaunchConfig_t cfg{};
                        cfg.gridDim = dim3(ctas);
                        cfg.blockDim = dim3(threads);
                        cfg.dynamicSmemBytes = smem_kb ? smem_kb * 1024 : 16;
                        cfg.stream = s;
                        cudaLaunchAttribute at[1];
                        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                        at[0].val.programmaticStreamSerializationAllowed = 1;
                        cfg.attrs = at;
                        cfg.numAttrs = pdl ? 1 : 0;
                        auto run = [&]() {
                            for (int i = 0; i < N; ++i)
                                cudaLaunchKernelEx(&cfg, k_link, (const float*)(i & 1 ? b : a), (i & 1 ? a : b), early, 0);
                        };
                        run();
                        // graph-captured chain, like the invoke graph
                        cudaGraph_t g;
                        cudaGraphExec_t ge;
                        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
                        run();
                        cudaStreamEndCapture(s, &g);
                        if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
                            printf("instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError()));
                            return 1;
                        }
                        cudaGraphLaunch(ge, s);
                        cudaStreamSynchronize(s);
                        cudaEventRecord(e0, s);
                        cudaGraphLaunch(ge, s);
                        cudaEventRecord(e1, s);
                        cudaEventSynchronize(e1);
                        float ms;
                        cudaEventElapsedTime(&ms, e0, e1);
                        printf("pdl=%d trigger=%s ctas=%3d threads=%3d smem=%3d KB: %.2f us per kernel\n", pdl,
                               early ? "entry" : "exit ", ctas, threads, smem_kb, ms * 1000 / N);
                        cudaGraphExecDestroy(ge);
                        cudaGraphDestroy(g);
                    }
    printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
