// device.cuh — sm_100a device helpers shared by the libfsw kernels (inline PTX).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#include "kernels.h"

namespace fsw {

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Streaming 128-bit load that does not allocate in L1 (host-mapped source, read once).
__device__ __forceinline__ uint4 ld_stream_v4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_v4(uint4* p, const uint4& v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// Device timeline (kernels.h kTraceStride), compiled in only for the tracing build of the library
// (FSW_TRACE_KERNELS: libfsw_trace.so, loaded by FSW_LIB for tools/timeline.py) — in the default build the
// stamps cost nothing (measured: the per-kernel stamps and their %globaltimer reads on the producer thread
// added ~27 us to resident BERT-base even with tracing off).  The layer kernels get the per-GPU buffer as a
// kernel parameter (Wait::trace, Args::trace); the swap kernels read g_trace, this translation unit's copy,
// once at kernel start.  One thread per CTA records, with atomicMax (min fields complemented).
static __device__ unsigned long long* g_trace = nullptr;
#ifdef FSW_TRACE_KERNELS
#define FSW_TRACE_MAX(t, layer, field, value)                                                          \
    do {                                                                                              \
        unsigned long long* t_ = (t);                                                                 \
        if (t_ && (layer) >= 0) atomicMax(t_ + (uint64_t)(layer) * kTraceStride + (field), (value));   \
    } while (0)
// Records the CTA's entry now and its exit when it goes out of scope (every return path); thread 0.
struct TraceExit {
    unsigned long long* t;
    int32_t layer;
    __device__ __forceinline__ TraceExit(unsigned long long* tr, int32_t l) : t(tr), layer(l) {
        if (threadIdx.x == 0) FSW_TRACE_MAX(t, layer, 0, ~globaltimer());
    }
    __device__ __forceinline__ ~TraceExit() {
        if (threadIdx.x == 0) FSW_TRACE_MAX(t, layer, 2, globaltimer());
    }
};
#else
#define FSW_TRACE_MAX(t, layer, field, value) do { } while (0)
struct TraceExit {
    __device__ __forceinline__ TraceExit(unsigned long long*, int32_t) {}
};
#endif

// Layer-kernel side of the ready-flag protocol: one thread spins with
// back-off until the layer's byte counter reaches its region size, then the caller does a
// CTA barrier.  The acquire pairs with the swap kernel's red.release; the barrier extends
// the ordering to the rest of the CTA.  A watchdog turns a lost release into an error word.
__device__ __forceinline__ void wait_ready_thread(const Wait& w) {
    auto load = [&](const uint32_t* p) { return w.sys ? ld_acquire_sys(p) : ld_acquire_gpu(p); };
    for (uint32_t j = 0; j < w.n; ++j) {
        if (load(w.ready[j]) >= w.target[j]) continue;
        const uint64_t t0 = globaltimer();
        uint32_t ns = 64;
        while (load(w.ready[j]) < w.target[j]) {
            __nanosleep(ns);
            if (ns < 1024) ns <<= 1;
            if (globaltimer() - t0 > kWatchdogNs) {
                atomicExch(&w.ctl->err, 1);
                atomicExch(&w.ctl->err_layer, w.layer);
                return;
            }
        }
    }
}

__device__ __forceinline__ void wait_ready_cta(const Wait& w) {
    if (w.n == 0) return;
    if (threadIdx.x == 0) {
        wait_ready_thread(w);
        FSW_TRACE_MAX(w.trace, w.layer, 1, globaltimer());
    }
    __syncthreads();
}

// Programmatic dependent launch (every layer kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): the GEMM lets its successor start once
// its MMAs are done (trigger before the epilogue; the other kernels trigger implicitly at exit),
// and every kernel waits for its predecessor's completion and memory before it touches any
// activation (wait).  Weight reads are ordered by the ready counters instead, so a GEMM streams
// its first weight stages while its predecessor is still in its epilogue.  (Triggering at kernel
// entry was measured: +19 % on BERT-base resident latency from early CTAs holding SMs.)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ float bf16_to_f32(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
__device__ __forceinline__ uint16_t f32_to_bf16(float f) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

__device__ __forceinline__ float gelu_erf(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_tanh(float x) {
    const float k0 = 0.7978845608028654f;  // sqrt(2/pi)
    return 0.5f * x * (1.0f + tanhf(k0 * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float apply_act(int act, float x) {
    switch (act) {
        case FSW_ACT_RELU: return fmaxf(x, 0.0f);
        case FSW_ACT_GELU_ERF: return gelu_erf(x);
        case FSW_ACT_GELU_TANH: return gelu_tanh(x);
        case FSW_ACT_TANH: return tanhf(x);
        default: return x;
    }
}

// Epilogue activation with the transcendental cases out of line: a GEMM epilogue applies it to every output
// element, and inlined erf / tanh expansions in an unrolled store loop made the epilogue code tens of KB —
// instruction-cache misses on every launch (measured in k_mega and k_gemm_ws: 4-7 us store phases).
static __device__ __noinline__ float4 act4_slow(int act, float4 v) {
    return make_float4(apply_act(act, v.x), apply_act(act, v.y), apply_act(act, v.z), apply_act(act, v.w));
}
__device__ __forceinline__ float4 act4(int act, float4 v) {
    if (act == FSW_ACT_NONE) return v;
    if (act == FSW_ACT_RELU) return make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
    return act4_slow(act, v);
}

// L2 prefetch of [p, p + bytes) (bulk, no completion; bytes multiple of 16)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Host side: launch with programmatic stream serialisation (PDL) so the kernel's prologue (and
// its weight prefetch) overlaps the previous layer kernel; captured into the invoke graph as a
// programmatic edge.
enum PdlKind { PDL_GEMM = 1, PDL_LN = 2, PDL_ATTN = 4, PDL_EMBED = 8, PDL_GEMV = 16, PDL_IM2COL = 32, PDL_POOL = 64 };
template <typename... KArgs, typename... Args>
static void launch_pdl_cluster(int kind, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                               dim3 cluster, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster.x;
    attr[1].val.clusterDim.y = cluster.y;
    attr[1].val.clusterDim.z = cluster.z;
    cfg.attrs = attr;
    // FSW_PDL_MASK = kinds launched with PDL (A/B switch of tools/pdl_ab.sh).  Default: all but
    // attention — launched early behind the QKV GEMM it cost ~19 us per layer on BERT-base
    // (profiles/r01/pdl_ab.txt); every other kind gains or is neutral.
    static const int mask = getenv("FSW_PDL_MASK") ? atoi(getenv("FSW_PDL_MASK")) : (0x7f & ~PDL_ATTN);
    const bool pdl = (mask & kind) != 0, clustered = cluster.x * cluster.y * cluster.z > 1;
    if (!pdl) cfg.attrs = attr + 1;
    cfg.numAttrs = (pdl ? 1 : 0) + (clustered ? 1 : 0);
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
static void launch_pdl(int kind, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    launch_pdl_cluster(kind, kernel, grid, block, smem, s, dim3(1, 1, 1), std::forward<Args>(args)...);
}

}  // namespace fsw
