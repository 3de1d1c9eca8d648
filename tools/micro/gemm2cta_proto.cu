// Prototype (tools only, not in libfsw): batch-1 GEMM on the 2-CTA UMMA (tcgen05.mma.cta_group::2),
// in the swap-AB form cuBLAS uses for these shapes: a CTA pair computes 128 weight rows x 32 tokens,
// each CTA holding 64 weight rows and 16 tokens of every K sub-tile in its shared memory, so an SM
// receives half the operand bytes of a 1-CTA tile (k_gemm vs cuBLAS).
//   Y[t][n] = sum_k X[t][k] * W[n][k] + b[n]      (bf16 in, fp32 accumulate, bf16 out)
// Weights use libfsw's pre-tiled K-major SWIZZLE_128B layout (one bulk copy per 64-row sub-tile).
// The peer CTA relays "my half of stage s landed" to the leader's barrier; the leader issues the
// MMAs and commits each stage to both CTAs' empty barriers (multicast).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/gemm2cta_proto tools/micro/gemm2cta_proto.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <vector>

#ifndef KSUB_
#define KSUB_ 4
#endif
#ifndef MAXST_
#define MAXST_ 5
#endif
#ifndef T_
#define T_ 32
#endif
constexpr int T = T_, TH = T / 2, WR = 64, KSUB = KSUB_;  // T tokens per pair tile (16 .. 128)
constexpr int TCOLS = TH < 32 ? 32 : TH;                   // TMEM columns (accumulator: T/2 per lane half)
__device__ unsigned long long g_stamp[512][6];  // per-CTA %globaltimer phase stamps (isolated launch)
__device__ __forceinline__ unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
#define STAMP(i) do { if (threadIdx.x == 0 && blockIdx.x + gridDim.x * blockIdx.y < 512) g_stamp[blockIdx.x + gridDim.x * blockIdx.y][i] = gtime(); } while (0)
constexpr uint32_t WSUB = WR * 128, XSUB = TH * 128, STAGE = KSUB * (WSUB + XSUB);

struct Args {
    const uint8_t* w;
    const uint16_t* bias;
    uint16_t* out;
    uint32_t M, N, K, n_pad;
    uint32_t wrow0;  // row of the weights in the weight map (0 unless POOL_GB places them in a big buffer)
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
    } while (!ok);
}
__device__ __forceinline__ uint64_t desc_sw128(const void* p) {
    return ((uint64_t)(su32(p) >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) k_g2(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, Args a, int stages, int teardown_sync) {
    extern __shared__ uint8_t raw[];
    STAMP(0);
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    uint64_t* lfull = (uint64_t*)(smem + stages * STAGE);
    uint64_t* pfull = lfull + stages;
    uint64_t* empty = pfull + stages;
    uint64_t* done = empty + stages;
    uint32_t* tslot = (uint32_t*)(done + 1);
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t w0 = (blockIdx.x >> 1) * 128 + rank * WR;  // this CTA's weight rows
    const uint32_t tb = blockIdx.y * T;                       // the pair's tokens
    const uint32_t nkt = a.K / 64, nst = (nkt + KSUB - 1) / KSUB;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&lfull[s], 1);
            mbar_init(&pfull[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t kstride = (uint64_t)(a.n_pad / 8) * 1024;
    // warp 0 issues the copies lane-parallel: lane 0 arms the stages' barriers, then lane l issues copy l
    // of the stages in [st0, st1) (one thread issuing every copy back to back was the critical path)
#ifdef DIRECT
    // DIRECT: both CTAs' copies complete on the LEADER's barrier (cta_group::2 TMA), which expects the
    // bytes of both halves; no relay
    constexpr uint32_t kArmMul = 2;
    const bool arms = rank == 0;
#else
    constexpr uint32_t kArmMul = 1;
    const bool arms = true;
#endif
    auto arm = [&](uint32_t st0, uint32_t st1) {
        if (lane == 0 && arms)
            for (uint32_t st = st0; st < st1; ++st) {
                const uint32_t nsub = min((uint32_t)KSUB, nkt - st * KSUB);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&lfull[st % stages])), "r"(kArmMul * nsub * (WSUB + XSUB)) : "memory");
            }
        __syncwarp();
    };
    auto bar_of = [&](uint32_t s) -> uint32_t {
#ifdef DIRECT
        uint32_t r;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(su32(&lfull[s])));
        return r;
#else
        return su32(&lfull[s]);
#endif
    };
    auto load_w = [&](uint32_t st0, uint32_t st1) {
        for (uint32_t i = lane; i < (st1 - st0) * KSUB; i += 32) {
            const uint32_t st = st0 + i / KSUB, j = i % KSUB, kt = st * KSUB + j, s = st % stages;
            if (kt >= nkt) continue;
// (measured: a plain cp.async.bulk whose mbarrier operand is the LEADER's barrier never completes it
//  (the kernel hangs), so the weights need a tensor map, or the relay, in the 2-CTA design)
#ifdef DIRECT
            asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                             su32(smem + s * STAGE + j * WSUB)), "l"(&tmW), "r"(0), "r"((int)(a.wrow0 + kt * a.n_pad + w0)), "r"(bar_of(s)) : "memory");
#else
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(smem + s * STAGE + j * WSUB)), "l"(a.w + kt * kstride + (uint64_t)(w0 / 8) * 1024), "r"(WSUB),
                         "r"(su32(&lfull[s])) : "memory");
#endif
        }
    };
    auto load_x = [&](uint32_t st0, uint32_t st1) {
        for (uint32_t i = lane; i < (st1 - st0) * KSUB; i += 32) {
            const uint32_t st = st0 + i / KSUB, j = i % KSUB, kt = st * KSUB + j, s = st % stages;
            if (kt >= nkt) continue;
#ifdef DIRECT
            asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                             su32(smem + s * STAGE + KSUB * WSUB + j * XSUB)), "l"(&tmX), "r"((int)(kt * 64)), "r"((int)(tb + rank * TH)),
                         "r"(bar_of(s)) : "memory");
#else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                             su32(smem + s * STAGE + KSUB * WSUB + j * XSUB)), "l"(&tmX), "r"((int)(kt * 64)), "r"((int)(tb + rank * TH)),
                         "r"(su32(&lfull[s])) : "memory");
#endif
        }
    };
    // the weights of the stages in flight are requested before anything else (they depend on nothing),
    // while warp 1 allocates the pair's TMEM
    const uint32_t pre = min((uint32_t)stages, nst);
    if (warp == 0) {
        if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
        arm(0, pre);
#ifndef DIRECT
        load_w(0, pre);  // DIRECT: the peer may only signal the leader's barrier after the cluster barrier
#endif
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "n"(TCOLS) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    STAMP(1);

    if (warp == 0) {  // producer (both CTAs): the tokens, then the rest of the ring
#ifdef DIRECT
        load_w(0, pre);
#endif
        asm volatile("griddepcontrol.wait;" ::: "memory");
        load_x(0, pre);
        for (uint32_t st = pre; st < nst; ++st) {
            if (lane == 0) mbar_wait(&empty[st % stages], ((st / stages) - 1) & 1);
            __syncwarp();
            arm(st, st + 1);
            load_w(st, st + 1);
            load_x(st, st + 1);
        }
        STAMP(2);
#ifndef DIRECT
    } else if (warp == 1 && lane == 0 && rank == 1) {  // relay: my half of stage s has landed
        for (uint32_t st = 0; st < nst; ++st) {
            const uint32_t s = st % stages;
            mbar_wait(&lfull[s], (st / stages) & 1);
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(su32(&pfull[s])));
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        }
#endif
    } else if (warp == 1 && lane == 0 && rank == 0) {  // MMA issuer: M = 128 (64 per CTA), N = 32 (16 per CTA)
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(T >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (uint32_t st = 0; st < nst; ++st) {
            const uint32_t s = st % stages, nsub = min((uint32_t)KSUB, nkt - st * KSUB);
            mbar_wait(&lfull[s], (st / stages) & 1);
#ifndef DIRECT
            mbar_wait(&pfull[s], (st / stages) & 1);
#endif
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t ad0 = desc_sw128(smem + s * STAGE), bd0 = desc_sw128(smem + s * STAGE + KSUB * WSUB);
            for (uint32_t j = 0; j < nsub; ++j)
                for (uint32_t kk = 0; kk < 4; ++kk) {
                    const uint64_t ad = ad0 + ((j * WSUB + kk * 32) >> 4), bd = bd0 + ((j * XSUB + kk * 32) >> 4);
                    const uint32_t acc = (st | j | kk) != 0;
                    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                }
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                             su32(&empty[s])), "h"((uint16_t)3) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(done)),
                     "h"((uint16_t)3) : "memory");
    }
    __syncwarp();
    // epilogue: this CTA's 64 weight rows x all 32 tokens; TMEM lane = m + 64·(token >= 16), column = token mod 16
    mbar_wait(done, 0);
    STAMP(3);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t m = (warp & 1) * 32 + lane, n = w0 + m, tok0 = tb + (warp >> 1) * TH;
    const float bias = n < a.N ? __uint_as_float((uint32_t)a.bias[n] << 16) : 0.0f;
#pragma unroll
    for (int c0 = 0; c0 < TH; c0 += 16) {
        uint32_t r[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                       "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(tmem + ((warp * 32u) << 16) + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (n < a.N)
            for (int c = 0; c < 16 && c0 + c < TH; ++c) {
                const uint32_t t = tok0 + c0 + c;
                if (t < a.M) {
                    const float v = __uint_as_float(r[c]) + bias;
                    const uint32_t u = __float_as_uint(v);
                    a.out[(uint64_t)t * a.N + n] = (uint16_t)((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
                }
            }
    }
    __syncthreads();
    STAMP(4);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (teardown_sync) cluster_sync();  // (both CTAs have seen `done`: no MMA can still target either TMEM)
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
    STAMP(5);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)((u + 0x7FFF + ((u >> 16) & 1)) >> 16); }
static float bf2f(uint16_t h) { uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4); return f; }

int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int tsync = getenv("NO_TEARDOWN_SYNC") ? 0 : 1;
    struct Shape { const char* name; uint32_t M, K, N; } shapes[] = {
        {"bert.qkv", 128, 768, 2304}, {"bert.o", 128, 768, 768}, {"bert.ffn1", 128, 768, 3072}, {"bert.ffn2", 128, 3072, 768},
        {"gpt.qkv", 128, 1600, 4800}, {"gpt.fc", 128, 1600, 6400}, {"gpt.proj2", 128, 6400, 1600}};
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncFn enc = (EncFn)fp;
    cudaFuncSetAttribute(k_g2, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (auto& sh : shapes) {
        if (argc > 1 && strcmp(argv[1], sh.name)) continue;
        const uint32_t n_pad = (sh.N + 127) / 128 * 128, nkt = sh.K / 64;
        std::vector<uint16_t> X((size_t)sh.M * sh.K), Wl((size_t)sh.N * sh.K), B(sh.N);
        uint32_t x = 7;
        auto rnd = [&]() { x = x * 1664525u + 1013904223u; return ((x >> 8) * (1.0f / 16777216.0f)) * 2.0f - 1.0f; };
        for (auto& v : X) v = f2bf(rnd());
        for (auto& v : Wl) v = f2bf(rnd() * 0.05f);
        for (auto& v : B) v = f2bf(rnd() * 0.1f);
        // pre-tiled weights: k tile kt, 8-row group g = n / 8: 1024 B at (kt·n_pad/8 + g)·1024, row n%8 at
        // +128·(n%8), its 16-B chunk c at chunk c ^ (n % 8)  (K-major SWIZZLE_128B)
        std::vector<uint16_t> Wt((size_t)nkt * n_pad * 64, 0);
        for (uint32_t n = 0; n < sh.N; ++n)
            for (uint32_t k = 0; k < sh.K; ++k) {
                const uint32_t kt = k / 64, kk = k % 64, c = kk / 8, e = kk % 8;
                const size_t byte = ((size_t)kt * (n_pad / 8) + n / 8) * 1024 + (n % 8) * 128 + ((c ^ (n % 8)) * 16) + e * 2;
                Wt[byte / 2] = Wl[(size_t)n * sh.K + k];
            }
        uint16_t *dX, *dB, *dO;
        uint8_t* dW;
        cudaMalloc(&dX, X.size() * 2);
        uint8_t* big = nullptr;
        const uint64_t big_bytes = getenv("POOL_GB") ? (uint64_t)atoi(getenv("POOL_GB")) << 30 : 0;
        if (big_bytes) {  // weights deep inside a pool-sized allocation, the map spanning all of it (libfsw's layout)
            cudaMalloc(&big, big_bytes);
            dW = big + big_bytes / 2 / 1024 * 1024;
        } else {
            cudaMalloc(&dW, Wt.size() * 2);
        }
        cudaMalloc(&dB, B.size() * 2);
        cudaMalloc(&dO, (size_t)sh.M * sh.N * 2);
        cudaMemcpy(dX, X.data(), X.size() * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(dW, Wt.data(), Wt.size() * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
        cudaMemset(dO, 0, (size_t)sh.M * sh.N * 2);
        CUtensorMap tm;
        const cuuint64_t dims[2] = {sh.K, sh.M}, strides[1] = {(cuuint64_t)sh.K * 2};
        const cuuint32_t box[2] = {64, TH}, es[2] = {1, 1};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dX, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("tensor map failed\n");
            return 1;
        }
        CUtensorMap tw;  // the pre-tiled weights as rows of 128 B (already swizzled: copied verbatim)
        const uint64_t wrow0 = big_bytes ? (uint64_t)(dW - big) / 128 : 0;
        const cuuint64_t wd[2] = {64, big_bytes ? big_bytes / 128 : (cuuint64_t)nkt * n_pad}, wsd[1] = {128};
        const cuuint32_t wbox[2] = {64, (cuuint32_t)WR};
        if (enc(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, big_bytes ? (void*)big : (void*)dW, wd, wsd, wbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("weight tensor map failed\n");
            return 1;
        }
        Args a{dW, dB, dO, sh.M, sh.N, sh.K, n_pad, (uint32_t)wrow0};
        const int nst = (int)((nkt + KSUB - 1) / KSUB), stages = nst < MAXST_ ? nst : MAXST_;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(n_pad / 128 * 2, (sh.M + T - 1) / T);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = stages * STAGE + 1024 + 256;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_g2, tm, tw, a, stages, tsync);
        cudaError_t e2 = cudaStreamSynchronize(s);
        if (e != cudaSuccess || e2 != cudaSuccess) {
            printf("%s: launch %s / %s\n", sh.name, cudaGetErrorString(e), cudaGetErrorString(e2));
            return 1;
        }
        {  // phases of one isolated launch
            cudaDeviceSynchronize();
            cudaLaunchKernelEx(&cfg, k_g2, tm, tw, a, stages, tsync);
            cudaDeviceSynchronize();
            static unsigned long long st[512][6];
            cudaMemcpyFromSymbol(st, g_stamp, sizeof st);
            const uint32_t nct = std::min(512u, cfg.gridDim.x * cfg.gridDim.y);
            double ph[5] = {0};
            unsigned long long t0 = ~0ull, t1 = 0;
            for (uint32_t c = 0; c < nct; ++c) {
                t0 = std::min(t0, st[c][0]); t1 = std::max(t1, st[c][5]);
                for (int p = 0; p < 5; ++p) ph[p] += (double)(st[c][p + 1] - st[c][p]);
            }
            printf("%-10s phases (us, mean over %u CTAs): setup %.2f  loads-issued %.2f  mma-done %.2f  epilogue %.2f  teardown %.2f | span %.2f\n",
                   sh.name, nct, ph[0] / nct / 1e3, ph[1] / nct / 1e3, ph[2] / nct / 1e3, ph[3] / nct / 1e3, ph[4] / nct / 1e3, (t1 - t0) / 1e3);
        }
        std::vector<uint16_t> O((size_t)sh.M * sh.N);
        cudaMemcpy(O.data(), dO, O.size() * 2, cudaMemcpyDeviceToHost);
        double err = 0, mx = 0;
        for (uint32_t t = 0; t < sh.M; t += 7)
            for (uint32_t n = 0; n < sh.N; ++n) {
                double ref = bf2f(B[n]);
                for (uint32_t k = 0; k < sh.K; ++k) ref += (double)bf2f(X[(size_t)t * sh.K + k]) * bf2f(Wl[(size_t)n * sh.K + k]);
                err = std::max(err, std::fabs(ref - bf2f(O[(size_t)t * sh.N + n])));
                mx = std::max(mx, std::fabs(ref));
            }
        // timing: back-to-back launches captured in a graph, with and without PDL
        for (int pdl = 1; pdl >= 0; --pdl) {
        cfg.numAttrs = pdl;
        const int reps = 50;
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, k_g2, tm, tw, a, stages, tsync);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-10s M=%4u K=%5u N=%5u ctas=%4u stages=%d: %6.2f us per GEMM (graph, %s)  max err %.2e of max |ref| %.2f  %s\n",
               sh.name, sh.M, sh.K, sh.N, cfg.gridDim.x * cfg.gridDim.y, stages, ms * 1000 / reps, pdl ? "PDL chain" : "no PDL   ",
               err, mx, err <= 1e-2 * mx ? "OK" : "MISMATCH");
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        }
        cudaFree(dX); cudaFree(big ? (void*)big : (void*)dW); cudaFree(dB); cudaFree(dO);
    }
    printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
