// gemm_tc.cu — K3: flag-gated bf16 GEMM on the 5th-generation tensor cores (tcgen05).
//
//   out[m][n] = act( Σ_k A[m][k]·W[n][k] + b[n] + res[m][n] )       fp32 accumulate in TMEM
//
// A (activations, row-major bf16 in the per-GPU workspace) arrives by TMA (SWIZZLE_128B).
// W (weights, in the model's pool extent) is stored in the host store — and therefore in
// HBM after the swap — already in the UMMA K-major SWIZZLE_128B tile order,
// so each [BN x 64] weight tile is ONE contiguous cp.async.bulk of BN·128 bytes: no tensor
// map is needed for weights and the graph stays valid whichever extent the model lands in.
//
// One CTA = one 128 x BN output tile; 4 warps.  Lane 0 of warp 0 is the producer: it first
// spins on the layer's ready counter (the swap kernel's release, PAPER.md:588-590
// pipelining), fences generic->async proxy, then streams the K loop through an mbarrier ring
// whose stages are KSUB x 64 wide (4 x 64 for BN <= 64): at batch-1 M the MMA chain is
// issue-bound (~47 cycles per tcgen05.mma for N <= 64, ~170 cycles per mbarrier wait, both
// measured: tools/micro/umma_micro.cu), so wide stages amortise the waits.  Lane 0 of warp 1
// issues tcgen05.mma (M=128, N=BN, K=16) into TMEM and commits each stage back to its empty
// barrier.  All 4 warps then drain TMEM (tcgen05.ld 32x32b) into a shared tile and apply the
// fused bias / residual / activation epilogue with 16-B coalesced global accesses.
//
// Two generalisations for the batch-1 shapes of the paper's models:
//   * split-K (gridDim.z > 1): small-M GEMMs (ResNet stages 3-4: M = 196 / 49, K up to 4608)
//     would otherwise run a long serial K loop on a handful of CTAs.  Each split writes an fp32
//     partial tile; the last CTA to arrive on the tile's counter sums the partials in split order
//     (deterministic, bit-identical run to run) and runs the epilogue.
//   * implicit-GEMM convolution (a.conv): the A tile of k-tile (r, s, c0) is Hb output rows x Q
//     output columns x 64 input channels, gathered straight from the NHWC activation by ONE 4-D
//     TMA load: start (c0, s − pad, p0·stride + r − pad), element strides = conv stride, and the
//     out-of-bounds zero fill is the conv padding.  No im2col buffer, no extra kernel.
// Every launch uses programmatic dependent launch (device.cuh): the prologue and the first
// stages' WEIGHT loads overlap the previous kernel; activations are touched only after
// griddepcontrol.wait.
#include "device.cuh"
#include "umma.cuh"

namespace fsw {

#ifdef FSW_GEMM_TIMING  // tools/gemm_bench.cu only: per-CTA phase stamps
__device__ unsigned long long g_gemm_stamp[1024][6];
#define STAMP(i) do { if (threadIdx.x == 0) g_gemm_stamp[((blockIdx.z * gridDim.x + blockIdx.x) * gridDim.y + blockIdx.y) & 1023][i] = globaltimer(); } while (0)
#else
#define STAMP(i) do { } while (0)
#endif

namespace {

template <int BN>
struct Cfg {
    static constexpr int kSub = BN <= 64 ? 4 : 2;            // 64-wide k sub-tiles per stage
    static constexpr uint32_t kA = kBM * kBK * 2;            // one A sub-tile: 16 KiB
    static constexpr uint32_t kB = BN * kBK * 2;             // one W sub-tile: BN x 128 B
    static constexpr int kLdc = BN + 4;                       // epilogue tile row stride (floats)
    static constexpr uint32_t kCtile = kBM * kLdc * 4;
    // runtime stage geometry: the A sub-tile occupies a_sub bytes of shared memory (16 KiB, or 8 KiB for
    // 64-row activation tiles, whose 16-KiB UMMA read then runs into the following sub-tile: rows whose
    // accumulators are never read), so 64-row tiles fit twice the k-tiles in flight
    __host__ __device__ static uint32_t a_sub(uint32_t m_rows, int conv) { return !conv && m_rows <= 64 ? kA / 2 : kA; }
    __host__ __device__ static uint32_t stage_bytes(uint32_t asub) { return kSub * (asub + kB); }
    __host__ __device__ static uint32_t ring_bytes(int stages, uint32_t asub = kA) {
        uint32_t r = stages * stage_bytes(asub);
        return r < kCtile ? (kCtile + 1023) / 1024 * 1024 : r;
    }
    __host__ __device__ static uint32_t smem_bytes(int stages, uint32_t asub = kA) {
        return ring_bytes(stages, asub) + 1024 /*barriers*/ + 1024 /*align*/;
    }
    __host__ static int max_stages(uint32_t asub) {
        const int fit = (int)((200 * 1024) / stage_bytes(asub));
        return fit > 8 ? 8 : fit;
    }
};

}  // namespace

constexpr int kGemmThreads = 512;  // warp 0 TMA producer, warp 1 MMA issuer, all 16 in the epilogue

template <int BN>
__global__ void __maxnreg__(96)  // 512 threads x 96 regs: a 256-thread swap CTA (<= 64 regs) still fits beside it
    k_gemm(const __grid_constant__ CUtensorMap tmA, const DevDesc* __restrict__ d, Wait w, GemmArgs a, int stages) {
    TraceExit tx(w.trace, w.layer);
    using C = Cfg<BN>;
    constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // stage s: A sub-tiles at smem + s*sstride + j*asub, W sub-tiles after the A sub-tiles
    const uint32_t asub = C::a_sub(a.m_rows, a.conv), sstride = C::stage_bytes(asub);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::ring_bytes(stages, asub));
    uint64_t* empty = full + stages;
    uint64_t* done = empty + stages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    uint32_t* last_flag = tmem_slot + 1;

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x * gridDim.y + blockIdx.y;
    const DevDesc dd = *d;  // the invoke descriptor: written by the graph's first node, before any kernel
    const uint32_t m0 = blockIdx.x * a.m_rows, n0 = blockIdx.y * BN;
    const uint32_t kt_begin = blockIdx.z * a.kt_per;
    const uint32_t nkt = min(a.K / kBK, kt_begin + a.kt_per) - kt_begin;  // >= 1 (host plan)
    const uint32_t nst = (nkt + C::kSub - 1) / C::kSub;                   // pipeline steps
    // TMA box bytes of one A sub-tile: Hb x Q conv rows, or m_rows activation rows (m_rows = 64 halves the
    // A bytes a CTA streams: the upper 64 rows of the 128-row UMMA tile then hold stale data whose
    // accumulator rows the epilogue never reads)
    const uint32_t a_bytes = a.conv ? a.Hb * a.Q * (kBK * 2) : a.m_rows * (kBK * 2);
    // A multicast over a cluster of mc CTAs along N: CTA r loads rows [r·128/mc, (r+1)·128/mc) of
    // every A sub-tile and broadcasts them to the whole cluster; a stage is free again only when
    // all mc CTAs' MMAs have read it (empty barriers count mc multicast commits).
    const uint32_t mc = a.mc > 1 ? a.mc : 1;
    const uint32_t crank = mc > 1 ? cluster_ctarank() : 0;
    const uint16_t cmask = (uint16_t)((1u << mc) - 1u);
    STAMP(0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], mc);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (mc > 1) cluster_sync();  // every CTA's barriers exist before any multicast lands
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    STAMP(1);

    // Role dispatch is warp-uniform: warp 0 produces (lane 0 arms each stage's barrier, then lane j issues
    // the copies of the stage's sub-tile j: one thread issuing every TMA / bulk copy back to back was the
    // producer's critical path), lane 0 of warp 1 issues the MMAs; the other lanes of warp 1 park.
    if (warp == 0) {
        if (lane == 0) {
            wait_ready_thread(w);
            FSW_TRACE_MAX(w.trace, w.layer, 1, globaltimer());
        }
        __syncwarp();  // the weights lane 0 acquired are visible to the warp
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const uint8_t* wt = weight_ptr(dd, a.w_off);
        const uint64_t ktile_stride = (uint64_t)(a.n_pad / 8) * 1024;
        auto load_w = [&](uint32_t st) {
            const int s = st % stages;
            const uint32_t kt0 = st * C::kSub, nsub = min((uint32_t)C::kSub, nkt - kt0);
            uint8_t* sb = smem + s * sstride + C::kSub * asub;
            if (lane == 0) mbar_expect_tx(&full[s], nsub * (a_bytes + C::kB));
            __syncwarp();
            if (lane < nsub)
                bulk_load(sb + lane * C::kB, wt + (kt_begin + kt0 + lane) * ktile_stride + (uint64_t)(n0 / 8) * 1024, C::kB,
                          &full[s]);
        };
        auto load_a = [&](uint32_t st) {
            const int s = st % stages;
            const uint32_t kt0 = st * C::kSub, nsub = min((uint32_t)C::kSub, nkt - kt0);
            uint8_t* sa = smem + s * sstride;
            if (lane < nsub) {
                const uint32_t j = lane, kk = (kt_begin + kt0 + j) * kBK;
                if (a.conv) {
                    const uint32_t tap = kk / a.Cin, c0 = kk - tap * a.Cin, r = tap / a.S, sx = tap - r * a.S;
                    tma_load_4d(sa + j * asub, &tmA, (int)c0, (int)sx - (int)a.pad,
                                (int)(blockIdx.x * a.Hb * a.stride + r) - (int)a.pad, 0, &full[s]);
                } else if (mc > 1) {
                    const uint32_t rows = kBM / mc;
                    tma_load_2d_mc(sa + j * asub + crank * rows * (kBK * 2), &tmA, (int)kk, (int)(m0 + crank * rows),
                                   &full[s], cmask);
                } else {
                    tma_load_2d(sa + j * asub, &tmA, (int)kk, (int)m0, &full[s]);
                }
            }
        };
        // weights of the first stages stream while the previous kernel is still running
        const uint32_t pre = min((uint32_t)stages, nst);
        for (uint32_t st = 0; st < pre; ++st) load_w(st);
        if (lane == 0 && a.pf_bytes && w.n == 0) {  // resident (FSW_GEMM_PF): this CTA's share of the next GEMM's weights into L2
            const uint32_t ncta = gridDim.x * gridDim.y * gridDim.z;
            const uint32_t cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
            const uint64_t share = ((a.pf_bytes + ncta - 1) / ncta + 255) & ~255ull;
            const uint64_t b0 = cta * share, b1 = a.pf_bytes < b0 + share ? a.pf_bytes : b0 + share;
            const uint8_t* pf = weight_ptr(dd, a.pf_off);
            for (uint64_t o = b0; o < b1; o += 65536) prefetch_l2(pf + o, (uint32_t)(b1 - o < 65536 ? b1 - o : 65536));
        }
        pdl_wait();
        if (lane == 0) FSW_TRACE_MAX(w.trace, w.layer, 5, globaltimer());
        asm volatile("fence.proxy.async.global;" ::: "memory");
        for (uint32_t st = 0; st < pre; ++st) load_a(st);
        for (uint32_t st = pre; st < nst; ++st) {
            const int s = st % stages;
            if (lane == 0) mbar_wait(&empty[s], ((st / stages) - 1) & 1);
            __syncwarp();
            load_w(st);
            load_a(st);
        }
        STAMP(2);
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(kBM, BN);
            for (uint32_t st = 0; st < nst; ++st) {
                const int s = st % stages;
                mbar_wait(&full[s], (st / stages) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t kt0 = st * C::kSub, nsub = min((uint32_t)C::kSub, nkt - kt0);
                const uint8_t* sa = smem + s * sstride;
                const uint8_t* sb = sa + C::kSub * asub;
                const uint64_t ad0 = umma_desc_sw128(sa), bd0 = umma_desc_sw128(sb);
                for (uint32_t j = 0; j < nsub; ++j) {
#pragma unroll
                    for (uint32_t kk = 0; kk < kBK / 16; ++kk) {
                        // advance the start address: 16-B units; sub-tile j, 32 B per K=16 step
                        const uint64_t ad = ad0 + ((j * asub + kk * 32) >> 4);
                        const uint64_t bd = bd0 + ((j * C::kB + kk * 32) >> 4);
                        umma_f16(tmem, ad, bd, idesc, (st | j | kk) != 0);
                    }
                }
                if (mc > 1) umma_commit_mc(&empty[s], cmask);
                else umma_commit(&empty[s]);
            }
            umma_commit(done);
        }
        __syncwarp();
    }

    // ---------------- epilogue ----------------
    // 1) TMEM -> registers -> shared tile [128][BN+4] fp32 (all MMAs are complete at `done`,
    //    so the stage buffers are free to reuse).
    mbar_wait(done, 0);
    pdl_trigger();  // the successor's prologue and weight prefetch overlap this epilogue
    if (threadIdx.x == 0) FSW_TRACE_MAX(w.trace, w.layer, 6, globaltimer());
    STAMP(3);
    // this thread's 4 bias columns (weights: acquired by the producer before the MMAs completed), loaded
    // now so the round trip overlaps the TMEM drain
    constexpr uint32_t upr = BN / 4;
    const uint32_t c_own = (threadIdx.x % upr) * 4;
    uint2 bias_raw = make_uint2(0u, 0u);
    if (a.has_bias && n0 + c_own < a.N && a.N % 4 == 0)
        bias_raw = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.b_off)) + n0 + c_own);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float* ct = reinterpret_cast<float*>(smem);
#pragma unroll
    // warp w reads TMEM lanes 32·(w mod 4) (its lane quarter) and every (w / 4)-th 32-column block
    for (int c0 = 32 * (int)(warp >> 2); c0 < BN; c0 += 32 * (kGemmThreads / 128)) {
        if ((warp & 3u) * 32u >= a.m_rows) break;  // TMEM lanes past the tile's rows (m_rows = 64)
        uint32_t r[32];
        tmem_ld32(tmem + (((warp & 3u) * 32u) << 16) + (uint32_t)c0, r);
        float4* dst = reinterpret_cast<float4*>(ct + ((warp & 3u) * 32 + lane) * C::kLdc + c0);
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (c0 + 4 * j < BN)
                dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                     __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    STAMP(4);
    pdl_wait();  // activations (residual in, output / partials out) only after the predecessor
    if (threadIdx.x == 0) FSW_TRACE_MAX(w.trace, w.layer, 7, globaltimer());
    uint32_t rows = min(a.m_rows, a.M - m0);
    const uint32_t cols = min((uint32_t)BN, a.N - n0);
    uint32_t rb = 0;  // first tile row this CTA's epilogue covers
    if (a.cz > 1) {
        // 2c) cluster split-K: the cz CTAs of a (1, 1, cz) cluster hold the partial tiles of one output
        //     tile in their shared memory; CTA z sums rows [z·rows/cz, (z+1)·rows/cz) of all of them over
        //     DSMEM in split order (deterministic) and runs the epilogue on those rows only.
        cluster_sync();
        const uint32_t z = blockIdx.z, per = (rows + a.cz - 1) / a.cz;
        rb = min(rows, z * per);
        const uint32_t re = min(rows, rb + per);
        for (uint32_t u = threadIdx.x; u < (re - rb) * upr; u += blockDim.x) {
            const uint32_t r = rb + u / upr, c = (u % upr) * 4;
            const float* src = ct + r * C::kLdc + c;
            float4 v[8];  // all peers' loads in flight at once, then the sum in split order
#pragma unroll
            for (uint32_t q = 0; q < 8; ++q)
                if (q < a.cz) v[q] = ld_dsmem_f4(src, q);
            float4 acc = v[0];
#pragma unroll
            for (uint32_t q = 1; q < 8; ++q) {
                if (q >= a.cz) break;
                acc.x += v[q].x;
                acc.y += v[q].y;
                acc.z += v[q].z;
                acc.w += v[q].w;
            }
            // peers read only their own row slices: overwriting this slice of the local tile is safe
            *reinterpret_cast<float4*>(const_cast<float*>(src)) = acc;
        }
        __syncthreads();
        rows = re - rb;
    } else if (a.splits > 1) {
        // 2a) split-K: publish this split's partial tile, the last arriving CTA reduces all splits
        //     in split order (fixed summation order: deterministic).  Loads are batched kB units
        //     per thread so the reduction is bandwidth- rather than latency-bound.
        float* part = a.part + (size_t)tile * a.splits * (kBM * BN);
        float4* mine = reinterpret_cast<float4*>(part + (size_t)blockIdx.z * (kBM * BN));
        for (uint32_t u = threadIdx.x; u < rows * upr; u += blockDim.x) {
            const uint32_t r = u / upr, c = (u - r * upr) * 4;
            mine[u] = *reinterpret_cast<const float4*>(ct + r * C::kLdc + c);
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) *last_flag = atomicAdd(&a.ctr[tile], 1u) == a.splits - 1;
        __syncthreads();
        if (!*last_flag) {
            if (mc > 1) cluster_sync();
            return;
        }
        __threadfence();
        constexpr int kB = 8;
        for (uint32_t u0 = threadIdx.x; u0 < rows * upr; u0 += blockDim.x * kB) {
            float4 acc[kB];
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                const uint32_t u = u0 + j * blockDim.x;
                acc[j] = u < rows * upr ? __ldcg(reinterpret_cast<const float4*>(part) + u) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            for (uint32_t z = 1; z < a.splits; ++z) {
                const float4* pz = reinterpret_cast<const float4*>(part + (size_t)z * (kBM * BN));
                float4 v[kB];
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    const uint32_t u = u0 + j * blockDim.x;
                    v[j] = u < rows * upr ? __ldcg(pz + u) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    acc[j].x += v[j].x;
                    acc[j].y += v[j].y;
                    acc[j].z += v[j].z;
                    acc[j].w += v[j].w;
                }
            }
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                const uint32_t u = u0 + j * blockDim.x;
                if (u < rows * upr) {
                    const uint32_t r = u / upr, c = (u - r * upr) * 4;
                    *reinterpret_cast<float4*>(ct + r * C::kLdc + c) = acc[j];
                }
            }
        }
        if (threadIdx.x == 0) a.ctr[tile] = 0;  // self-reset for the next GEMM (ordered by PDL wait)
        __syncthreads();
    }
    // 2b) row-major pass over 4-column units: consecutive threads take consecutive units, so the
    //     bias / residual loads and the output stores are 8-16 B and coalesced.  Because
    //     blockDim.x is a multiple of BN/4, a thread always owns the same 4 columns: its bias is
    //     loaded once, and its residual rows are loaded kE at a time before any of their stores
    //     (measured: a load -> store chain per unit cost ~0.3 us per unit, 9.8 us at BN = 128).
    const uint16_t* __restrict__ bias = a.has_bias ? reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.b_off)) : nullptr;
    const bool vec = (a.N % 4 == 0) && (a.ld_out % 4 == 0) && (a.res == nullptr || a.ld_res % 4 == 0);
    if (vec) {
        constexpr int kE = 8;
        const uint32_t units = rows * upr, c = (threadIdx.x % upr) * 4;
        const bool col_ok = c < cols;
        float4 bsum = make_float4(0.f, 0.f, 0.f, 0.f);
        if (bias && col_ok) {  // c == c_own: prefetched after the MMAs
            const uint2 bv = bias_raw;
            bsum = make_float4(__uint_as_float(bv.x << 16), __uint_as_float(bv.x & 0xffff0000u),
                               __uint_as_float(bv.y << 16), __uint_as_float(bv.y & 0xffff0000u));
        }
        const float* __restrict__ resf = a.res && !a.res_bf16 ? reinterpret_cast<const float*>(a.res) : nullptr;
        const uint16_t* __restrict__ resh = a.res && a.res_bf16 ? reinterpret_cast<const uint16_t*>(a.res) : nullptr;
        for (uint32_t u0 = threadIdx.x; u0 < units; u0 += blockDim.x * kE) {
            uint4 raw[kE];
#pragma unroll
            for (int j = 0; j < kE; ++j) {
                const uint32_t u = u0 + j * blockDim.x, r = rb + u / upr;
                raw[j] = make_uint4(0, 0, 0, 0);
                if (u < units && col_ok) {
                    const uint64_t ri = (uint64_t)(m0 + r) * a.ld_res + n0 + c;
                    if (resf) raw[j] = *reinterpret_cast<const uint4*>(resf + ri);
                    else if (resh) {
                        const uint2 h = *reinterpret_cast<const uint2*>(resh + ri);
                        raw[j] = make_uint4(h.x << 16, h.x & 0xffff0000u, h.y << 16, h.y & 0xffff0000u);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < kE; ++j) {
                const uint32_t u = u0 + j * blockDim.x, r = rb + u / upr;
                if (!(u < units && col_ok)) continue;
                float4 v = *reinterpret_cast<const float4*>(ct + r * C::kLdc + c);
                // (acc + bias) + residual, the order of the unfused definition
                v.x = (v.x + bsum.x) + __uint_as_float(raw[j].x);
                v.y = (v.y + bsum.y) + __uint_as_float(raw[j].y);
                v.z = (v.z + bsum.z) + __uint_as_float(raw[j].z);
                v.w = (v.w + bsum.w) + __uint_as_float(raw[j].w);
                v = act4(a.act, v);
                const uint64_t oi = (uint64_t)(m0 + r) * a.ld_out + n0 + c;
                const uint2 pk = make_uint2((uint32_t)f32_to_bf16(v.x) | ((uint32_t)f32_to_bf16(v.y) << 16),
                                            (uint32_t)f32_to_bf16(v.z) | ((uint32_t)f32_to_bf16(v.w) << 16));
                if (a.out_bf16) *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(a.out) + oi) = pk;
                else *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + oi) = v;
                if (a.out2) *reinterpret_cast<uint2*>(a.out2 + oi) = pk;
            }
        }
    } else {
        for (uint32_t idx = threadIdx.x; idx < rows * BN; idx += blockDim.x) {
            const uint32_t r = rb + idx / BN, c = idx - (idx / BN) * BN;
            if (c >= cols) continue;
            const uint32_t m = m0 + r, n = n0 + c;
            float x = ct[r * C::kLdc + c];
            if (bias) x += bf16_to_f32(bias[n]);
            if (a.res)
                x += a.res_bf16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(a.res)[(uint64_t)m * a.ld_res + n])
                                : reinterpret_cast<const float*>(a.res)[(uint64_t)m * a.ld_res + n];
            x = apply_act(a.act, x);
            const uint64_t oi = (uint64_t)m * a.ld_out + n;
            if (a.out_bf16) reinterpret_cast<uint16_t*>(a.out)[oi] = f32_to_bf16(x);
            else reinterpret_cast<float*>(a.out)[oi] = x;
            if (a.out2) a.out2[oi] = f32_to_bf16(x);
        }
    }
#ifdef FSW_GEMM_TIMING
    __syncthreads();
    STAMP(5);
#endif
    if (mc > 1 || a.cz > 1) cluster_sync();  // no CTA leaves while a peer may still read / target its smem
}

// ---- K3b: the 2-CTA (cta_group::2) swap-AB GEMM for batch-1 transformer linears ---------------
// out[t][n] = act(Σ_k A[t][k]·W[n][k] + b[n] + res[t][n]) over a CTA PAIR: the pair owns 128 weight rows
// (the UMMA M operand, 64 per CTA) and T tokens (the N operand, T/2 per CTA); each CTA holds only its
// halves of every K sub-tile in shared memory and the leader's tcgen05.mma.cta_group::2 reads the
// peer's, so an SM receives half the operand bytes of a 1-CTA tile (per-SM operand
// bytes set the batch-1 GEMM time).  Both CTAs' TMA loads complete on the LEADER's full barrier
// (cp.async.bulk.tensor.cta_group::2), which expects both halves' bytes; the weights come through one
// tensor map over the GPU's whole weight pool (rows of 128 B of the pre-tiled layout, copied verbatim),
// addressed by the row of the layer's extent, so no per-extent map is needed.  The leader commits each
// stage to both CTAs' empty barriers (multicast).  TMEM layout of the pair's M=128 accumulator in each
// CTA: lane m + 64·(token ≥ T/2), column token mod T/2 (CUTLASS's 2SM "2x2" atom).
constexpr int kG2WR = 64, kG2KSub = 4;
template <int TT>
struct G2Cfg {
    static constexpr int TH = TT / 2;
    static constexpr uint32_t kW = kG2WR * 128, kX = TH * 128, kStage = kG2KSub * (kW + kX);
    static constexpr int kTmemCols = TH < 32 ? 32 : TH;
    __host__ static int max_stages() { const int f = (int)((200 * 1024) / kStage); return f > 5 ? 5 : f; }
};


template <int TT>
__global__ void __launch_bounds__(128) k_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
                                               const DevDesc* __restrict__ d, Wait w, GemmArgs a, int stages) {
    TraceExit tx(w.trace, w.layer);
    using C = G2Cfg<TT>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * C::kStage);
    uint64_t* empty = full + stages;
    uint64_t* done = empty + stages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    const uint32_t rank = cluster_ctarank(), warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t w0 = (blockIdx.x >> 1) * 128 + rank * kG2WR;  // this CTA's weight rows (tile columns)
    const uint32_t tb = blockIdx.y * TT;                          // the pair's tokens (tile rows)
    const uint32_t nkt = a.K / kBK, nst = (nkt + kG2KSub - 1) / kG2KSub;
    const DevDesc dd = *d;
    // issued now so their latency hides under the setup: the weight row of this CTA in the pool map, the
    // bias of this thread's epilogue row
    const uint64_t wrow = (uint64_t)(weight_ptr(dd, a.w_off) - reinterpret_cast<const uint8_t*>(a.wpool)) / 128 + w0;
    const uint32_t n_ep = w0 + (warp & 1) * 32 + lane;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "n"(C::kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();  // both CTAs' barriers exist before any copy completes on the leader's
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        // producer (both CTAs), lane-parallel: lane 0 of the LEADER arms a stage for both halves' bytes
        uint32_t lead[8];  // the leader's full barriers, in the cluster window
        for (int s = 0; s < stages && s < 8; ++s)
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead[s]) : "r"(smem_u32(&full[s])));
        if (lane == 0) {
            wait_ready_thread(w);
            FSW_TRACE_MAX(w.trace, w.layer, 1, globaltimer());
        }
        __syncwarp();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        auto arm = [&](uint32_t st0, uint32_t st1) {
            if (lane == 0 && rank == 0)
                for (uint32_t st = st0; st < st1; ++st) {
                    const uint32_t nsub = min((uint32_t)kG2KSub, nkt - st * kG2KSub);
                    mbar_expect_tx(&full[st % stages], 2 * nsub * (C::kW + C::kX));
                }
            __syncwarp();
        };
        auto load = [&](uint32_t st0, uint32_t st1, bool wts) {
            for (uint32_t i = lane; i < (st1 - st0) * kG2KSub; i += 32) {
                const uint32_t st = st0 + i / kG2KSub, j = i % kG2KSub, kt = st * kG2KSub + j, s = st % stages;
                if (kt >= nkt) continue;
                if (wts)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                        "%3}], [%4];" ::"r"(smem_u32(smem + s * C::kStage + j * C::kW)),
                        "l"(&tmW), "r"(0), "r"((int)(wrow + (uint64_t)kt * a.n_pad)), "r"(lead[s])
                        : "memory");
                else
                    asm volatile(
                        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                        "%3}], [%4];" ::"r"(smem_u32(smem + s * C::kStage + kG2KSub * C::kW + j * C::kX)),
                        "l"(&tmA), "r"((int)(kt * kBK)), "r"((int)(tb + rank * C::TH)), "r"(lead[s])
                        : "memory");
            }
        };
        const uint32_t pre = min((uint32_t)stages, nst);
        arm(0, pre);
        load(0, pre, true);  // weights first: they do not depend on the predecessor
        pdl_wait();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        load(0, pre, false);
        for (uint32_t st = pre; st < nst; ++st) {
            if (lane == 0) mbar_wait(&empty[st % stages], ((st / stages) - 1) & 1);
            __syncwarp();
            arm(st, st + 1);
            load(st, st + 1, true);
            load(st, st + 1, false);
        }
    } else if (warp == 1 && lane == 0 && rank == 0) {  // MMA issuer: M = 128 (64 per CTA), N = TT (TT/2 per CTA)
        constexpr uint32_t idesc = umma_idesc_bf16(128, TT);
        for (uint32_t st = 0; st < nst; ++st) {
            const uint32_t s = st % stages, nsub = min((uint32_t)kG2KSub, nkt - st * kG2KSub);
            mbar_wait(&full[s], (st / stages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t ad0 = umma_desc_sw128(smem + s * C::kStage), bd0 = umma_desc_sw128(smem + s * C::kStage + kG2KSub * C::kW);
            for (uint32_t j = 0; j < nsub; ++j)
#pragma unroll
                for (uint32_t kk = 0; kk < kBK / 16; ++kk) {
                    const uint64_t ad = ad0 + ((j * C::kW + kk * 32) >> 4), bd = bd0 + ((j * C::kX + kk * 32) >> 4);
                    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)((st | j | kk) != 0)));
                }
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                             smem_u32(&empty[s])), "h"((uint16_t)3) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         smem_u32(done)), "h"((uint16_t)3) : "memory");
    }
    __syncwarp();
    // epilogue: this CTA's 64 weight rows x the pair's TT tokens, straight from TMEM.  (Barrier waits
    // are cta-scope, as for the 1-CTA kernel: an .acquire.cluster poll executes CCTL.IVALL, an L1
    // invalidate, on every try; it was the top warp stall of the first in-graph ncu capture.)
    mbar_wait(done, 0);
    pdl_trigger();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    pdl_wait();  // activations (residual in, output out) only after the predecessor
    const uint32_t n = n_ep, tok0 = tb + (warp >> 1) * C::TH;
    const float bias = a.has_bias && n < a.N ? bf16_to_f32(reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.b_off))[n]) : 0.0f;
#pragma unroll
    for (int c0 = 0; c0 < C::TH; c0 += 16) {
        uint32_t r[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                       "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(tmem + ((warp * 32u) << 16) + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (n < a.N) {
            // every residual load of the 16 tokens before any store: the output may alias the residual as far
            // as the compiler knows, so a load after a store waits for it (one round trip per token otherwise)
            float rv[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const uint32_t t = tok0 + c0 + c;
                rv[c] = 0.0f;
                if (a.res && c0 + c < C::TH && t < a.M)
                    rv[c] = a.res_bf16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(a.res)[(uint64_t)t * a.ld_res + n])
                                       : reinterpret_cast<const float*>(a.res)[(uint64_t)t * a.ld_res + n];
            }
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const uint32_t t = tok0 + c0 + c;
                if (c0 + c >= C::TH || t >= a.M) break;
                const float v = apply_act(a.act, (__uint_as_float(r[c]) + bias) + rv[c]);
                const uint64_t oi = (uint64_t)t * a.ld_out + n;
                if (a.out_bf16) reinterpret_cast<uint16_t*>(a.out)[oi] = f32_to_bf16(v);
                else reinterpret_cast<float*>(a.out)[oi] = v;
                if (a.out2) a.out2[oi] = f32_to_bf16(v);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    // both CTAs saw `done`: no MMA can still target either TMEM, and no copy or MMA touches the peer's
    // shared memory any more
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols) : "memory");
}

template <int TT>
static void launch_g2(cudaStream_t s, const DevDesc* d, Wait w, const CUtensorMap* tmA, const CUtensorMap* tmW, const GemmArgs& a) {
    using C = G2Cfg<TT>;
    const int nst = (int)((a.K / kBK + kG2KSub - 1) / kG2KSub), ms = C::max_stages();
    const int stages = nst < ms ? nst : ms;
    const dim3 grid((a.n_pad + 127) / 128 * 2, (a.M + TT - 1) / TT);
    launch_pdl_cluster(PDL_GEMM, k_gemm2<TT>, grid, dim3(128), stages * C::kStage + 2048, s, dim3(2, 1, 1), *tmA, *tmW, d, w, a,
                       stages);
}

template <int BN>
static void launch_bn(cudaStream_t s, const DevDesc* d, Wait w, const CUtensorMap* tmA, const GemmArgs& a) {
    using C = Cfg<BN>;
    const int nst = (int)((a.kt_per + C::kSub - 1) / C::kSub);
    const uint32_t asub = C::a_sub(a.m_rows, a.conv);
    const int ms = C::max_stages(asub);
    const int stages = nst < ms ? nst : ms;
    dim3 grid((a.M + a.m_rows - 1) / a.m_rows, a.n_pad / BN, a.splits);
    launch_pdl_cluster(PDL_GEMM, k_gemm<BN>, grid, dim3(kGemmThreads), C::smem_bytes(stages, asub), s,
                       dim3(1, a.mc > 1 ? a.mc : 1, a.cz > 1 ? a.cz : 1), *tmA, d, w, a, stages);
}

void init_gemm_attrs() {  // once per device at fsw_init (kernel preloading)
    cudaFuncSetAttribute(k_gemm<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_gemm<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_gemm<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_gemm<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_gemm2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_gemm2<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_gemm2<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_gemm2<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

template <int BN>
static int max_clusters_bn(int cz) {
    using C = Cfg<BN>;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1, 1, cz);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = C::smem_bytes(C::max_stages(C::kA));
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 1;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = cz;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_gemm<BN>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Clusters of cz GEMM CTAs that can be resident at once on the current device (one wave).
int gemm_max_active_clusters(int bn, int cz) {
    switch (bn) {
        case 16: return max_clusters_bn<16>(cz);
        case 32: return max_clusters_bn<32>(cz);
        case 64: return max_clusters_bn<64>(cz);
        default: return max_clusters_bn<128>(cz);
    }
}

void launch_gemm(cudaStream_t s, const DevDesc* d, Wait w, const CUtensorMap* tmA, const GemmArgs& a, const CUtensorMap* tmW) {
    if (a.ws_tt) {
        launch_gemm_ws(s, d, w, tmA, a);
        return;
    }
    if (a.pair_t) {
        switch (a.pair_t) {
            case 16: launch_g2<16>(s, d, w, tmA, tmW, a); break;
            case 32: launch_g2<32>(s, d, w, tmA, tmW, a); break;
            case 64: launch_g2<64>(s, d, w, tmA, tmW, a); break;
            default: launch_g2<128>(s, d, w, tmA, tmW, a); break;
        }
        return;
    }
    switch (a.bn) {
        case 16: launch_bn<16>(s, d, w, tmA, a); break;
        case 32: launch_bn<32>(s, d, w, tmA, a); break;
        case 64: launch_bn<64>(s, d, w, tmA, a); break;
        default: launch_bn<128>(s, d, w, tmA, a); break;
    }
}

// ---- TMA descriptor for a row-major bf16 activation [rows][cols] (row pitch ld_elems) ----
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool make_tmap_act(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems, uint32_t box_rows) {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return false;
        fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {ld_elems * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows ? box_rows : (cuuint32_t)kBM};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The GPU's whole weight pool as rows of 128 B (the pre-tiled weight layout, copied verbatim by the
// 2-CTA GEMM: no swizzle on the copy, the bytes already are in SWIZZLE_128B order), 64-row boxes.
bool make_tmap_pool(CUtensorMap* map, const void* pool, uint64_t bytes) {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return false;
        fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    if (bytes / 128 >= (1ull << 31)) return false;  // TMA row coordinates are int32
    const cuuint64_t dims[2] = {64, bytes / 128};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {64, (cuuint32_t)kG2WR};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_conv(CUtensorMap* map, const void* base, uint32_t H, uint32_t W, uint32_t C, uint32_t Q, uint32_t Hb,
                    uint32_t stride) {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return false;
        fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    if (Q * stride > 256 || Hb * stride > 256 || Hb * Q > (uint32_t)kBM || C % kBK) return false;
    const cuuint64_t dims[4] = {C, W, H, 1};
    const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    const cuuint32_t box[4] = {(cuuint32_t)kBK, Q * stride, Hb * stride, 1};
    const cuuint32_t estr[4] = {1, stride, stride, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


}  // namespace fsw
