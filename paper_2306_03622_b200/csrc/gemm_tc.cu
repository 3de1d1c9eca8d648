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
// One CTA = one 128 x BN output tile; 4 warps.  Thread 0 is the TMA producer: it first
// spins on the layer's ready counter (the swap kernel's release, PAPER.md:588-590
// pipelining), fences generic->async proxy, then streams the K loop through a 4-stage
// mbarrier ring.  Thread 32 issues tcgen05.mma (M=128, N=BN, K=16) into TMEM and commits
// each stage back to its empty barrier.  All 4 warps then drain TMEM (tcgen05.ld 32x32b)
// through the fused bias / residual / activation epilogue.
#include "device.cuh"

namespace fsw {

namespace {

constexpr int kBM = 128, kBK = 64, kStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    const uint32_t a = smem_u32(b);
    uint32_t ok = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms 1024 B apart (SBO),
// LBO unused for swizzled K-major, version 1 (sm_100), base offset 0 (1024-B aligned tiles).
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* p) {
    const uint64_t addr = smem_u32(p);
    return ((addr >> 4) & 0x3FFFull) | (0ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}
// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
        "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int BN>
struct Smem {
    static constexpr uint32_t kA = kBM * kBK * 2;  // 16 KiB
    static constexpr uint32_t kB = BN * kBK * 2;   // BN x 128 B
    static constexpr uint32_t kBytes = kStages * (kA + kB) + 1024 /*barriers*/ + 1024 /*align slack*/;
};

}  // namespace

template <int BN>
__global__ void __launch_bounds__(128, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const DevDesc* __restrict__ d, Wait w, GemmArgs a) {
    using S = Smem<BN>;
    constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * S::kA;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * S::kB);
    uint64_t* empty = full + kStages;
    uint64_t* done = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t m0 = blockIdx.x * kBM, n0 = blockIdx.y * BN;
    const uint32_t nk = a.K / kBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
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
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (threadIdx.x == 0) {
        // ---------------- producer: ready flag -> proxy fence -> TMA(A) + bulk(W) ring ----------------
        wait_ready_thread(w);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const uint8_t* wt = d->wbase + a.w_off;
        const uint64_t ktile_stride = (uint64_t)(a.n_pad / 8) * 1024;
        for (uint32_t kb = 0; kb < nk; ++kb) {
            const int s = kb % kStages;
            if (kb >= (uint32_t)kStages) mbar_wait(&empty[s], ((kb / kStages) - 1) & 1);
            mbar_expect_tx(&full[s], S::kA + S::kB);
            tma_load_2d(sA + s * S::kA, &tmA, (int)(kb * kBK), (int)m0, &full[s]);
            bulk_load(sB + s * S::kB, wt + kb * ktile_stride + (uint64_t)(n0 / 8) * 1024, S::kB, &full[s]);
        }
    } else if (threadIdx.x == 32) {
        // ---------------- MMA issuer: one thread drives the tensor core ----------------
        constexpr uint32_t idesc = umma_idesc_bf16(kBM, BN);
        for (uint32_t kb = 0; kb < nk; ++kb) {
            const int s = kb % kStages;
            mbar_wait(&full[s], (kb / kStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
                const uint64_t ad = umma_desc_sw128(sA + s * S::kA + kk * 32);
                const uint64_t bd = umma_desc_sw128(sB + s * S::kB + kk * 32);
                umma_f16(tmem, ad, bd, idesc, (kb | kk) != 0);
            }
            umma_commit(&empty[s]);
        }
        umma_commit(done);
    }

    // ---------------- epilogue: TMEM -> registers -> bias/residual/act -> global ----------------
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t row = m0 + warp * 32 + lane;
    const uint16_t* bias = a.has_bias ? reinterpret_cast<const uint16_t*>(d->wbase + a.b_off) : nullptr;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((warp * 32u) << 16) + (uint32_t)c0, r);
        if (row >= a.M) continue;
        const uint32_t nb = n0 + c0;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        const uint32_t ncols = min(32u, (uint32_t)(BN - c0));  // valid accumulator columns in this chunk
        const bool full_vec = ncols == 32 && (nb + 32 <= a.N) && (a.ld_out % 8 == 0) && (a.res == nullptr || a.ld_res % 8 == 0);
        if (full_vec) {
            if (bias) {
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                    const uint4 bv = *reinterpret_cast<const uint4*>(bias + nb + j);
                    const uint32_t bu[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        v[j + 2 * h] += __uint_as_float(bu[h] << 16);
                        v[j + 2 * h + 1] += __uint_as_float(bu[h] & 0xffff0000u);
                    }
                }
            }
            if (a.res) {
                if (a.res_bf16) {
                    const uint4* rp = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.res) +
                                                                     (uint64_t)row * a.ld_res + nb);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint4 rv = rp[j];
                        const uint32_t ru[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            v[8 * j + 2 * h] += __uint_as_float(ru[h] << 16);
                            v[8 * j + 2 * h + 1] += __uint_as_float(ru[h] & 0xffff0000u);
                        }
                    }
                } else {
                    const float4* rp =
                        reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.res) + (uint64_t)row * a.ld_res + nb);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float4 rv = rp[j];
                        v[4 * j] += rv.x;
                        v[4 * j + 1] += rv.y;
                        v[4 * j + 2] += rv.z;
                        v[4 * j + 3] += rv.w;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = apply_act(a.act, v[j]);
            if (a.out_bf16 || a.out2) {
                uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    pk[j] = (uint32_t)f32_to_bf16(v[2 * j]) | ((uint32_t)f32_to_bf16(v[2 * j + 1]) << 16);
                uint16_t* dst = a.out_bf16 ? reinterpret_cast<uint16_t*>(a.out) : a.out2;
                uint4* op = reinterpret_cast<uint4*>(dst + (uint64_t)row * a.ld_out + nb);
#pragma unroll
                for (int j = 0; j < 4; ++j) op[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            }
            if (!a.out_bf16) {
                float4* op = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + (uint64_t)row * a.ld_out + nb);
#pragma unroll
                for (int j = 0; j < 8; ++j) op[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t n = nb + j;
                if (n >= a.N || (uint32_t)j >= ncols) break;
                float x = v[j];
                if (bias) x += bf16_to_f32(bias[n]);
                if (a.res)
                    x += a.res_bf16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(a.res)[(uint64_t)row * a.ld_res + n])
                                    : reinterpret_cast<const float*>(a.res)[(uint64_t)row * a.ld_res + n];
                x = apply_act(a.act, x);
                const uint64_t oi = (uint64_t)row * a.ld_out + n;
                if (a.out_bf16) reinterpret_cast<uint16_t*>(a.out)[oi] = f32_to_bf16(x);
                else reinterpret_cast<float*>(a.out)[oi] = x;
                if (a.out2) a.out2[oi] = f32_to_bf16(x);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
}

template <int BN>
static void launch_bn(cudaStream_t s, const DevDesc* d, Wait w, const CUtensorMap* tmA, const GemmArgs& a) {
    const int smem = (int)Smem<BN>::kBytes;
    dim3 grid((a.M + kBM - 1) / kBM, a.n_pad / BN);
    k_gemm<BN><<<grid, 128, smem, s>>>(*tmA, d, w, a);
}

void init_gemm_attrs() {  // once per device at fsw_init (kernel preloading)
    cudaFuncSetAttribute(k_gemm<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Smem<16>::kBytes);
    cudaFuncSetAttribute(k_gemm<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Smem<32>::kBytes);
    cudaFuncSetAttribute(k_gemm<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Smem<64>::kBytes);
    cudaFuncSetAttribute(k_gemm<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Smem<128>::kBytes);
}

void launch_gemm(cudaStream_t s, const DevDesc* d, Wait w, const CUtensorMap* tmA, const GemmArgs& a) {
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

bool make_tmap_act(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems) {
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
    const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)kBM};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace fsw
