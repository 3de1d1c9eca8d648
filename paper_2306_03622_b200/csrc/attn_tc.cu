// attn_tc.cu — K6b: single-tile attention on the 5th-generation tensor cores (tcgen05 / TMEM / TMA), T <= 128,
// head width 64: one CTA per head, 256 threads, threads q and q + 128 = query row q = TMEM lane q (one per key half).
//
//   S = Q·Kᵀ (UMMA M = 128 queries, N = 128 keys, K = 64) -> TMEM columns [0, 128)
//   each thread: its S row from TMEM, scale 1/√64, causal / length mask, max, P = exp(S − max) rounded to bf16,
//                l = Σ exp (fp32) — P is written to shared memory as the K-major SWIZZLE_128B A operand
//   O = P·V (UMMA M = 128, N = 64, K = 128 keys; V is the MN-major B operand exactly as TMA loaded it: rows =
//            keys, 64 head columns contiguous) -> TMEM columns [128, 192)
//   out[q][h·64 + d] = O[q][d] / l  (bf16)
// Q, K and V come from the QKV activation [T][3·H·64] by three TMA boxes of 64 columns x 128 rows (rows past T
// zero-filled).  Against the mma.sync kernel (k_attention_mma2: 4 warps per (head, 16 query rows), S and P·V in
// registers), this holds a whole head's S in TMEM and issues 12 MMAs from one thread.
#include "device.cuh"
#include "umma.cuh"

namespace fsw {

constexpr uint32_t kAtT = 128, kAtDh = 64;
__device__ __forceinline__ uint32_t pack_bf16x2_tc(float lo, float hi) {
    return (uint32_t)f32_to_bf16(lo) | ((uint32_t)f32_to_bf16(hi) << 16);
}
constexpr uint32_t kAtTile = kAtT * kAtDh * 2;  // one 128 x 64 bf16 tile: 16 KiB
// shared memory: Q | K | V | barriers; P (two 64-key sub-tiles, 32 KiB) reuses Q | K once S = Q·Kᵀ is complete (52 KiB
// in all: a CTA fits beside the next GEMM's early-resident CTAs)
constexpr uint32_t kAtSmem = 3 * kAtTile + 3072 + 1024;  // + barriers, TMEM slot, 2 KiB of row max / sum, alignment

// UMMA shared-memory descriptor of an MN-major SWIZZLE_128B operand whose rows (stride 128 B, 8-row atoms 1024 B
// apart along K) hold 64 contiguous MN elements: LBO unused (one 128-B atom column), SBO = 1024 B.
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(const void* p) {
    const uint64_t addr = smem_u32(p);
    return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void __launch_bounds__(256) k_attention_tc(const __grid_constant__ CUtensorMap tmQKV, AttnArgs a) {
    TraceExit tx(a.trace, a.layer);
    pdl_trigger();  // the O-projection sets up and loads its weights during attention (as FSW_EARLY_TRIGGER bit 1)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sQ = smem, *sK = smem + kAtTile, *sV = smem + 2 * kAtTile, *sP = smem;  // P over Q | K (after S)
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 3 * kAtTile);  // [0] loads, [1] S done, [2] O done (+ tslot, red)
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
    // 256 threads: thread t handles query row q = t mod 128 (TMEM lane quarter = warp mod 4) and key half
    // kh = t / 128 (keys [64 kh, 64 kh + 64)) of the softmax, and head columns [32 kh, 32 kh + 32) of the output
    const uint32_t tid = threadIdx.x, warp = tid >> 5, h = blockIdx.x;
    const uint32_t T = a.T, D = a.H * kAtDh, q = tid & 127u, kh = tid >> 7;
    float* red = reinterpret_cast<float*>(tslot + 4);  // [2 halves][128 rows] row max, then row sum

    if (tid == 0) {
        for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQKV) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    pdl_wait();  // the QKV activation comes from the predecessor

    if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_expect_tx(&bar[0], 3 * kAtTile);
        tma_load_2d(sQ, &tmQKV, (int)(h * kAtDh), 0, &bar[0]);
        tma_load_2d(sK, &tmQKV, (int)(D + h * kAtDh), 0, &bar[0]);
        tma_load_2d(sV, &tmQKV, (int)(2 * D + h * kAtDh), 0, &bar[0]);
        mbar_wait(&bar[0], 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        constexpr uint32_t idesc = umma_idesc_bf16(128, 128);
        const uint64_t qd = umma_desc_sw128(sQ), kd = umma_desc_sw128(sK);
#pragma unroll
        for (uint32_t ks = 0; ks < kAtDh / 16; ++ks) umma_f16(tmem, qd + ks * 2, kd + ks * 2, idesc, ks != 0);
        umma_commit(&bar[1]);
    }
    __syncwarp();
    mbar_wait(&bar[1], 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // softmax of this thread's half row (fp32); the halves combine max and sum through shared memory; P rounded to
    // bf16 into the K-major SWIZZLE_128B A operand (sub-tile kh holds keys [64 kh, 64 kh + 64))
    float s[kAtT / 2];
#pragma unroll
    for (uint32_t c0 = 0; c0 < kAtT / 2; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + (((warp & 3u) * 32u) << 16) + kh * 64 + c0, v);
#pragma unroll
        for (int c = 0; c < 32; ++c) s[c0 + c] = __uint_as_float(v[c]);
    }
    const float sc = 0.125f * 1.4426950408889634f;  // 1/√64, in log2 units
    const uint32_t kend = a.causal ? min(T, q + 1) : T;  // keys [0, kend) are visible
    float m = -INFINITY;
#pragma unroll
    for (uint32_t k = 0; k < kAtT / 2; ++k) {
        s[k] = kh * 64 + k < kend ? s[k] * sc : -INFINITY;
        m = fmaxf(m, s[k]);
    }
    red[kh * 128 + q] = m;
    __syncthreads();
    m = fmaxf(red[q], red[128 + q]);  // finite: key 0 is always visible
    float l = 0.f;
    uint8_t* prow = sP + kh * (kAtT * 128) + (q / 8) * 1024 + (q % 8) * 128;
#pragma unroll
    for (uint32_t c = 0; c < 8; ++c) {  // 8 chunks of 8 keys: 16-B swizzled stores
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float p0 = exp2f(s[8 * c + 2 * j] - m), p1 = exp2f(s[8 * c + 2 * j + 1] - m);
            l += p0 + p1;
            w[j] = pack_bf16x2_tc(p0, p1);
        }
        *reinterpret_cast<uint4*>(prow + ((c ^ (q % 8)) * 16)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    __syncthreads();  // every max read before the sums overwrite nothing: the sums go to the other row of red
    red[256 + kh * 128 + q] = l;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P (generic stores) -> the MMA (async proxy)
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        constexpr uint32_t idesc = umma_idesc_bf16(128, kAtDh) | (1u << 16);  // B (V) MN-major
        const uint64_t vd = umma_desc_sw128_mn(sV);
#pragma unroll
        for (uint32_t ks = 0; ks < kAtT / 16; ++ks) {
            // A: sub-tile ks / 4 (64 keys), 32 B per 16-key step inside it; B: 16 key rows = 2 atoms = 2 KiB
            const uint64_t pd = umma_desc_sw128(sP + (ks / 4) * (kAtT * 128)) + ((ks % 4) * 32 >> 4);
            umma_f16(tmem + 128, pd, vd + ((ks * 2048) >> 4), idesc, ks != 0);
        }
        umma_commit(&bar[2]);
    }
    __syncwarp();
    mbar_wait(&bar[2], 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const float inv = 1.0f / (red[256 + q] + red[384 + q]);
    uint16_t* orow = a.out + (uint64_t)q * D + h * kAtDh;
    {
        const uint32_t c0 = kh * 32;
        uint32_t v[32];
        tmem_ld32(tmem + (((warp & 3u) * 32u) << 16) + 128 + c0, v);
        if (q < T) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint4 o;
                o.x = pack_bf16x2_tc(__uint_as_float(v[8 * j]) * inv, __uint_as_float(v[8 * j + 1]) * inv);
                o.y = pack_bf16x2_tc(__uint_as_float(v[8 * j + 2]) * inv, __uint_as_float(v[8 * j + 3]) * inv);
                o.z = pack_bf16x2_tc(__uint_as_float(v[8 * j + 4]) * inv, __uint_as_float(v[8 * j + 5]) * inv);
                o.w = pack_bf16x2_tc(__uint_as_float(v[8 * j + 6]) * inv, __uint_as_float(v[8 * j + 7]) * inv);
                *reinterpret_cast<uint4*>(orow + c0 + 8 * j) = o;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}


bool attention_tc_ok(const AttnArgs& a) { return a.T >= 1 && a.T <= kAtT && a.dh == kAtDh; }

void launch_attention_tc(cudaStream_t s, const CUtensorMap* tm, const AttnArgs& a) {
    launch_pdl(PDL_ATTN, k_attention_tc, dim3(a.H), dim3(256), kAtSmem, s, *tm, a);
}

void init_attn_tc_attrs() { cudaFuncSetAttribute(k_attention_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kAtSmem); }

}  // namespace fsw
