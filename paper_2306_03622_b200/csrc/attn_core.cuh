// attn_core.cuh — the tensor-core attention core shared by the per-layer kernel (ops.cu,
// k_attention_mma2) and the persistent transformer kernel (mega.cu): one task = (head h, 16 query rows
// from q0) run by 128 threads (4 warps) with `sync` as their barrier and `sm_kv2` as their shared memory.
#pragma once
#include <math.h>

#include "device.cuh"

namespace fsw {

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    return (uint32_t)f32_to_bf16(lo) | ((uint32_t)f32_to_bf16(hi) << 16);
}

constexpr int kAttnMmaMaxT = 128;
template <bool CG>
__device__ __forceinline__ uint32_t ldq(const uint16_t* p) {
    return CG ? __ldcg(reinterpret_cast<const unsigned int*>(p)) : *reinterpret_cast<const uint32_t*>(p);
}
// Key-split variant: one CTA per (head, 16 query rows); its 4 warps take a quarter of the keys each
// (S, softmax and P·V over 32 keys at T = 128: a quarter of the dependent MMA chain of the kernel
// above), then combine through shared memory with the usual max / sum rescaling:
//   m = max_w m_w,  O = Σ_w e^(m_w − m) O_w,  l = Σ_w e^(m_w − m) l_w,  out = O / l.
constexpr int kAttnSplitRows = 16, kAttnSplitWarps = 4;

template <int DH, bool CG = false, typename Sync>
__device__ __forceinline__ void attn_split_core(const AttnArgs& a, uint32_t h, uint32_t q0, uint16_t* sm_kv2, uint32_t tid,
                                                Sync sync) {
    constexpr int KS = DH / 16, NO = DH / 8, LD = DH + 8;
    constexpr int NSW = kAttnMmaMaxT / 8 / kAttnSplitWarps;  // key n-tiles per warp (4 at T <= 128)
    // CG: activations through L2 only (ld.global.cg) — in the persistent kernel (mega.cu) another SM may have
    // rewritten this slot since an earlier layer's task cached it in this SM's L1
    const uint32_t T = a.T, D = a.H * DH, W3 = 3 * D;
    const uint32_t kend = a.causal ? min(T, q0 + kAttnSplitRows) : T;
    const uint32_t kpad = (kend + 15) & ~15u;
    const uint32_t kper = (((kpad + kAttnSplitWarps - 1) / kAttnSplitWarps) + 15) & ~15u;  // keys per warp, x16
    uint16_t* Ks = sm_kv2;
    uint16_t* Vs = Ks + kper * kAttnSplitWarps * LD;
    float* Os = reinterpret_cast<float*>(Vs + kper * kAttnSplitWarps * LD);  // [warp][16][DH]
    float* Ms = Os + kAttnSplitWarps * 16 * DH;                                // [warp][16]
    float* Ls = Ms + kAttnSplitWarps * 16;
    constexpr uint32_t C8 = DH / 8;
    const uint32_t kstage = kper * kAttnSplitWarps;
    for (uint32_t i = tid; i < kstage * C8; i += 128u) {
        const uint32_t j = i / C8, c = (i - j * C8) * 8;
        uint4 kv = make_uint4(0, 0, 0, 0), vv = kv;
        if (j < kend) {
            const uint16_t* row = a.qkv + (uint64_t)j * W3 + h * DH + c;
            kv = CG ? __ldcg(reinterpret_cast<const uint4*>(row + D)) : *reinterpret_cast<const uint4*>(row + D);
            vv = CG ? __ldcg(reinterpret_cast<const uint4*>(row + 2 * D)) : *reinterpret_cast<const uint4*>(row + 2 * D);
        }
        *reinterpret_cast<uint4*>(Ks + j * LD + c) = kv;
        *reinterpret_cast<uint4*>(Vs + j * LD + c) = vv;
    }
    const uint32_t warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const uint32_t ra = q0 + g, rb = ra + 8;
    uint32_t qa[KS][4];
    {
        const uint16_t* pa = a.qkv + (uint64_t)ra * W3 + h * DH;
        const uint16_t* pb = a.qkv + (uint64_t)rb * W3 + h * DH;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            const uint32_t c = kk * 16 + 2 * t;
            qa[kk][0] = ra < T ? ldq<CG>(pa + c) : 0u;
            qa[kk][1] = rb < T ? ldq<CG>(pb + c) : 0u;
            qa[kk][2] = ra < T ? ldq<CG>(pa + c + 8) : 0u;
            qa[kk][3] = rb < T ? ldq<CG>(pb + c + 8) : 0u;
        }
    }
    sync();
    // this warp's keys [k0, k0 + kper) ∩ [0, kend)
    const uint32_t k0 = warp * kper;
    const uint32_t nst = k0 < kend ? (min(kend - k0, kper) + 7) / 8 : 0;
    const float scale = rsqrtf((float)DH);
    float s[NSW][4];
#pragma unroll
    for (int n = 0; n < NSW; ++n) {
        s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.0f;
        if ((uint32_t)n < nst) {
            const uint16_t* kr = Ks + (k0 + n * 8 + g) * LD + 2 * t;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk)
                mma_bf16_16816(s[n], qa[kk], *reinterpret_cast<const uint32_t*>(kr + kk * 16),
                               *reinterpret_cast<const uint32_t*>(kr + kk * 16 + 8));
        }
    }
    float mxa = -INFINITY, mxb = -INFINITY;
#pragma unroll
    for (int n = 0; n < NSW; ++n) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t j = k0 + n * 8 + 2 * t + (e & 1), r = e < 2 ? ra : rb;
            const bool ok = (uint32_t)n < nst && j < kend && j < T && (!a.causal || j <= r);
            s[n][e] = ok ? s[n][e] * scale : -INFINITY;
        }
        mxa = fmaxf(mxa, fmaxf(s[n][0], s[n][1]));
        mxb = fmaxf(mxb, fmaxf(s[n][2], s[n][3]));
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
        mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, o));
        mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, o));
    }
    // a row with no valid key in this warp's range contributes nothing (weight e^-inf = 0 below)
    const float ba = mxa == -INFINITY ? 0.0f : mxa, bb = mxb == -INFINITY ? 0.0f : mxb;
    float za = 0.0f, zb = 0.0f;
#pragma unroll
    for (int n = 0; n < NSW; ++n) {
        s[n][0] = __expf(s[n][0] - ba);
        s[n][1] = __expf(s[n][1] - ba);
        s[n][2] = __expf(s[n][2] - bb);
        s[n][3] = __expf(s[n][3] - bb);
        za += s[n][0] + s[n][1];
        zb += s[n][2] + s[n][3];
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
        za += __shfl_xor_sync(0xffffffffu, za, o);
        zb += __shfl_xor_sync(0xffffffffu, zb, o);
    }
    float o[NO][4];
#pragma unroll
    for (int n = 0; n < NO; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.0f;
    const uint32_t nkk = (nst + 1) / 2;
#pragma unroll
    for (int kk = 0; kk < NSW / 2; ++kk) {
        if ((uint32_t)kk >= nkk) break;
        const uint32_t pa[4] = {pack_bf16x2(s[2 * kk][0], s[2 * kk][1]), pack_bf16x2(s[2 * kk][2], s[2 * kk][3]),
                                pack_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                                pack_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
        const uint32_t mi = lane >> 3, rr = lane & 7;
#pragma unroll
        for (int n = 0; n < NO; n += 2) {
            const uint16_t* p = Vs + (k0 + kk * 16 + (mi & 1) * 8 + rr) * LD + (n + (mi >> 1)) * 8;
            uint32_t b0, b1, b2, b3;
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                         : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                         : "r"((uint32_t)__cvta_generic_to_shared(p)));
            mma_bf16_16816(o[n], pa, b0, b1);
            if (n + 1 < NO) mma_bf16_16816(o[n + 1], pa, b2, b3);
        }
    }
    // partial results to shared memory: O_w rows g and g+8, m_w (-inf when empty), l_w
    float* ow = Os + warp * 16 * DH;
#pragma unroll
    for (int n = 0; n < NO; ++n) {
        const uint32_t c = n * 8 + 2 * t;
        *reinterpret_cast<float2*>(ow + g * DH + c) = make_float2(o[n][0], o[n][1]);
        *reinterpret_cast<float2*>(ow + (g + 8) * DH + c) = make_float2(o[n][2], o[n][3]);
    }
    if (t == 0) {
        Ms[warp * 16 + g] = mxa;
        Ms[warp * 16 + g + 8] = mxb;
        Ls[warp * 16 + g] = za;
        Ls[warp * 16 + g + 8] = zb;
    }
    sync();
    // combine: thread i handles (row, 8 columns) units, warps' contributions in warp order
    for (uint32_t u = tid; u < 16u * (DH / 8); u += 128u) {
        const uint32_t r = u / (DH / 8), c = (u % (DH / 8)) * 8;
        if (q0 + r >= T) continue;
        float m = -INFINITY;
#pragma unroll
        for (int w = 0; w < kAttnSplitWarps; ++w) m = fmaxf(m, Ms[w * 16 + r]);
        float l = 0.0f, acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int w = 0; w < kAttnSplitWarps; ++w) {
            const float mw = Ms[w * 16 + r];
            if (mw == -INFINITY) continue;
            const float f = __expf(mw - m);
            l += f * Ls[w * 16 + r];
            const float4 x0 = *reinterpret_cast<const float4*>(Os + (w * 16 + r) * DH + c);
            const float4 x1 = *reinterpret_cast<const float4*>(Os + (w * 16 + r) * DH + c + 4);
            acc[0] += f * x0.x; acc[1] += f * x0.y; acc[2] += f * x0.z; acc[3] += f * x0.w;
            acc[4] += f * x1.x; acc[5] += f * x1.y; acc[6] += f * x1.z; acc[7] += f * x1.w;
        }
        const float il = 1.0f / l;
        const uint4 pk = make_uint4(pack_bf16x2(acc[0] * il, acc[1] * il), pack_bf16x2(acc[2] * il, acc[3] * il),
                                    pack_bf16x2(acc[4] * il, acc[5] * il), pack_bf16x2(acc[6] * il, acc[7] * il));
        *reinterpret_cast<uint4*>(a.out + (uint64_t)(q0 + r) * D + h * DH + c) = pk;
    }
}

template <int DH>
__host__ __device__ constexpr size_t attn2_smem_bytes(uint32_t T) {
    return 2ull * ((((((T + 15) & ~15u) + kAttnSplitWarps - 1) / kAttnSplitWarps) + 15) & ~15u) * kAttnSplitWarps * (DH + 8) *
               sizeof(uint16_t) +
           sizeof(float) * (kAttnSplitWarps * 16 * DH + 2 * kAttnSplitWarps * 16);
}

}  // namespace fsw
