// ops.cu — the non-GEMM layer kernels (HBM/latency-bound at batch 1): embedding gather,
// LayerNorm, GEMV (M = 1 linears: MLP, pooler, fc, LM head), attention core, im2col,
// max/avg pooling.  Each kernel that reads weights first waits on its layer's ready
// counter (device.cuh), which is how "each layer's kernels start as soon as its weights
// land" (BASELINE.json north_star).
#include "device.cuh"

namespace fsw {

// ------------------------------------------------------------------------------------------
// EMBED: out[t][c] = Σ_j table_j[row_j(t)][c]   (fp32 sum of bf16 rows)
// ------------------------------------------------------------------------------------------
__global__ void k_embed(const DevDesc* __restrict__ d, Wait w, EmbedArgs a) {
    wait_ready_cta(w);
    pdl_wait();
    const uint32_t t = blockIdx.x;
    const DevDesc dd = *d;
    uint32_t row[4];
    for (int j = 0; j < a.n_tables; ++j) {
        uint32_t r = a.rule[j] == FSW_RULE_IDS ? (uint32_t)a.ids[t] : (a.rule[j] == FSW_RULE_POSITION ? t : 0u);
        if (r >= a.table_rows[j]) {  // out-of-range id: flag it, read row 0
            if (threadIdx.x == 0) atomicExch(&w.ctl->err, 3);
            r = 0;
        }
        row[j] = r;
    }
    for (uint32_t c = threadIdx.x; c < a.C; c += blockDim.x) {
        float s = 0.0f;
        for (int j = 0; j < a.n_tables; ++j) {
            const uint16_t* tab = reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.table_off[j]));
            s += bf16_to_f32(tab[(uint64_t)row[j] * a.C + c]);
        }
        if (a.out) a.out[(uint64_t)t * a.C + c] = s;
        if (a.out_bf16) a.out_bf16[(uint64_t)t * a.C + c] = f32_to_bf16(s);
    }
}

void launch_embed(cudaStream_t s, const DevDesc* d, Wait w, const EmbedArgs& a) {
    launch_pdl(PDL_EMBED, k_embed, dim3(a.T), dim3(256), 0, s, d, w, a);
}

// ------------------------------------------------------------------------------------------
// LAYERNORM: one warp per row, the row held in registers as float4 (NV per lane, C <= 128·NV),
// fp32 two-pass statistics (mean, then centred variance), 8-B vector loads of γ/β.
// ------------------------------------------------------------------------------------------
template <int NV>
__global__ void __launch_bounds__(128) k_layernorm(const DevDesc* __restrict__ d, Wait w, LnArgs a) {
    wait_ready_cta(w);
    pdl_wait();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t r = blockIdx.x * (blockDim.x >> 5) + warp;
    if (r >= a.rows) return;
    const uint32_t n4 = a.C >> 2;
    const float4* x = reinterpret_cast<const float4*>(a.in + (uint64_t)r * a.C);
    float4 v[NV];
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const uint32_t c = lane + 32u * j;
        v[j] = c < n4 ? x[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    }
    const float mu = warp_sum(s) / (float)a.C;
    float q = 0.0f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        if (lane + 32u * j < n4) {
            const float d0 = v[j].x - mu, d1 = v[j].y - mu, d2 = v[j].z - mu, d3 = v[j].w - mu;
            q += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
        }
    }
    const float inv = rsqrtf(warp_sum(q) / (float)a.C + a.eps);
    const uint2* g = reinterpret_cast<const uint2*>(weight_ptr(*d, a.g_off));
    const uint2* b = reinterpret_cast<const uint2*>(weight_ptr(*d, a.b_off));
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const uint32_t c = lane + 32u * j;
        if (c < n4) {
            const uint2 gv = g[c], bv = b[c];
            float4 y;
            y.x = (v[j].x - mu) * inv * __uint_as_float(gv.x << 16) + __uint_as_float(bv.x << 16);
            y.y = (v[j].y - mu) * inv * __uint_as_float(gv.x & 0xffff0000u) + __uint_as_float(bv.x & 0xffff0000u);
            y.z = (v[j].z - mu) * inv * __uint_as_float(gv.y << 16) + __uint_as_float(bv.y << 16);
            y.w = (v[j].w - mu) * inv * __uint_as_float(gv.y & 0xffff0000u) + __uint_as_float(bv.y & 0xffff0000u);
            if (a.out_f32) reinterpret_cast<float4*>(a.out_f32 + (uint64_t)r * a.C)[c] = y;
            if (a.out_bf16) {
                const uint32_t lo = (uint32_t)f32_to_bf16(y.x) | ((uint32_t)f32_to_bf16(y.y) << 16);
                const uint32_t hi = (uint32_t)f32_to_bf16(y.z) | ((uint32_t)f32_to_bf16(y.w) << 16);
                reinterpret_cast<uint2*>(a.out_bf16 + (uint64_t)r * a.C)[c] = make_uint2(lo, hi);
            }
        }
    }
}

void launch_layernorm(cudaStream_t s, const DevDesc* d, Wait w, const LnArgs& a) {
    const unsigned grid = (a.rows + 3) / 4;
    const uint32_t nv = (a.C / 4 + 31) / 32;
    if (nv <= 2) launch_pdl(PDL_LN, k_layernorm<2>, dim3(grid), dim3(128), 0, s, d, w, a);
    else if (nv <= 4) launch_pdl(PDL_LN, k_layernorm<4>, dim3(grid), dim3(128), 0, s, d, w, a);
    else if (nv <= 6) launch_pdl(PDL_LN, k_layernorm<6>, dim3(grid), dim3(128), 0, s, d, w, a);
    else if (nv <= 8) launch_pdl(PDL_LN, k_layernorm<8>, dim3(grid), dim3(128), 0, s, d, w, a);
    else if (nv <= 13) launch_pdl(PDL_LN, k_layernorm<13>, dim3(grid), dim3(128), 0, s, d, w, a);
    else launch_pdl(PDL_LN, k_layernorm<16>, dim3(grid), dim3(128), 0, s, d, w, a);
}

// ------------------------------------------------------------------------------------------
// GEMV (rows <= 8): one warp per output feature, 16-B coalesced weight loads along K,
// x staged once per CTA in shared memory as fp32.  HBM-bound: bytes = N·K·2.
// ------------------------------------------------------------------------------------------
constexpr int kGemvMaxRows = 8;

template <int R>
__global__ void __launch_bounds__(256) k_gemv(const DevDesc* __restrict__ d, Wait w, GemvArgs a) {
    extern __shared__ float xs[];  // [R][K]
    pdl_wait();
    for (uint32_t i = threadIdx.x; i < R * a.K; i += blockDim.x) {
        const uint32_t r = i / a.K, k = i - r * a.K;
        const uint64_t src = (uint64_t)(a.r0 + r) * a.ldx + k;
        xs[i] = r >= a.rows ? 0.0f : a.x_bf16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(a.x)[src])
                         : reinterpret_cast<const float*>(a.x)[src];
    }
    if (threadIdx.x == 0) wait_ready_thread(w);
    __syncthreads();  // publishes xs and the acquired weights to the CTA
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gwarp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    const uint8_t* wmat = weight_ptr(*d, a.w_off);
    const uint16_t* bvec = a.has_bias ? reinterpret_cast<const uint16_t*>(weight_ptr(*d, a.b_off)) : nullptr;
    const uint32_t k8n = a.K >> 3;
    for (uint32_t o = gwarp; o < a.N; o += nwarps) {
        const uint4* wr = reinterpret_cast<const uint4*>(wmat + (uint64_t)o * a.K * 2);
        float acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0f;
#pragma unroll 4
        for (uint32_t k8 = lane; k8 < k8n; k8 += 32) {
            const uint4 wv = __ldcg(wr + k8);
            const uint32_t wu[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const float w0 = __uint_as_float(wu[h] << 16), w1 = __uint_as_float(wu[h] & 0xffff0000u);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float* xr = xs + r * a.K + k8 * 8 + 2 * h;
                    acc[r] = fmaf(w0, xr[0], acc[r]);
                    acc[r] = fmaf(w1, xr[1], acc[r]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = warp_sum(acc[r]);
        if (lane < R && lane < a.rows) {
            float v = 0.0f;
#pragma unroll
            for (int r = 0; r < R; ++r) v = (r == (int)lane) ? acc[r] : v;
            const uint64_t oi = (uint64_t)lane * a.N + o;
            if (bvec) v += bf16_to_f32(bvec[o]);
            if (a.res) v += a.res_bf16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(a.res)[oi])
                                       : reinterpret_cast<const float*>(a.res)[oi];
            v = apply_act(a.act, v);
            if (a.out_bf16) reinterpret_cast<uint16_t*>(a.out)[oi] = f32_to_bf16(v);
            else reinterpret_cast<float*>(a.out)[oi] = v;
            if (a.out2) a.out2[oi] = f32_to_bf16(v);
        }
    }
}

void launch_gemv(cudaStream_t s, const DevDesc* d, Wait w, const GemvArgs& a) {
    const size_t smem = sizeof(float) * a.K * (a.rows <= 1 ? 1 : kGemvMaxRows);
    int ctas = (int)((a.N + 7) / 8);
    if (ctas > 148 * 4) ctas = 148 * 4;
    if (ctas < 1) ctas = 1;
    if (a.rows <= 1) {
        launch_pdl(PDL_GEMV, k_gemv<1>, dim3(ctas), dim3(256), smem, s, d, w, a);
    } else {
        launch_pdl(PDL_GEMV, k_gemv<kGemvMaxRows>, dim3(ctas), dim3(256), smem, s, d, w, a);
    }
}

// ------------------------------------------------------------------------------------------
// ATTENTION core.  One CTA per (head, 16 query rows), 8 warps x 2 rows.  K and V of the head
// are staged in shared memory as bf16 (K rows padded by 4 B: conflict-free column reads);
// scores, softmax and the P·V accumulation are fp32 (SURVEY §8c reading #1).
// ------------------------------------------------------------------------------------------
constexpr int kAttnRows = 16;

__global__ void __launch_bounds__(256) k_attention(AttnArgs a) {
    extern __shared__ __align__(16) uint8_t sm_attn[];
    pdl_wait();
    const uint32_t T = a.T, dh = a.dh, D = a.H * dh, W3 = 3 * D;
    const uint32_t h = blockIdx.x, t0 = blockIdx.y * kAttnRows;
    const uint32_t nwarp = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tend = min(T, t0 + kAttnRows);
    const uint32_t kend = a.causal ? tend : T;  // keys this CTA needs
    const uint32_t kst = dh / 2 + 1;           // K row stride in 32-bit words (padded)
    uint32_t* Ks = reinterpret_cast<uint32_t*>(sm_attn);     // [T][kst]   bf16x2
    uint32_t* Vs = Ks + ((T * kst + 3) & ~3u);                // [T][dh/2]  bf16x2, 16-B aligned (uint4 stores)
    float* Ps = reinterpret_cast<float*>(Vs + T * (dh / 2));  // [nwarp][T]
    float* Qs = Ps + nwarp * T;                               // [nwarp][dh]
    const uint32_t dh8 = dh / 8;
    for (uint32_t i = threadIdx.x; i < kend * dh8; i += blockDim.x) {
        const uint32_t j = i / dh8, c8 = i - j * dh8;
        const uint16_t* row = a.qkv + (uint64_t)j * W3 + h * dh + c8 * 8;
        const uint4 kv = *reinterpret_cast<const uint4*>(row + D);
        const uint4 vv = *reinterpret_cast<const uint4*>(row + 2 * D);
        uint32_t* kd = Ks + j * kst + c8 * 4;
        kd[0] = kv.x; kd[1] = kv.y; kd[2] = kv.z; kd[3] = kv.w;
        *reinterpret_cast<uint4*>(Vs + j * (dh / 2) + c8 * 4) = vv;
    }
    __syncthreads();
    const float scale = rsqrtf((float)dh);
    float* P = Ps + warp * T;
    float* q = Qs + warp * dh;
    for (uint32_t t = t0 + warp; t < tend; t += nwarp) {
        for (uint32_t c = lane; c < dh; c += 32) q[c] = bf16_to_f32(a.qkv[(uint64_t)t * W3 + h * dh + c]) * scale;
        __syncwarp();
        const uint32_t jmax = a.causal ? t + 1 : T;
        float mx = -INFINITY;
        for (uint32_t j = lane; j < jmax; j += 32) {
            const uint32_t* kr = Ks + j * kst;
            float s0 = 0.0f, s1 = 0.0f;
            for (uint32_t c2 = 0; c2 < dh / 2; ++c2) {
                const uint32_t k2 = kr[c2];
                const float2 q2 = *reinterpret_cast<const float2*>(q + 2 * c2);
                s0 = fmaf(q2.x, __uint_as_float(k2 << 16), s0);
                s1 = fmaf(q2.y, __uint_as_float(k2 & 0xffff0000u), s1);
            }
            const float sc = s0 + s1;
            P[j] = sc;
            mx = fmaxf(mx, sc);
        }
        mx = warp_max(mx);
        float z = 0.0f;
        for (uint32_t j = lane; j < jmax; j += 32) {
            const float e = __expf(P[j] - mx);
            P[j] = e;
            z += e;
        }
        z = warp_sum(z);
        __syncwarp();
        const float iz = 1.0f / z;
        for (uint32_t c2 = lane; c2 < dh / 2; c2 += 32) {
            float o0 = 0.0f, o1 = 0.0f;
            for (uint32_t j = 0; j < jmax; ++j) {
                const float pj = P[j];
                const uint32_t v2 = Vs[j * (dh / 2) + c2];
                o0 = fmaf(pj, __uint_as_float(v2 << 16), o0);
                o1 = fmaf(pj, __uint_as_float(v2 & 0xffff0000u), o1);
            }
            const uint32_t pk = (uint32_t)f32_to_bf16(o0 * iz) | ((uint32_t)f32_to_bf16(o1 * iz) << 16);
            *reinterpret_cast<uint32_t*>(a.out + (uint64_t)t * D + h * dh + 2 * c2) = pk;
        }
        __syncwarp();
    }
}

void launch_attention(cudaStream_t s, const AttnArgs& a) {
    const int threads = 256, nwarp = threads / 32;
    const size_t smem = 4 * (((a.T * (a.dh / 2 + 1) + 3) & ~3u) + a.T * (a.dh / 2)) + sizeof(float) * (nwarp * a.T + nwarp * a.dh);
    dim3 grid(a.H, (a.T + kAttnRows - 1) / kAttnRows);
    launch_pdl(PDL_ATTN, k_attention, grid, dim3(threads), smem, s, a);
}

// ------------------------------------------------------------------------------------------
// IM2COL (NHWC bf16 -> [P·Q][Kpad] bf16, k = (r·S + s)·C + c, zero padding / tail)
// ------------------------------------------------------------------------------------------
__global__ void k_im2col_vec8(Im2colArgs a) {  // C % 8 == 0: one 16-B chunk per thread
    pdl_wait();
    const uint32_t k8n = a.Kpad >> 3;
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (uint64_t)a.P * a.Q * k8n) return;
    const uint32_t pq = (uint32_t)(idx / k8n), k = (uint32_t)(idx - (uint64_t)pq * k8n) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (k < a.K) {
        const uint32_t rs = k / a.C, c = k - rs * a.C, r = rs / a.S, s = rs - r * a.S;
        const uint32_t p = pq / a.Q, q = pq - p * a.Q;
        const int ih = (int)(p * a.stride) - (int)a.pad + (int)r, iw = (int)(q * a.stride) - (int)a.pad + (int)s;
        if (ih >= 0 && iw >= 0 && ih < (int)a.H && iw < (int)a.W)
            v = *reinterpret_cast<const uint4*>(a.in + ((uint64_t)ih * a.W + iw) * a.C + c);
    }
    *reinterpret_cast<uint4*>(a.out + (uint64_t)pq * a.Kpad + k) = v;
}

__global__ void k_im2col_scalar(Im2colArgs a) {
    pdl_wait();
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (uint64_t)a.P * a.Q * a.Kpad) return;
    const uint32_t pq = (uint32_t)(idx / a.Kpad), k = (uint32_t)(idx - (uint64_t)pq * a.Kpad);
    uint16_t v = 0;
    if (k < a.K) {
        const uint32_t rs = k / a.C, c = k - rs * a.C, r = rs / a.S, s = rs - r * a.S;
        const uint32_t p = pq / a.Q, q = pq - p * a.Q;
        const int ih = (int)(p * a.stride) - (int)a.pad + (int)r, iw = (int)(q * a.stride) - (int)a.pad + (int)s;
        if (ih >= 0 && iw >= 0 && ih < (int)a.H && iw < (int)a.W) v = a.in[((uint64_t)ih * a.W + iw) * a.C + c];
    }
    a.out[idx] = v;
}

void launch_im2col(cudaStream_t s, const Im2colArgs& a) {
    if (a.C % 8 == 0) {
        const uint64_t n = (uint64_t)a.P * a.Q * (a.Kpad / 8);
        launch_pdl(PDL_IM2COL, k_im2col_vec8, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, a);
    } else {
        const uint64_t n = (uint64_t)a.P * a.Q * a.Kpad;
        launch_pdl(PDL_IM2COL, k_im2col_scalar, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, a);
    }
}

// ------------------------------------------------------------------------------------------
// pooling (NHWC bf16)
// ------------------------------------------------------------------------------------------
__global__ void k_maxpool(PoolArgs a) {
    pdl_wait();
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (uint64_t)a.P * a.Q * a.C) return;
    const uint32_t c = (uint32_t)(idx % a.C), pq = (uint32_t)(idx / a.C), p = pq / a.Q, q = pq - p * a.Q;
    float m = -INFINITY;
    for (uint32_t r = 0; r < a.k; ++r)
        for (uint32_t s = 0; s < a.k; ++s) {
            const int ih = (int)(p * a.stride) - (int)a.pad + (int)r, iw = (int)(q * a.stride) - (int)a.pad + (int)s;
            if (ih < 0 || iw < 0 || ih >= (int)a.H || iw >= (int)a.W) continue;
            m = fmaxf(m, bf16_to_f32(a.in[((uint64_t)ih * a.W + iw) * a.C + c]));
        }
    a.out[idx] = f32_to_bf16(m);
}

void launch_maxpool(cudaStream_t s, const PoolArgs& a) {
    const uint64_t n = (uint64_t)a.P * a.Q * a.C;
    launch_pdl(PDL_POOL, k_maxpool, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, a);
}

__global__ void k_avgpool(PoolArgs a) {
    pdl_wait();
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= a.C) return;
    const uint32_t hw = a.H * a.W;
    float s = 0.0f;
    for (uint32_t i = 0; i < hw; ++i) s += bf16_to_f32(a.in[(uint64_t)i * a.C + c]);
    a.out_f32[c] = s / (float)hw;
}

void launch_avgpool(cudaStream_t s, const PoolArgs& a) {
    launch_pdl(PDL_POOL, k_avgpool, dim3((a.C + 127) / 128), dim3(128), 0, s, a);
}

void init_ops_attrs() {
    cudaFuncSetAttribute(k_gemv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_gemv<kGemvMaxRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

}  // namespace fsw
