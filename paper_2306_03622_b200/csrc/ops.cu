// ops.cu — the non-GEMM layer kernels (HBM/latency-bound at batch 1): embedding gather,
// LayerNorm, GEMV (M = 1 linears: MLP, pooler, fc, LM head), attention core, im2col,
// max/avg pooling.  Each kernel that reads weights first waits on its layer's ready
// counter (device.cuh), which is how "each layer's kernels start as soon as its weights
// land" (BASELINE.json north_star).
#include "device.cuh"
#include "attn_core.cuh"

namespace fsw {

// programmatic-launch trigger at kernel entry for LayerNorm (bit 0) / attention (bit 1): FSW_EARLY_TRIGGER
static __device__ int g_early_trigger = 0;


// ------------------------------------------------------------------------------------------
// EMBED: out[t][c] = Σ_j table_j[row_j(t)][c]   (fp32 sum of bf16 rows)
// ------------------------------------------------------------------------------------------
__global__ void k_embed(const DevDesc* __restrict__ d, Wait w, EmbedArgs a) {
    TraceExit tx(w.trace, w.layer);
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
// fp32 two-pass statistics (mean, then centred variance), 8-B vector loads of γ/β.  γ/β are
// weights (ordered by the ready counter, not by PDL): they are loaded before griddepcontrol.wait,
// so their round trip overlaps the previous kernel instead of following the statistics.
// ------------------------------------------------------------------------------------------
template <int NV>
__global__ void __launch_bounds__(128) k_layernorm(const DevDesc* __restrict__ d, Wait w, LnArgs a) {
    TraceExit tx(w.trace, w.layer);
    if (g_early_trigger & 1) pdl_trigger();  // the successor GEMM sets up and loads its weights during this LN
    wait_ready_cta(w);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t r = blockIdx.x * (blockDim.x >> 5) + warp;
    const uint32_t n4 = a.C >> 2;
    uint2 gv[NV], bv[NV];
    {
        const uint2* g = reinterpret_cast<const uint2*>(weight_ptr(*d, a.g_off));
        const uint2* b = reinterpret_cast<const uint2*>(weight_ptr(*d, a.b_off));
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const uint32_t c = lane + 32u * j;
            gv[j] = c < n4 ? g[c] : make_uint2(0u, 0u);
            bv[j] = c < n4 ? b[c] : make_uint2(0u, 0u);
        }
    }
    pdl_wait();
    if (r >= a.rows) return;
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
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const uint32_t c = lane + 32u * j;
        if (c < n4) {
            float4 y;
            y.x = (v[j].x - mu) * inv * __uint_as_float(gv[j].x << 16) + __uint_as_float(bv[j].x << 16);
            y.y = (v[j].y - mu) * inv * __uint_as_float(gv[j].x & 0xffff0000u) + __uint_as_float(bv[j].x & 0xffff0000u);
            y.z = (v[j].z - mu) * inv * __uint_as_float(gv[j].y << 16) + __uint_as_float(bv[j].y << 16);
            y.w = (v[j].w - mu) * inv * __uint_as_float(gv[j].y & 0xffff0000u) + __uint_as_float(bv[j].y & 0xffff0000u);
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
    TraceExit tx(w.trace, w.layer);
    extern __shared__ float xs[];  // [R][K]
    pdl_wait();
    for (uint32_t i = threadIdx.x; i < R * a.K; i += blockDim.x) {
        const uint32_t r = i / a.K, k = i - r * a.K;
        const uint64_t src = (uint64_t)(a.r0 + r) * a.ldx + k;
        xs[i] = r >= a.rows ? 0.0f : a.x_bf16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(a.x)[src])
                         : reinterpret_cast<const float*>(a.x)[src];
    }
    if (threadIdx.x == 0) {
        wait_ready_thread(w);
        FSW_TRACE_MAX(w.trace, w.layer, 1, globaltimer());
    }
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
    TraceExit tx(a.trace, a.layer);
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

// ------------------------------------------------------------------------------------------
// ATTENTION on the tensor cores for the batch-1 shapes of the paper's transformers (T <= 128,
// dh in {16, 32, 64, 128}).  One CTA per (head, 64 query rows), 4 warps x 16 rows.  K and V of
// the keys the CTA needs are staged in shared memory (rows padded to dh + 8 elements: the
// 32-bit fragment loads and ldmatrix are bank-conflict free).  Per warp, everything stays in
// registers: S = Q·Kᵀ by mma.sync m16n8k16 (bf16 in, fp32 accumulate; Q fragments loaded straight
// from the qkv rows), the scale, causal / length mask and softmax in fp32 (row max and sum over
// the lane quad), P rounded to bf16 and fed back as the A operand of O = P·V (V fragments by
// ldmatrix.trans), O / Σ stored bf16.  At T = 128 the whole problem is ~10 µs of latency chains on
// the old scalar kernel; the warp-level MMA keeps every dependent step in registers.  (tcgen05 would
// need a TMEM allocation and mbarrier round trips per tile for a 16x128 problem: no gain here.)
// ------------------------------------------------------------------------------------------
constexpr int kAttnMmaRows = 64;

template <int DH>
__global__ void __launch_bounds__(128) k_attention_mma(AttnArgs a) {
    TraceExit tx(a.trace, a.layer);
    constexpr int KS = DH / 16;        // k-steps of Q·Kᵀ
    constexpr int NO = DH / 8;         // n-tiles of O
    constexpr int NS = kAttnMmaMaxT / 8;  // n-tiles of S (keys)
    constexpr int LD = DH + 8;         // smem row stride (elements)
    extern __shared__ __align__(16) uint16_t sm_kv[];
    uint16_t* Ks = sm_kv;                           // [kpad][LD]
    pdl_wait();
    const uint32_t T = a.T, D = a.H * DH, W3 = 3 * D;
    const uint32_t h = blockIdx.x, r0 = blockIdx.y * kAttnMmaRows;
    const uint32_t kend = a.causal ? min(T, r0 + kAttnMmaRows) : T;
    const uint32_t kpad = (kend + 15) & ~15u;
    uint16_t* Vs = Ks + kpad * LD;                  // [kpad][LD]
    // stage K and V rows [0, kpad) (rows >= T zero), 16-B chunks
    constexpr uint32_t C8 = DH / 8;
    for (uint32_t i = threadIdx.x; i < kpad * C8; i += blockDim.x) {
        const uint32_t j = i / C8, c = (i - j * C8) * 8;
        uint4 kv = make_uint4(0, 0, 0, 0), vv = kv;
        if (j < kend) {
            const uint16_t* row = a.qkv + (uint64_t)j * W3 + h * DH + c;
            kv = *reinterpret_cast<const uint4*>(row + D);
            vv = *reinterpret_cast<const uint4*>(row + 2 * D);
        }
        *reinterpret_cast<uint4*>(Ks + j * LD + c) = kv;
        *reinterpret_cast<uint4*>(Vs + j * LD + c) = vv;
    }
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const uint32_t q0 = r0 + warp * 16;
    // Q fragments (A operand, row-major 16 x DH) straight from the qkv rows q0+g and q0+g+8
    uint32_t qa[KS][4];
    {
        const uint32_t ra = q0 + g, rb = q0 + g + 8;
        const uint16_t* pa = a.qkv + (uint64_t)ra * W3 + h * DH;
        const uint16_t* pb = a.qkv + (uint64_t)rb * W3 + h * DH;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            const uint32_t c = kk * 16 + 2 * t;
            qa[kk][0] = ra < T ? *reinterpret_cast<const uint32_t*>(pa + c) : 0u;
            qa[kk][1] = rb < T ? *reinterpret_cast<const uint32_t*>(pb + c) : 0u;
            qa[kk][2] = ra < T ? *reinterpret_cast<const uint32_t*>(pa + c + 8) : 0u;
            qa[kk][3] = rb < T ? *reinterpret_cast<const uint32_t*>(pb + c + 8) : 0u;
        }
    }
    __syncthreads();
    if (q0 >= T) return;  // after the barrier: every thread helped stage
    // keys this warp needs: all (non-causal) or up to its last row (causal)
    const uint32_t kw = a.causal ? min(kend, q0 + 16) : kend;
    const uint32_t nst = (kw + 7) / 8;
    const float scale = rsqrtf((float)DH);
    float s[NS][4];
#pragma unroll
    for (int n = 0; n < NS; ++n) {
        s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.0f;
        if ((uint32_t)n < nst) {
            const uint16_t* kr = Ks + (n * 8 + g) * LD + 2 * t;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk)
                mma_bf16_16816(s[n], qa[kk], *reinterpret_cast<const uint32_t*>(kr + kk * 16),
                               *reinterpret_cast<const uint32_t*>(kr + kk * 16 + 8));
        }
    }
    // scale, mask, row max / sum (rows q0+g: elements 0,1; q0+g+8: elements 2,3)
    const uint32_t ra = q0 + g, rb = ra + 8;
    float mxa = -INFINITY, mxb = -INFINITY;
#pragma unroll
    for (int n = 0; n < NS; ++n) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t j = n * 8 + 2 * t + (e & 1), r = e < 2 ? ra : rb;
            const bool ok = (uint32_t)n < nst && j < T && (!a.causal || j <= r);
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
    float za = 0.0f, zb = 0.0f;
#pragma unroll
    for (int n = 0; n < NS; ++n) {
        s[n][0] = __expf(s[n][0] - mxa);
        s[n][1] = __expf(s[n][1] - mxa);
        s[n][2] = __expf(s[n][2] - mxb);
        s[n][3] = __expf(s[n][3] - mxb);
        za += s[n][0] + s[n][1];
        zb += s[n][2] + s[n][3];
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
        za += __shfl_xor_sync(0xffffffffu, za, o);
        zb += __shfl_xor_sync(0xffffffffu, zb, o);
    }
    // O = P·V: the S accumulators of key tiles 2kk, 2kk+1 are the A fragment of k-step kk
    float o[NO][4];
#pragma unroll
    for (int n = 0; n < NO; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.0f;
    const uint32_t nkk = (nst + 1) / 2;
#pragma unroll
    for (int kk = 0; kk < NS / 2; ++kk) {
        if ((uint32_t)kk >= nkk) break;
        const uint32_t pa[4] = {pack_bf16x2(s[2 * kk][0], s[2 * kk][1]), pack_bf16x2(s[2 * kk][2], s[2 * kk][3]),
                                pack_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                                pack_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
        // ldmatrix.x4.trans: matrices (keys kk·16 + 0..7 | 8..15) x (cols n·8 | (n+1)·8)
        const uint32_t mi = lane >> 3, rr = lane & 7;
#pragma unroll
        for (int n = 0; n < NO; n += 2) {
            const uint16_t* p = Vs + (kk * 16 + (mi & 1) * 8 + rr) * LD + (n + (mi >> 1)) * 8;
            uint32_t b0, b1, b2, b3;
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                         : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                         : "r"((uint32_t)__cvta_generic_to_shared(p)));
            mma_bf16_16816(o[n], pa, b0, b1);
            if (n + 1 < NO) mma_bf16_16816(o[n + 1], pa, b2, b3);
        }
    }
    const float ia = 1.0f / za, ib = 1.0f / zb;
#pragma unroll
    for (int n = 0; n < NO; ++n) {
        const uint32_t c = h * DH + n * 8 + 2 * t;
        if (ra < T) *reinterpret_cast<uint32_t*>(a.out + (uint64_t)ra * D + c) = pack_bf16x2(o[n][0] * ia, o[n][1] * ia);
        if (rb < T) *reinterpret_cast<uint32_t*>(a.out + (uint64_t)rb * D + c) = pack_bf16x2(o[n][2] * ib, o[n][3] * ib);
    }
}

template <int DH>
__global__ void __launch_bounds__(128) k_attention_mma2(AttnArgs a) {
    TraceExit tx(a.trace, a.layer);
    extern __shared__ __align__(16) uint16_t sm_kv2[];
    if (g_early_trigger & 2) pdl_trigger();  // the O-projection sets up and loads its weights during attention
    pdl_wait();
    attn_split_core<DH>(a, blockIdx.x, blockIdx.y * kAttnSplitRows, sm_kv2, threadIdx.x, []() { __syncthreads(); });
}

template <int DH>
static size_t attn2_smem(uint32_t T) {
    const uint32_t kpad = (T + 15) & ~15u;
    const uint32_t kper = (((kpad + kAttnSplitWarps - 1) / kAttnSplitWarps) + 15) & ~15u;
    return 2ull * kper * kAttnSplitWarps * (DH + 8) * sizeof(uint16_t) +
           sizeof(float) * (kAttnSplitWarps * 16 * DH + 2 * kAttnSplitWarps * 16);
}

template <int DH>
static void launch_attention_mma2(cudaStream_t s, const AttnArgs& a) {
    dim3 grid(a.H, (a.T + kAttnSplitRows - 1) / kAttnSplitRows);
    launch_pdl(PDL_ATTN, k_attention_mma2<DH>, grid, dim3(32 * kAttnSplitWarps), attn2_smem<DH>(a.T), s, a);
}

template <int DH>
static void launch_attention_mma(cudaStream_t s, const AttnArgs& a) {
    const uint32_t kmax = (a.T + 15) & ~15u;  // keys staged by the CTA that needs the most
    const size_t smem = 2ull * kmax * (DH + 8) * sizeof(uint16_t);
    dim3 grid(a.H, (a.T + kAttnMmaRows - 1) / kAttnMmaRows);
    launch_pdl(PDL_ATTN, k_attention_mma<DH>, grid, dim3(128), smem, s, a);
}

void launch_attention(cudaStream_t s, const AttnArgs& a) {
    static const bool scalar = getenv("FSW_ATTN_SCALAR") != nullptr;  // A/B hooks: the scalar kernel,
    static const bool nosplit = getenv("FSW_ATTN_NOSPLIT") != nullptr; // the MMA kernel without key split
    if (a.T <= (uint32_t)kAttnMmaMaxT && !scalar && !nosplit) {
        switch (a.dh) {
            case 16: return launch_attention_mma2<16>(s, a);
            case 32: return launch_attention_mma2<32>(s, a);
            case 64: return launch_attention_mma2<64>(s, a);
            case 128: return launch_attention_mma2<128>(s, a);
            default: break;
        }
    }
    if (a.T <= (uint32_t)kAttnMmaMaxT && !scalar) {
        switch (a.dh) {
            case 16: return launch_attention_mma<16>(s, a);
            case 32: return launch_attention_mma<32>(s, a);
            case 64: return launch_attention_mma<64>(s, a);
            case 128: return launch_attention_mma<128>(s, a);
            default: break;
        }
    }
    const int threads = 256, nwarp = threads / 32;
    const size_t smem = 4 * (((a.T * (a.dh / 2 + 1) + 3) & ~3u) + a.T * (a.dh / 2)) + sizeof(float) * (nwarp * a.T + nwarp * a.dh);
    dim3 grid(a.H, (a.T + kAttnRows - 1) / kAttnRows);
    launch_pdl(PDL_ATTN, k_attention, grid, dim3(threads), smem, s, a);
}

// ------------------------------------------------------------------------------------------
// IM2COL (NHWC bf16 -> [P·Q][Kpad] bf16, k = (r·S + s)·C + c, zero padding / tail)
// ------------------------------------------------------------------------------------------
__global__ void k_im2col_vec8(Im2colArgs a) {  // C % 8 == 0: one 16-B chunk per thread
    TraceExit tx(a.trace, a.layer);
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
    TraceExit tx(a.trace, a.layer);
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
    TraceExit tx(a.trace, a.layer);
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
    TraceExit tx(a.trace, a.layer);
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
    {  // LayerNorm (bit 0) and attention (bit 1) let their successor launch at entry (FSW_EARLY_TRIGGER, A/B hook;
       // default both: resident BERT-base 0.562 -> 0.502 ms, profiles/r02/gemm/ws_sweep.txt)
        static const int early = getenv("FSW_EARLY_TRIGGER") ? atoi(getenv("FSW_EARLY_TRIGGER")) : 3;
        cudaMemcpyToSymbol(g_early_trigger, &early, sizeof early);
    }
    cudaFuncSetAttribute(k_gemv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_gemv<kGemvMaxRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_attention_mma<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_attention_mma<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_attention_mma<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_attention_mma<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_attention_mma2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_attention_mma2<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_attention_mma2<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_attention_mma2<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}


}  // namespace fsw
