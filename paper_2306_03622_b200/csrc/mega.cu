// mega.cu — k_mega: the persistent transformer kernel.  ONE launch runs every layer of a BERT / GPT-2
// style layer table (EMBED, LAYERNORM, LINEAR, ATTENTION) on one CTA per SM, instead of one kernel
// per layer op (~86 launches for BERT-base, each paying its setup, first-data latency and epilogue
// tail: resident BERT-base measured 52 us per encoder layer against ~2 us of weight bytes at HBM rate,
// profiles/r02/timeline_*).  It is the same flag-gated pipelined execution: every op
// waits for its layer's ready counter before it touches weights, so on a cold invoke it runs behind
// the swap exactly like the per-op kernels.
//
// Work: op i of the table is n_tasks tasks; CTA c takes tasks c, c + grid, ... of every op, in op
// order.  Dependencies are op-level: a task reads activations only after op i − 1 has counted all of
// its tasks done (red.release on a per-op counter, ld.acquire by the consumer; chained, so every
// earlier op is done too).  Weights are not activations: the producer warp streams the weight tiles
// of a CTA's next GEMM task into the shared-memory ring BEFORE that dependency resolves, so the HBM
// weight stream of op i overlaps the tail of op i − 1.
//
// Warp roles (192 threads): warp 0 = producer (one thread: weight bulk copies of the pre-tiled layout,
// DESIGN.md §4, and TMA loads of the activation tile), warp 1 = tcgen05.mma issuer (one thread),
// warps 2-5 = epilogue of GEMM tasks (TMEM lane quarter = warp mod 4) and the CUDA-core tasks
// (embedding gather, LayerNorm, attention core, small-M GEMV) with named barrier 1.
//
// GEMM tiles are swap-AB: the UMMA M operand is 128 weight rows, N is tt tokens (16 / 32 / 64), so a
// task streams 128·K_range·2 weight bytes and tt·K_range·2 activation bytes; D = [weight row][token]
// sits in one of two TMEM buffers (the MMA of the next task overlaps this task's epilogue).  Split-K
// tasks write fp32 partials; the last split to arrive sums them in split order (deterministic).
#include "attn_core.cuh"
#include "umma.cuh"

namespace fsw {

constexpr int kMkThreads = 192, kMkStages = 5;
constexpr uint32_t kMkW = 128 * 128;               // one weight k-tile: 128 rows x 64 k bf16
constexpr uint32_t kMkA = kMkTT * 128;             // one activation k-tile: <= 64 tokens x 64 k bf16
constexpr uint32_t kMkStage = kMkW + kMkA;
constexpr uint32_t kMkCompute = 56 * 1024;         // attention (dh <= 64, T <= 128) / GEMV staging
constexpr uint32_t kMkRing = kMkStages * kMkStage;
constexpr uint32_t kMkTmemCols = 2 * kMkTT;        // two accumulator buffers
constexpr uint64_t kMkWatchdogNs = 4ull * 1000 * 1000 * 1000;

static_assert(sizeof(MkOp) <= 1024, "MkOp must fit its shared-memory slot");
constexpr uint32_t kMkOpSmem = 1024;  // the epilogue warps' copy of the current op (sizeof(MkOp) <= 1 KiB)
size_t mega_smem_bytes() { return 1024 + kMkRing + kMkCompute + kMkOpSmem + 256; }

// Phase stamps (FSW_MEGA_STAMPS=1, tools/mega_phases.py): per (op, CTA) the %globaltimer of
// [0] producer: dependency resolved (activation loads issued), [1] MMA: first stage full, [2] MMA: last
// commit, [3] epilogue: accumulator ready, [4] epilogue: split-K partials published / output stored,
// [5] task done (counter released), [6] compute task: dependency resolved, [7] compute task: body done.
__device__ unsigned long long* g_mk_stamp = nullptr;
__device__ __forceinline__ void mk_stamp(uint32_t op, uint32_t k) {
    unsigned long long* p = g_mk_stamp;
    if (p) p[((uint64_t)op * gridDim.x + blockIdx.x) * 8 + k] = globaltimer();
}
void set_mega_stamps(unsigned long long* p) { cudaMemcpyToSymbol(g_mk_stamp, &p, sizeof p); }

__device__ __forceinline__ void mk_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// mbarrier wait with a watchdog (a lost arrival must end the kernel, not hang the GPU)
__device__ __forceinline__ void mk_wait(uint64_t* b, uint32_t parity, DevCtl* ctl) {
    const uint32_t a = smem_u32(b);
    uint32_t ok = 0, n = 0;
    uint64_t t0 = 0;
    for (;;) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(a), "r"(parity) : "memory");
        if (ok) return;
        if (++n == 64) t0 = globaltimer();
        if (n > 64 && (n & 255) == 0 && globaltimer() - t0 > kMkWatchdogNs) {
            atomicExch(&ctl->err, 4);
            return;
        }
    }
}

// Op completion (DESIGN.md §5 k_mega): every task adds 1 to its op's counter (acq_rel); the task that
// brings it to n_tasks then publishes "ops 0..i are done" into every CTA's own epoch word (a fence, then
// one store per CTA), so each CTA polls a private 128-B line instead of 300 threads polling one counter
// (measured: that polling saturated the counter's L2 slice and slowed every load that hashed to it, the
// split-K reductions 10-25 us).  Counters and epoch words are 128 B apart (kMkLine u32).
constexpr uint32_t kMkLine = 32;
__device__ __forceinline__ void mk_wait_op(const uint32_t* epoch, uint32_t dep, DevCtl* ctl) {
    const uint32_t need = dep + 1;
    if (ld_acquire_gpu(epoch) >= need) return;
    const uint64_t t0 = globaltimer();
    uint32_t ns = 32;
    while (ld_acquire_gpu(epoch) < need) {
        __nanosleep(ns);
        if (ns < 128) ns <<= 1;
        if (globaltimer() - t0 > kWatchdogNs) {
            atomicExch(&ctl->err, 4);
            return;
        }
    }
}

__device__ __forceinline__ void mk_done(uint32_t* cnt, uint32_t n_tasks, uint32_t* epochs, uint32_t op) {
    __threadfence();
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    if (old + 1 == n_tasks) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (uint32_t c = 0; c < gridDim.x; ++c)
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(epochs + (uint64_t)c * kMkLine), "r"(op + 1) : "memory");
    }
}

struct MkTile {
    uint32_t r, j, z, kt0, nk, rows_w;
};
__device__ __forceinline__ MkTile mk_tile(const MkOp& op, uint32_t g) {
    MkTile t;
    t.z = g % op.splits;
    const uint32_t rem = g / op.splits;
    t.j = rem % op.n_tt;
    t.r = rem / op.n_tt;
    t.kt0 = t.z * op.kt_per;
    t.nk = min(op.gemm.K / 64, t.kt0 + op.kt_per) - t.kt0;
    t.rows_w = min(128u, op.gemm.n_pad - t.r * 128);
    return t;
}

// Activation with the transcendental cases out of line: k_mega is one large kernel whose warps run
// different code at once, so every inlined erf / tanh expansion costs instruction-cache space (measured:
// the inlined apply_act made a 4-unit epilogue pass 7 us instead of 2.8, even for act = NONE).
__device__ __noinline__ float mk_act_slow(int act, float x) { return apply_act(act, x); }
__device__ __forceinline__ float mk_act(int act, float x) {
    if (act == FSW_ACT_NONE) return x;
    if (act == FSW_ACT_RELU) return fmaxf(x, 0.0f);
    return mk_act_slow(act, x);
}

// ---- GEMM epilogue from the staged tile T[token][row] (fp32, row stride kMkLdt) ------------------------
// Units of (token, 4 consecutive output features), consecutive threads on consecutive features, kE units
// per thread with every residual load in flight before any store: out = act((acc + b) + res), the order of
// the unfused definition, as 8-B (bf16) or 16-B (f32) stores.
constexpr uint32_t kMkLdt = 132;
__device__ __forceinline__ void mk_out_tile(const DevDesc& dd, const GemmArgs& a, const float* T, uint32_t tok0, uint32_t n0,
                                            uint32_t tt, uint32_t e) {
    const uint16_t* bptr = a.has_bias ? reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.b_off)) : nullptr;
    const bool vec = (a.N % 4 == 0) && (a.ld_out % 4 == 0) && (!a.res || a.ld_res % 4 == 0);
    constexpr uint32_t kE = 4;
    const uint32_t units = tt * 32;
    for (uint32_t u0 = 0; u0 < units; u0 += kE * 128) {
        float4 rv[kE];
#pragma unroll
        for (uint32_t k = 0; k < kE; ++k) {
            const uint32_t u = u0 + k * 128 + e, tok = tok0 + (u >> 5), n = n0 + (u & 31) * 4;
            rv[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (vec && a.res && u < units && tok < a.M && n < a.N) {
                const uint64_t ri = (uint64_t)tok * a.ld_res + n;
                if (a.res_bf16) {
                    const uint2 h = __ldcg(reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(a.res) + ri));
                    rv[k] = make_float4(__uint_as_float(h.x << 16), __uint_as_float(h.x & 0xffff0000u), __uint_as_float(h.y << 16),
                                        __uint_as_float(h.y & 0xffff0000u));
                } else {
                    rv[k] = __ldcg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.res) + ri));
                }
            }
        }
#pragma unroll
        for (uint32_t k = 0; k < kE; ++k) {
            const uint32_t u = u0 + k * 128 + e, c = u >> 5, tok = tok0 + c, n = n0 + (u & 31) * 4;
            if (u >= units || tok >= a.M || n >= a.N) continue;
            const float4 x = *reinterpret_cast<const float4*>(T + c * kMkLdt + (u & 31) * 4);
            if (vec) {
                float y[4] = {x.x, x.y, x.z, x.w};
                const float r[4] = {rv[k].x, rv[k].y, rv[k].z, rv[k].w};
                if (bptr) {
                    const uint2 bv = *reinterpret_cast<const uint2*>(bptr + n);
                    y[0] += __uint_as_float(bv.x << 16);
                    y[1] += __uint_as_float(bv.x & 0xffff0000u);
                    y[2] += __uint_as_float(bv.y << 16);
                    y[3] += __uint_as_float(bv.y & 0xffff0000u);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) y[q] = mk_act(a.act, y[q] + r[q]);
                const uint64_t oi = (uint64_t)tok * a.ld_out + n;
                const uint2 pk = make_uint2((uint32_t)f32_to_bf16(y[0]) | ((uint32_t)f32_to_bf16(y[1]) << 16),
                                            (uint32_t)f32_to_bf16(y[2]) | ((uint32_t)f32_to_bf16(y[3]) << 16));
                if (a.out_bf16) *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(a.out) + oi) = pk;
                else *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + oi) = make_float4(y[0], y[1], y[2], y[3]);
                if (a.out2) *reinterpret_cast<uint2*>(a.out2 + oi) = pk;
            } else {  // N or a leading dimension not a multiple of 4 (e.g. a 2-wide QA head): scalar
                const float xs[4] = {x.x, x.y, x.z, x.w};
                for (uint32_t q = 0; q < 4 && n + q < a.N; ++q) {
                    float v = xs[q] + (bptr ? bf16_to_f32(bptr[n + q]) : 0.0f);
                    if (a.res) {
                        const uint64_t ri = (uint64_t)tok * a.ld_res + n + q;
                        v += a.res_bf16 ? bf16_to_f32(__ldcg(reinterpret_cast<const unsigned short*>(a.res) + ri))
                                        : __ldcg(reinterpret_cast<const float*>(a.res) + ri);
                    }
                    v = mk_act(a.act, v);
                    const uint64_t oi = (uint64_t)tok * a.ld_out + n + q;
                    if (a.out_bf16) reinterpret_cast<uint16_t*>(a.out)[oi] = f32_to_bf16(v);
                    else reinterpret_cast<float*>(a.out)[oi] = v;
                    if (a.out2) a.out2[oi] = f32_to_bf16(v);
                }
            }
        }
    }
}

// ---- CUDA-core tasks (128 threads, tid e) --------------------------------------------------------------
__device__ __forceinline__ void mk_embed(const DevDesc& dd, const EmbedArgs& a, uint32_t t, uint32_t e, DevCtl* ctl) {
    uint32_t row[4];
    for (int j = 0; j < a.n_tables; ++j) {
        uint32_t r = a.rule[j] == FSW_RULE_IDS ? (uint32_t)__ldcg(a.ids + t) : (a.rule[j] == FSW_RULE_POSITION ? t : 0u);
        if (r >= a.table_rows[j]) {
            if (e == 0) atomicExch(&ctl->err, 3);
            r = 0;
        }
        row[j] = r;
    }
    // 8 columns per thread per pass, every table load of the pass in flight before the stores
    for (uint32_t c0 = 0; c0 < a.C; c0 += 8 * 128) {
        float s[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] = 0.0f;
        for (int j = 0; j < a.n_tables; ++j) {
            const unsigned short* tab = reinterpret_cast<const unsigned short*>(weight_ptr(dd, a.table_off[j])) + (uint64_t)row[j] * a.C;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t c = c0 + e + u * 128;
                if (c < a.C) s[u] += bf16_to_f32(__ldcg(tab + c));
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t c = c0 + e + u * 128;
            if (c >= a.C) break;
            if (a.out) a.out[(uint64_t)t * a.C + c] = s[u];
            if (a.out_bf16) a.out_bf16[(uint64_t)t * a.C + c] = f32_to_bf16(s[u]);
        }
    }
}

__device__ __forceinline__ void mk_ln_out(const LnArgs& a, uint32_t r, uint32_t c, float4 v, float mu, float inv, uint2 gv,
                                          uint2 bv) {
    float4 y;
    y.x = (v.x - mu) * inv * __uint_as_float(gv.x << 16) + __uint_as_float(bv.x << 16);
    y.y = (v.y - mu) * inv * __uint_as_float(gv.x & 0xffff0000u) + __uint_as_float(bv.x & 0xffff0000u);
    y.z = (v.z - mu) * inv * __uint_as_float(gv.y << 16) + __uint_as_float(bv.y << 16);
    y.w = (v.w - mu) * inv * __uint_as_float(gv.y & 0xffff0000u) + __uint_as_float(bv.y & 0xffff0000u);
    if (a.out_f32) reinterpret_cast<float4*>(a.out_f32 + (uint64_t)r * a.C)[c] = y;
    if (a.out_bf16) {
        const uint32_t lo = (uint32_t)f32_to_bf16(y.x) | ((uint32_t)f32_to_bf16(y.y) << 16);
        const uint32_t hi = (uint32_t)f32_to_bf16(y.z) | ((uint32_t)f32_to_bf16(y.w) << 16);
        reinterpret_cast<uint2*>(a.out_bf16 + (uint64_t)r * a.C)[c] = make_uint2(lo, hi);
    }
}

// one warp per row: the row held in registers (NV float4 per lane, all loads in flight at once), fp32
// two-pass statistics (mean, then centred variance) as k_layernorm
template <int NV>
__device__ __forceinline__ void mk_layernorm_nv(const DevDesc& dd, const LnArgs& a, uint32_t r, uint32_t lane) {
    if (r >= a.rows) return;
    const float4* x = reinterpret_cast<const float4*>(a.in + (uint64_t)r * a.C);
    const uint2* g = reinterpret_cast<const uint2*>(weight_ptr(dd, a.g_off));
    const uint2* b = reinterpret_cast<const uint2*>(weight_ptr(dd, a.b_off));
    const uint32_t n4 = a.C >> 2;
    float4 v[NV];
    uint2 gv[NV], bv[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const uint32_t c = lane + 32u * j;
        v[j] = c < n4 ? __ldcg(x + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        gv[j] = c < n4 ? g[c] : make_uint2(0u, 0u);
        bv[j] = c < n4 ? b[c] : make_uint2(0u, 0u);
    }
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < NV; ++j) s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
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
        if (c >= n4) break;
        mk_ln_out(a, r, c, v[j], mu, inv, gv[j], bv[j]);
    }
}

__device__ __forceinline__ void mk_layernorm(const DevDesc& dd, const LnArgs& a, uint32_t r, uint32_t lane) {
    const uint32_t nv = (a.C / 4 + 31) / 32;  // C <= 1664 (plan eligibility): BERT-base 768, GPT-2-XL 1600
    if (nv <= 6) mk_layernorm_nv<6>(dd, a, r, lane);
    else mk_layernorm_nv<13>(dd, a, r, lane);
}

// GEMV task: features [o0, o0 + 64) of a rows <= 8 linear; x staged in shared memory as fp32
constexpr uint32_t kMkGemvFeat = 64;
template <int R>
__device__ __forceinline__ void mk_gemv(const DevDesc& dd, const GemvArgs& a, uint32_t o0, float* xs, uint32_t e) {
    for (uint32_t i = e; i < R * a.K; i += 128) {
        const uint32_t r = i / a.K, k = i - r * a.K;
        const uint64_t src = (uint64_t)(a.r0 + r) * a.ldx + k;
        xs[i] = r >= a.rows ? 0.0f
                : a.x_bf16  ? bf16_to_f32(__ldcg(reinterpret_cast<const unsigned short*>(a.x) + src))
                            : __ldcg(reinterpret_cast<const float*>(a.x) + src);
    }
    mk_bar();
    const uint32_t lane = e & 31, wq = e >> 5;
    const uint8_t* wmat = weight_ptr(dd, a.w_off);
    const uint16_t* bvec = a.has_bias ? reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.b_off)) : nullptr;
    const uint32_t k8n = a.K >> 3;
    for (uint32_t f = wq; f < kMkGemvFeat; f += 4) {
        const uint32_t o = o0 + f;
        if (o >= a.N) break;
        const uint4* wr = reinterpret_cast<const uint4*>(wmat + (uint64_t)o * a.K * 2);
        float acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0f;
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
        if (lane < (uint32_t)R && lane < a.rows) {
            float v = 0.0f;
#pragma unroll
            for (int r = 0; r < R; ++r) v = (r == (int)lane) ? acc[r] : v;
            const uint64_t oi = (uint64_t)lane * a.N + o;
            if (bvec) v += bf16_to_f32(bvec[o]);
            if (a.res) v += a.res_bf16 ? bf16_to_f32(__ldcg(reinterpret_cast<const unsigned short*>(a.res) + oi))
                                       : __ldcg(reinterpret_cast<const float*>(a.res) + oi);
            v = mk_act(a.act, v);
            if (a.out_bf16) reinterpret_cast<uint16_t*>(a.out)[oi] = f32_to_bf16(v);
            else reinterpret_cast<float*>(a.out)[oi] = v;
            if (a.out2) a.out2[oi] = f32_to_bf16(v);
        }
    }
    mk_bar();  // xs is rewritten by the next task
}

// 168 registers: 192 x 168 + a 256-thread swap CTA x 64 fit one SM's register file (cold invokes)
__global__ void __maxnreg__(168)
    k_mega(const DevDesc* __restrict__ d, const MkOp* __restrict__ ops, uint32_t n_ops, uint32_t* op_cnt,
           const CUtensorMap* __restrict__ tmaps, uint32_t* tile_ctr, float* part) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned by pointer arithmetic on the __shared__ array (not an integer round trip), so the
    // compiler keeps every derived pointer in the shared address space: LDS / STS that global stores
    // cannot alias (generic loads after global stores were ordered behind them: ~1 us per store)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* ring = smem;
    uint8_t* cmp = smem + kMkRing;  // compute region
    MkOp* sop = reinterpret_cast<MkOp*>(cmp + kMkCompute);  // epilogue warps: the current op, in shared memory
    uint64_t* full = reinterpret_cast<uint64_t*>(cmp + kMkCompute + kMkOpSmem);
    uint64_t* empty = full + kMkStages;
    uint64_t* tfull = empty + kMkStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    uint32_t* flag = tmem_slot + 1;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const DevDesc dd = *d;
    DevCtl* ctl = ops[0].w.ctl;
    [[maybe_unused]] unsigned long long* const g_tr = g_trace;
    uint32_t* epochs = op_cnt + (uint64_t)n_ops * kMkLine;  // [ctas] epoch words after the op counters
    const uint32_t* my_epoch = epochs + (uint64_t)blockIdx.x * kMkLine;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kMkStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kMkTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ================= producer =================
        if (lane == 0) {
            uint32_t it = 0;
            for (uint32_t i = 0; i < n_ops; ++i) {
                const MkOp op = ops[i];  // a register / local copy: never reloaded after asm memory clobbers or stores
                if (op.kind != MK_GEMM || blockIdx.x >= op.n_tasks) continue;
                wait_ready_thread(op.w);  // the layer's weights landed (cold); no-op when resident
                FSW_TRACE_MAX(g_tr, op.layer, 1, globaltimer());
                asm volatile("fence.proxy.async.global;" ::: "memory");
                const GemmArgs a = op.gemm;
                const uint8_t* wt = weight_ptr(dd, a.w_off);
                const uint64_t ktile_stride = (uint64_t)(a.n_pad / 8) * 1024;
                const CUtensorMap* tm = tmaps + op.tmap;
                bool dep_ok = op.dep < 0;
                for (uint32_t g = blockIdx.x; g < op.n_tasks; g += gridDim.x) {
                    const MkTile t = mk_tile(op, g);
                    const uint32_t wbytes = t.rows_w * 128, abytes = op.tt * 128;
                    const uint32_t pre = dep_ok ? 0u : min(t.nk, (uint32_t)kMkStages);
                    // weights of the first stages before the activation dependency resolves
                    for (uint32_t q = 0; q < pre; ++q) {
                        const uint32_t s = (it + q) % kMkStages;
                        mk_wait(&empty[s], (((it + q) / kMkStages) & 1) ^ 1, ctl);
                        mbar_expect_tx(&full[s], wbytes + abytes);
                        bulk_load(ring + s * kMkStage, wt + (t.kt0 + q) * ktile_stride + (uint64_t)(t.r * 16) * 1024, wbytes,
                                  &full[s]);
                    }
                    if (!dep_ok) {
                        mk_wait_op(my_epoch, (uint32_t)op.dep, ctl);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        dep_ok = true;
                    }
                    mk_stamp(i, 0);
                    for (uint32_t q = 0; q < pre; ++q) {
                        const uint32_t s = (it + q) % kMkStages;
                        tma_load_2d(ring + s * kMkStage + kMkW, tm, (int)((t.kt0 + q) * 64), (int)(t.j * op.tt), &full[s]);
                    }
                    for (uint32_t q = pre; q < t.nk; ++q) {
                        const uint32_t s = (it + q) % kMkStages;
                        mk_wait(&empty[s], (((it + q) / kMkStages) & 1) ^ 1, ctl);
                        mbar_expect_tx(&full[s], wbytes + abytes);
                        bulk_load(ring + s * kMkStage, wt + (t.kt0 + q) * ktile_stride + (uint64_t)(t.r * 16) * 1024, wbytes,
                                  &full[s]);
                        tma_load_2d(ring + s * kMkStage + kMkW, tm, (int)((t.kt0 + q) * 64), (int)(t.j * op.tt), &full[s]);
                    }
                    it += t.nk;
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ================= MMA issuer =================
        if (lane == 0) {
            uint32_t it = 0, acc = 0;
            for (uint32_t i = 0; i < n_ops; ++i) {
                const MkOp op = ops[i];  // a register / local copy: never reloaded after asm memory clobbers or stores
                if (op.kind != MK_GEMM) continue;
                const uint32_t idesc = umma_idesc_bf16(128, (int)op.tt);
                for (uint32_t g = blockIdx.x; g < op.n_tasks; g += gridDim.x) {
                    const MkTile t = mk_tile(op, g);
                    const uint32_t b = acc & 1;
                    mk_wait(&tempty[b], ((acc >> 1) & 1) ^ 1, ctl);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t dcol = tmem + b * kMkTT;
                    for (uint32_t q = 0; q < t.nk; ++q) {
                        const uint32_t s = it % kMkStages;
                        mk_wait(&full[s], (it / kMkStages) & 1, ctl);
                        if (q == 0) mk_stamp(i, 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint64_t ad = umma_desc_sw128(ring + s * kMkStage), bd = umma_desc_sw128(ring + s * kMkStage + kMkW);
#pragma unroll
                        for (uint32_t kk = 0; kk < 4; ++kk) umma_f16(dcol, ad + kk * 2, bd + kk * 2, idesc, (q | kk) != 0);
                        umma_commit(&empty[s]);
                        ++it;
                    }
                    umma_commit(&tfull[b]);
                    mk_stamp(i, 2);
                    ++acc;
                }
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue / CUDA-core tasks (warps 2-5) =================
        const uint32_t e = threadIdx.x - 64, quarter = warp & 3, ew = e >> 5;
        uint32_t acc = 0;
        for (uint32_t i = 0; i < n_ops; ++i) {
            if (blockIdx.x >= ops[i].n_tasks) continue;
            // the op's arguments in shared memory: global reads of them would miss L1 after every fence
            // (CCTL.IVALL) and could not be kept in registers across the epilogue's stores
            mk_bar();  // the previous op's readers are done with sop
            for (uint32_t k = e; k < sizeof(MkOp) / 4; k += 128)
                reinterpret_cast<uint32_t*>(sop)[k] = reinterpret_cast<const uint32_t*>(ops + i)[k];
            mk_bar();
            const MkOp op = *sop;  // thread-local copy: stores through generic pointers cannot alias it
            // activations of op i - 1 and this op's weights are visible to the 128 threads
            if (e == 0) {
                if (op.dep >= 0) mk_wait_op(my_epoch, (uint32_t)op.dep, ctl);
                wait_ready_thread(op.w);
                if (op.kind != MK_GEMM) FSW_TRACE_MAX(g_tr, op.layer, 1, globaltimer());
                mk_stamp(i, 6);
            }
            mk_bar();
            for (uint32_t g = blockIdx.x; g < op.n_tasks; g += gridDim.x) {
                if (e == 0) FSW_TRACE_MAX(g_tr, op.layer, 0, ~globaltimer());
                switch (op.kind) {
                    case MK_GEMM: {
                        const GemmArgs a = op.gemm;
                        const MkTile t = mk_tile(op, g);
                        const uint32_t b = acc & 1;
                        mk_wait(&tfull[b], (acc >> 1) & 1, ctl);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        if (e == 0) mk_stamp(i, 3);
                        // 1) TMEM -> shared tile T[token][row] (fp32, row stride kMkLdt): the accumulator is
                        //    free for the next task's MMAs as soon as it is read
                        float* T = reinterpret_cast<float*>(cmp);
                        const uint32_t row = quarter * 32 + lane;
                        for (uint32_t c0 = 0; c0 < op.tt; c0 += 32) {
                            uint32_t v[32];
                            tmem_ld32(tmem + ((quarter * 32) << 16) + b * kMkTT + c0, v);
#pragma unroll
                            for (uint32_t c = 0; c < 32; ++c)
                                if (c0 + c < op.tt) T[(c0 + c) * kMkLdt + row] = __uint_as_float(v[c]);
                        }
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        mk_bar();
                        if (e == 0) mbar_arrive(&tempty[b]);
                        if (e == 0 && op.splits == 1) mk_stamp(i, 6);
                        ++acc;
                        const uint32_t tile = t.r * op.n_tt + t.j;
                        bool out_now = op.splits == 1;
                        if (!out_now) {
                            // 2a) split-K: publish this split's partial [token][row] (float4, coalesced); the last
                            //     split to arrive sums all of them in split order into T and runs the epilogue
                            float4* myp = reinterpret_cast<float4*>(part + ((uint64_t)tile * op.splits + t.z) * (128 * kMkTT));
                            for (uint32_t u = e; u < op.tt * 32; u += 128)
                                __stcg(myp + u, *reinterpret_cast<const float4*>(T + (u >> 5) * kMkLdt + (u & 31) * 4));
                            __threadfence();
                            mk_bar();
                            if (e == 0) *flag = atomicAdd(tile_ctr + (uint64_t)tile * kMkLine, 1u) == op.splits - 1;
                            mk_bar();
                            if (e == 0) mk_stamp(i, 6);
                            out_now = *flag != 0;
                            if (out_now) {
                                __threadfence();
                                const float4* p0 = reinterpret_cast<const float4*>(part + (uint64_t)tile * op.splits * (128 * kMkTT));
                                const uint32_t nq = op.tt * 32;
                                for (uint32_t u0 = 0; u0 < nq; u0 += 4 * 128) {
                                    float4 x[4];
#pragma unroll
                                    for (uint32_t k = 0; k < 4; ++k) {
                                        const uint32_t u = u0 + k * 128 + e;
                                        x[k] = u < nq ? __ldcg(p0 + u) : make_float4(0.f, 0.f, 0.f, 0.f);
                                    }
                                    for (uint32_t z = 1; z < op.splits; ++z) {
                                        const float4* pz = p0 + (uint64_t)z * (128 * kMkTT / 4);
                                        float4 y[4];
#pragma unroll
                                        for (uint32_t k = 0; k < 4; ++k) {
                                            const uint32_t u = u0 + k * 128 + e;
                                            y[k] = u < nq ? __ldcg(pz + u) : make_float4(0.f, 0.f, 0.f, 0.f);
                                        }
#pragma unroll
                                        for (uint32_t k = 0; k < 4; ++k) {
                                            x[k].x += y[k].x;
                                            x[k].y += y[k].y;
                                            x[k].z += y[k].z;
                                            x[k].w += y[k].w;
                                        }
                                    }
#pragma unroll
                                    for (uint32_t k = 0; k < 4; ++k) {
                                        const uint32_t u = u0 + k * 128 + e;
                                        if (u < nq) *reinterpret_cast<float4*>(T + (u >> 5) * kMkLdt + (u & 31) * 4) = x[k];
                                    }
                                }
                                if (e == 0) tile_ctr[(uint64_t)tile * kMkLine] = 0;  // self-reset for the next GEMM
                                mk_bar();
                                if (e == 0) mk_stamp(i, 7);
                            }
                        }
                        if (out_now) {
                            // 2b) row-major pass over (token, 4 features) units: bias, residual (4 units' loads in
                            //     flight per thread), activation, 8-B (bf16) / 16-B (f32) stores
                            mk_out_tile(dd, a, T, t.j * op.tt, t.r * 128, op.tt, e);
                            if (e == 0 && op.splits == 1) mk_stamp(i, 7);
                        }
                        if (e == 0) mk_stamp(i, 4);
                        break;
                    }
                    case MK_LN:
                        mk_layernorm(dd, op.ln, g * 4 + ew, lane);
                        break;
                    case MK_EMBED:
                        mk_embed(dd, op.embed, g, e, ctl);
                        break;
                    case MK_GEMV:
                        mk_gemv<1>(dd, op.gemv, g * kMkGemvFeat, reinterpret_cast<float*>(cmp), e);  // rows == 1 (plan)
                        break;
                    case MK_ATTN: {
                        const AttnArgs a = op.attn;
                        const uint32_t h = g % a.H, q0 = (g / a.H) * kAttnSplitRows;
                        uint16_t* kv = reinterpret_cast<uint16_t*>(cmp);
                        attn_split_core<64, true>(a, h, q0, kv, e, mk_bar);  // dh = 64 only (plan eligibility)
                        mk_bar();  // the staging buffers are rewritten by the next task
                        break;
                    }
                    default:
                        break;
                }
                mk_bar();
                if (e == 0) {
                    if (op.kind != MK_GEMM) mk_stamp(i, 7);
                    mk_done(op_cnt + (uint64_t)i * kMkLine, op.n_tasks, epochs, i);
                    mk_stamp(i, 5);
                    FSW_TRACE_MAX(g_tr, op.layer, 2, globaltimer());
                }
            }
        }
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kMkTmemCols) : "memory");
}

void launch_mega(cudaStream_t s, int ctas, const DevDesc* d, const MkOp* ops, uint32_t n_ops, uint32_t* op_cnt,
                 const CUtensorMap* tmaps, uint32_t* tile_ctr, float* part) {
    k_mega<<<ctas, kMkThreads, mega_smem_bytes(), s>>>(d, ops, n_ops, op_cnt, tmaps, tile_ctr, part);
}

void init_mega_attrs() {
    cudaFuncSetAttribute(k_mega, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mega_smem_bytes());
}

void set_trace_mega(unsigned long long* t) { cudaMemcpyToSymbol(g_trace, &t, sizeof t); }

}  // namespace fsw
