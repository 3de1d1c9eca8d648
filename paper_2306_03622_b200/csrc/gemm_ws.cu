// gemm_ws.cu — K3c: the weight-stationary swap-AB tcgen05 GEMM for batch-1 transformer linears.
//
//   out[t][n] = act( Σ_k X[t][k]·W[n][k] + b[n] + res[t][n] )          fp32 accumulate in TMEM
//
// Why another GEMM ("k_gemm_ws"): at batch 1 a linear is a chain of latencies, and in the
// invoke graph its successor can only start its arithmetic once its predecessor's activations are out
// (griddepcontrol.wait).  k_gemm puts 128 TOKENS on the UMMA M operand, so every CTA streams the whole
// 128 x K activation (196 KB at K = 768) AFTER that wait, through a ring whose stages it reuses.  Here the
// roles are swapped and nothing the CTA needs after the wait is large:
//   * the UMMA M operand is 128 WEIGHT rows (the store's pre-tiled K-major SWIZZLE_128B layout makes one
//     128-row x 64-k sub-tile one contiguous 16-KiB bulk copy), the N operand is a tile of TT tokens;
//   * a CTA owns ONE K range (split-K over a (1, 1, S) cluster) and ALL of its weight sub-tiles live in
//     shared memory at once — no ring, no stage reuse, one mbarrier per k sub-tile.  They are loaded
//     right after the layer's readiness wait (PAPER.md:588-590 pipelining), i.e. before the predecessor
//     finishes when the CTA is resident early (programmatic dependent launch);
//   * after the wait only the TT x K_range activation slice moves (TMA, one box per k sub-tile), and each
//     sub-tile's 4 MMAs issue as soon as it lands;
//   * the S partial tiles of a cluster are reduced over distributed shared memory: each CTA pushes every row's
//     partial into the receive region of the CTA that owns the row's sum (CTA z owns weight-row quads
//     [z·per, (z+1)·per), per = ceil(32/S)); after one cluster barrier the owner sums its rows in split order
//     (deterministic) and runs the fused bias / residual / activation epilogue with 8-16-B coalesced accesses.
// The grid is one wave: (ceil(N/128), ceil(M/TT), S) CTAs of 512 threads (16 warps share the epilogue: with one
// warp per scheduler its dependent ALU chains — the GELU — were latency-bound, 4-5 us per epilogue).
#include "device.cuh"
#include "umma.cuh"

namespace fsw {

namespace {
constexpr int kWsMaxKt = 16;          // k sub-tiles one CTA holds (kt_per)
constexpr uint32_t kWsW = 128 * 128;  // one 128-row x 64-k weight sub-tile: 16 KiB
template <int TT>
struct WsCfg {
    static constexpr uint32_t kX = TT * 128;               // one TT-token x 64-k activation sub-tile
    static constexpr uint32_t kTmemCols = TT < 32 ? 32 : TT;
    // rows of the weight tile whose split-K sum CTA z of S owns: quads [z·per, (z+1)·per), per = ceil(32 / S)
    __host__ __device__ static uint32_t rows_owned(uint32_t S) { return 4u * ((32u + S - 1u) / S); }
    // receive region: every split's partial of the owned rows, [S][TT][rows_owned] fp32
    __host__ __device__ static uint32_t rbytes(uint32_t S) { return S * TT * rows_owned(S) * 4u; }
    // slots = k sub-tiles resident at once: all of the CTA's K range (weight-stationary), or a ring of that many
    __host__ __device__ static uint32_t smem(uint32_t slots, uint32_t S) { return slots * kWsW + slots * kX + rbytes(S) + 1024 + 1024; }
};
}  // namespace

constexpr int kWsThreads = 512;  // thread 0 loads, thread 32 issues the MMAs; all 16 warps drain TMEM and run the epilogue
// folded LayerNorm (a.ln_x): warps 4..15 build the normalised operand tiles; (μ, rstd) of the tile's tokens in the
// extra KiB after the control block
constexpr uint32_t kLnWarp0 = 4, kLnWarps = kWsThreads / 32 - kLnWarp0;

// Per-token partial of a folded LayerNorm's statistics over the nq lanes (a power of two dividing 32) that hold one
// token's output columns: (mean, M2) of their 4·nq values, two shuffle passes (the LN kernel's two-pass form).
__device__ __forceinline__ float2 ln_partial(const float4 v, uint32_t nq) {
    float s = (v.x + v.y) + (v.z + v.w);
    for (uint32_t o = 1; o < nq; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / (float)(4u * nq);
    const float d0 = v.x - mu, d1 = v.y - mu, d2 = v.z - mu, d3 = v.w - mu;
    float q = (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
    for (uint32_t o = 1; o < nq; o <<= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    return make_float2(mu, q);
}

// LN: the folded-LayerNorm instantiation (FSW_LN_FUSE; stationary mode only), so the default kernels carry none of its
// code (measured: 0.26 us per launch when they did)
template <int TT, bool RING, bool LN>
__global__ void __launch_bounds__(kWsThreads, 2) k_gemm_ws(const __grid_constant__ CUtensorMap tmX, const DevDesc* __restrict__ d, Wait w,
                                                 GemmArgs a) {
    TraceExit tx(w.trace, w.layer);
    using C = WsCfg<TT>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t kt0 = blockIdx.z * a.kt_per;
    const uint32_t nkt = min(a.K / kBK, kt0 + a.kt_per) - kt0;  // >= 1 (host plan)
    const uint32_t S = gridDim.z;
    // NS sub-tile slots: the whole K range (weight-stationary, ws_stages = 0) or a ring of ws_stages slots for K
    // ranges too long to hold (the first NS slots' weights still load before the predecessor finishes)
    const uint32_t NS = RING ? a.ws_stages : a.kt_per;
    const bool ring = RING && NS < nkt;
    uint8_t* sw = smem;                                          // weight sub-tiles
    uint8_t* sx = smem + NS * kWsW;                              // activation sub-tiles
    float* recv = reinterpret_cast<float*>(sx + NS * C::kX);     // split partials of the owned rows
    // 1-KiB control block: full[kWsMaxKt] | done | TMEM slot | (at +256) the tile's 128 bias values | (at +768, ring)
    // empty[kWsMaxKt]
    uint8_t* ctl = reinterpret_cast<uint8_t*>(recv) + C::rbytes(S);
    uint64_t* full = reinterpret_cast<uint64_t*>(ctl);
    uint64_t* done = full + kWsMaxKt;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    float* bias_s = reinterpret_cast<float*>(ctl + 256);
    uint64_t* empty = reinterpret_cast<uint64_t*>(ctl + 768);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t n0 = blockIdx.x * 128, t0 = blockIdx.y * TT;
    const DevDesc dd = *d;

    if (threadIdx.x == 0) {
        for (uint32_t j = 0; j < NS && j < nkt; ++j) {
            mbar_init(&full[j], LN && a.ln_x ? 1 + kLnWarps : 1);  // + the operand-building warps' arrivals
            if (RING) mbar_init(&empty[j], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "n"(C::kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    if (a.trig_early) pdl_trigger();

    if (threadIdx.x == 0) {
        // producer: the layer's weights (ordered by the ready counters), then — after the predecessor — the
        // activation slice.  Rows past the weight's padded height are not copied (their accumulators are
        // never stored).
        wait_ready_thread(w);
        FSW_TRACE_MAX(w.trace, w.layer, 1, globaltimer());
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const uint32_t wrows = min(128u, a.n_pad - n0);
        const uint8_t* wt = weight_ptr(dd, a.w_off) + (uint64_t)(n0 / 8) * 1024;
        const uint64_t ktile_stride = (uint64_t)(a.n_pad / 8) * 1024;
        const uint32_t pre = min(NS, nkt);
        const uint32_t xbytes = LN && a.ln_x ? 0u : C::kX;  // a folded LayerNorm builds the operand in place
        for (uint32_t j = 0; j < pre; ++j) {
            mbar_expect_tx(&full[j], wrows * 128 + xbytes);
            bulk_load(sw + j * kWsW, wt + (kt0 + j) * ktile_stride, wrows * 128, &full[j]);
        }
        if (a.pf_bytes && w.n == 0) {  // resident: this CTA's share of the next GEMM's weights into L2
            const uint32_t ncta = gridDim.x * gridDim.y * gridDim.z;
            const uint32_t cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
            const uint64_t share = ((a.pf_bytes + ncta - 1) / ncta + 255) & ~255ull;
            const uint64_t b0 = cta * share, b1 = a.pf_bytes < b0 + share ? a.pf_bytes : b0 + share;
            const uint8_t* pf = weight_ptr(dd, a.pf_off);
            for (uint64_t o = b0; o < b1; o += 65536) prefetch_l2(pf + o, (uint32_t)(b1 - o < 65536 ? b1 - o : 65536));
        }
        pdl_wait();
        FSW_TRACE_MAX(w.trace, w.layer, 5, globaltimer());
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (xbytes)
            for (uint32_t j = 0; j < pre; ++j) tma_load_2d(sx + j * C::kX, &tmX, (int)((kt0 + j) * kBK), (int)t0, &full[j]);
        // ring: refill slot j mod NS once the MMAs of its previous use are done (slot / phase counted, no division:
        // this thread and the MMA issuer are on the critical path)
        if (RING)
        for (uint32_t j = pre, sl = 0, ph = 0; j < nkt; ++j) {
            mbar_wait(&empty[sl], ph);
            mbar_expect_tx(&full[sl], wrows * 128 + C::kX);
            bulk_load(sw + sl * kWsW, wt + (kt0 + j) * ktile_stride, wrows * 128, &full[sl]);
            tma_load_2d(sx + sl * C::kX, &tmX, (int)((kt0 + j) * kBK), (int)t0, &full[sl]);
            if (++sl == NS) sl = 0, ph ^= 1u;
        }
    } else if (threadIdx.x == 32) {
        constexpr uint32_t idesc = umma_idesc_bf16(kBM, TT);
        if (RING) {
            for (uint32_t j = 0, sl = 0, ph = 0; j < nkt; ++j) {
                mbar_wait(&full[sl], ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t ad = umma_desc_sw128(sw + sl * kWsW), bd = umma_desc_sw128(sx + sl * C::kX);
#pragma unroll
                for (uint32_t kk = 0; kk < kBK / 16; ++kk) umma_f16(tmem, ad + kk * 2, bd + kk * 2, idesc, (j | kk) != 0);
                if (ring && j + NS < nkt) umma_commit(&empty[sl]);  // the slot is free once these MMAs have read it
                if (++sl == NS) sl = 0, ph ^= 1u;
            }
        } else {  // every k sub-tile has its own slot and barrier
            for (uint32_t j = 0; j < nkt; ++j) {
                mbar_wait(&full[j], 0);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t ad = umma_desc_sw128(sw + j * kWsW), bd = umma_desc_sw128(sx + j * C::kX);
#pragma unroll
                for (uint32_t kk = 0; kk < kBK / 16; ++kk) umma_f16(tmem, ad + kk * 2, bd + kk * 2, idesc, (j | kk) != 0);
            }
        }
        umma_commit(done);
    } else if (LN && a.ln_x && warp >= kLnWarp0) {
        // Folded LayerNorm: the operand is LN(x) of this CTA's tokens over its K range, built here.
        // (1) per token, (μ, rstd) merged from the producer's per-slot (mean, M2) partials (Chan's formula, slots in
        // order: deterministic); (2) per k sub-tile, 8 columns per thread: (x − μ)·rstd·γ + β rounded to bf16 and
        // stored at the SWIZZLE_128B position the TMA box would have used (16-B chunk c of row r at c ^ (r & 7)),
        // then a proxy fence and one arrival per warp on the sub-tile's barrier.
        const uint32_t lw = warp - kLnWarp0, K = a.K;
        float* mu_s = reinterpret_cast<float*>(ctl + 1024);
        float* rs_s = mu_s + 128;
        if (lane == 0) wait_ready_thread(w);  // the LayerNorm's γ / β (the Wait includes its layer)
        __syncwarp();
        const uint16_t* gam = reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.ln_g_off));
        const uint16_t* bet = reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.ln_b_off));
        pdl_wait();
        const float cnt = (float)a.ln_cnt, inv_k = 1.0f / (float)K;
        for (uint32_t tok = lw; tok < TT; tok += kLnWarps) {
            const uint32_t t = min(t0 + tok, a.M - 1);
            const float2 p0 = lane < a.ln_slots ? a.ln_st[(uint64_t)lane * a.M + t] : make_float2(0.f, 0.f);
            const float2 p1 = lane + 32 < a.ln_slots ? a.ln_st[(uint64_t)(lane + 32) * a.M + t] : make_float2(0.f, 0.f);
            const float mu = warp_sum(p0.x + p1.x) * cnt * inv_k;
            const float e0 = p0.x - mu, e1 = p1.x - mu;
            float q = (lane < a.ln_slots ? p0.y + cnt * e0 * e0 : 0.f) + (lane + 32 < a.ln_slots ? p1.y + cnt * e1 * e1 : 0.f);
            const float rs = rsqrtf(warp_sum(q) * inv_k + a.ln_eps);
            if (lane == 0) {
                mu_s[tok] = mu;
                rs_s[tok] = rs;
                if (a.ln_musig && blockIdx.x == 0 && blockIdx.z == 0 && t0 + tok < a.M) a.ln_musig[t0 + tok] = make_float2(mu, rs);
            }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kLnWarps * 32) : "memory");  // every (μ, rstd) of the tile is in shared memory
        for (uint32_t j = 0; j < nkt; ++j) {
            uint8_t* xs = sx + j * C::kX;
            for (uint32_t c = lw * 32 + lane; c < TT * 8; c += kLnWarps * 32) {
                const uint32_t tok = c >> 3, ch = c & 7, t = t0 + tok, k = (kt0 + j) * kBK + ch * 8;
                uint4 pk = make_uint4(0u, 0u, 0u, 0u);
                if (t < a.M) {
                    const float4* xp = reinterpret_cast<const float4*>(a.ln_x + (uint64_t)t * K + k);
                    const float4 x0 = xp[0], x1 = xp[1];
                    const uint4 gv = *reinterpret_cast<const uint4*>(gam + k), bv = *reinterpret_cast<const uint4*>(bet + k);
                    const float mu = mu_s[tok], rs = rs_s[tok];
                    auto y = [&](float x, uint32_t g2, uint32_t b2, bool hi) {
                        const float gg = __uint_as_float(hi ? g2 & 0xffff0000u : g2 << 16), bb = __uint_as_float(hi ? b2 & 0xffff0000u : b2 << 16);
                        return (uint32_t)f32_to_bf16((x - mu) * rs * gg + bb);
                    };
                    pk.x = y(x0.x, gv.x, bv.x, false) | (y(x0.y, gv.x, bv.x, true) << 16);
                    pk.y = y(x0.z, gv.y, bv.y, false) | (y(x0.w, gv.y, bv.y, true) << 16);
                    pk.z = y(x1.x, gv.z, bv.z, false) | (y(x1.y, gv.z, bv.z, true) << 16);
                    pk.w = y(x1.z, gv.w, bv.w, false) | (y(x1.w, gv.w, bv.w, true) << 16);
                }
                *reinterpret_cast<uint4*>(xs + tok * 128u + ((ch ^ (tok & 7u)) << 4)) = pk;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> the tensor core's reads
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[j]);
        }
    }
    __syncwarp();

    mbar_wait(done, 0);
    if (!a.trig_early) pdl_trigger();  // the successor's prologue and weight loads overlap this epilogue
    if (threadIdx.x == 0) FSW_TRACE_MAX(w.trace, w.layer, 6, globaltimer());
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 3) {  // bias of the tile's 128 rows into shared memory (weights are ready: `done` follows the acquire)
        const uint16_t* bias = a.has_bias ? reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.b_off)) : nullptr;
        for (uint32_t r = lane * 4; r < 128; r += 128) {
            float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
            if (bias && n0 + r < a.N) {
                const uint2 v = *reinterpret_cast<const uint2*>(bias + n0 + r);
                b = make_float4(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u), __uint_as_float(v.y << 16),
                                __uint_as_float(v.y & 0xffff0000u));
            }
            *reinterpret_cast<float4*>(bias_s + r) = b;
        }
    }
    // TMEM (lane = weight row, column = token) -> PUSHED into the receive region of the CTA of the cluster that owns
    // the row's split-K sum: recv[my split][token][row - owner's first row] (st.shared::cluster; the own CTA too).
    // The receive region is nobody's operand memory, so a peer may push before this CTA's MMAs are done, and one
    // cluster barrier orders every push before every reduction — no second barrier before exit (a pulling
    // reduction needs one so that no CTA leaves while a peer still reads its shared memory).
    // Warp w reads TMEM lane quarter w mod 4 and every (w / 4)-th 16-column block.
    const uint32_t RO = C::rows_owned(S), rank = blockIdx.z;
    {
        const uint32_t q4 = warp & 3u, r = q4 * 32 + lane, zown = r / RO, rl = r - zown * RO;
        uint32_t dst;  // element (src = rank, token 0, row rl) in the owner's receive region
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(smem_u32(recv + (rank * TT) * RO + rl)), "r"(zown));
        auto push = [&](uint32_t c, uint32_t v) {
            asm volatile("st.shared::cluster.b32 [%0], %1;" ::"r"(dst + c * RO * 4u), "r"(v) : "memory");
        };
        // 16-column chunks dealt over the 4 warp groups: for TT >= 64 every warp pushes (32-column chunks left half
        // the warps idle at TT = 64 and the push was the epilogue's longest phase)
#pragma unroll 1
        for (int c0 = 16 * (int)(warp >> 2); c0 < TT; c0 += 16 * (kWsThreads / 128)) {
            uint32_t v[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
                           "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                         : "r"(tmem + ((q4 * 32u) << 16) + (uint32_t)c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int c = 0; c < 16; ++c) push((uint32_t)(c0 + c), v[c]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) FSW_TRACE_MAX(w.trace, w.layer, 11, globaltimer());
    if (S > 1) cluster_sync();  // every split's pushes have landed (release / acquire over the cluster)
    else __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols) : "memory");
    pdl_wait();  // residual in / output out: only after the predecessor
    if (threadIdx.x == 0) FSW_TRACE_MAX(w.trace, w.layer, 7, globaltimer());

    // reduction (split order) + epilogue over this CTA's weight-row quads x the tile's tokens
    const uint32_t q0 = min(32u, rank * (RO / 4)), nq = min(32u, q0 + RO / 4) - q0;
    const uint32_t units = nq * TT;
    const float* __restrict__ resf = a.res && !a.res_bf16 ? reinterpret_cast<const float*>(a.res) : nullptr;
    const uint16_t* __restrict__ resh = a.res && a.res_bf16 ? reinterpret_cast<const uint16_t*>(a.res) : nullptr;
    constexpr int kE = 2;
    for (uint32_t u0 = threadIdx.x; u0 < units; u0 += kWsThreads * kE) {
        float4 acc[kE];
        uint4 rr[kE];
#pragma unroll
        for (int e = 0; e < kE; ++e) {
            const uint32_t u = u0 + e * kWsThreads;
            acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
            rr[e] = make_uint4(0, 0, 0, 0);
            if (u >= units) continue;
            const uint32_t tok = u / nq, q = q0 + (u - tok * nq), n = n0 + 4 * q, t = t0 + tok;
            // splits in order (deterministic): recv[z][tok][4 (q - q0) .. + 3]
            const float* src = recv + tok * RO + 4 * (q - q0);
            acc[e] = *reinterpret_cast<const float4*>(src);
            for (uint32_t z = 1; z < S; ++z) {
                const float4 v = *reinterpret_cast<const float4*>(src + z * TT * RO);
                acc[e].x += v.x;
                acc[e].y += v.y;
                acc[e].z += v.z;
                acc[e].w += v.w;
            }
            if (t < a.M && n < a.N) {
                const uint64_t ri = (uint64_t)t * a.ld_res + n;
                if (resf) rr[e] = *reinterpret_cast<const uint4*>(resf + ri);
                else if (resh) {
                    const uint2 h = *reinterpret_cast<const uint2*>(resh + ri);
                    rr[e] = make_uint4(h.x << 16, h.x & 0xffff0000u, h.y << 16, h.y & 0xffff0000u);
                }
                if (LN && a.res_musig) {  // a folded LayerNorm's output as the residual: LN(res) from (μ, rstd), γ, β
                    const float2 ms = a.res_musig[t];
                    const uint2 g = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.res_g_off)) + n);
                    const uint2 b = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(weight_ptr(dd, a.res_b_off)) + n);
                    rr[e].x = __float_as_uint((__uint_as_float(rr[e].x) - ms.x) * ms.y * __uint_as_float(g.x << 16) + __uint_as_float(b.x << 16));
                    rr[e].y = __float_as_uint((__uint_as_float(rr[e].y) - ms.x) * ms.y * __uint_as_float(g.x & 0xffff0000u) + __uint_as_float(b.x & 0xffff0000u));
                    rr[e].z = __float_as_uint((__uint_as_float(rr[e].z) - ms.x) * ms.y * __uint_as_float(g.y << 16) + __uint_as_float(b.y << 16));
                    rr[e].w = __float_as_uint((__uint_as_float(rr[e].w) - ms.x) * ms.y * __uint_as_float(g.y & 0xffff0000u) + __uint_as_float(b.y & 0xffff0000u));
                }
            }
        }
        if (threadIdx.x == 0 && u0 == 0) FSW_TRACE_MAX(w.trace, w.layer, 8, globaltimer());
#pragma unroll
        for (int e = 0; e < kE; ++e) {
            const uint32_t u = u0 + e * kWsThreads;
            if (LN && a.st_out && u0 + e * kWsThreads - lane < units) {
                // a folded LayerNorm's producer: (mean, M2) of this token's columns in this slot (the plan allows it only
                // when every slot holds 128 / splits valid columns of every token, nq a power of two); whole warps
                const uint32_t tok = u / nq, q = q0 + (u - tok * nq), n = n0 + 4 * q, t = t0 + tok;
                float4 v = acc[e];
                if (u < units) {
                    const float4 b = *reinterpret_cast<const float4*>(bias_s + 4 * q);
                    v.x = (v.x + b.x) + __uint_as_float(rr[e].x);
                    v.y = (v.y + b.y) + __uint_as_float(rr[e].y);
                    v.z = (v.z + b.z) + __uint_as_float(rr[e].z);
                    v.w = (v.w + b.w) + __uint_as_float(rr[e].w);
                    v = act4(a.act, v);
                }
                const float2 pm = ln_partial(v, nq);
                if ((u & (nq - 1)) == 0 && u < units && t < a.M && n < a.N)
                    a.st_out[(uint64_t)(blockIdx.x * S + rank) * a.M + t] = pm;
            }
            if (u >= units) continue;
            const uint32_t tok = u / nq, q = q0 + (u - tok * nq), n = n0 + 4 * q, t = t0 + tok;
            if (t >= a.M || n >= a.N) continue;
            const float4 b = *reinterpret_cast<const float4*>(bias_s + 4 * q);
            float4 v = acc[e];
            // (acc + bias) + residual, the order of the unfused definition (as k_gemm)
            v.x = (v.x + b.x) + __uint_as_float(rr[e].x);
            v.y = (v.y + b.y) + __uint_as_float(rr[e].y);
            v.z = (v.z + b.z) + __uint_as_float(rr[e].z);
            v.w = (v.w + b.w) + __uint_as_float(rr[e].w);
            v = act4(a.act, v);
            const uint64_t oi = (uint64_t)t * a.ld_out + n;
            const uint2 pk = make_uint2((uint32_t)f32_to_bf16(v.x) | ((uint32_t)f32_to_bf16(v.y) << 16),
                                        (uint32_t)f32_to_bf16(v.z) | ((uint32_t)f32_to_bf16(v.w) << 16));
            if (a.out_bf16) *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(a.out) + oi) = pk;
            else *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + oi) = v;
            if (a.out2) *reinterpret_cast<uint2*>(a.out2 + oi) = pk;
        }
    }
    if (threadIdx.x == 0) FSW_TRACE_MAX(w.trace, w.layer, 9, globaltimer());
}

template <int TT>
static void launch_ws(cudaStream_t s, const DevDesc* d, Wait w, const CUtensorMap* tmX, const GemmArgs& a) {
    using C = WsCfg<TT>;
    const dim3 grid((a.n_pad + 127) / 128, (a.M + TT - 1) / TT, a.splits);
    if (a.ws_stages)
        launch_pdl_cluster(PDL_GEMM, k_gemm_ws<TT, true, false>, grid, dim3(kWsThreads), C::smem(a.ws_stages, a.splits), s,
                           dim3(1, 1, a.splits), *tmX, d, w, a);
    else if (a.ln_x || a.st_out || a.res_musig)  // + 1 KiB for a folded LayerNorm's (μ, rstd) per token
        launch_pdl_cluster(PDL_GEMM, k_gemm_ws<TT, false, true>, grid, dim3(kWsThreads), C::smem(a.kt_per, a.splits) + 1024u, s,
                           dim3(1, 1, a.splits), *tmX, d, w, a);
    else
        launch_pdl_cluster(PDL_GEMM, k_gemm_ws<TT, false, false>, grid, dim3(kWsThreads), C::smem(a.kt_per, a.splits), s,
                           dim3(1, 1, a.splits), *tmX, d, w, a);
}

void launch_gemm_ws(cudaStream_t s, const DevDesc* d, Wait w, const CUtensorMap* tmX, const GemmArgs& a) {
    switch (a.ws_tt) {
        case 16: launch_ws<16>(s, d, w, tmX, a); break;
        case 32: launch_ws<32>(s, d, w, tmX, a); break;
        case 64: launch_ws<64>(s, d, w, tmX, a); break;
        default: launch_ws<128>(s, d, w, tmX, a); break;
    }
}

uint32_t gemm_ws_smem(uint32_t tt, uint32_t slots, uint32_t splits) {
    switch (tt) {
        case 16: return WsCfg<16>::smem(slots, splits);
        case 32: return WsCfg<32>::smem(slots, splits);
        case 64: return WsCfg<64>::smem(slots, splits);
        default: return WsCfg<128>::smem(slots, splits);
    }
}

template <int TT>
static int ws_max_clusters(uint32_t slots, int cz) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1, 1, cz);
    cfg.blockDim = dim3(kWsThreads);
    cfg.dynamicSmemBytes = WsCfg<TT>::smem(slots, (uint32_t)cz);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 1;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = cz;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_gemm_ws<TT, false, false>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int gemm_ws_max_active_clusters(uint32_t tt, uint32_t kt_per, int cz) {
    switch (tt) {
        case 16: return ws_max_clusters<16>(kt_per, cz);
        case 32: return ws_max_clusters<32>(kt_per, cz);
        case 64: return ws_max_clusters<64>(kt_per, cz);
        default: return ws_max_clusters<128>(kt_per, cz);
    }
}

template <int TT>
static void ws_attrs() {
    for (auto k : {k_gemm_ws<TT, false, false>, k_gemm_ws<TT, true, false>, k_gemm_ws<TT, false, true>}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);  // split-K clusters up to 16
    }
}

void init_gemm_ws_attrs() {
    ws_attrs<16>();
    ws_attrs<32>();
    ws_attrs<64>();
    ws_attrs<128>();
}

}  // namespace fsw
