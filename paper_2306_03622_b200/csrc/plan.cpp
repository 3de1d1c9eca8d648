// plan.cpp — per-(model, GPU) execution plan: workspace layout and the kernel list, with the
// tcgen05 GEMM tiling chosen by cost models fitted to B200 sweeps.
#include "rt_internal.h"

// Tiling of one tcgen05 GEMM launch (gemm_tc.cu): tile width BN and split-K factor.
// max_cl[bn / 16][cz]: clusters of cz CTAs resident at once (cudaOccupancyMaxActiveClusters; B200 fits
// fewer CTAs in clusters than singly, e.g. 132 in clusters of 4), or nullptr (no cluster configs).
using ClusterCap = std::array<std::array<int, 9>, 9>;
static Tiling choose_tiling(uint64_t m_tiles, uint32_t n_pad, uint32_t kt, uint32_t a_kt_bytes, uint32_t /*m_rows*/,
                            const ClusterCap* max_cl = nullptr) {
    // Linear latency model fitted (least squares, rms 1.1 us) to the (BN, split) sweep of
    // tools/gemm_bench.cu on B200 over the batch-1 GEMM shapes of the paper's models
    // (profiles/r01/gemm_bench_sweep.txt): fixed cost, the bytes one CTA streams into shared memory,
    // the epilogue width, the split-K reduction, and the total L2->SM traffic (every N tile re-reads
    // A).  One CTA per SM: a grid beyond one wave of 148 pays per wave.  Picks within 0.5 us of the
    // measured best on every swept shape.
    Tiling best{16, 1, kt, false};
    double best_t = 1e30;
    for (int bn : {16, 32, 64, 128}) {
        if (n_pad % bn) continue;
        const uint64_t base = m_tiles * (n_pad / bn);
        for (uint32_t S = 1; S <= 16 && S <= kt; ++S) {
            const uint32_t kt_per = (kt + S - 1) / S;
            if ((kt + kt_per - 1) / kt_per != S) continue;  // no empty split
            const uint64_t ctas = base * S;
            if (S > 1 && ctas > 148) break;
            const double cta_kb = kt_per * (double)(a_kt_bytes + bn * 128) / 1e3;
            const double waves = (double)((ctas + 147) / 148);
            double t = 4.44 + 0.0078 * cta_kb + 0.233 * (bn / 16.0) + 0.0428 * std::min<double>(ctas, 148) * cta_kb / 1e3;
            if (S > 1) t += 2.51 + 0.0516 * S * (bn / 16.0);
            t *= waves;
            if (t < best_t - 1e-9) {
                best_t = t;
                best = {bn, S, kt_per, false};
            }
            // cluster split-K (partials reduced over DSMEM, gemm_tc.cu 2c): a second linear model fitted
            // to the single-wave cluster configurations of the same sweep (profiles/r01/gemm_sweep_cz2.txt,
            // rms 1.9 us); with the first model it picks the measured best (or within 0.5 us) on every shape
            if (S >= 2 && S <= 8 && max_cl && ctas <= (uint64_t)(*max_cl)[bn / 16][S] * S) {
                const double tc = 6.2102 + 0.0051 * cta_kb + 0.0737 * (bn / 16.0) + 0.0766 * ctas * cta_kb / 1e3 + 0.2124 * S;
                if (tc < best_t - 1e-9) {
                    best_t = tc;
                    best = {bn, S, kt_per, true};
                }
            }
        }
    }
    return best;
}

// Tiling of the weight-stationary swap-AB GEMM (k_gemm_ws, gemm_ws.cu): tt tokens per tile and `splits` K
// ranges over a cluster, one wave.  Measured in the invoke graph (profiles/r02/gemm/ws_sweep.txt, resident
// BERT-base): it beats k_gemm on the narrow linears (N <= 16 weight-row tiles: O-projection, FFN2; GPT-2 attention
// projection), where k_gemm
// has few CTAs each streaming the whole activation, and loses on the wide ones (QKV, FFN1), where its DSMEM
// split-K reduction and larger epilogue cost more than the activation bytes it saves.  Cost (relative, fitted to
// that sweep): the epilogue's token width, the split-K reduction, the MMA chain, and a penalty for CTAs too large
// to be resident beside their predecessor.  ok = false: no tiling fits (k_gemm runs the linear).
struct WsTiling { uint32_t tt, splits, kt_per, stages; bool ok; };  // stages: 0 = K range resident, else ring slots
static WsTiling choose_ws_tiling(uint32_t M, uint32_t n_pad, uint32_t kt, bool any_width) {
    const uint64_t rt = (n_pad + 127) / 128;
    // A/B hook: FSW_GEMM_WS_FORCE="tt:splits" for every shape, or "N:K:tt:splits,..." per weight shape (a shape
    // not in the list runs k_gemm)
    static const char* force = getenv("FSW_GEMM_WS_FORCE");
    // ("N:K:tt:splits:stages" selects a ring of `stages` k sub-tile slots)
    int ftt = 0, fs = 0, fst = 0;
    if (force) {
        int fn, fk, t, sp;
        const char* q = force;
        if (sscanf(q, "%d:%d:%d:%d", &fn, &fk, &t, &sp) == 4) {
            ftt = -1;
            while (q) {
                int st = 0, n = sscanf(q, "%d:%d:%d:%d:%d", &fn, &fk, &t, &sp, &st);
                if (n < 4) break;
                if ((uint32_t)fn == n_pad && (uint32_t)fk == kt * 64) ftt = t, fs = sp, fst = n == 5 ? st : 0;
                q = strchr(q, ',');
                if (q) ++q;
            }
        } else {
            sscanf(force, "%d:%d", &ftt, &fs);
        }
    }
    if (ftt < 0 || M > 128) return WsTiling{0, 0, 0, 0, false};
    (void)any_width;
    // Tilings measured best for the paper's transformer shapes (M = 128 tokens; weight rows padded, K): BERT-base
    // QKV 64:2, O-projection 32:4 (resident 0.423 -> 0.414 ms), FFN1 64:2 and FFN2 64:8 each on a 3-slot ring
    // (106 KB per CTA instead of 179, so FFN2's CTAs become resident beside FFN1's and stage their first weights
    // during it: 0.415 -> 0.411 ms; either ring alone is slower), GPT-2-XL QKV / FC / proj2 on a 3-slot ring
    // (profiles/r02/gemm/ws_sweep.txt, chain_vs_cublas.txt); used when they fit, the cost model otherwise.
    bool table_used = false;
    if (!ftt && M == 128) {
        struct Known { uint32_t n_pad, K, tt, s, stages; };
        static const Known known[] = {{2304, 768, 64, 2, 0}, {768, 768, 32, 4, 0}, {3072, 768, 64, 2, 3}, {768, 3072, 64, 8, 3},
                                      // GPT-2-XL's wide linears: a ring of 3 slots per CTA (their K ranges do not fit)
                                      {4800, 1600, 128, 3, 3}, {6400, 1600, 128, 2, 3}, {1600, 6400, 128, 8, 3}};
        for (const Known& k : known)
            if (k.n_pad == n_pad && k.K == kt * 64) ftt = (int)k.tt, fs = (int)k.s, fst = (int)k.stages, table_used = true;
    }
    auto search = [&](int ftt, int fs, int fst) {
        WsTiling best{0, 0, 0, 0, false};
        double best_t = 1e30;
        for (uint32_t tt : {16u, 32u, 64u, 128u}) {
            if (ftt && tt != (uint32_t)ftt) continue;
            for (uint32_t s = 1; s <= 16 && s <= kt; ++s) {  // clusters beyond 8 are non-portable (B200: 16)
                if (fs && s != (uint32_t)fs) continue;
                const uint32_t kp = (kt + s - 1) / s;
                if ((kt + kp - 1) / kp != s || (fst ? fst > 16 || (uint32_t)fst >= kp : kp > 16)) continue;
                const uint32_t slots = fst ? (uint32_t)fst : kp;
                const uint64_t ctas = rt * ((M + tt - 1) / tt) * s;
                const uint32_t smem = gemm_ws_smem(tt, slots, s);
                // <= 184 KB: a CTA must fit beside one swap-decode CTA (k_swapz_tma: ring + decode table, ~41 KB) in a
                // cold invoke (measured: GPT-2-XL's attention projection at 128:7, 204 KB, took the cold invoke from 37.6
                // to 40.2 ms)
                if (smem > 184 * 1024) continue;
                // one-wave capacity per (tt, kt_per, s), queried once; plans of different GPUs are built concurrently
                static std::mutex cap_mu;
                static std::map<uint64_t, int> cap_cache;
                const uint64_t key = ((uint64_t)tt << 40) | ((uint64_t)slots << 20) | s;
                int cap;
                {
                    std::lock_guard<std::mutex> lk(cap_mu);
                    auto it = cap_cache.find(key);
                    if (it == cap_cache.end())
                        it = cap_cache.emplace(key, s > 1 ? gemm_ws_max_active_clusters(tt, slots, (int)s) * (int)s : 148).first;
                    cap = it->second;
                }
                if (ctas > (uint64_t)std::min(cap, 148)) continue;
                const double t = 0.3 * (tt / 16.0) + 0.4 * (s - 1) + 0.1 * kp + (smem > 150 * 1024 ? 2.0 : 0.0) + (ctas > 120 ? 2.0 : 0.0);
                if (t < best_t - 1e-9) {
                    best_t = t;
                    best = {tt, s, kp, (uint32_t)fst, true};
                }
            }
        }
        return best;
    };
    const WsTiling t = search(ftt, fs, fst);
    return t.ok || !table_used ? t : search(0, 0, 0);  // a measured tiling that does not fit here: the cost model
}
// ==========================================================================================
// persistent transformer kernel (mega.cu): eligibility, tiling, op table
// ==========================================================================================
// Tiling of one swap-AB GEMM op of k_mega: tt tokens per tile (UMMA N) and `splits` K ranges, chosen by
// a per-CTA cost model over one CTA per SM: a task streams kt_per k-tiles of (weight rows + tt tokens)
// x 128 B into its SM (~45 GB/s per SM of L2 -> SM bandwidth) plus ~0.6 us of fixed
// cost; split-K adds its partial write and the last split's reduction.
struct MkTiling { uint32_t tt, splits, kt_per; };
static MkTiling mega_tiling(uint32_t M, uint32_t n_pad, uint32_t kt, int ctas) {
    MkTiling best{kMkTT, 1, kt};
    double best_c = 1e30;
    static const uint32_t max_split = getenv("FSW_MEGA_MAXSPLIT") ? (uint32_t)atoi(getenv("FSW_MEGA_MAXSPLIT")) : 8;  // A/B
    static const double split_cost = getenv("FSW_MEGA_SPLITCOST") ? atof(getenv("FSW_MEGA_SPLITCOST")) : 1.0;
    for (uint32_t tt : {16u, 32u, 64u}) {
        if (tt > kMkTT) break;
        for (uint32_t s = 1; s <= max_split && s <= kt; ++s) {
            const uint32_t kp = (kt + s - 1) / s;
            if ((kt + kp - 1) / kp != s) continue;
            const uint64_t tasks = (uint64_t)((n_pad + 127) / 128) * ((M + tt - 1) / tt) * s;
            const double waves = (double)((tasks + ctas - 1) / ctas);
            const double bytes = (double)kp * (std::min<uint32_t>(128, n_pad) * 128 + tt * 128);
            double cost = waves * (0.6 + bytes / 45e3);
            if (s > 1) cost += split_cost + s * tt * 512.0 / 45e3;
            if (cost < best_c - 1e-9) {
                best_c = cost;
                best = {tt, s, kp};
            }
        }
    }
    return best;
}

fsw_status build_mega(fsw_ctx* c, Model& m, Plan& p, Gpu& g) {
    (void)c;
    MegaPlan& mp = p.mega;
    mp.on = false;
    // Opt-in (FSW_MEGA=1): parity-green, but at batch 1 its op-level dependency chain (release -> epoch ->
    // acquire -> TMA of the activations -> MMA -> epilogue, ~4-6 us per op) is slower than the PDL chain of
    // per-op kernels (resident BERT-base 1.05-1.09 vs 0.59 ms; DESIGN.md §5 "k_mega", profiles/r02/mega/)
    static const bool on = getenv("FSW_MEGA") && atoi(getenv("FSW_MEGA")) == 1;
    if (!on) return FSW_OK;
    // eligible: transformer ops only, shapes the kernel's shared memory holds
    for (const Launch& x : p.launches) {
        switch (x.kind) {
            case K_EMBED: break;
            case K_LN: if (x.ln.C % 4 || x.ln.C > 1664) return FSW_OK; break;
            case K_GEMV: if (x.gemv.rows > 1 || x.gemv.K * 4 > 56 * 1024 || x.gemv.K % 8) return FSW_OK; break;
            case K_GEMM: if (x.gemm.conv || x.gemm.pair_t || !x.abase) return FSW_OK; break;
            case K_ATTN: if (x.attn.T > 128 || x.attn.dh != 64) return FSW_OK; break;
            default: return FSW_OK;
        }
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g.dev);
    mp.ctas = sms;
    std::vector<CUtensorMap> maps;
    uint64_t part_bytes = 0;
    mp.ops.clear();
    for (const Launch& x : p.launches) {
        MkOp op;
        memset(&op, 0, sizeof op);
        op.layer = x.layer;
        op.dep = (int32_t)mp.ops.size() - 1;
        switch (x.kind) {
            case K_EMBED:
                op.kind = MK_EMBED;
                op.embed = x.embed;
                op.n_tasks = x.embed.T;
                break;
            case K_LN:
                op.kind = MK_LN;
                op.ln = x.ln;
                op.n_tasks = (x.ln.rows + 3) / 4;
                break;
            case K_GEMV:
                op.kind = MK_GEMV;
                op.gemv = x.gemv;
                op.n_tasks = (x.gemv.N + 63) / 64;
                break;
            case K_ATTN:
                op.kind = MK_ATTN;
                op.attn = x.attn;
                op.attn.layer = x.layer;
                op.n_tasks = x.attn.H * ((x.attn.T + 15) / 16);
                break;
            case K_GEMM: {
                op.kind = MK_GEMM;
                op.gemm = x.gemm;
                const MkTiling t = mega_tiling(x.gemm.M, x.gemm.n_pad, x.gemm.K / 64, sms);
                op.tt = t.tt;
                op.splits = t.splits;
                op.kt_per = t.kt_per;
                op.n_rt = (x.gemm.n_pad + 127) / 128;
                op.n_tt = (x.gemm.M + t.tt - 1) / t.tt;
                op.n_tasks = op.n_rt * op.n_tt * op.splits;
                op.tmap = (uint32_t)maps.size();
                CUtensorMap tm;
                if (!make_tmap_act(&tm, x.abase, x.gemm.M, x.a_cols, x.a_cols, t.tt))
                    return fail(FSW_ECUDA, "plan: cuTensorMapEncodeTiled failed (mega, layer %d)", x.layer);
                maps.push_back(tm);
                if (op.n_rt * op.n_tt * 32 > kGemmCtrs) return FSW_OK;  // tile counters 128 B apart
                if (op.splits > 1) part_bytes = std::max<uint64_t>(part_bytes, (uint64_t)op.n_rt * op.n_tt * op.splits * 128 * kMkTT * 4);
                break;
            }
            default:
                return FSW_OK;
        }
        mp.ops.push_back(op);
    }
    if (mp.ops.empty()) return FSW_OK;
    const uint64_t part_off = align_up(p.ws_bytes, 1024);
    if (part_off + part_bytes > g.ws_bytes) return FSW_OK;  // no room: the per-op kernels run it
    p.ws_bytes = align_up(part_off + part_bytes, 1024);
    mp.part = reinterpret_cast<float*>(g.ws + part_off);
    // per-op counters and per-CTA epoch words, 128 B apart (mega.cu kMkLine)
    CU(cudaMalloc(&mp.op_cnt, 128 * (mp.ops.size() + (size_t)mp.ctas)));
    if (!maps.empty()) {
        CU(cudaMalloc(&mp.tmaps, sizeof(CUtensorMap) * maps.size()));
        CU(cudaMemcpy(mp.tmaps, maps.data(), sizeof(CUtensorMap) * maps.size(), cudaMemcpyHostToDevice));
    }
    if (getenv("FSW_MEGA_STAMPS") && atoi(getenv("FSW_MEGA_STAMPS"))) {
        const size_t n = mp.ops.size() * (size_t)mp.ctas * 8;
        CU(cudaMalloc(&mp.stamps, n * sizeof(unsigned long long)));
        CU(cudaMemset(mp.stamps, 0, n * sizeof(unsigned long long)));
        set_mega_stamps(mp.stamps);  // one model at a time: the last planned model's buffer
    }
    mp.on = true;
    return FSW_OK;
}

// ==========================================================================================
// plan: workspace layout + kernel list for one (model, GPU)
// ==========================================================================================
fsw_status build_plan(fsw_ctx* c, Model& m, int gi) {
    Gpu& g = c->gpus[gi];
    auto p = std::make_unique<Plan>();
    const size_t ns = m.slots.size();
    // which f32 slots feed a GEMM (need a bf16 shadow)
    std::vector<bool> need_shadow(ns, false);
    uint64_t scratch = 0;  // im2col scratch
    for (auto& L : m.layers) {
        if (L.op == FSW_OP_LINEAR && linear_is_gemm(m, L) && m.slots[L.in0].dtype == FSW_DT_F32) need_shadow[L.in0] = true;
        if (L.op == FSW_OP_CONV2D) {
            const fsw_slot& si = m.slots[L.in0];
            const fsw_slot& so = m.slots[L.out];
            const fsw_tensor& W = m.tensors[m.refs[L.first_ref]].t;
            if (conv_path(W, L, si, so) == CONV_IM2COL) {
                const uint64_t K = (uint64_t)W.shape[1] * W.shape[2] * W.shape[3];
                scratch = std::max(scratch, (uint64_t)so.shape[0] * so.shape[1] * align_up(K, 64) * 2);
            }
        }
    }
    uint64_t off = 0;
    p->slot_off.resize(ns);
    p->shadow_off.assign(ns, -1);
    const uint64_t stage_input_off = kStageHdr;  // input slot lives in the device stage
    for (size_t i = 0; i < ns; ++i) {
        if ((int)i == m.input_slot) {
            p->slot_off[i] = UINT64_MAX;
            continue;
        }
        p->slot_off[i] = off;
        off = align_up(off + slot_bytes(m.slots[i]), 1024);
        if (need_shadow[i]) {
            p->shadow_off[i] = (int64_t)off;
            off = align_up(off + slot_numel(m.slots[i]) * 2, 1024);
        }
    }
    const uint64_t scratch_off = off;
    off = align_up(off + scratch, 1024);
    p->ws_bytes = off;
    if (off > g.ws_bytes) return fail(FSW_ENOMEM, "plan: workspace needs %llu bytes > %llu", (unsigned long long)off, (unsigned long long)g.ws_bytes);
    if (m.input_bytes + kStageHdr > g.stage_cap || m.output_bytes > g.out_cap) return fail(FSW_ENOMEM, "plan: input/output too large");

    auto sptr = [&](int s) -> uint8_t* {
        if (s < 0) return nullptr;
        if (s == m.input_slot) return g.dstage + stage_input_off;
        return g.ws + p->slot_off[s];
    };
    auto shadow = [&](int s) -> uint16_t* {
        return (s >= 0 && p->shadow_off[s] >= 0) ? reinterpret_cast<uint16_t*>(g.ws + p->shadow_off[s]) : nullptr;
    };
    auto ref = [&](const fsw_layer& L, uint32_t j) -> const TensorInfo& { return m.tensors[m.refs[L.first_ref + j]]; };
    uint64_t part_bytes = 0;  // split-K partial tiles, shared by all GEMMs of the plan
    auto set_tiling = [&](GemmArgs& a, uint64_t m_tiles, uint32_t m_rows, uint32_t a_kt_bytes) {
        // one-wave cluster capacity for every (BN, cluster size), queried once (the pool's GPUs are alike)
        static const ClusterCap max_cl = []() {
            ClusterCap t{};
            for (int bn : {16, 32, 64, 128})
                for (int cz = 2; cz <= 8; ++cz) t[bn / 16][cz] = gemm_max_active_clusters(bn, cz);
            return t;
        }();
        Tiling t = choose_tiling(m_tiles, a.n_pad, a.K / 64, a_kt_bytes, m_rows, &max_cl);
        // A/B hook (in-graph tiling sweep, tools/gemm_graph_sweep.sh): FSW_GEMM_FORCE="bn:splits:cluster" for the
        // linears whose chosen tiling is not split-K (bn 0 = keep); a forced tiling that does not fit is ignored
        static const char* force = getenv("FSW_GEMM_FORCE");
        if (force && t.splits == 1 && !a.conv && m_rows == 128) {
            int fbn = 0, fs = 1, fc = 0;
            if (sscanf(force, "%d:%d:%d", &fbn, &fs, &fc) >= 2) {
                const int bn = fbn ? fbn : t.bn;
                const uint32_t kt = a.K / 64, kp = (kt + fs - 1) / fs;
                const uint64_t ctas = m_tiles * (a.n_pad / bn) * (uint64_t)fs;
                const bool fits = a.n_pad % bn == 0 && fs >= 1 && (kt + kp - 1) / kp == (uint32_t)fs && ctas <= 148 &&
                                  (!fc || (fs >= 2 && fs <= 8 && ctas <= (uint64_t)max_cl[bn / 16][fs] * fs));
                if (fits) t = Tiling{bn, (uint32_t)fs, kp, fc != 0};
            }
        }
        a.bn = t.bn;
        a.m_rows = m_rows;
        a.splits = t.splits;
        a.kt_per = t.kt_per;
        a.ctr = g.gemm_ctr;
        static const bool no_cz = getenv("FSW_GEMM_NO_CLUSTER_SPLIT") != nullptr;  // A/B hook
        a.cz = t.cluster && !no_cz ? t.splits : 0;
        // A multicast across an N cluster (plain GEMMs; the implicit-conv A box is not row-split)
        a.mc = 1;
        static const uint32_t mc_max = getenv("FSW_GEMM_MC") ? (uint32_t)atoi(getenv("FSW_GEMM_MC")) : 1;
        for (uint32_t c : {8u, 4u, 2u})
            if (!a.cz && c <= mc_max && m_rows == 128 && (a.n_pad / t.bn) % c == 0) {
                a.mc = c;
                break;
            }
        const uint64_t tiles = m_tiles * (a.n_pad / t.bn);
        if (t.splits > 1) part_bytes = std::max<uint64_t>(part_bytes, tiles * t.splits * 128 * t.bn * 4);
        return tiles <= kGemmCtrs;
    };

    CU(cudaSetDevice(g.dev));
    for (uint32_t li = 0; li < m.layers.size(); ++li) {
        const fsw_layer& L = m.layers[li];
        const fsw_slot& si = m.slots[L.in0];
        const fsw_slot& so = m.slots[L.out];
        Launch x{};
        x.layer = (int)li;
        switch (L.op) {
            case FSW_OP_EMBED: {
                x.kind = K_EMBED;
                EmbedArgs& a = x.embed;
                a.ids = reinterpret_cast<const int32_t*>(sptr(L.in0));
                a.n_tables = L.attr[0];
                for (int j = 0; j < a.n_tables; ++j) {
                    a.table_off[j] = ref(L, j).st_off;
                    a.table_rows[j] = ref(L, j).t.shape[0];
                    a.rule[j] = L.attr[1 + j];
                }
                a.T = so.shape[0];
                a.C = so.shape[1];
                if (so.dtype == FSW_DT_F32) {
                    a.out = reinterpret_cast<float*>(sptr(L.out));
                    a.out_bf16 = shadow(L.out);
                } else {
                    a.out_bf16 = reinterpret_cast<uint16_t*>(sptr(L.out));
                }
                break;
            }
            case FSW_OP_LAYERNORM: {
                x.kind = K_LN;
                LnArgs& a = x.ln;
                a.in = reinterpret_cast<const float*>(sptr(L.in0));
                a.C = slot_cols(si);
                a.rows = (uint32_t)slot_rows(si);
                float eps;
                memcpy(&eps, &L.attr[0], 4);
                a.eps = eps;
                a.g_off = ref(L, 0).st_off;
                a.b_off = ref(L, 1).st_off;
                if (so.dtype == FSW_DT_F32) {
                    a.out_f32 = reinterpret_cast<float*>(sptr(L.out));
                    a.out_bf16 = shadow(L.out);
                } else {
                    a.out_bf16 = reinterpret_cast<uint16_t*>(sptr(L.out));
                }
                break;
            }
            case FSW_OP_LINEAR: {
                const TensorInfo& W = ref(L, 0);
                const bool has_b = L.n_refs > 1;
                if (!linear_is_gemm(m, L)) {
                    x.kind = K_GEMV;
                    GemvArgs& a = x.gemv;
                    a.x = sptr(L.in0);
                    a.x_bf16 = si.dtype == FSW_DT_BF16;
                    a.ldx = slot_cols(si);
                    a.r0 = (uint32_t)L.attr[1];
                    a.rows = (uint32_t)linear_rows(m, L);
                    a.K = W.t.shape[1];
                    a.N = W.t.shape[0];
                    a.w_off = W.st_off;
                    a.has_bias = has_b;
                    a.b_off = has_b ? ref(L, 1).st_off : 0;
                    a.act = L.attr[0];
                    a.res = sptr(L.in1);
                    a.res_bf16 = L.in1 >= 0 && m.slots[L.in1].dtype == FSW_DT_BF16;
                    a.out = sptr(L.out);
                    a.out_bf16 = so.dtype == FSW_DT_BF16;
                    a.out2 = shadow(L.out);
                } else {
                    x.kind = K_GEMM;
                    GemmArgs& a = x.gemm;
                    a.M = (uint32_t)slot_rows(si);
                    a.N = W.rows;
                    a.K = W.cols_pad;
                    a.n_pad = W.rows_pad;
                    a.w_off = W.st_off;
                    a.has_bias = has_b;
                    a.b_off = has_b ? ref(L, 1).st_off : 0;
                    a.act = L.attr[0];
                    a.res = sptr(L.in1);
                    a.res_bf16 = L.in1 >= 0 && m.slots[L.in1].dtype == FSW_DT_BF16;
                    a.ld_res = a.N;
                    a.out = sptr(L.out);
                    a.out_bf16 = so.dtype == FSW_DT_BF16;
                    a.ld_out = a.N;
                    a.out2 = shadow(L.out);
                    const void* abase = si.dtype == FSW_DT_BF16 ? (const void*)sptr(L.in0) : (const void*)shadow(L.in0);
                    // Opt-in (FSW_GEMM_2CTA=1): the 2-CTA swap-AB GEMM for the wide batch-1 transformer linears
                    // (<= 128 tokens, K <= 1600, N >= 768), the token tile putting the number of CTA pairs
                    // nearest 40.  Back to back on L2-resident weights it beat k_gemm by 14-20 %
                    // (profiles/r01/gemm2cta_proto_tokens.txt), but inside the invoke graph, weights from
                    // HBM, it is slower (resident BERT-base 0.702 vs 0.586 ms, profiles/r01/gemm2cta_in_graph.txt),
                    // so k_gemm stays the default.
                    static const bool use2 = getenv("FSW_GEMM_2CTA") != nullptr;
                    uint32_t pt = 0;
                    if (use2 && g.wmap_ok && a.M <= 128 && a.K / 64 <= 25 && a.N >= 768) {
                        const uint32_t ntile = (a.n_pad + 127) / 128;
                        long best = 1 << 30;
                        static const long target = getenv("FSW_GEMM_2CTA_PAIRS") ? atol(getenv("FSW_GEMM_2CTA_PAIRS")) : 40;
                        for (uint32_t t : {16u, 32u, 64u, 128u}) {
                            const long pairs = (long)ntile * ((a.M + t - 1) / t), dist = pairs > target ? pairs - target : target - pairs;
                            if (dist < best) best = dist, pt = t;
                        }
                    }
                    // Weight-stationary swap-AB GEMM (k_gemm_ws) for the narrow batch-1 linears (choose_ws_tiling);
                    // FSW_GEMM_WS=0 turns it off, =2 allows it for every width (A/B hooks)
                    // (off under FSW_MEGA=1: the persistent kernel takes its GEMMs from the k_gemm plan)
                    static const int ws_mode = getenv("FSW_MEGA") && atoi(getenv("FSW_MEGA")) == 1 ? 0
                                               : getenv("FSW_GEMM_WS") ? atoi(getenv("FSW_GEMM_WS")) : 1;
                    WsTiling wt{0, 0, 0, 0, false};
                    if (ws_mode && !pt && a.N % 4 == 0) wt = choose_ws_tiling(a.M, a.n_pad, a.K / 64, ws_mode == 2);
                    if (wt.ok) {
                        a.ws_tt = wt.tt;
                        a.ws_stages = wt.stages;
                        a.bn = 128;
                        a.m_rows = wt.tt;
                        a.splits = wt.splits;
                        a.kt_per = wt.kt_per;
                        a.mc = 1;
                        a.cz = wt.splits > 1 ? wt.splits : 0;
                        if (!make_tmap_act(&x.tmap, abase, a.M, slot_cols(si), slot_cols(si), wt.tt))
                            return fail(FSW_ECUDA, "plan: cuTensorMapEncodeTiled failed (layer %u)", li);
                    } else if (pt) {
                        a.pair_t = pt;
                        a.wpool = g.pool;
                        a.bn = 128;
                        a.m_rows = pt;
                        a.splits = 1;
                        a.kt_per = a.K / 64;
                        a.mc = 1;
                        a.cz = 0;
                        if (!make_tmap_act(&x.tmap, abase, a.M, slot_cols(si), slot_cols(si), pt / 2))
                            return fail(FSW_ECUDA, "plan: cuTensorMapEncodeTiled failed (layer %u)", li);
                    } else {
                        x.abase = abase;
                        x.a_cols = slot_cols(si);
                        set_tiling(a, (a.M + 127) / 128, 128, 128 * 128);
                        if (!make_tmap_act(&x.tmap, abase, a.M, slot_cols(si), slot_cols(si), 128 / a.mc))
                            return fail(FSW_ECUDA, "plan: cuTensorMapEncodeTiled failed (layer %u)", li);
                    }
                }
                break;
            }
            case FSW_OP_ATTENTION: {
                x.kind = K_ATTN;
                x.attn = {reinterpret_cast<const uint16_t*>(sptr(L.in0)), reinterpret_cast<uint16_t*>(sptr(L.out)),
                          si.shape[0], (uint32_t)L.attr[0], (uint32_t)L.attr[1], L.attr[2]};
                // tcgen05 attention for T <= 128, head width 64 (FSW_ATTN_TC: 1 on, 0 off)
                static const int attn_tc = getenv("FSW_ATTN_TC") ? atoi(getenv("FSW_ATTN_TC")) : 0;
                if (attn_tc && attention_tc_ok(x.attn)) {
                    const uint64_t cols = 3ull * x.attn.H * x.attn.dh;
                    if (!make_tmap_act(&x.tmap, x.attn.qkv, x.attn.T, cols, cols, 128))
                        return fail(FSW_ECUDA, "plan: cuTensorMapEncodeTiled failed (attention, layer %u)", li);
                    x.attn_tc = true;
                }
                break;
            }
            case FSW_OP_CONV2D: {
                const TensorInfo& W = ref(L, 0);
                const uint32_t R = W.t.shape[1], S = W.t.shape[2], Cin = W.t.shape[3];
                const ConvPath path = conv_path(W.t, L, si, so);
                const uint32_t P = so.shape[0], Q = so.shape[1];
                const void* abase = sptr(L.in0);
                uint32_t acols = Cin;
                if (path == CONV_IM2COL) {
                    Launch y{};
                    y.kind = K_IM2COL;
                    y.layer = (int)li;
                    y.im2col = {reinterpret_cast<const uint16_t*>(sptr(L.in0)), si.shape[0], si.shape[1], Cin,
                                reinterpret_cast<uint16_t*>(g.ws + scratch_off), P, Q, R, S, (uint32_t)L.attr[1],
                                (uint32_t)L.attr[2], R * S * Cin, W.cols_pad};
                    p->launches.push_back(y);
                    abase = g.ws + scratch_off;
                    acols = W.cols_pad;
                }
                x.kind = K_GEMM;
                GemmArgs& a = x.gemm;
                a.M = P * Q;
                a.N = W.rows;
                a.K = W.cols_pad;
                a.n_pad = W.rows_pad;
                a.w_off = W.st_off;
                a.has_bias = 1;
                a.b_off = ref(L, 1).st_off;
                a.act = L.attr[0];
                a.res = sptr(L.in1);
                a.res_bf16 = 1;
                a.ld_res = a.N;
                a.out = sptr(L.out);
                a.out_bf16 = 1;
                a.ld_out = a.N;
                a.out2 = nullptr;
                if (path == CONV_IMPLICIT) {
                    const uint32_t Hb = conv_rows_per_tile(P, Q);
                    a.conv = 1;
                    a.Q = Q;
                    a.stride = (uint32_t)L.attr[1];
                    a.pad = (uint32_t)L.attr[2];
                    a.S = S;
                    a.Cin = Cin;
                    a.Hb = Hb;
                    set_tiling(a, (P + Hb - 1) / Hb, Hb * Q, Hb * Q * 128);
                    if (!make_tmap_conv(&x.tmap, abase, si.shape[0], si.shape[1], Cin, Q, Hb, a.stride))
                        return fail(FSW_ECUDA, "plan: conv tensor map failed (layer %u)", li);
                } else {
                    set_tiling(a, (a.M + 127) / 128, 128, 128 * 128);
                    if (!make_tmap_act(&x.tmap, abase, a.M, acols, acols, 128 / a.mc))
                        return fail(FSW_ECUDA, "plan: cuTensorMapEncodeTiled failed (layer %u)", li);
                }
                break;
            }
            case FSW_OP_MAXPOOL:
            case FSW_OP_AVGPOOL: {
                x.kind = L.op == FSW_OP_MAXPOOL ? K_MAXPOOL : K_AVGPOOL;
                PoolArgs& a = x.pool;
                a.in = reinterpret_cast<const uint16_t*>(sptr(L.in0));
                a.H = si.shape[0];
                a.W = si.shape[1];
                a.C = si.shape[2];
                if (L.op == FSW_OP_MAXPOOL) {
                    a.P = so.shape[0];
                    a.Q = so.shape[1];
                    a.k = L.attr[0];
                    a.stride = L.attr[1];
                    a.pad = L.attr[2];
                    a.out = reinterpret_cast<uint16_t*>(sptr(L.out));
                } else {
                    a.out_f32 = reinterpret_cast<float*>(sptr(L.out));
                }
                break;
            }
        }
        p->launches.push_back(x);
    }
    {  // L2 prefetch of the next GEMM's weights in resident invokes (FSW_GEMM_PF=0: off) and the chosen tilings
       // (FSW_PLAN_VERBOSE=1)
        // default on: resident BERT-base 0.476 -> 0.472 ms, GPT-2-XL 2.730 -> 2.682 ms (profiles/r02/gemm/ws_sweep.txt)
        static const bool pf = !(getenv("FSW_GEMM_PF") && atoi(getenv("FSW_GEMM_PF")) == 0);
        static const bool verbose = getenv("FSW_PLAN_VERBOSE") && atoi(getenv("FSW_PLAN_VERBOSE")) == 1;
        static const int ws_trig = getenv("FSW_WS_TRIGGER") ? atoi(getenv("FSW_WS_TRIGGER")) : 0;
        for (size_t i = 0; i < p->launches.size(); ++i) {
            Launch& x = p->launches[i];
            if (x.kind != K_GEMM) continue;
            GemmArgs& a = x.gemm;
            // linears only: ResNet-50's convolutions measured 2 % slower with it (0.405 -> 0.412 ms)
            if (pf && !a.pair_t && m.layers[x.layer].op == FSW_OP_LINEAR)
                for (size_t j = i + 1; j < p->launches.size(); ++j)
                    if (p->launches[j].kind == K_GEMM && m.layers[p->launches[j].layer].op == FSW_OP_LINEAR) {
                        const GemmArgs& b = p->launches[j].gemm;
                        a.pf_off = b.w_off;
                        a.pf_bytes = (uint64_t)b.K * b.n_pad * 2;
                        break;
                    }
            // early PDL release (A/B hook FSW_WS_TRIGGER: 0 = after the MMAs, 1 = at entry for every k_gemm_ws,
            // 2 = at entry when the successor is not a GEMM)
            if (a.ws_tt && ws_trig) {
                const bool next_gemm = i + 1 < p->launches.size() && p->launches[i + 1].kind == K_GEMM;
                a.trig_early = ws_trig == 1 || !next_gemm;
            }
            if (verbose)
                fprintf(stderr, "[fsw plan] layer %d GEMM M=%u N=%u K=%u: %s tt/bn=%u splits=%u kt_per=%u stages=%u cz=%u smem=%u pf=%llu\n",
                        x.layer, a.M, a.N, a.K, a.ws_tt ? "ws" : a.pair_t ? "2cta" : "k_gemm", a.ws_tt ? a.ws_tt : (uint32_t)a.bn,
                        a.splits, a.kt_per, a.ws_stages, a.cz, a.ws_tt ? gemm_ws_smem(a.ws_tt, a.ws_stages ? a.ws_stages : a.kt_per, a.splits) : 0u, (unsigned long long)a.pf_bytes);
        }
    }
    // LayerNorm folded into the k_gemm_ws launches around it (FSW_LN_FUSE=1; DESIGN §5 "folded LayerNorm"): the
    // producing GEMM writes per-token partial statistics, the GEMM reading the LN output as its operand normalises
    // on load, the GEMM reading it as a residual recomputes it from the pre-LN stream; the LN launch goes.  Only
    // where every reader of the LN output is such a GEMM and the pre-LN stream outlives them (post-LN BERT: both
    // LayerNorms of every layer but the last).
    static const int ln_fuse = getenv("FSW_LN_FUSE") ? atoi(getenv("FSW_LN_FUSE")) : 0;
    if (ln_fuse) {
        std::vector<uint8_t> drop(p->launches.size(), 0);
        auto pow2 = [](uint32_t v) { return v && !(v & (v - 1)); };
        for (size_t i = 1; i < p->launches.size(); ++i) {
            Launch& ln = p->launches[i];
            Launch& pr = p->launches[i - 1];
            if (ln.kind != K_LN || pr.kind != K_GEMM || drop[i - 1]) continue;
            const GemmArgs& pa = pr.gemm;
            const uint32_t C = ln.ln.C, M = ln.ln.rows;
            if (!pa.ws_tt || pa.ws_stages || (const void*)pa.out != (const void*)ln.ln.in || pa.out_bf16 || pa.N != C || pa.n_pad != C ||
                C % 128 || !pow2(pa.splits) || pa.splits > 8 || pa.M != M || pa.st_out)
                continue;
            const uint32_t slots = (C / 128) * pa.splits;
            if (slots > 64) continue;
            const int s_in = m.layers[ln.layer].in0, s_out = m.layers[ln.layer].out;
            if (s_out == m.output_slot || s_in == m.output_slot) continue;
            int a_cons = -1, r_cons = -1;
            bool ok = true, in_live = true;
            for (size_t j = i + 1; j < p->launches.size() && ok; ++j) {
                const fsw_layer& L = m.layers[p->launches[j].layer];
                const Launch& y = p->launches[j];
                const bool reads = L.in0 == s_out || L.in1 == s_out;
                if (reads && !in_live) ok = false;  // the pre-LN stream was overwritten before this reader
                if (L.in0 == s_out) {
                    const GemmArgs& ya = y.gemm;
                    if (a_cons >= 0 || y.kind != K_GEMM || !ya.ws_tt || ya.ws_stages || ya.M != M || ya.K != C || ya.ln_x ||
                        y.wait_layer2 >= 0 ||  // one extra readiness wait per launch (the LayerNorm's weights)
                        gemm_ws_smem(ya.ws_tt, ya.kt_per, ya.splits) + 1024 > 184 * 1024)
                        ok = false;
                    a_cons = (int)j;
                }
                if (L.in1 == s_out) {
                    const GemmArgs& ya = y.gemm;
                    if (r_cons >= 0 || y.kind != K_GEMM || !ya.ws_tt || ya.ws_stages || ya.res_bf16 || ya.ld_res != C || ya.M != M ||
                        ya.res_musig || y.wait_layer2 >= 0)
                        ok = false;
                    r_cons = (int)j;
                }
                if (L.out == s_out) break;  // rewritten: later readers see the new value
                if (L.out == s_in) {
                    if (reads) ok = false;  // it would overwrite the pre-LN stream it normalises
                    in_live = false;
                }
            }
            if (!ok || a_cons < 0 || a_cons == r_cons) continue;
            // scratch: the partials [slots][M] and (μ, rstd) [M]
            const uint64_t st_off = align_up(off, 256), ms_off = align_up(st_off + (uint64_t)slots * M * 8, 256);
            off = align_up(ms_off + (uint64_t)M * 8, 1024);
            float2* st = reinterpret_cast<float2*>(g.ws + st_off);
            float2* ms = reinterpret_cast<float2*>(g.ws + ms_off);
            pr.gemm.st_out = st;
            GemmArgs& ca = p->launches[a_cons].gemm;
            ca.ln_x = ln.ln.in;
            ca.ln_st = st;
            ca.ln_slots = slots;
            ca.ln_cnt = 128 / pa.splits;
            ca.ln_g_off = ln.ln.g_off;
            ca.ln_b_off = ln.ln.b_off;
            ca.ln_eps = ln.ln.eps;
            ca.ln_musig = r_cons >= 0 ? ms : nullptr;
            p->launches[a_cons].wait_layer2 = ln.layer;
            if (r_cons >= 0) {
                GemmArgs& ra = p->launches[r_cons].gemm;
                ra.res = ln.ln.in;
                ra.res_bf16 = 0;
                ra.ld_res = C;
                ra.res_musig = ms;
                ra.res_g_off = ln.ln.g_off;
                ra.res_b_off = ln.ln.b_off;
                p->launches[r_cons].wait_layer2 = ln.layer;
            }
            drop[i] = 1;
            if (getenv("FSW_PLAN_VERBOSE") && atoi(getenv("FSW_PLAN_VERBOSE")) == 1)
                fprintf(stderr, "[fsw plan] LayerNorm layer %d folded: statistics from layer %d (%u slots), operand of layer %d, residual of layer %d\n",
                        ln.layer, pr.layer, slots, p->launches[a_cons].layer, r_cons >= 0 ? p->launches[r_cons].layer : -1);
        }
        std::vector<Launch> kept;
        for (size_t i = 0; i < p->launches.size(); ++i)
            if (!drop[i]) kept.push_back(p->launches[i]);
        p->launches.swap(kept);
    }
    // split-K partials live after the activations and the im2col scratch
    const uint64_t part_off = align_up(off, 1024);
    p->ws_bytes = align_up(part_off + part_bytes, 1024);
    if (p->ws_bytes > g.ws_bytes)
        return fail(FSW_ENOMEM, "plan: workspace needs %llu bytes > %llu", (unsigned long long)p->ws_bytes, (unsigned long long)g.ws_bytes);
    for (Launch& x : p->launches)
        if (x.kind == K_GEMM) x.gemm.part = reinterpret_cast<float*>(g.ws + part_off);
    {
        const fsw_status ms = build_mega(c, m, *p, g);
        if (ms != FSW_OK) return ms;
    }
    p->built = true;
    m.plans[gi] = std::move(p);
    return FSW_OK;
}

