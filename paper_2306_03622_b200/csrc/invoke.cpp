// invoke.cpp — pool residency (heavy / light, invalidation, extents, partial caching, eviction),
// Algorithm 1 placement and fsw_invoke / fsw_invoke_ex.
#include "rt_internal.h"

// ==========================================================================================
// pool residency
// ==========================================================================================
// Heavy / light: set by the caller, else heavy_by_slo (policy.h) on the
// swap's added latency = mean cold − mean resident device time, measured; before both were measured
// the swap time is estimated from the bytes that cross the link (the coded store for a link-coded model)
// at 55 GB/s (the copy engine's measured PCIe rate) and the resident time as 0.
bool model_heavy(const fsw_ctx* c, const Model& m) {
    if (m.heavy >= 0) return m.heavy != 0;
    double swap_ms, res_ms = 0.0;
    if (m.n_cold_runs && m.n_warm_runs) {
        res_ms = m.warm_ms_sum / (double)m.n_warm_runs;
        swap_ms = std::max(0.0, m.cold_ms_sum / (double)m.n_cold_runs - res_ms);
    } else {
        swap_ms = (double)(m.zstore ? m.zbytes : m.store_bytes) / 55e6;
    }
    return heavy_by_slo(swap_ms, res_ms, m.slo_ms, c->queue_budget_ms, c->heavy_theta);
}

extern "C" fsw_status fsw_model_set_slo(fsw_ctx* c, uint32_t id, double deadline_ms) {
    if (!c || !(deadline_ms > 0.0)) return fail(FSW_EINVAL, "model_set_slo: bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    Model* m = c->models.size() > id ? c->models[id].get() : nullptr;
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    m->slo_ms = m->slo_ms > 0.0 ? std::min(m->slo_ms, deadline_ms) : deadline_ms;
    return FSW_OK;
}

extern "C" fsw_status fsw_set_heavy_policy(fsw_ctx* c, double theta, double queue_budget_ms) {
    if (!c || !(theta > 0.0) || !(queue_budget_ms >= 0.0)) return fail(FSW_EINVAL, "set_heavy_policy: bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    c->heavy_theta = theta;
    c->queue_budget_ms = queue_budget_ms;
    return FSW_OK;
}

extern "C" fsw_status fsw_model_set_heavy(fsw_ctx* c, uint32_t id, int32_t heavy) {
    if (!c || heavy < -1 || heavy > 1) return fail(FSW_EINVAL, "model_set_heavy: bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    Model* m = c->models.size() > id ? c->models[id].get() : nullptr;
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    m->heavy = heavy;
    return FSW_OK;
}

extern "C" fsw_status fsw_model_is_heavy(fsw_ctx* c, uint32_t id, int32_t* heavy) {
    if (!c || !heavy) return fail(FSW_EINVAL, "model_is_heavy: bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    Model* m = c->models.size() > id ? c->models[id].get() : nullptr;
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    *heavy = model_heavy(c, *m) ? 1 : 0;
    return FSW_OK;
}

// Eviction invalidates, it never copies back.  The suffix (or whole model)
// extent goes; with keep_prefix a cached prefix stays (partial caching), else it goes too.
void invalidate(fsw_ctx* c, Model& m, int gi, bool keep_prefix) {
    if (m.extent[gi] >= 0) {
        fsw_arena_free(c->gpus[gi].arena, (uint64_t)m.extent[gi]);
        m.extent[gi] = -1;
    }
    m.complete[gi] = 0;
    if (!keep_prefix && m.pextent[gi] >= 0) {
        fsw_arena_free(c->gpus[gi].arena, (uint64_t)m.pextent[gi]);
        m.pextent[gi] = -1;
        m.pvalid[gi] = 0;
    }
}

// Pool extents for a cold invoke of m on GPU gi: the suffix (or the whole model), plus the prefix
// when m caches one that is not here yet.  Makes room by evicting idle models, heaviness-aware LRU
// (PAPER.md:885-897): their suffixes / whole extents first (cached prefixes survive), and only
// then cached prefixes, least recently used first.
static fsw_status ensure_extent(fsw_ctx* c, Model& m, int gi) {
    Gpu& g = c->gpus[gi];
    const uint64_t need_p = m.split && m.pextent[gi] < 0 ? m.split : 0, need_s = m.store_bytes - m.split;
    for (;;) {
        uint64_t po = 0, so = 0;
        if (need_p == 0 || fsw_arena_alloc(g.arena, need_p, &po) == FSW_OK) {
            if (fsw_arena_alloc(g.arena, need_s, &so) == FSW_OK) {
                if (need_p) {
                    m.pextent[gi] = (int64_t)po;
                    m.pvalid[gi] = 0;
                }
                m.extent[gi] = (int64_t)so;
                m.complete[gi] = 0;  // a resident copy only once the cold invoke succeeded
                return FSW_OK;
            }
            if (need_p) fsw_arena_free(g.arena, po);
        }
        std::vector<Model*> cand;
        std::vector<uint8_t> heavy, in_use;
        std::vector<uint32_t> copies;
        std::vector<uint64_t> last;
        for (auto& o : c->models) {
            if (!o || o.get() == &m || o->extent[gi] < 0) continue;
            cand.push_back(o.get());
            heavy.push_back(model_heavy(c, *o));
            uint32_t k = 0;
            for (size_t i = 0; i < o->extent.size(); ++i) k += o->extent[i] >= 0 && o->complete[i];
            copies.push_back(k);
            last.push_back(o->last_use[gi]);
            in_use.push_back(o->inflight != 0);
        }
        const std::vector<uint32_t> order = eviction_order(heavy, copies, last, in_use);
        if (!order.empty()) {
            invalidate(c, *cand[order[0]], gi, /*keep_prefix=*/true);
            g.n_evictions++;
            g.n_evictions_heavy += heavy[order[0]];
            continue;
        }
        Model* pv = nullptr;  // then the least recently used idle cached prefix
        for (auto& o : c->models)
            if (o && o.get() != &m && o->pextent[gi] >= 0 && o->extent[gi] < 0 && o->inflight == 0 &&
                (!pv || o->last_use[gi] < pv->last_use[gi]))
                pv = o.get();
        if (!pv)
            return fail(FSW_ENOMEM, "pool on gpu %d cannot hold %llu bytes even after evicting every idle model", g.dev,
                        (unsigned long long)(need_p + need_s));
        invalidate(c, *pv, gi);
        g.n_evictions++;
    }
}

// Partial-parameter caching (the paper's future work).
extern "C" fsw_status fsw_model_set_cache_prefix(fsw_ctx* c, uint32_t id, uint64_t bytes, uint64_t* actual) {
    if (!c) return fail(FSW_EINVAL, "NULL ctx");
    std::lock_guard<std::mutex> lk(c->mu);
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    for (size_t i = 0; i < m->extent.size(); ++i)
        if (m->extent[i] >= 0 || m->pextent[i] >= 0)
            return fail(FSW_ESTATE, "model %u is resident on gpu %zu: evict it before changing its cached prefix", id, i);
    // the largest layer boundary <= bytes that leaves a non-empty suffix
    uint64_t split = 0;
    for (size_t li = 0; li < m->layers.size(); ++li)
        if (m->region_off[li] <= bytes && m->region_off[li] < m->store_bytes) split = m->region_off[li];
    m->split = split;  // graphs and copy plans are keyed by the swapped range and the split
    if (actual) *actual = split;
    return FSW_OK;
}

extern "C" fsw_status fsw_evict_ex(fsw_ctx* c, uint32_t id, int32_t gpu, uint32_t flags) {
    if (!c) return fail(FSW_EINVAL, "NULL ctx");
    std::lock_guard<std::mutex> lk(c->mu);
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (m->inflight) return fail(FSW_EBUSY, "model %u has an invoke in flight", id);
    if (gpu >= (int)c->gpus.size() || gpu < -1) return fail(FSW_EINVAL, "bad gpu %d", gpu);
    const bool keep = (flags & FSW_EVICT_KEEP_PREFIX) != 0;
    if (gpu >= 0) {
        if (m->extent[gpu] < 0 && (keep || m->pextent[gpu] < 0))
            return fail(FSW_ESTATE, "model %u is not resident on gpu %d", id, gpu);
        invalidate(c, *m, gpu, keep);
        c->gpus[gpu].n_evictions++;
        return FSW_OK;
    }
    for (size_t i = 0; i < c->gpus.size(); ++i)
        if (m->extent[i] >= 0 || (!keep && m->pextent[i] >= 0)) {
            invalidate(c, *m, (int)i, keep);
            c->gpus[i].n_evictions++;
        }
    return FSW_OK;
}

extern "C" fsw_status fsw_evict(fsw_ctx* c, uint32_t id, int32_t gpu) { return fsw_evict_ex(c, id, gpu, 0); }

// ==========================================================================================
// invoke
// ==========================================================================================
// Algorithm 1 over the pool's live state; NVLink through NVSwitch is uniform.
static Decision pick_gpu(fsw_ctx* c, Model& m) {
    const size_t n = c->gpus.size();
    std::vector<uint8_t> avail(n), hosts(n), loading(n);
    for (size_t i = 0; i < n; ++i) {
        avail[i] = !c->gpus[i].busy;
        hosts[i] = m.extent[i] >= 0 && m.complete[i];  // an extent still being swapped in is no copy
        loading[i] = (uint8_t)c->gpus[i].loading;
    }
    std::vector<float> link(n * n, 0.0f);
    for (size_t g = 0; g < n; ++g)
        for (size_t s = 0; s < n; ++s) link[g * n + s] = c->peer[g][s] ? 1.0f : 0.0f;
    return schedule(avail, hosts, c->neighbor, loading, link);
}

// A CUDA profiling / checking tool is attached: ncu's libcuda-injection or compute-sanitizer's
// interceptor is mapped into the process (or FSW_PROFILER_SAFE=1 asks for the same behaviour).
static bool profiler_attached() {
    if (getenv("FSW_PROFILER_SAFE") && atoi(getenv("FSW_PROFILER_SAFE")) != 0) return true;
    if (getenv("CUDA_INJECTION64_PATH")) return true;
    FILE* f = fopen("/proc/self/maps", "r");
    if (!f) return false;
    char line[4096];
    bool found = false;
    while (!found && fgets(line, sizeof line, f))
        found = strstr(line, "libcuda-injection") || strstr(line, "InterceptorInjectionTarget");
    fclose(f);
    return found;
}

extern "C" fsw_status fsw_invoke_ex(fsw_ctx* c, uint32_t id, const fsw_invoke_opts* opts, const void* input,
                                    uint64_t input_bytes, void* output, uint64_t output_cap, fsw_invoke_stats* stats) {
    NvtxRange nv_invoke("fsw_invoke");
    const double t_entry = now_ms();
    if (!c || !input || !output) return fail(FSW_EINVAL, "invoke: NULL argument");
    if (c->gpus.empty()) return fail(FSW_ECUDA, "invoke: context has no GPU (FSW_HOST_ONLY)");
    fsw_invoke_opts o{};
    o.gpu = -1;
    if (opts) o = *opts;
    Model* m = nullptr;
    int gi = -1;
    bool cold = false;
    std::vector<int> srcs;          // striped swap sources (pool GPU indices), empty = not striped
    int peer = -1;                  // GPU->GPU swap source (pool GPU index), -1 = from the host
    bool pcached = false;           // the model's cached prefix is already on the target
    std::vector<SrcSlot*> slots;    // their swap-kernel slots
    {
        std::unique_lock<std::mutex> lk(c->mu);
        m = find_model(c, id);
        if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
        if (input_bytes != m->input_bytes) return fail(FSW_EINVAL, "invoke: input_bytes %llu != %llu", (unsigned long long)input_bytes, (unsigned long long)m->input_bytes);
        if (output_cap < m->output_bytes) return fail(FSW_EINVAL, "invoke: output_cap too small (%llu < %llu)", (unsigned long long)output_cap, (unsigned long long)m->output_bytes);
        if (o.gpu >= (int)c->gpus.size()) return fail(FSW_EINVAL, "invoke: bad gpu %d", o.gpu);
        Decision dec;
        for (;;) {
            if (o.gpu >= 0) {
                gi = c->gpus[o.gpu].busy ? -1 : o.gpu;
            } else {
                gi = (dec = pick_gpu(c, *m)).gpu;
                // a host swap prefers an idle GPU that still caches the model's prefix (NEXT #4)
                if (dec.kind == 1 && m->split)
                    for (int i = 0; i < (int)c->gpus.size(); ++i)
                        if (!c->gpus[i].busy && m->pvalid[i] && m->pextent[i] >= 0) {
                            gi = i;
                            break;
                        }
            }
            if (gi >= 0) break;
            c->cv.wait(lk);
        }
        Gpu& g = c->gpus[gi];
        g.busy = true;
        m->inflight++;
        cold = m->extent[gi] < 0;
        pcached = cold && m->split && m->pextent[gi] >= 0 && m->pvalid[gi];
        if (cold) {
            fsw_status s = ensure_extent(c, *m, gi);
            if (s != FSW_OK) {
                g.busy = false;
                m->inflight--;
                c->cv.notify_all();
                return s;
            }
        }
        m->last_use[gi] = ++c->clock;
        fsw_status ss = FSW_OK;
        // GPU->GPU swap from a resident copy (Alg. 1 case 2): explicit, or policy
        if (cold && o.peer_src) {
            const int s = (int)o.peer_src - 1;
            if (s < 0 || s >= (int)c->gpus.size() || s == gi) ss = fail(FSW_EINVAL, "invoke: bad peer_src %d", s);
            else if (m->extent[s] < 0 || !m->complete[s]) ss = fail(FSW_ESTATE, "invoke: model %u is not resident on gpu %d", id, s);
            else if (!c->peer[gi][s]) ss = fail(FSW_ETOPO, "invoke: gpu %d cannot read gpu %d", gi, s);
            else peer = s;
        } else if (cold && !o.n_stripe_src && !((o.flags | c->cfg.flags) & FSW_NO_PEER_SWAP)) {
            if (o.gpu < 0 && dec.kind == 2) peer = dec.src;  // Algorithm 1, line 11
            for (int s = 0; s < (int)c->gpus.size() && peer < 0; ++s)
                if (s != gi && m->extent[s] >= 0 && m->complete[s] && c->peer[gi][s]) peer = s;
        }
        // striped swap: explicit sources, or the ctx policy for large stores
        if (ss != FSW_OK || peer >= 0) {
        } else if (cold && o.n_stripe_src) {
            if (!o.stripe_src || o.n_stripe_src > 16) ss = fail(FSW_EINVAL, "invoke: stripe_src");
            for (uint32_t j = 0; ss == FSW_OK && j < o.n_stripe_src; ++j) {
                const int sgi = o.stripe_src[j];
                if (sgi < 0 || sgi >= (int)c->gpus.size()) ss = fail(FSW_EINVAL, "invoke: stripe source %d", sgi);
                else if (!c->peer[sgi][gi]) ss = fail(FSW_ETOPO, "invoke: gpu %d cannot store into gpu %d", sgi, gi);
                else srcs.push_back(sgi);
            }
        } else if (cold && c->gpus.size() > 1 && m->store_bytes >= c->cfg.stripe_min_bytes) {
            srcs.push_back(gi);
            for (int i = 0; i < (int)c->gpus.size(); ++i)
                if (i != gi && c->peer[i][gi]) srcs.push_back(i);
        }
        if (srcs.size() == 1 && srcs[0] == gi) srcs.clear();
        for (size_t j = 0; ss == FSW_OK && j < srcs.size(); ++j) {
            SrcSlot* free_slot = nullptr;
            for (SrcSlot& sl : c->gpus[srcs[j]].src)
                if (!sl.busy) {
                    free_slot = &sl;
                    break;
                }
            if (!free_slot) {
                if (o.n_stripe_src) ss = fail(FSW_EBUSY, "invoke: no free swap slot on gpu %d", srcs[j]);
                else srcs.erase(srcs.begin() + j--);  // policy: that link is busy feeding other swaps
                continue;
            }
            free_slot->busy = true;
            slots.push_back(free_slot);
        }
        if (srcs.size() == 1 && srcs[0] == gi) {
            slots[0]->busy = false;
            srcs.clear();
            slots.clear();
        }
        if (ss == FSW_OK && cold && peer < 0) g.loading = model_heavy(c, *m) ? 2 : 1;  // host link in use
        if (ss != FSW_OK) {
            for (SrcSlot* sl : slots) sl->busy = false;
            if (cold) invalidate(c, *m, gi);
            g.busy = false;
            m->inflight--;
            c->cv.notify_all();
            return ss;
        }
    }
    Gpu& g = c->gpus[gi];
    const bool striped = !srcs.empty();
    fsw_status st = FSW_OK;
    auto finish = [&](fsw_status s) {
        std::lock_guard<std::mutex> lk(c->mu);
        g.loading = 0;
        if (s != FSW_OK && cold) invalidate(c, *m, gi);  // failed swap: extent is not valid
        for (SrcSlot* sl : slots) sl->busy = false;
        g.busy = false;
        m->inflight--;
        c->cv.notify_all();
        return s;
    };
    if (cudaSetDevice(g.dev) != cudaSuccess) return finish(fail(FSW_ECUDA, "cudaSetDevice"));
    if (!m->plans[gi]) {
        st = build_plan(c, *m, gi);
        if (st != FSW_OK) return finish(st);
    }
    Plan& p = *m->plans[gi];
    // Profiler-safe mode: under ncu / compute-sanitizer (a CUDA injection library is attached) kernels
    // run serialised, so nothing may wait on work the tool orders after it: every invoke runs no-overlap
    // (DMAZ then decodes after its last copy group, on the copy stream).
    static const bool profiled = profiler_attached();
    const uint32_t flags = o.flags | c->cfg.flags | (profiled ? FSW_NO_OVERLAP : 0u);
    const bool baseline = (flags & FSW_DMA_BASELINE) != 0;
    int engine = (int)(o.engine ? o.engine : c->cfg.engine);
    if (baseline) engine = FSW_ENGINE_DMA;
    const bool big = m->store_bytes >= c->cfg.dma_min_bytes;
    if (engine == FSW_ENGINE_AUTO)
        engine = m->zstore ? (m->store_bytes >= c->cfg.dmaz_min_bytes ? FSW_ENGINE_DMAZT : FSW_ENGINE_SMZ)
                           : (big ? FSW_ENGINE_DMA : FSW_ENGINE_SM);
    if (engine_coded(engine) && !m->zstore) return finish(fail(FSW_EINVAL, "invoke: model %u is not link-coded (FSW_REG_LINK_CODE)", id));
    // striped: sources store into the target with SM kernels (decoding ones for the coded engines):
    // DMAZ sources copy their runs into their own staging buffer with their copy engine and decode from
    // there (the copy engine's larger PCIe read requests: 55 vs 51.3 GB/s per link), SMZ
    // sources read the coded store zero-copy, plain stores use k_swap
    if (striped) engine = engine_coded(engine) ? (engine_dmaz(engine) ? FSW_ENGINE_DMAZ : FSW_ENGINE_SMZ) : FSW_ENGINE_SM;
    if (peer >= 0) engine = FSW_ENGINE_DMA;  // NVLink copy-engine transfer from the peer's extent
    const uint64_t dgrp = baseline ? (2ull << 20) : o.dma_group_bytes ? o.dma_group_bytes : c->cfg.dma_group_bytes;
    const uint32_t dstr = baseline ? 1u : o.dma_streams ? o.dma_streams : c->cfg.dma_streams;
    if (engine > FSW_ENGINE_DMAZT || dgrp == 0 || dgrp % 256 || dstr == 0 || dstr > (uint32_t)kMaxWaitSrc)
        return finish(fail(FSW_EINVAL, "invoke: bad engine / dma_group_bytes / dma_streams"));
    if (cold && engine == FSW_ENGINE_DMAZT && dstr != 1)
        return finish(fail(FSW_EINVAL, "invoke: DMAZT uses one copy stream (its tail kernel runs on the second)"));
    auto extents = [&](int i) {  // the model's extents on pool GPU i
        return DevDesc{c->gpus[i].pool + (m->pextent[i] >= 0 ? m->pextent[i] : 0), c->gpus[i].pool + m->extent[i], m->split, 0};
    };
    InvokeCfg ic{cold, (flags & FSW_NO_OVERLAP) != 0, engine,
                 o.chunk_bytes ? o.chunk_bytes : c->cfg.chunk_bytes, (int)o.order, o.order_seed,
                 o.copy_ctas                     ? o.copy_ctas
                 : engine_dmaz(engine)           ? std::max(c->cfg.copy_ctas, m->htab.empty() ? kDmazCtas : dmaz_huff_ctas())
                 : engine == FSW_ENGINE_SMZ      ? std::max(c->cfg.copy_ctas, m->htab.empty() ? kSmzCtas : smz_huff_ctas())
                                                 : c->cfg.copy_ctas,
                 extents(gi), nullptr};
    ic.from = pcached ? m->split : 0;
    if (ic.chunk % 256 || ic.chunk == 0 || ic.chunk >= (1ull << 32)) return finish(fail(FSW_EINVAL, "invoke: bad chunk_bytes"));
    if (cold && engine == FSW_ENGINE_DMA) ic.dma_plan = &get_dma_plan(*m, p, dgrp, dstr, ic.from);
    ic.zgrp = dgrp;
    ic.zstreams = dstr;
    ic.tail_ctas = engine == FSW_ENGINE_DMAZT && !striped ? (m->htab.empty() ? kSmzCtas : dmazt_huff_tail_ctas()) : 0;
    if (cold && engine_dmaz(engine) && !striped && g.zstage_cap < m->zbytes) {
        // grow the staging buffer (graphs bake its address: the generation is part of their key)
        cudaFree(g.zstage);
        g.zstage = nullptr;
        g.zstage_cap = 0;
        const uint64_t cap = align_up(m->zbytes, 64ull << 20);
        if (cudaMalloc(&g.zstage, cap) != cudaSuccess) {
            cudaGetLastError();
            return finish(fail(FSW_ENOMEM, "invoke: staging buffer of %llu bytes", (unsigned long long)cap));
        }
        g.zstage_cap = cap;
        g.zstage_gen++;
    }
    if (peer >= 0) {
        ic.src = extents(peer);
        ic.src_host = false;
    }
    const bool sm = engine_bytes_ready(engine);  // a swap kernel releases per-layer byte counters
    // striped: every source claims pieces of >= 256 KiB (one system-scope fence + release each)
    const uint64_t schunk = std::max<uint64_t>(ic.chunk, 256ull << 10);
    std::vector<PieceSet*> sps(srcs.size(), nullptr);
    std::vector<ZPieceSet*> zps(srcs.size(), nullptr);
    std::vector<int> src_node;
    for (int sgi : srcs) src_node.push_back(c->gpu_node[sgi]);
    for (size_t j = 0; j < srcs.size(); ++j) {
        if (engine == FSW_ENGINE_SMZ)
            st = get_zstripe_pieces(*m, p, src_node, (uint32_t)j, c->gpus[srcs[j]].dev, ic.from, &zps[j]);
        else if (engine == FSW_ENGINE_DMAZ)
            st = get_zstripe_dma(*m, p, src_node, (uint32_t)j, c->gpus[srcs[j]].dev, ic.from, kStripeRunBytes, &zps[j]);
        else
            st = get_stripe_pieces(*m, p, schunk, src_node, (uint32_t)j, c->gpus[srcs[j]].dev, ic.from, &sps[j]);
        if (st != FSW_OK) return finish(st);
    }
    for (size_t j = 0; striped && engine == FSW_ENGINE_DMAZ && j < srcs.size(); ++j) {
        SrcSlot& sl = *slots[j];  // grow the source's staging buffer to its share of the coded bytes
        if (sl.stage_cap >= zps[j]->cend) continue;
        cudaSetDevice(c->gpus[srcs[j]].dev);
        cudaFree(sl.stage);
        sl.stage = nullptr;
        sl.stage_cap = 0;
        const uint64_t cap = align_up(std::max<uint64_t>(zps[j]->cend, 1), 64ull << 20);
        if (cudaMalloc(&sl.stage, cap) != cudaSuccess) {
            cudaGetLastError();
            return finish(fail(FSW_ENOMEM, "invoke: striped staging buffer of %llu bytes on gpu %d", (unsigned long long)cap,
                               c->gpus[srcs[j]].dev));
        }
        sl.stage_cap = cap;
    }
    if (striped) {
        cudaSetDevice(g.dev);
        ic.striped = true;
        ic.local_ctas = ic.ctas * (uint32_t)srcs.size();  // the gate waits for every source kernel
    }
    const bool coded = engine_coded(engine);
    GraphKey key{cold, (int)(flags & FSW_NO_OVERLAP), cold && sm && !striped ? ic.order : 0, cold ? engine + (striped ? 8 : 0) : 0,
                 cold && !striped ? (engine == FSW_ENGINE_SM ? ic.chunk : engine == FSW_ENGINE_SMZ ? 0 : dgrp) : 0,
                 cold && sm && !striped ? ic.seed : 0, cold ? (striped ? ic.local_ctas : sm ? ic.ctas : dstr) : 0, 0};
    key.from = cold ? ic.from : 0;
    if (cold && engine_dmaz(engine) && !striped) {
        key.extra = g.zstage_gen;  // baked staging address
        key.pext = dstr;           // copy streams
    }
    if (cold && !sm) {  // DMA graphs bake addresses: the target extents and a peer source's extents
        key.ext = m->extent[gi];
        key.pext = m->pextent[gi];
        if (peer >= 0) {
            key.order = peer + 1;
            key.src_ext = m->extent[peer];
            key.src_pext = m->pextent[peer];
        }
    }
    key.fault = c->fault_gen;
    auto it = p.graphs.find(key);
    cudaGraphExec_t exec = nullptr;
    if (it == p.graphs.end()) {
        if (key.baked()) {
            // graphs baked for other placements: keep the kMaxBakedGraphs - 1 most recently used (the
            // placement changes under eviction churn; none of them is executing: this GPU is ours)
            std::vector<std::pair<uint64_t, GraphKey>> baked;
            for (auto& kv : p.graphs)
                if (kv.first.baked()) baked.push_back({kv.second.last_use, kv.first});
            std::sort(baked.begin(), baked.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
            for (size_t i = 0; i + kMaxBakedGraphs <= baked.size(); ++i) {
                cudaGraphExecDestroy(p.graphs[baked[i].second].exec);
                cudaFree(p.graphs[baked[i].second].mk_ops);
                p.graphs.erase(baked[i].second);
            }
        }
        p.last_mk_ops = nullptr;
        {
            NvtxRange nv_build("build invoke graph");
            st = build_graph(c, *m, p, g, ic, &exec);
        }
        if (st != FSW_OK) {
            cudaFree(p.last_mk_ops);
            p.last_mk_ops = nullptr;
            return finish(st);
        }
        p.graphs[key] = GraphEntry{exec, ++p.graph_clock, p.last_mk_ops};
    } else {
        exec = it->second.exec;
        it->second.last_use = ++p.graph_clock;
    }
    // Test mode (FSW_DEBUG_POISON): every byte this invoke's swap must write, the DMAZ staging buffer
    // and the model's activation workspace start as a per-invoke pattern, so an omitted store can never
    // pass as the stale correct byte an earlier invoke left (the allocator hands back the same extent).
    // Ordered before the graph on the launching stream, outside the timed events.
    if (c->cfg.flags & FSW_DEBUG_POISON) {
        const uint32_t pat = 0xA5C30000u ^ (uint32_t)((g.generation + 1) * 2654435761u);
        launch_poison(g.sx, g.ws, p.ws_bytes, pat ^ 0x10u);
        if (cold) {
            launch_poison(g.sx, g.pool + m->extent[gi], m->store_bytes - m->split, pat);
            if (m->split && !pcached) launch_poison(g.sx, g.pool + m->pextent[gi], m->split, pat);
            if (engine_dmaz(engine) && !striped && g.zstage) launch_poison(g.sx, g.zstage, g.zstage_cap, pat ^ 0x20u);
        }
    }
    if (g.trace)  // device timeline of this invoke (FSW_TRACE): every field starts at 0
        cudaMemsetAsync(g.trace, 0, sizeof(unsigned long long) * kTraceStride * m->layers.size(), g.sx);
    // stage: descriptor + input (pinned), one H2D node in the graph
    DevDesc dd = ic.dst;
    dd.generation = ++g.generation;
    memcpy(g.hstage, &dd, sizeof dd);
    memcpy(g.hstage + kStageHdr, input, input_bytes);
    cudaEventRecord(g.ev0, g.sx);
    cudaError_t e = cudaSuccess;
    if (striped) {
        // Reset the target's counters, then every source loads its share of the pieces over its own
        // host link and stores it into the target's extent (peer stores over NVLink for remote
        // sources), releasing each piece on the target's layer counter at system scope.
        cudaMemsetAsync(g.ready, 0, sizeof(uint32_t) * m->layers.size(), g.sx);
        cudaMemsetAsync(g.ctl, 0, sizeof(DevCtl), g.sx);
        cudaEventRecord(g.evs0, g.sx);
        cudaEventRecord(g.evfork, g.sx);
        for (size_t j = 0; j < srcs.size(); ++j) {
            Gpu& sg = c->gpus[srcs[j]];
            SrcSlot& sl = *slots[j];
            cudaSetDevice(sg.dev);
            cudaStreamWaitEvent(sl.st, g.evfork, 0);
            cudaMemsetAsync(sl.ctl, 0, sizeof(DevCtl), sl.st);
            // an empty share still starts its CTAs: the target's gate counts every source kernel
            if (engine == FSW_ENGINE_DMAZ) {
                // copy engine: the source's runs, back to back, into its staging buffer, a fenced write of
                // the run count after each; the decode kernel (own stream) waits per piece for its run
                static PFN_writeValue32 wv = get_write_value32();
                cudaMemsetAsync(sl.progress, 0, 128, sl.st);
                if (c->cfg.flags & FSW_DEBUG_POISON) launch_poison(sl.st, sl.stage, sl.stage_cap, 0x5A5A0000u ^ (uint32_t)j);
                cudaEventRecord(sl.evfork, sl.st);
                cudaStreamWaitEvent(sl.sdec, sl.evfork, 0);
                launch_swapz(sl.sdec, (int)ic.ctas, (int)c->cfg.copy_threads, sl.stage, 0, ic.dst, nullptr, zps[j]->dev,
                             (uint32_t)zps[j]->host.size(), g.ready, sl.ctl, g.ctl, 1, 1, sl.progress, zps[j]->htab);
                uint32_t cnt = 0;
                uint64_t soff = 0;  // run k sits at the sum of the earlier runs' bytes (get_zstripe_dma)
                for (size_t gi2 = 0; gi2 < zps[j]->groups.size(); ++gi2) {
                    const auto& gr = zps[j]->groups[gi2];
                    if (!(c->fault_kind == FSW_FAULT_DROP_GROUP && c->fault_index == gi2))
                        cudaMemcpyAsync(sl.stage + soff, m->zstore + gr.lo, gr.hi - gr.lo, cudaMemcpyHostToDevice, sl.st);
                    wv(sl.st, (CUdeviceptr)sl.progress, (cuuint32_t)(++cnt), 0);
                    soff += gr.hi - gr.lo;
                }
                cudaEventRecord(sl.evjoin, sl.sdec);
                cudaStreamWaitEvent(sl.st, sl.evjoin, 0);
            } else if (engine == FSW_ENGINE_SMZ)
                launch_swapz(sl.st, (int)ic.ctas, (int)c->cfg.copy_threads, m->zstore, 0, ic.dst, nullptr, zps[j]->dev,
                             (uint32_t)zps[j]->host.size(), g.ready, sl.ctl, g.ctl, 1, 0, nullptr, zps[j]->htab);
            else
                launch_swap(sl.st, (int)ic.ctas, (int)c->cfg.copy_threads, m->store, ic.dst, nullptr, sps[j]->dev,
                            (uint32_t)sps[j]->host.size(), g.ready, sl.ctl, g.ctl, 1);
            cudaEventRecord(sl.done, sl.st);
        }
        cudaSetDevice(g.dev);
        for (size_t j = 0; j < srcs.size(); ++j) cudaStreamWaitEvent(g.sc, slots[j]->done, 0);
        cudaEventRecord(g.evs1, g.sc);
        if (ic.no_overlap) cudaStreamWaitEvent(g.sx, g.evs1, 0);
        e = cudaGraphLaunch(exec, g.sx);
        cudaStreamWaitEvent(g.sx, g.evs1, 0);
    } else {
        e = cudaGraphLaunch(exec, g.sx);
    }
    cudaEventRecord(g.ev1, g.sx);
    const double t_launched = now_ms();
    if (e == cudaSuccess) {
        NvtxRange nv_wait(cold ? "wait (cold: swap + layers)" : "wait (resident)");
        e = cudaEventSynchronize(g.ev1);
    }
    if (e != cudaSuccess) return finish(fail(FSW_ECUDA, "invoke: graph launch/sync: %s", cudaGetErrorString(e)));
    const DevCtl ctl = *g.hctl;
    if (ctl.err) {
        const char* what = ctl.err == 1 ? "ready-flag watchdog" : ctl.err == 2 ? "swap-gate watchdog" : "embedding id out of range";
        return finish(fail(ctl.err == 3 ? FSW_EINVAL : FSW_ETIMEOUT, "invoke: %s (layer %d)", what, ctl.err_layer));
    }
    memcpy(output, g.hout, m->output_bytes);
    const double t_out = now_ms();
    if (stats) {
        memset(stats, 0, sizeof *stats);
        stats->host_setup_ms = t_launched - t_entry;
        stats->host_wait_ms = t_out - t_launched;
        float ms = 0;
        cudaEventElapsedTime(&ms, g.ev0, g.ev1);
        stats->device_ms = ms;
        stats->gpu = gi;
        stats->n_sources = cold ? (striped ? (uint32_t)srcs.size() : 1) : 0;
        stats->swap_kind = cold ? (striped ? FSW_SWAP_STRIPED : peer >= 0 ? FSW_SWAP_PEER : FSW_SWAP_HOST) : FSW_SWAP_RESIDENT;
        stats->n_kernels = (p.mega.on ? 1u : (uint32_t)p.launches.size()) + 1 /*finish*/;  // k_mega: one launch
        if (cold) {
            float swap_ms = 0;
            cudaEventElapsedTime(&swap_ms, g.evs0, g.evs1);
            stats->swap_ms = swap_ms;
            stats->bytes_swapped = m->store_bytes - ic.from;
            stats->link_gbps = swap_ms > 0 ? stats->bytes_swapped / (swap_ms * 1e6) : 0;
            stats->wire_bytes = stats->bytes_swapped;
            stats->engine = (uint32_t)engine;
            if (striped) {
                float tail = 0;
                cudaEventElapsedTime(&tail, g.evs1, g.ev1);
                stats->swap_span_ms = swap_ms;
                stats->compute_tail_ms = tail > 0 ? tail : 0;
                stats->n_kernels += (uint32_t)srcs.size() + (ic.no_overlap ? 0 : 1);  // sources (+ gate)
                for (size_t j = 0; j < srcs.size(); ++j) stats->n_copies += (uint32_t)(engine == FSW_ENGINE_DMAZ ? zps[j]->groups.size() : coded ? zps[j]->host.size() : sps[j]->host.size());
                if (coded) {
                    stats->wire_bytes = 0;
                    for (ZPieceSet* zs : zps)
                        for (const ZPiece& pc : zs->host) stats->wire_bytes += pc.cbytes;
                }
            } else if (coded) {
                if (ctl.t_last > ctl.t_first) stats->swap_span_ms = (ctl.t_last - ctl.t_first) * 1e-6;
                if (ctl.t_end > ctl.t_last) stats->compute_tail_ms = (ctl.t_end - ctl.t_last) * 1e-6;
                stats->n_kernels += (ic.no_overlap ? 1 : 2) + (engine == FSW_ENGINE_DMAZT ? 1 : 0);  // decode (+ gate, + tail)
                ZPieceSet* zs = nullptr;
                if (get_zpieces(*m, p, g, ic.order, ic.seed, ic.from, engine_dmaz(engine) ? dgrp : 0,
                                engine_dmaz(engine) ? dstr : 1, &zs,
                                engine == FSW_ENGINE_DMAZT ? dmazt_tail_permille() : 0) == FSW_OK) {
                    // copy groups (+ the zero-copy tail's pieces for DMAZT), or pieces
                    stats->n_copies = (uint32_t)(engine_dmaz(engine) ? zs->groups.size() + (zs->host.size() - zs->n_body)
                                                                     : zs->host.size());
                    stats->wire_bytes = zs->cend - zs->cfrom;
                }
            } else if (engine == FSW_ENGINE_SM) {
                if (ctl.t_last > ctl.t_first) stats->swap_span_ms = (ctl.t_last - ctl.t_first) * 1e-6;
                if (ctl.t_end > ctl.t_last) stats->compute_tail_ms = (ctl.t_end - ctl.t_last) * 1e-6;
                stats->n_kernels += ic.no_overlap ? 1 : 2;  // swap (+ gate)
                PieceSet* ps = nullptr;
                if (get_pieces(*m, p, g, ic.chunk, ic.order, ic.seed, ic.from, &ps) == FSW_OK) stats->n_copies = (uint32_t)ps->host.size();
            } else {
                float tail = 0;
                cudaEventElapsedTime(&tail, g.evs1, g.ev1);
                stats->swap_span_ms = swap_ms;
                stats->compute_tail_ms = tail > 0 ? tail : 0;
                stats->n_copies = (uint32_t)ic.dma_plan->groups.size();
            }
        }
    }
    {
        std::lock_guard<std::mutex> lk(c->mu);
        float dms = 0;
        cudaEventElapsedTime(&dms, g.ev0, g.ev1);
        if (cold) {
            g.n_cold++;
            g.bytes_swapped_total += m->store_bytes - ic.from;
            if (m->split) m->pvalid[gi] = 1;  // the prefix bytes have landed
            m->complete[gi] = 1;              // now a resident copy (peer swaps may read it)
            if (peer < 0 && !striped) {
                m->cold_ms_sum += dms;
                m->n_cold_runs++;
            }
        } else {
            g.n_warm++;
            m->warm_ms_sum += dms;
            m->n_warm_runs++;
        }
    }
    finish(FSW_OK);
    if (stats) stats->total_ms = now_ms() - t_entry;
    return FSW_OK;
}

extern "C" fsw_status fsw_debug_set_fault(fsw_ctx* c, uint32_t kind, uint32_t index) {
    if (!c || kind > FSW_FAULT_DROP_GROUP) return fail(FSW_EINVAL, "set_fault: bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    for (Gpu& g : c->gpus) {
        if (g.busy) return fail(FSW_EBUSY, "set_fault: an invoke is in flight on gpu %d", g.dev);
        CU(cudaSetDevice(g.dev));
        set_drop_piece(kind == FSW_FAULT_DROP_PIECE ? index : 0xffffffffu);
        CU(cudaDeviceSynchronize());
    }
    c->fault_kind = kind;
    c->fault_index = index;
    c->fault_gen++;  // cached graphs (DMA groups are baked into them) are keyed by it
    return FSW_OK;
}

extern "C" fsw_status fsw_invoke(fsw_ctx* c, uint32_t id, const void* input, uint64_t input_bytes, void* output,
                                 uint64_t output_cap, fsw_invoke_stats* stats) {
    return fsw_invoke_ex(c, id, nullptr, input, input_bytes, output, output_cap, stats);
}

