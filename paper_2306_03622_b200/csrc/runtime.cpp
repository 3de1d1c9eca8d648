// runtime.cpp — libfsw host runtime behind include/fsw.h: errors, the pool arena, init / shutdown,
// pool stats and the debug read-backs.  The rest: store.cpp (registration, host store, link code),
// plan.cpp (layer plans, GEMM tiling), graph.cpp (swap plans, invoke graphs), invoke.cpp (residency,
// eviction, placement, fsw_invoke).
//
// Layers: C-ABI -> host runtime (host store, weight pool, invoke orchestrator,
// per-(model, GPU) execution plans and CUDA graphs) -> sm_100a kernels (kernels.h).
//
// Paper mapping:
//   model repository in host memory ........ HostStore
//   GPU executor, one shared runtime/GPU .... Gpu
//   pre-allocated pool + block management ... Arena
//   late binding + on-demand swapping ....... invoke()
//   pipelined model execution ............... cold graph: swap kernel ‖ flag-gated layers
//   eviction by invalidation ................ evict()
//   one request per GPU ..................... Gpu::busy
#include "rt_internal.h"

// ==========================================================================================
// errors
// ==========================================================================================
static thread_local std::string g_err;

fsw_status fail(fsw_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}


extern "C" const char* fsw_last_error(void) { return g_err.c_str(); }
extern "C" const char* fsw_version(void) { return "fsw 0.1 (sm_100a)"; }
// ==========================================================================================
struct fsw_arena {
    uint64_t capacity, align;
    std::map<uint64_t, uint64_t> free_;   // offset -> size
    std::map<uint64_t, uint64_t> used_;   // offset -> size
};

extern "C" fsw_arena* fsw_arena_create(uint64_t capacity, uint64_t align) {
    if (align == 0 || (align & (align - 1))) return nullptr;
    auto* a = new fsw_arena{capacity / align * align, align, {}, {}};
    if (a->capacity) a->free_[0] = a->capacity;
    return a;
}
extern "C" void fsw_arena_destroy(fsw_arena* a) { delete a; }

extern "C" fsw_status fsw_arena_alloc(fsw_arena* a, uint64_t bytes, uint64_t* offset) {
    if (!a || !offset || bytes == 0) return fail(FSW_EINVAL, "arena_alloc: bad argument");
    const uint64_t need = align_up(bytes, a->align);
    auto best = a->free_.end();
    for (auto it = a->free_.begin(); it != a->free_.end(); ++it)
        if (it->second >= need && (best == a->free_.end() || it->second < best->second)) best = it;
    if (best == a->free_.end()) return fail(FSW_ENOMEM, "arena_alloc: no free extent of %llu bytes", (unsigned long long)need);
    const uint64_t off = best->first, sz = best->second;
    a->free_.erase(best);
    if (sz > need) a->free_[off + need] = sz - need;
    a->used_[off] = need;
    *offset = off;
    return FSW_OK;
}

extern "C" fsw_status fsw_arena_free(fsw_arena* a, uint64_t offset) {
    if (!a) return fail(FSW_EINVAL, "arena_free: null arena");
    auto it = a->used_.find(offset);
    if (it == a->used_.end()) return fail(FSW_EINVAL, "arena_free: %llu is not an allocated extent", (unsigned long long)offset);
    uint64_t off = it->first, sz = it->second;
    a->used_.erase(it);
    auto nx = a->free_.lower_bound(off);
    if (nx != a->free_.end() && off + sz == nx->first) {
        sz += nx->second;
        a->free_.erase(nx);
    }
    auto pv = a->free_.lower_bound(off);
    if (pv != a->free_.begin()) {
        --pv;
        if (pv->first + pv->second == off) {
            off = pv->first;
            sz += pv->second;
            a->free_.erase(pv);
        }
    }
    a->free_[off] = sz;
    return FSW_OK;
}

extern "C" void fsw_arena_stats(const fsw_arena* a, uint64_t* used, uint64_t* largest_free, uint32_t* n_allocated) {
    uint64_t u = 0, lf = 0;
    if (a) {
        for (auto& kv : a->used_) u += kv.second;
        for (auto& kv : a->free_) lf = std::max(lf, kv.second);
    }
    if (used) *used = u;
    if (largest_free) *largest_free = lf;
    if (n_allocated) *n_allocated = a ? (uint32_t)a->used_.size() : 0;
}

// ==========================================================================================
// init / shutdown
// ==========================================================================================
static fsw_status init_gpu(fsw_ctx* c, Gpu& g) {
    CU(cudaSetDevice(g.dev));
    CU(cudaFree(nullptr));  // create the context now (one shared runtime per GPU)
    init_gemm_attrs();
    init_gemm_ws_attrs();
    init_attn_tc_attrs();
    init_mega_attrs();
    init_ops_attrs();
    init_swap_attrs();
    CU(cudaStreamCreateWithFlags(&g.sx, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&g.sc, cudaStreamNonBlocking));
    g.sd[0] = g.sc;
    CU(cudaStreamCreateWithFlags(&g.sz, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&g.evz, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&g.evset, cudaEventDisableTiming));
    for (int j = 1; j < kMaxWaitSrc; ++j) CU(cudaStreamCreateWithFlags(&g.sd[j], cudaStreamNonBlocking));
    for (int j = 0; j < kMaxWaitSrc; ++j) CU(cudaEventCreateWithFlags(&g.evd[j], cudaEventDisableTiming));
    CU(cudaMalloc(&g.progress, 128 * kMaxWaitSrc));
    CU(cudaMalloc(&g.gemm_ctr, sizeof(uint32_t) * kGemmCtrs));
    for (SrcSlot& sl : g.src) {
        CU(cudaMalloc(&sl.ctl, sizeof(DevCtl)));
        CU(cudaMalloc(&sl.progress, 128));
        CU(cudaStreamCreateWithFlags(&sl.st, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&sl.sdec, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&sl.evfork, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&sl.evjoin, cudaEventDisableTiming));
    }
    CU(cudaMemset(g.gemm_ctr, 0, sizeof(uint32_t) * kGemmCtrs));
    CU(cudaMemset(g.progress, 0, 128 * kMaxWaitSrc));
    size_t free_b = 0, total_b = 0;
    CU(cudaMemGetInfo(&free_b, &total_b));
    uint64_t want = c->cfg.pool_bytes_per_gpu ? c->cfg.pool_bytes_per_gpu : (64ull << 30);
    want = std::min<uint64_t>(want, (uint64_t)(free_b * 0.6));
    g.pool_bytes = want / (64 << 10) * (64 << 10);
    CU(cudaMalloc(&g.pool, g.pool_bytes));
    g.wmap_ok = make_tmap_pool(&g.wmap, g.pool, g.pool_bytes);
    g.arena = fsw_arena_create(g.pool_bytes, 64 << 10);
    g.ws_bytes = c->cfg.workspace_bytes_per_gpu ? c->cfg.workspace_bytes_per_gpu : (512ull << 20);
    CU(cudaMalloc(&g.ws, g.ws_bytes));
    g.ready_cap = 1u << 16;
    CU(cudaMalloc(&g.ready, sizeof(uint32_t) * g.ready_cap));
    CU(cudaMemset(g.ready, 0, sizeof(uint32_t) * g.ready_cap));
    CU(cudaMalloc(&g.ctl, sizeof(DevCtl)));
    CU(cudaMemset(g.ctl, 0, sizeof(DevCtl)));
    CU(cudaMalloc(&g.ctl_tail, sizeof(DevCtl)));
    CU(cudaMemset(g.ctl_tail, 0, sizeof(DevCtl)));
    g.stage_cap = 16ull << 20;
    g.out_cap = 16ull << 20;
    CU(cudaMalloc(&g.dstage, g.stage_cap));
    CU(cudaHostAlloc(&g.hstage, g.stage_cap, cudaHostAllocPortable));
    CU(cudaHostAlloc(&g.hout, g.out_cap, cudaHostAllocPortable | cudaHostAllocMapped));
    CU(cudaHostAlloc(reinterpret_cast<void**>(&g.hctl), sizeof(DevCtl), cudaHostAllocPortable | cudaHostAllocMapped));
    memset(g.hstage, 0, kStageHdr);
    for (cudaEvent_t* e : {&g.ev0, &g.ev1, &g.evs0, &g.evs1}) CU(cudaEventCreate(e));
    if (c->cfg.flags & FSW_TRACE) {  // device timeline: every kernel of this device records into it
        CU(cudaMalloc(&g.trace, sizeof(unsigned long long) * kTraceStride * g.ready_cap));
        CU(cudaMemset(g.trace, 0, sizeof(unsigned long long) * kTraceStride * g.ready_cap));
        set_trace_swap(g.trace);  // the layer kernels get it through their parameters (graph.cpp)
        set_trace_mega(g.trace);
    }
    CU(cudaEventCreateWithFlags(&g.evfork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&g.evjoin, cudaEventDisableTiming));
    return FSW_OK;
}

extern "C" fsw_status fsw_init(const fsw_config* cfg, fsw_ctx** out) {
    if (!out) return fail(FSW_EINVAL, "fsw_init: out is NULL");
    *out = nullptr;
    if (cfg && (cfg->flags & FSW_HOST_ONLY)) {
        auto c = std::make_unique<fsw_ctx>();
        c->cfg = *cfg;
        c->cfg.gpu_ids = nullptr;
        if (c->cfg.chunk_bytes == 0) c->cfg.chunk_bytes = 256 << 10;
        *out = c.release();
        return FSW_OK;
    }
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(FSW_ECUDA, "fsw_init: no CUDA device (%s)", e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
    auto c = std::make_unique<fsw_ctx>();
    if (cfg) c->cfg = *cfg;
    if (getenv("FSW_DEBUG_POISON") && atoi(getenv("FSW_DEBUG_POISON")) != 0) c->cfg.flags |= FSW_DEBUG_POISON;
    if (getenv("FSW_TRACE") && atoi(getenv("FSW_TRACE")) != 0) c->cfg.flags |= FSW_TRACE;
    if (c->cfg.copy_ctas == 0) c->cfg.copy_ctas = 16;
    if (c->cfg.copy_threads == 0) c->cfg.copy_threads = 256;
    if (c->cfg.chunk_bytes == 0) c->cfg.chunk_bytes = 16 << 10;
    if (c->cfg.stripe_min_bytes == 0) c->cfg.stripe_min_bytes = 256ull << 20;
    if (c->cfg.dma_min_bytes == 0) c->cfg.dma_min_bytes = 32ull << 20;
    if (c->cfg.dmaz_min_bytes == 0) c->cfg.dmaz_min_bytes = 128ull << 20;
    if (c->cfg.dma_group_bytes == 0) c->cfg.dma_group_bytes = 64ull << 20;
    if (c->cfg.dma_streams == 0) c->cfg.dma_streams = 1;
    if (c->cfg.engine > FSW_ENGINE_DMAZT || c->cfg.dma_streams > (uint32_t)kMaxWaitSrc || c->cfg.dma_group_bytes % 256)
        return fail(FSW_EINVAL, "fsw_init: engine, dma_streams (1..4) or dma_group_bytes (multiple of 256) invalid");
    if (c->cfg.chunk_bytes % 256 || c->cfg.copy_threads % 32 || c->cfg.copy_threads > 512)
        return fail(FSW_EINVAL, "fsw_init: chunk_bytes must be a multiple of 256, copy_threads a multiple of 32 <= 512");
    uint32_t n = c->cfg.n_gpus ? c->cfg.n_gpus : (uint32_t)ndev;
    c->gpus.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
        c->gpus[i].dev = c->cfg.gpu_ids ? c->cfg.gpu_ids[i] : (int)i;
        if (c->gpus[i].dev < 0 || c->gpus[i].dev >= ndev) return fail(FSW_EINVAL, "fsw_init: bad gpu id %d", c->gpus[i].dev);
        fsw_status s = init_gpu(c.get(), c->gpus[i]);
        if (s != FSW_OK) return s;
    }
    c->neighbor.assign(n, -1);
    {
        const char* fk = getenv("FSW_FAKE_NUMA");
        c->fake_numa = fk && atoi(fk) > 1;
        for (uint32_t i = 0; i < n; ++i)
            c->gpu_node.push_back(c->fake_numa ? (int)(i % (uint32_t)atoi(fk)) : gpu_numa_node(c->gpus[i].dev));
        for (int v : c->gpu_node)
            if (v >= 0 && std::find(c->nodes.begin(), c->nodes.end(), v) == c->nodes.end()) c->nodes.push_back(v);
        std::sort(c->nodes.begin(), c->nodes.end());
    }
    if (cfg && cfg->pcie_neighbor)
        for (uint32_t i = 0; i < n; ++i) c->neighbor[i] = cfg->pcie_neighbor[i] < (int32_t)n ? cfg->pcie_neighbor[i] : -1;
    c->cfg.pcie_neighbor = nullptr;
    // NVLink peer access between the pool's GPUs (striped swap stores into a peer's extent)
    c->peer.assign(n, std::vector<char>(n, 0));
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < n; ++j) {
            if (c->gpus[i].dev == c->gpus[j].dev) {
                c->peer[i][j] = 1;
                continue;
            }
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, c->gpus[i].dev, c->gpus[j].dev);
            if (ok) {
                CU(cudaSetDevice(c->gpus[i].dev));
                cudaError_t e = cudaDeviceEnablePeerAccess(c->gpus[j].dev, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e != cudaSuccess) ok = 0;
            }
            c->peer[i][j] = (char)ok;
        }
    c->cfg.gpu_ids = nullptr;
    *out = c.release();
    return FSW_OK;
}

void free_plan(Gpu& g, Plan& p) {
    cudaSetDevice(g.dev);
    for (auto& kv : p.graphs) {
        cudaGraphExecDestroy(kv.second.exec);
        cudaFree(kv.second.mk_ops);
    }
    p.graphs.clear();
    cudaFree(p.mega.tmaps);
    cudaFree(p.mega.op_cnt);
    cudaFree(p.mega.stamps);
    p.mega.stamps = nullptr;
    p.mega.tmaps = nullptr;
    p.mega.op_cnt = nullptr;
    for (auto& kv : p.pieces) cudaFree(kv.second.dev);
    p.pieces.clear();
    for (auto& kv : p.stripe) cudaFree(kv.second.dev);  // UVA: any current device
    p.stripe.clear();
    for (auto& kv : p.zp) cudaFree(kv.second.dev), cudaFree(kv.second.htab);
    p.zp.clear();
    for (auto& kv : p.zstripe) cudaFree(kv.second.dev), cudaFree(kv.second.htab);
    p.zstripe.clear();
    for (auto& kv : p.zstripe_dma) cudaFree(kv.second.dev), cudaFree(kv.second.htab);
    p.zstripe_dma.clear();
}

void free_store(Model& m, bool host_only) {
    if (m.zstore) {
        if (!host_only) cudaHostUnregister(m.zstore);
        munmap(m.zstore, m.zalloc);
        m.zstore = nullptr;
    }
    if (!m.store) return;
    if (m.store_wc) {
        cudaFreeHost(m.store);
    } else {
        if (!host_only) cudaHostUnregister(m.store);
        munmap(m.store, m.store_alloc);
    }
    m.store = nullptr;
}

extern "C" void fsw_shutdown(fsw_ctx* c) {
    if (!c) return;
    for (auto& m : c->models) {
        if (!m) continue;
        for (size_t i = 0; i < c->gpus.size(); ++i)
            if (m->plans[i]) free_plan(c->gpus[i], *m->plans[i]);
        free_store(*m, (c->cfg.flags & FSW_HOST_ONLY) != 0);
    }
    for (auto& g : c->gpus) {
        cudaSetDevice(g.dev);
        cudaStreamSynchronize(g.sx);
        cudaStreamSynchronize(g.sc);
        cudaFree(g.pool);
        cudaFree(g.ws);
        cudaFree(g.ready);
        cudaFree(g.trace);
        cudaFree(g.ctl);
        cudaFree(g.ctl_tail);
        cudaFree(g.dstage);
        cudaFree(g.zstage);
        cudaStreamDestroy(g.sz);
        cudaEventDestroy(g.evz);
        cudaEventDestroy(g.evset);
        cudaFreeHost(g.hstage);
        cudaFreeHost(g.hout);
        cudaFreeHost(g.hctl);
        for (cudaEvent_t e : {g.ev0, g.ev1, g.evs0, g.evs1, g.evfork, g.evjoin}) cudaEventDestroy(e);
        for (int j = 0; j < kMaxWaitSrc; ++j) cudaEventDestroy(g.evd[j]);
        for (int j = 1; j < kMaxWaitSrc; ++j) cudaStreamDestroy(g.sd[j]);
        cudaFree(g.progress);
        cudaFree(g.gemm_ctr);
        for (SrcSlot& sl : g.src) {
            cudaFree(sl.ctl);
            cudaFree(sl.progress);
            cudaFree(sl.stage);
            cudaStreamDestroy(sl.st);
            cudaStreamDestroy(sl.sdec);
            cudaEventDestroy(sl.done);
            cudaEventDestroy(sl.evfork);
            cudaEventDestroy(sl.evjoin);
        }
        cudaStreamDestroy(g.sx);
        cudaStreamDestroy(g.sc);
        fsw_arena_destroy(g.arena);
    }
    delete c;
}

extern "C" fsw_status fsw_n_gpus(fsw_ctx* c, uint32_t* n) {
    if (!c || !n) return fail(FSW_EINVAL, "fsw_n_gpus: NULL");
    *n = (uint32_t)c->gpus.size();
    return FSW_OK;
}

Model* find_model(fsw_ctx* c, uint32_t id) {
    if (!c || id >= c->models.size()) return nullptr;
    return c->models[id].get();
}

extern "C" fsw_status fsw_pool_stats_get(fsw_ctx* c, int32_t gpu, fsw_pool_stats* out) {
    if (!c || !out || gpu < 0 || gpu >= (int)c->gpus.size()) return fail(FSW_EINVAL, "pool_stats: bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    Gpu& g = c->gpus[gpu];
    memset(out, 0, sizeof *out);
    out->capacity = g.pool_bytes;
    fsw_arena_stats(g.arena, &out->used, &out->largest_free, &out->n_extents);
    for (auto& m : c->models) {
        if (m && m->extent[gpu] >= 0) out->n_resident++;
        if (m && m->pextent[gpu] >= 0 && m->pvalid[gpu]) out->prefix_bytes_cached += m->split;
    }
    out->n_evictions = g.n_evictions;
    out->n_evictions_heavy = g.n_evictions_heavy;
    out->bytes_swapped_total = g.bytes_swapped_total;
    out->n_invokes_cold = g.n_cold;
    out->n_invokes_warm = g.n_warm;
    return FSW_OK;
}

// ==========================================================================================
// debug read-back
// ==========================================================================================
extern "C" fsw_status fsw_debug_read_resident(fsw_ctx* c, uint32_t id, int32_t gpu, void* dst, uint64_t cap) {
    if (!c || !dst || gpu < 0 || gpu >= (int)c->gpus.size()) return fail(FSW_EINVAL, "read_resident: bad argument");
    std::lock_guard<std::mutex> lk(c->mu);
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (m->extent[gpu] < 0) return fail(FSW_ESTATE, "model %u not resident on gpu %d", id, gpu);
    if (cap < m->store_bytes) return fail(FSW_EINVAL, "read_resident: cap too small");
    CU(cudaSetDevice(c->gpus[gpu].dev));
    uint8_t* pool = c->gpus[gpu].pool;
    if (m->split) CU(cudaMemcpy(dst, pool + m->pextent[gpu], m->split, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(static_cast<uint8_t*>(dst) + m->split, pool + m->extent[gpu], m->store_bytes - m->split,
                  cudaMemcpyDeviceToHost));
    return FSW_OK;
}

extern "C" fsw_status fsw_debug_trace_read(fsw_ctx* c, uint32_t id, int32_t gpu, uint64_t* out, uint32_t cap_layers,
                                           uint64_t* t_invoke) {
    if (!c || !out || gpu < 0 || gpu >= (int)c->gpus.size()) return fail(FSW_EINVAL, "trace_read: bad argument");
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    Gpu& g = c->gpus[gpu];
    if (!g.trace) return fail(FSW_ESTATE, "trace_read: context not created with FSW_TRACE");
    const size_t nl = m->layers.size();
    if (cap_layers < nl) return fail(FSW_EINVAL, "trace_read: cap %u < %zu layers", cap_layers, nl);
    CU(cudaSetDevice(g.dev));
    std::vector<unsigned long long> raw(nl * kTraceStride);
    CU(cudaMemcpy(raw.data(), g.trace, sizeof(unsigned long long) * raw.size(), cudaMemcpyDeviceToHost));
    for (size_t l = 0; l < nl; ++l) {  // [entry, wait done, exit, first release, last release, GEMM phases]; 0 = none
        const unsigned long long* r = &raw[l * kTraceStride];
        for (uint32_t i = 0; i < 16; ++i) out[16 * l + i] = r[i];
        out[16 * l + 0] = r[0] ? ~r[0] : 0;
        out[16 * l + 3] = r[3] ? ~r[3] : 0;
    }
    if (t_invoke) {  // the last invoke's control block: first piece claimed, last released, graph end
        DevCtl ctl{};
        CU(cudaMemcpy(&ctl, g.ctl, sizeof ctl, cudaMemcpyDeviceToHost));
        t_invoke[0] = ctl.t_first;
        t_invoke[1] = ctl.t_last;
        t_invoke[2] = ctl.t_end;
    }
    return FSW_OK;
}

// Phase stamps of the persistent kernel's last run (FSW_MEGA_STAMPS=1; tools/mega_phases.py): out receives
// [n_ops][ctas][8] u64 and ops[n_ops][4] = (kind, n_tasks, tt, splits).  *n_ops / *ctas always set.
extern "C" fsw_status fsw_debug_mega_stamps(fsw_ctx* c, uint32_t id, int32_t gpu, uint64_t* out, uint32_t* ops_out,
                                            uint64_t cap, uint32_t* n_ops, uint32_t* ctas) {
    if (!c || !n_ops || !ctas || gpu < 0 || gpu >= (int)c->gpus.size()) return fail(FSW_EINVAL, "mega_stamps: bad argument");
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (!m->plans[gpu] || !m->plans[gpu]->mega.on) return fail(FSW_ESTATE, "mega_stamps: no persistent-kernel plan");
    const MegaPlan& mp = m->plans[gpu]->mega;
    *n_ops = (uint32_t)mp.ops.size();
    *ctas = (uint32_t)mp.ctas;
    if (!mp.stamps) return fail(FSW_ESTATE, "mega_stamps: FSW_MEGA_STAMPS was not set");
    const size_t n = mp.ops.size() * (size_t)mp.ctas * 8;
    if (!out || cap < n) return fail(FSW_EINVAL, "mega_stamps: cap");
    CU(cudaSetDevice(c->gpus[gpu].dev));
    CU(cudaMemcpy(out, mp.stamps, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (ops_out)
        for (size_t i = 0; i < mp.ops.size(); ++i) {
            ops_out[4 * i] = mp.ops[i].kind;
            ops_out[4 * i + 1] = mp.ops[i].n_tasks;
            ops_out[4 * i + 2] = mp.ops[i].tt;
            ops_out[4 * i + 3] = mp.ops[i].splits;
        }
    return FSW_OK;
}

extern "C" fsw_status fsw_debug_read_coded(fsw_ctx* c, uint32_t id, void* dst, uint64_t cap) {
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (!m->zstore) return fail(FSW_ESTATE, "model %u is not link-coded", id);
    if (!dst || cap < m->zbytes) return fail(FSW_EINVAL, "read_coded: cap %llu < %llu", (unsigned long long)cap, (unsigned long long)m->zbytes);
    memcpy(dst, m->zstore, m->zbytes);
    return FSW_OK;
}

extern "C" fsw_status fsw_debug_coded_code(fsw_ctx* c, uint32_t id, uint8_t* lengths_out) {
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (!m->zstore) return fail(FSW_ESTATE, "model %u is not link-coded", id);
    if (!lengths_out) return fail(FSW_EINVAL, "coded_code: lengths_out is NULL");
    memcpy(lengths_out, m->hlen, 16);
    return FSW_OK;
}

extern "C" fsw_status fsw_debug_coded_pieces(fsw_ctx* c, uint32_t id, fsw_coded_piece* out, uint32_t cap, uint32_t* n) {
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (!m->zstore) return fail(FSW_ESTATE, "model %u is not link-coded", id);
    if (!n) return fail(FSW_EINVAL, "coded_pieces: n is NULL");
    *n = (uint32_t)m->zpieces.size();
    if (m->zpieces.size() > cap || (!out && cap)) return fail(FSW_EINVAL, "coded_pieces: cap %u < %u", cap, *n);
    for (size_t i = 0; i < m->zpieces.size(); ++i) {
        const ZPiece& z = m->zpieces[i];
        out[i] = {z.off, z.coff, z.bytes, z.cbytes, z.layer, 0, {}};
        memcpy(out[i].hdr, z.hdr, sizeof z.hdr);
    }
    return FSW_OK;
}

extern "C" fsw_status fsw_debug_read_store(fsw_ctx* c, uint32_t id, void* dst, uint64_t cap) {
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (!dst || cap < m->store_bytes) return fail(FSW_EINVAL, "read_store: cap too small");
    memcpy(dst, m->store, m->store_bytes);
    return FSW_OK;
}

extern "C" fsw_status fsw_debug_read_slot(fsw_ctx* c, uint32_t id, int32_t gpu, int32_t slot, void* dst, uint64_t cap) {
    if (!c || !dst || gpu < 0 || gpu >= (int)c->gpus.size()) return fail(FSW_EINVAL, "read_slot: bad argument");
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (slot < 0 || slot >= (int)m->slots.size()) return fail(FSW_EINVAL, "read_slot: bad slot");
    if (!m->plans[gpu]) return fail(FSW_ESTATE, "read_slot: model never ran on gpu %d", gpu);
    const uint64_t b = slot_bytes(m->slots[slot]);
    if (cap < b) return fail(FSW_EINVAL, "read_slot: cap too small");
    Gpu& g = c->gpus[gpu];
    CU(cudaSetDevice(g.dev));
    const uint8_t* src = slot == m->input_slot ? g.dstage + kStageHdr : g.ws + m->plans[gpu]->slot_off[slot];
    CU(cudaMemcpy(dst, src, b, cudaMemcpyDeviceToHost));
    return FSW_OK;
}

