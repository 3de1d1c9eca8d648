// litmus.cpp — fsw_debug_litmus: the readiness-protocol litmus test (test infrastructure; the product
// path never calls it).  DESIGN.md §5 "Memory ordering" states the protocol; this runs it in the
// overlapped mode thousands of times against a consumer that reads the weights exactly as a layer
// kernel does (acquire -> fence.proxy.async -> bulk copy), with the destination poisoned first, so a
// release that overtakes its stores, or a missing proxy fence, shows up as a stale (poison) word.
#include "rt_internal.h"

extern "C" fsw_status fsw_debug_litmus(fsw_ctx* c, uint32_t id, int32_t gpu, uint32_t engine, uint32_t ctas, uint32_t iters,
                                       uint64_t* bad_words, uint64_t* checked_bytes) {
    if (!c || !bad_words || !checked_bytes || gpu < 0 || gpu >= (int)c->gpus.size() || engine < FSW_ENGINE_SM ||
        engine > FSW_ENGINE_DMAZT || ctas == 0 || ctas > 1024 || iters == 0)
        return fail(FSW_EINVAL, "litmus: bad argument");
    Model* m = nullptr;
    Gpu& g = c->gpus[gpu];
    uint64_t off = 0;
    {
        std::unique_lock<std::mutex> lk(c->mu);
        m = find_model(c, id);
        if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
        if (m->inflight) return fail(FSW_EBUSY, "litmus: model %u has an invoke in flight", id);
        if (engine_coded((int)engine) && !m->zstore) return fail(FSW_EINVAL, "litmus: model %u is not link-coded", id);
        c->cv.wait(lk, [&] { return !g.busy; });
        if (fsw_arena_alloc(g.arena, m->store_bytes, &off) != FSW_OK)
            return fail(FSW_ENOMEM, "litmus: no room for a %llu-byte scratch extent", (unsigned long long)m->store_bytes);
        g.busy = true;
        m->inflight++;
    }
    uint8_t* golden = nullptr;
    uint8_t* stage = nullptr;
    LitmusLayer* dlayers = nullptr;
    unsigned long long* dcnt = nullptr;
    cudaGraphExec_t exec = nullptr;
    auto finish = [&](fsw_status s) {
        cudaDeviceSynchronize();
        if (exec) cudaGraphExecDestroy(exec);
        cudaFree(golden);
        cudaFree(stage);
        cudaFree(dlayers);
        cudaFree(dcnt);
        std::lock_guard<std::mutex> lk(c->mu);
        fsw_arena_free(g.arena, off);
        g.busy = false;
        m->inflight--;
        c->cv.notify_all();
        return s;
    };
    if (cudaSetDevice(g.dev) != cudaSuccess) return finish(fail(FSW_ECUDA, "cudaSetDevice"));
    if (!m->plans[gpu]) {
        fsw_status st = build_plan(c, *m, gpu);
        if (st != FSW_OK) return finish(st);
    }
    Plan& p = *m->plans[gpu];
    const DevDesc dst{g.pool + off, g.pool + off, 0, 0};
    const uint64_t grp = 1ull << 20;  // copy groups of the DMA engines: many publish events per swap
    PieceSet* ps = nullptr;
    ZPieceSet* zs = nullptr;
    fsw_status st = FSW_OK;
    if (engine == FSW_ENGINE_SM) st = get_pieces(*m, p, g, c->cfg.chunk_bytes, FSW_ORDER_EXEC, 0, 0, &ps);
    if (engine_coded((int)engine))
        st = get_zpieces(*m, p, g, FSW_ORDER_EXEC, 0, 0, engine_dmaz((int)engine) ? grp : 0, 1, &zs,
                         engine == FSW_ENGINE_DMAZT ? dmazt_tail_permille() : 0);
    if (st != FSW_OK) return finish(st);
    const DmaPlan* dp = engine == FSW_ENGINE_DMA ? &get_dma_plan(*m, p, grp, 1, 0) : nullptr;
    // the consumer's table: every non-empty layer region with its wait targets
    std::vector<LitmusLayer> ly;
    for (uint32_t li = 0; li < m->layers.size(); ++li) {
        if (!m->region_bytes[li]) continue;
        LitmusLayer x{m->region_off[li], (uint32_t)m->region_bytes[li], li, {}};
        x.target[0] = dp ? dp->target[li][0] : (uint32_t)m->region_bytes[li];
        ly.push_back(x);
    }
    Wait wb{};
    wb.ctl = g.ctl;
    wb.n = 1;
    wb.ready[0] = dp ? g.progress : g.ready;
    const int per_layer = dp ? 0 : 1;
    if (cudaMalloc(&golden, m->store_bytes) != cudaSuccess || cudaMalloc(&dlayers, sizeof(LitmusLayer) * ly.size()) != cudaSuccess ||
        cudaMalloc(&dcnt, 2 * sizeof(unsigned long long)) != cudaSuccess)
        return finish(fail(FSW_ENOMEM, "litmus: device buffers"));
    if (cudaMemcpy(golden, m->store, m->store_bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(dlayers, ly.data(), sizeof(LitmusLayer) * ly.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemset(dcnt, 0, 2 * sizeof(unsigned long long)) != cudaSuccess)
        return finish(fail(FSW_ECUDA, "litmus: setup copies"));
    uint64_t stage_bytes = 0;
    if (engine_dmaz((int)engine)) {
        stage_bytes = zs->cend - zs->cfrom;
        if (cudaMalloc(&stage, stage_bytes) != cudaSuccess) return finish(fail(FSW_ENOMEM, "litmus: staging buffer"));
    }
    static PFN_writeValue32 wv = get_write_value32();
    if (!wv) return finish(fail(FSW_ECUDA, "cuStreamWriteValue32 entry point unavailable"));
    // one iteration as a graph: poison, reset, then producer (copy stream) || consumer (layer stream)
    cudaStream_t sx = g.sx, sc = g.sc;
    const uint32_t pat = 0x5EED0000u ^ (iters * 2654435761u);
    if (cudaStreamBeginCapture(sx, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        return finish(fail(FSW_ECUDA, "litmus: capture"));
    launch_poison(sx, g.pool + off, m->store_bytes, pat);
    if (stage) launch_poison(sx, stage, stage_bytes, pat ^ 0x20u);
    cudaMemsetAsync(g.ready, 0, sizeof(uint32_t) * m->layers.size(), sx);
    cudaMemsetAsync(g.ctl, 0, sizeof(DevCtl), sx);
    cudaMemsetAsync(g.ctl_tail, 0, sizeof(DevCtl), sx);
    cudaMemsetAsync(g.progress, 0, 128 * kMaxWaitSrc, sx);
    cudaEventRecord(g.evfork, sx);
    cudaStreamWaitEvent(sc, g.evfork, 0);
    const int threads = (int)c->cfg.copy_threads;
    uint32_t gate = (uint32_t)ctas;
    if (engine == FSW_ENGINE_SM) {
        launch_swap(sc, (int)ctas, threads, m->store, dst, nullptr, ps->dev, (uint32_t)ps->host.size(), g.ready, g.ctl, g.ctl, 0);
    } else if (engine == FSW_ENGINE_SMZ) {
        launch_swapz(sc, (int)ctas, threads, m->zstore, 0, dst, nullptr, zs->dev, (uint32_t)zs->host.size(), g.ready, g.ctl, g.ctl,
                     0, 0, nullptr, zs->htab);
    } else if (engine == FSW_ENGINE_DMA) {
        gate = 0;  // no producer kernel: the copy engine publishes with fenced stream writes
        uint32_t cnt = 0;
        for (size_t gi = 0; gi < dp->groups.size(); ++gi) {
            const auto& gr = dp->groups[gi];
            if (!(c->fault_kind == FSW_FAULT_DROP_GROUP && c->fault_index == gi))
                cudaMemcpyAsync(weight_ptr(dst, gr.lo), m->store + gr.lo, gr.hi - gr.lo, cudaMemcpyHostToDevice, sc);
            wv(sc, (CUdeviceptr)g.progress, (cuuint32_t)(++cnt), 0);
        }
    } else {  // DMAZ / DMAZT: copy-engine groups into the staging buffer, decode kernel on its own stream
        cudaEventRecord(g.evd[0], sc);
        cudaStreamWaitEvent(g.sz, g.evd[0], 0);
        launch_swapz(g.sz, (int)ctas, threads, stage, zs->cfrom, dst, nullptr, zs->dev, zs->n_body, g.ready, g.ctl,
                     g.ctl, 0, 1, g.progress, zs->htab);
        if (engine == FSW_ENGINE_DMAZT) {  // + the zero-copy tail after the last body group
            cudaStreamWaitEvent(g.sd[1], g.evd[0], 0);
            launch_swapz_after(g.sd[1], (int)kSmzCtas, m->zstore, dst, nullptr, zs->dev + zs->n_body,
                               (uint32_t)zs->host.size() - zs->n_body, g.ready, g.ctl_tail, g.ctl, g.progress,
                               (uint32_t)zs->groups.size(), zs->htab);
            gate += kSmzCtas;
        }
        uint32_t cnt = 0;
        for (size_t gi = 0; gi < zs->groups.size(); ++gi) {
            const auto& gr = zs->groups[gi];
            if (!(c->fault_kind == FSW_FAULT_DROP_GROUP && c->fault_index == gi))
                cudaMemcpyAsync(stage + (gr.lo - zs->cfrom), m->zstore + gr.lo, gr.hi - gr.lo, cudaMemcpyHostToDevice, sc);
            wv(sc, (CUdeviceptr)g.progress, (cuuint32_t)(++cnt), 0);
        }
        cudaEventRecord(g.evz, g.sz);
        cudaStreamWaitEvent(sc, g.evz, 0);
        if (engine == FSW_ENGINE_DMAZT) {
            cudaEventRecord(g.evd[1], g.sd[1]);
            cudaStreamWaitEvent(sc, g.evd[1], 0);
        }
    }
    launch_litmus_check(sx, (int)ctas, dst, golden, dlayers, (uint32_t)ly.size(), wb, per_layer, g.ctl, gate, dcnt, dcnt + 1);
    cudaEventRecord(g.evjoin, sc);
    cudaStreamWaitEvent(sx, g.evjoin, 0);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(sx, &graph);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return finish(fail(FSW_ECUDA, "litmus: capture failed: %s", cudaGetErrorString(e)));
    }
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return finish(fail(FSW_ECUDA, "litmus: instantiate: %s", cudaGetErrorString(e)));
    for (uint32_t it = 0; it < iters; ++it) {
        e = cudaGraphLaunch(exec, sx);
        if (e == cudaSuccess && (it % 1024) == 1023) e = cudaStreamSynchronize(sx);
        if (e != cudaSuccess) return finish(fail(FSW_ECUDA, "litmus: iteration %u: %s", it, cudaGetErrorString(e)));
        if ((it % 1024) == 1023) {
            DevCtl ctl{};
            cudaMemcpy(&ctl, g.ctl, sizeof ctl, cudaMemcpyDeviceToHost);
            if (ctl.err) return finish(fail(FSW_ETIMEOUT, "litmus: watchdog (err %d, layer %d)", ctl.err, ctl.err_layer));
        }
    }
    if ((e = cudaStreamSynchronize(sx)) != cudaSuccess) return finish(fail(FSW_ECUDA, "litmus: %s", cudaGetErrorString(e)));
    DevCtl ctl{};
    unsigned long long cnt[2] = {0, 0};
    cudaMemcpy(&ctl, g.ctl, sizeof ctl, cudaMemcpyDeviceToHost);
    cudaMemcpy(cnt, dcnt, sizeof cnt, cudaMemcpyDeviceToHost);
    *bad_words = cnt[0];
    *checked_bytes = cnt[1];
    if (ctl.err) return finish(fail(FSW_ETIMEOUT, "litmus: watchdog (err %d, layer %d)", ctl.err, ctl.err_layer));
    return finish(FSW_OK);
}
