// graph.cpp — swap plans of every engine (SM pieces, DMA groups, link-coded pieces and groups,
// striped shares) and the capture of one CUDA graph per (model, GPU, invoke mode).
#include "rt_internal.h"

// Swap pieces for one chunk size / order: execution order, never straddling a layer region.
fsw_status get_pieces(Model& m, Plan& p, Gpu& g, uint64_t chunk, int order, uint32_t seed, uint64_t from,
                             PieceSet** out) {
    auto key = std::make_tuple(chunk, order, seed, from);
    auto it = p.pieces.find(key);
    if (it != p.pieces.end()) {
        *out = &it->second;
        return FSW_OK;
    }
    PieceSet ps;
    for (uint32_t li = 0; li < m.layers.size(); ++li) {
        if (m.region_off[li] < from) continue;  // cached prefix
        for (uint64_t o = 0; o < m.region_bytes[li]; o += chunk)
            ps.host.push_back({m.region_off[li] + o, (uint32_t)std::min<uint64_t>(chunk, m.region_bytes[li] - o), li});
    }
    if (order == FSW_ORDER_REVERSE) std::reverse(ps.host.begin(), ps.host.end());
    if (order == FSW_ORDER_RANDOM) {
        std::mt19937_64 rng(seed);
        std::shuffle(ps.host.begin(), ps.host.end(), rng);
    }
    CU(cudaSetDevice(g.dev));
    CU(cudaMalloc(&ps.dev, sizeof(Piece) * ps.host.size()));
    CU(cudaMemcpy(ps.dev, ps.host.data(), sizeof(Piece) * ps.host.size(), cudaMemcpyHostToDevice));
    auto res = p.pieces.emplace(key, std::move(ps));
    *out = &res.first->second;
    return FSW_OK;
}

// Copy groups of the DMA engine: whole layers are merged in execution order until a group holds
// at least `grp` bytes; a layer region larger than 2·grp is split into ≈grp pieces (256-B
// aligned).  Layer regions are contiguous in the store, so groups tile [0, store_bytes).
static DmaPlan make_dma_plan(const Model& m, uint64_t grp, uint32_t streams, uint64_t from, uint64_t split) {
    DmaPlan d;
    d.streams = streams;
    const size_t nl = m.layers.size();
    std::vector<uint32_t> last_group(nl, 0);
    uint64_t lo = from, hi = from;  // open group [lo, hi); groups tile [from, store_bytes)
    auto close = [&]() {
        if (hi > lo) {
            d.groups.push_back({lo, hi, (uint32_t)(d.groups.size() % streams)});
            lo = hi;
        }
    };
    // Taper: a group starting at `lo` aims at min(grp, max(tail_min, remaining / 2)) bytes, so the
    // groups shrink geometrically towards the end of the store.  The compute that trails the last
    // byte is then only the last small group's layers (big groups amortise the ~8 us per-copy
    // setup of the copy engine; small ones bound the tail).  Ramp: at a layer boundary a group also
    // closes once it holds ramp x the bytes already planned (>= tail_min), so the first layers land
    // early and their compute starts while the rest streams (a layer larger than the ramp is not split
    // for it: its kernel waits for its last byte anyway).
    const uint64_t total = m.store_bytes, tail_min = std::min<uint64_t>(grp, 1ull << 20);
    static const double frac = getenv("FSW_DMA_TAPER") ? atof(getenv("FSW_DMA_TAPER")) : 0.5;  // sweep hook
    // sweep hook, default off: measured (tools/linkcode_bench.py, profiles/r01/linkcode/) ramp 1-4 cost the
    // plain DMA engine 2-5 % on ResNet-50 and was neutral on BERT-base
    static const double ramp = getenv("FSW_DMA_RAMP") ? atof(getenv("FSW_DMA_RAMP")) : 0.0;    // 0 = no ramp
    auto want = [&](uint64_t at) {
        return std::min(grp, std::max(tail_min, align_up((uint64_t)((double)(total - at) * frac), 256)));
    };
    auto want_close = [&](uint64_t at) {
        if (ramp <= 0) return want(at);
        return std::min(want(at), std::max(tail_min, (uint64_t)((double)(at - from) * ramp)));
    };
    for (size_t li = 0; li < nl; ++li) {
        const uint64_t ro = m.region_off[li], rb = m.region_bytes[li];
        if (!rb || ro < from) continue;
        if (ro == split) close();  // a group never straddles the prefix / suffix extents
        if (rb > 2 * want(ro)) {
            close();
            for (uint64_t o = 0; o < rb;) {
                const uint64_t w = want(ro + o);
                const uint64_t step = rb - o <= 2 * w ? rb - o : w;
                o += step;
                hi = ro + o;
                close();
            }
        } else {
            hi = ro + rb;
            if (hi - lo >= want_close(lo)) close();
        }
        last_group[li] = hi > lo ? (uint32_t)d.groups.size() : (uint32_t)d.groups.size() - 1;
    }
    close();
    d.target.assign(nl, {});
    for (size_t li = 0; li < nl; ++li) {
        if (!m.region_bytes[li] || m.region_off[li] < from) continue;
        const uint32_t gl = last_group[li];
        for (uint32_t j = 0; j < streams; ++j) d.target[li][j] = gl >= j ? (gl - j) / streams + 1 : 0;
    }
    return d;
}

const DmaPlan& get_dma_plan(Model& m, Plan& p, uint64_t grp, uint32_t streams, uint64_t from) {
    const auto key = std::make_tuple(grp, streams, from, m.split);
    auto it = p.dma.find(key);
    if (it != p.dma.end()) return it->second;
    return p.dma.emplace(key, make_dma_plan(m, grp, streams, from, m.split)).first->second;
}

// Host-only inspection of the DMA engine's copy plan (tests; no GPU needed).
extern "C" fsw_status fsw_debug_dma_plan(fsw_ctx* c, uint32_t id, uint64_t group_bytes, uint32_t streams,
                                         uint64_t* group_lo_hi, uint32_t* group_stream, uint32_t cap_groups,
                                         uint32_t* n_groups, uint32_t* layer_targets /* [n_layers][4] */) {
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (!n_groups || group_bytes == 0 || group_bytes % 256 || streams == 0 || streams > (uint32_t)kMaxWaitSrc)
        return fail(FSW_EINVAL, "dma_plan: bad argument");
    const DmaPlan d = make_dma_plan(*m, group_bytes, streams, 0, m->split);
    *n_groups = (uint32_t)d.groups.size();
    if (d.groups.size() > cap_groups) return fail(FSW_EINVAL, "dma_plan: %zu groups > cap %u", d.groups.size(), cap_groups);
    for (size_t i = 0; i < d.groups.size(); ++i) {
        if (group_lo_hi) {
            group_lo_hi[2 * i] = d.groups[i].lo;
            group_lo_hi[2 * i + 1] = d.groups[i].hi;
        }
        if (group_stream) group_stream[i] = d.groups[i].stream;
    }
    if (layer_targets)
        for (size_t li = 0; li < m->layers.size(); ++li)
            for (int j = 0; j < kMaxWaitSrc; ++j) layer_targets[4 * li + j] = d.target[li][j];
    return FSW_OK;
}

// Coded pieces of one link-coded swap (store offsets >= from) in the claim order.  DMAZ (grp > 0):
// copy groups of whole pieces over the coded bytes, in execution order, tapered like the DMA engine's
// (a group starting at coded offset `at` aims at min(grp, max(1 MiB, remaining / 2)) bytes), so the
// decode and compute that trail the last group are short.  Groups are dealt round-robin to `streams`
// copy streams; each piece records its group as (stream << 24 | index of the group on its stream).
// Host part of a link-coded swap plan (no device memory): the pieces >= from in execution order, and
// for DMAZ (grp > 0) the copy groups.  Used by get_zpieces and by the host-only debug export.
// DMAZT (tail > 0): the last `tail` KiB of coded bytes (whole pieces, at most a quarter of them) form the
// zero-copy tail (n_body = the first tail piece); the copy groups cover only the body.  Measured
// (tools/resnet_engine_probe.py): BERT-base 2.832 -> 2.771 ms with a 7-MB tail (it replaces the body's last,
// tapered copy groups, ~8 us each, and the decode lag behind the last one); GPT-2-XL is unchanged within
// noise; a 51-MB store (ResNet-50) gains nothing over SMZ.  FSW_DMAZT_TAIL_MB overrides (MB of coded bytes).
uint32_t dmazt_tail_permille() {  // the tail in KiB (name kept for the key tuple)
    static const uint32_t v = getenv("FSW_DMAZT_TAIL_MB") ? (uint32_t)(atof(getenv("FSW_DMAZT_TAIL_MB")) * 1024.0 + 0.5) : 7168u;
    return v;
}

// The model's entropy-code decode table on the current device, beside a piece set (nullptr: no entropy-coded piece).
static cudaError_t upload_htab(const Model& m, ZPieceSet& zs) {
    zs.htab = nullptr;
    if (m.htab.empty()) return cudaSuccess;
    cudaError_t e = cudaMalloc(&zs.htab, m.htab.size());
    if (e == cudaSuccess) e = cudaMemcpy(zs.htab, m.htab.data(), m.htab.size(), cudaMemcpyHostToDevice);
    return e;
}

static fsw_status make_zplan(const Model& m, uint64_t from, uint64_t grp, uint32_t streams, ZPieceSet& zs,
                             uint32_t tail_permille = 0) {
    for (const ZPiece& pc : m.zpieces)
        if (pc.off >= from) zs.host.push_back(pc);
    if (zs.host.empty()) return fail(FSW_EINVAL, "link-coded swap with nothing to move");
    zs.cfrom = zs.host.front().coff;
    zs.cend = align_up(zs.host.back().coff + zs.host.back().cbytes, 128);  // the coded store is 128-B padded
    zs.n_body = (uint32_t)zs.host.size();
    uint64_t body_end = zs.cend;
    if (grp && tail_permille) {
        const uint64_t tail = std::min<uint64_t>((uint64_t)tail_permille << 10, (zs.cend - zs.cfrom) / 4);
        uint32_t k = (uint32_t)zs.host.size();
        while (k > 1 && zs.cend - zs.host[k - 1].coff <= tail) --k;
        zs.n_body = k;  // at least one body piece
        body_end = k < zs.host.size() ? zs.host[k].coff : zs.cend;
    }
    if (grp) {
        // the DMA engine's plan (make_dma_plan) over coded bytes: tail taper inside layers, head ramp
        // at layer boundaries
        // head ramp on by default here (measured: DMAZ ResNet-50 0.890 -> 0.809 ms at ramp 4, BERT-base
        // neutral); off for the plain DMA engine, where it cost ResNet-50 2-5 %
        static const double ramp = getenv("FSW_DMAZ_RAMP") ? atof(getenv("FSW_DMAZ_RAMP")) : 4.0;
        static const double taper = getenv("FSW_DMAZ_TAPER") ? atof(getenv("FSW_DMAZ_TAPER")) : 0.5;  // sweep hook
        const uint64_t tail_min = std::min<uint64_t>(grp, 1ull << 20);
        uint64_t lo = zs.cfrom;
        for (size_t i = 0; i < zs.n_body; ++i) {
            ZPiece& pc = zs.host[i];
            const uint32_t gi = (uint32_t)zs.groups.size();
            pc.grp = ((gi % streams) << 24) | (gi / streams);
            const bool last = i + 1 == zs.n_body;
            const uint64_t hi = last ? body_end : zs.host[i + 1].coff;
            const uint64_t want = std::min(grp, std::max(tail_min, (uint64_t)((double)(zs.cend - lo) * taper)));
            const uint64_t want_close =
                ramp > 0 ? std::min(want, std::max(tail_min, (uint64_t)((double)(lo - zs.cfrom) * ramp))) : want;
            const bool boundary = last || zs.host[i + 1].layer != pc.layer;
            if (last || hi - lo >= want || (boundary && hi - lo >= want_close)) {
                zs.groups.push_back({lo, hi, gi % streams});
                lo = hi;
            }
        }
    }
    return FSW_OK;
}

fsw_status get_zpieces(Model& m, Plan& p, Gpu& g, int order, uint32_t seed, uint64_t from, uint64_t grp,
                       uint32_t streams, ZPieceSet** out, uint32_t tail_permille) {
    const auto key = std::make_tuple(order, seed, from, grp, streams, tail_permille);
    auto it = p.zp.find(key);
    if (it != p.zp.end()) {
        *out = &it->second;
        return FSW_OK;
    }
    ZPieceSet zs;
    fsw_status st = make_zplan(m, from, grp, streams, zs, tail_permille);
    if (st != FSW_OK) return st;
    // claim orders permute within the body and within the tail (each kernel claims from its own table)
    if (order == FSW_ORDER_REVERSE) {
        std::reverse(zs.host.begin(), zs.host.begin() + zs.n_body);
        std::reverse(zs.host.begin() + zs.n_body, zs.host.end());
    }
    if (order == FSW_ORDER_RANDOM) {
        std::mt19937_64 rng(seed);
        std::shuffle(zs.host.begin(), zs.host.begin() + zs.n_body, rng);
        std::shuffle(zs.host.begin() + zs.n_body, zs.host.end(), rng);
    }
    CU(cudaSetDevice(g.dev));
    CU(cudaMalloc(&zs.dev, sizeof(ZPiece) * zs.host.size()));
    CU(upload_htab(m, zs));
    CU(cudaMemcpy(zs.dev, zs.host.data(), sizeof(ZPiece) * zs.host.size(), cudaMemcpyHostToDevice));
    *out = &p.zp.emplace(key, std::move(zs)).first->second;
    return FSW_OK;
}

// Host-only inspection of the DMAZ copy plan (tests; no GPU needed).
extern "C" fsw_status fsw_debug_dmaz_plan(fsw_ctx* c, uint32_t id, uint64_t group_bytes, uint32_t streams,
                                          uint64_t* group_lo_hi, uint32_t* group_stream, uint32_t cap_groups,
                                          uint32_t* n_groups, uint32_t* piece_group) {
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (!m->zstore) return fail(FSW_ESTATE, "model %u is not link-coded", id);
    if (!n_groups || group_bytes == 0 || streams == 0 || streams > (uint32_t)kMaxWaitSrc)
        return fail(FSW_EINVAL, "dmaz_plan: bad argument");
    ZPieceSet zs;
    fsw_status st = make_zplan(*m, 0, group_bytes, streams, zs);
    if (st != FSW_OK) return st;
    *n_groups = (uint32_t)zs.groups.size();
    if (zs.groups.size() > cap_groups) return fail(FSW_EINVAL, "dmaz_plan: %zu groups > cap %u", zs.groups.size(), cap_groups);
    for (size_t i = 0; i < zs.groups.size(); ++i) {
        if (group_lo_hi) {
            group_lo_hi[2 * i] = zs.groups[i].lo;
            group_lo_hi[2 * i + 1] = zs.groups[i].hi;
        }
        if (group_stream) group_stream[i] = zs.groups[i].stream;
    }
    if (piece_group)
        for (size_t i = 0; i < zs.host.size(); ++i) piece_group[i] = zs.host[i].grp;
    return FSW_OK;
}

// Striped link-coded swap: runs of 16 consecutive coded pieces (256 KiB of store) dealt round-robin to
// n sources; source j's table lives on its device.
static uint64_t nodes_key(const std::vector<int>& src_node) {  // FNV-1a of the sources' nodes
    uint64_t h = 1469598103934665603ull;
    for (int v : src_node) h = (h ^ (uint64_t)(uint32_t)(v + 7)) * 1099511628211ull;
    return h ^ src_node.size();
}

fsw_status get_zstripe_pieces(Model& m, Plan& p, const std::vector<int>& src_node, uint32_t j, int dev, uint64_t from,
                              ZPieceSet** out) {
    const auto key = std::make_tuple(nodes_key(src_node), j, dev, from);
    auto it = p.zstripe.find(key);
    if (it != p.zstripe.end()) {
        *out = &it->second;
        return FSW_OK;
    }
    // units = runs of 16 coded pieces (256 KiB of store); each goes to a source on the NUMA node of its
    // first coded byte (stripe_deal: round-robin among them; over all sources on a single-node host)
    std::vector<const ZPiece*> sel;
    for (const ZPiece& pc : m.zpieces)
        if (pc.off >= from) sel.push_back(&pc);
    std::vector<int> unit_node;
    for (size_t q = 0; q < sel.size(); q += 16) unit_node.push_back(chunk_node(m.zstore_node, sel[q]->coff));
    const std::vector<uint32_t> owner = stripe_deal(unit_node, src_node);
    ZPieceSet zs;
    for (size_t q = 0; q < sel.size(); ++q)
        if (owner[q / 16] == j) zs.host.push_back(*sel[q]);
    CU(cudaSetDevice(dev));
    if (!zs.host.empty()) {
        CU(cudaMalloc(&zs.dev, sizeof(ZPiece) * zs.host.size()));
        CU(upload_htab(m, zs));
        CU(cudaMemcpy(zs.dev, zs.host.data(), sizeof(ZPiece) * zs.host.size(), cudaMemcpyHostToDevice));
    }
    *out = &p.zstripe.emplace(key, std::move(zs)).first->second;
    return FSW_OK;
}

// DMAZ striped swap: the coded pieces >= from cut into runs of ~run_bytes contiguous coded bytes (whole
// pieces, execution order), each run dealt to a source on the NUMA node of its first byte (stripe_deal).
// Source j copies its runs with its copy engine, back to back, into its own staging buffer (run k at
// staging offset Σ earlier runs), publishing the run count after each, and its decode kernel decodes the
// run's pieces from there into the target.  groups = the runs [lo, hi) of the coded store; each piece's
// coff is rewritten to its staging offset and grp to its run's index (stream 0).
fsw_status get_zstripe_dma(Model& m, Plan& p, const std::vector<int>& src_node, uint32_t j, int dev, uint64_t from,
                           uint64_t run_bytes, ZPieceSet** out) {
    const auto key = std::make_tuple(nodes_key(src_node), j, dev, from, run_bytes);
    auto it = p.zstripe_dma.find(key);
    if (it != p.zstripe_dma.end()) {
        *out = &it->second;
        return FSW_OK;
    }
    std::vector<const ZPiece*> sel;
    for (const ZPiece& pc : m.zpieces)
        if (pc.off >= from) sel.push_back(&pc);
    if (sel.empty()) return fail(FSW_EINVAL, "link-coded swap with nothing to move");
    const uint64_t cend = align_up(sel.back()->coff + sel.back()->cbytes, 128);
    std::vector<std::pair<size_t, size_t>> runs;  // [first, last) piece index
    for (size_t a = 0; a < sel.size();) {
        size_t b = a + 1;
        while (b < sel.size() && sel[b]->coff - sel[a]->coff < run_bytes) ++b;
        runs.push_back({a, b});
        a = b;
    }
    std::vector<int> unit_node;
    for (auto& r : runs) unit_node.push_back(chunk_node(m.zstore_node, sel[r.first]->coff));
    const std::vector<uint32_t> owner = stripe_deal(unit_node, src_node);
    ZPieceSet zs;
    uint64_t soff = 0;
    for (size_t k = 0; k < runs.size(); ++k) {
        if (owner[k] != j) continue;
        const uint64_t lo = sel[runs[k].first]->coff, hi = runs[k].second < sel.size() ? sel[runs[k].second]->coff : cend;
        const uint32_t gi = (uint32_t)zs.groups.size();
        zs.groups.push_back({lo, hi, 0});
        for (size_t q = runs[k].first; q < runs[k].second; ++q) {
            ZPiece pc = *sel[q];
            pc.coff = soff + (pc.coff - lo);
            pc.grp = gi;
            zs.host.push_back(pc);
        }
        soff += hi - lo;
    }
    zs.cfrom = 0;
    zs.cend = soff;  // staging bytes this source needs
    CU(cudaSetDevice(dev));
    if (!zs.host.empty()) {
        CU(cudaMalloc(&zs.dev, sizeof(ZPiece) * zs.host.size()));
        CU(upload_htab(m, zs));
        CU(cudaMemcpy(zs.dev, zs.host.data(), sizeof(ZPiece) * zs.host.size(), cudaMemcpyHostToDevice));
    }
    *out = &p.zstripe_dma.emplace(key, std::move(zs)).first->second;
    return FSW_OK;
}

// Striped swap: the execution-order piece list of the SM engine dealt round-robin to n sources
// (piece q goes to source q mod n), so every source streams a share of every layer and all of them
// advance through the model together; source j's table is allocated on source j's device.
fsw_status get_stripe_pieces(Model& m, Plan& p, uint64_t chunk, const std::vector<int>& src_node, uint32_t j, int dev,
                             uint64_t from, PieceSet** out) {
    const auto key = std::make_tuple(chunk, nodes_key(src_node), j, dev, from);
    auto it = p.stripe.find(key);
    if (it != p.stripe.end()) {
        *out = &it->second;
        return FSW_OK;
    }
    // units = pieces; each goes to a source on the NUMA node of its first byte (stripe_deal)
    std::vector<Piece> all;
    std::vector<int> unit_node;
    for (uint32_t li = 0; li < m.layers.size(); ++li)
        for (uint64_t o = 0; m.region_off[li] >= from && o < m.region_bytes[li]; o += chunk) {
            all.push_back({m.region_off[li] + o, (uint32_t)std::min<uint64_t>(chunk, m.region_bytes[li] - o), li});
            unit_node.push_back(chunk_node(m.store_node, m.region_off[li] + o));
        }
    const std::vector<uint32_t> owner = stripe_deal(unit_node, src_node);
    PieceSet ps;
    for (size_t q = 0; q < all.size(); ++q)
        if (owner[q] == j) ps.host.push_back(all[q]);
    CU(cudaSetDevice(dev));
    if (!ps.host.empty()) {
        CU(cudaMalloc(&ps.dev, sizeof(Piece) * ps.host.size()));
        CU(cudaMemcpy(ps.dev, ps.host.data(), sizeof(Piece) * ps.host.size(), cudaMemcpyHostToDevice));
    }
    *out = &p.stripe.emplace(key, std::move(ps)).first->second;
    return FSW_OK;
}

// The readiness wait of a kernel of layer `layer` for this invoke configuration.
static Wait layer_wait(Model& m, Gpu& g, const InvokeCfg& ic, int layer) {
    Wait w{};
    w.ctl = g.ctl;
    w.layer = layer;
    w.trace = g.trace;
    if (ic.cold && m.region_bytes[layer] > 0 && m.region_off[layer] >= ic.from) {
        if (engine_bytes_ready(ic.engine)) {
            w.n = 1;
            w.ready[0] = g.ready + layer;
            w.target[0] = (uint32_t)m.region_bytes[layer];
            w.sys = ic.striped ? 1 : 0;
        } else {
            w.n = ic.dma_plan->streams;
            for (uint32_t j = 0; j < w.n; ++j) {
                w.ready[j] = g.progress + 32 * j;
                w.target[j] = ic.dma_plan->target[layer][j];
            }
        }
    }
    return w;
}

static fsw_status enqueue_layers(Model& m, Plan& p, Gpu& g, const InvokeCfg& ic, cudaStream_t s) {
    const DevDesc* d = reinterpret_cast<const DevDesc*>(g.dstage);
    if (p.mega.on) {
        // the persistent transformer kernel: one launch; its op table (this invoke configuration's waits)
        // was written to device memory by build_graph before the capture began
        cudaMemsetAsync(p.mega.op_cnt, 0, 128 * (p.mega.ops.size() + (size_t)p.mega.ctas), s);
        launch_mega(s, p.mega.ctas, d, reinterpret_cast<const MkOp*>(p.last_mk_ops), (uint32_t)p.mega.ops.size(),
                    p.mega.op_cnt, p.mega.tmaps, g.gemm_ctr, p.mega.part);
        return FSW_OK;
    }
    for (const Launch& x : p.launches) {
        Wait w = layer_wait(m, g, ic, x.layer);
        if (x.wait_layer2 >= 0) {  // a folded LayerNorm: its γ / β must have landed too
            const Wait w2 = layer_wait(m, g, ic, x.wait_layer2);
            for (uint32_t j = 0; j < w2.n; ++j) {
                uint32_t k = 0;
                while (k < w.n && w.ready[k] != w2.ready[j]) ++k;
                if (k < w.n) {
                    w.target[k] = std::max(w.target[k], w2.target[j]);  // the same counter (DMA group counts)
                } else if (w.n < (uint32_t)kMaxWaitSrc) {
                    w.ready[w.n] = w2.ready[j];
                    w.target[w.n++] = w2.target[j];
                    w.sys = w.sys | w2.sys;
                } else {
                    return fail(FSW_EINVAL, "plan: too many readiness counters for layer %d", x.layer);
                }
            }
        }
        switch (x.kind) {
            case K_EMBED: launch_embed(s, d, w, x.embed); break;
            case K_LN: launch_layernorm(s, d, w, x.ln); break;
            case K_GEMV: launch_gemv(s, d, w, x.gemv); break;
            case K_GEMM: launch_gemm(s, d, w, &x.tmap, x.gemm, &g.wmap); break;
            case K_ATTN: {
                AttnArgs a = x.attn;
                a.layer = x.layer;
                a.trace = g.trace;
                if (x.attn_tc) launch_attention_tc(s, &x.tmap, a);
                else launch_attention(s, a);
                break;
            }
            case K_IM2COL: {
                Im2colArgs a = x.im2col;
                a.layer = x.layer;
                a.trace = g.trace;
                launch_im2col(s, a);
                break;
            }
            case K_MAXPOOL:
            case K_AVGPOOL: {
                PoolArgs a = x.pool;
                a.layer = x.layer;
                a.trace = g.trace;
                if (x.kind == K_MAXPOOL) launch_maxpool(s, a);
                else launch_avgpool(s, a);
                break;
            }
        }
    }
    return FSW_OK;
}

PFN_writeValue32 get_write_value32() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess) return nullptr;
    return reinterpret_cast<PFN_writeValue32>(p);
}

// Capture the invoke graph of (model, GPU, cfg).  Root: H2D of [desc | input]; cold adds the
// ready/ctl reset, the swap kernel on its own stream (bracketed by external event nodes for
// timing) and the gate; then the flag-gated layer kernels; then D2H of output and ctl.
fsw_status build_graph(fsw_ctx* c, Model& m, Plan& p, Gpu& g, const InvokeCfg& ic, cudaGraphExec_t* out) {
    PieceSet* ps = nullptr;
    ZPieceSet* zs = nullptr;
    if (ic.cold && ic.engine == FSW_ENGINE_SM && !ic.striped) {
        fsw_status s = get_pieces(m, p, g, ic.chunk, ic.order, ic.seed, ic.from, &ps);
        if (s != FSW_OK) return s;
    }
    if (ic.cold && engine_coded(ic.engine) && !ic.striped) {
        fsw_status s = get_zpieces(m, p, g, ic.order, ic.seed, ic.from, engine_dmaz(ic.engine) ? ic.zgrp : 0,
                                   engine_dmaz(ic.engine) ? ic.zstreams : 1, &zs,
                                   ic.engine == FSW_ENGINE_DMAZT ? dmazt_tail_permille() : 0);
        if (s != FSW_OK) return s;
        if (engine_dmaz(ic.engine) && zs->cend - zs->cfrom > g.zstage_cap) return fail(FSW_EINVAL, "staging buffer too small");
    }
    if (ic.cold && (engine_bytes_ready(ic.engine) || ic.striped) && m.layers.size() > g.ready_cap)
        return fail(FSW_EINVAL, "too many layers");
    CU(cudaSetDevice(g.dev));
    if (p.mega.on) {  // the persistent kernel's op table with this configuration's waits (no allocation in a capture)
        std::vector<MkOp> ops = p.mega.ops;
        for (MkOp& op : ops) op.w = layer_wait(m, g, ic, op.layer);
        void* dev = nullptr;
        CU(cudaMalloc(&dev, sizeof(MkOp) * ops.size()));
        p.last_mk_ops = dev;
        CU(cudaMemcpy(dev, ops.data(), sizeof(MkOp) * ops.size(), cudaMemcpyHostToDevice));
    }
    cudaStream_t sx = g.sx, sc = g.sc;
    CU(cudaStreamBeginCapture(sx, cudaStreamCaptureModeThreadLocal));
    // The swap starts as early as possible: the DMA engine needs only its counters reset; the SM
    // engine also reads the invoke descriptor and the control block.  The input (up to 300 KB for
    // ResNet-50) is copied after the fork, overlapping the swap.
    const bool dma_cold = ic.cold && !ic.striped && ic.engine == FSW_ENGINE_DMA;
    // DMAZ: the copy engine also needs only its group counters reset; the decode kernel waits for the
    // rest of the setup (descriptor, control block, ready counters) through evset
    const bool dmaz_cold = ic.cold && !ic.striped && engine_dmaz(ic.engine);
    if (dma_cold || dmaz_cold) cudaMemsetAsync(g.progress, 0, 128 * kMaxWaitSrc, sx);
    if (dmaz_cold) {
        cudaEventRecord(g.evfork, sx);
        cudaStreamWaitEvent(sc, g.evfork, 0);
    }
    if (!dma_cold) cudaMemcpyAsync(g.dstage, g.hstage, kStageHdr, cudaMemcpyHostToDevice, sx);
    // striped: the counters and the control block are reset before the sources start (outside)
    if (!ic.striped && !dma_cold) cudaMemsetAsync(g.ctl, 0, sizeof(DevCtl), sx);
    if (ic.cold && ic.engine == FSW_ENGINE_DMAZT) cudaMemsetAsync(g.ctl_tail, 0, sizeof(DevCtl), sx);
    if (ic.cold && ic.striped && !ic.no_overlap && ic.local_ctas) launch_gate(sx, g.ctl, ic.local_ctas);
    if (ic.cold && !ic.striped) {
        if (engine_bytes_ready(ic.engine)) cudaMemsetAsync(g.ready, 0, sizeof(uint32_t) * m.layers.size(), sx);
        if (dmaz_cold) {
            cudaEventRecord(g.evset, sx);
        } else {
            cudaEventRecord(g.evfork, sx);
            cudaStreamWaitEvent(sc, g.evfork, 0);
        }
        cudaEventRecordWithFlags(g.evs0, sc, cudaEventRecordExternal);
        const DevDesc* desc = reinterpret_cast<const DevDesc*>(g.dstage);
        if (ic.engine == FSW_ENGINE_SM) {
            launch_swap(sc, (int)ic.ctas, (int)c->cfg.copy_threads, m.store, DevDesc{}, desc, ps->dev,
                        (uint32_t)ps->host.size(), g.ready, g.ctl, g.ctl, 0);
        } else if (ic.engine == FSW_ENGINE_SMZ) {
            // zero-copy decode: coded pieces straight from the mapped coded store over the host link
            launch_swapz(sc, (int)ic.ctas, (int)c->cfg.copy_threads, m.zstore, 0, DevDesc{}, desc, zs->dev,
                         (uint32_t)zs->host.size(), g.ready, g.ctl, g.ctl, 0, 0, nullptr, zs->htab);
        } else if (engine_dmaz(ic.engine)) {
            // copy engine moves coded groups into the staging buffer (a fenced stream write of the group
            // count after each); the decode kernel, forked onto its own stream, waits per piece for its
            // group and decodes from HBM into the extent
            static PFN_writeValue32 wv = get_write_value32();
            if (!wv) return fail(FSW_ECUDA, "cuStreamWriteValue32 entry point unavailable");
            // no-overlap: the decode kernel follows the copies on the copy stream (it then waits on nothing,
            // which also keeps the graph safe under tools that serialise kernels)
            const bool serial = ic.no_overlap;
            cudaStream_t sdec = serial ? sc : g.sz;
            cudaEventRecord(g.evd[0], sc);
            if (!serial) {
                cudaStreamWaitEvent(g.sz, g.evd[0], 0);
                cudaStreamWaitEvent(g.sz, g.evset, 0);
            }
            for (uint32_t j = 1; j < ic.zstreams; ++j) cudaStreamWaitEvent(g.sd[j], g.evd[0], 0);
            auto decode = [&]() {
                launch_swapz(sdec, (int)ic.ctas, (int)c->cfg.copy_threads, g.zstage, zs->cfrom, DevDesc{}, desc, zs->dev,
                             zs->n_body, g.ready, g.ctl, g.ctl, 0, 1, g.progress, zs->htab);
            };
            // DMAZT: the zero-copy tail kernel on copy stream 1, resident from the start (the gate counts its CTAs);
            // it reads the host store only once the last body group has landed (one transfer on the link at a time)
            const uint32_t n_tail = (uint32_t)zs->host.size() - zs->n_body;
            auto tail = [&](cudaStream_t st) {
                launch_swapz_after(st, (int)ic.tail_ctas, m.zstore, DevDesc{}, desc, zs->dev + zs->n_body, n_tail, g.ready, g.ctl_tail,
                                   g.ctl, g.progress, (uint32_t)zs->groups.size(), zs->htab);
            };
            if (ic.engine == FSW_ENGINE_DMAZT && !serial) {
                cudaStreamWaitEvent(g.sd[1], g.evd[0], 0);
                cudaStreamWaitEvent(g.sd[1], g.evset, 0);
                tail(g.sd[1]);
            }
            if (!serial) decode();
            uint32_t cnt[kMaxWaitSrc] = {};
            for (size_t gi = 0; gi < zs->groups.size(); ++gi) {
                const auto& gr = zs->groups[gi];
                cudaStream_t sj = g.sd[gr.stream];
                if (!(c->fault_kind == FSW_FAULT_DROP_GROUP && c->fault_index == gi))  // fault injection (tests)
                    cudaMemcpyAsync(g.zstage + (gr.lo - zs->cfrom), m.zstore + gr.lo, gr.hi - gr.lo, cudaMemcpyHostToDevice, sj);
                wv(sj, (CUdeviceptr)(g.progress + 32 * gr.stream), (cuuint32_t)(++cnt[gr.stream]), 0);
            }
            for (uint32_t j = 1; j < ic.zstreams; ++j) {
                cudaEventRecord(g.evd[j], g.sd[j]);
                cudaStreamWaitEvent(sc, g.evd[j], 0);
            }
            if (serial) {
                cudaStreamWaitEvent(sc, g.evset, 0);  // the decode reads the descriptor and ready counters
                decode();
                if (ic.engine == FSW_ENGINE_DMAZT) tail(sc);
            } else {
                cudaEventRecord(g.evz, g.sz);
                cudaStreamWaitEvent(sc, g.evz, 0);
                if (ic.engine == FSW_ENGINE_DMAZT) {
                    cudaEventRecord(g.evd[1], g.sd[1]);
                    cudaStreamWaitEvent(sc, g.evd[1], 0);
                }
            }
        } else {
            // Copy-engine DMA from the pinned store (the paper's transfer) in
            // layer-aligned groups (its "group" pipelining unit), dealt round-robin
            // to the copy streams so one engine's per-copy setup overlaps another's transfer.  After
            // each group a stream memory write (no kernel, so no SM is needed while layer kernels
            // spin) publishes that stream's group count; its default flags fence the copy first.
            static PFN_writeValue32 wv = get_write_value32();
            if (!wv) return fail(FSW_ECUDA, "cuStreamWriteValue32 entry point unavailable");
            const DmaPlan& dp = *ic.dma_plan;
            cudaEventRecord(g.evd[0], sc);
            for (uint32_t j = 1; j < dp.streams; ++j) cudaStreamWaitEvent(g.sd[j], g.evd[0], 0);
            uint32_t cnt[kMaxWaitSrc] = {};
            for (size_t gi = 0; gi < dp.groups.size(); ++gi) {
                const auto& gr = dp.groups[gi];
                cudaStream_t sj = g.sd[gr.stream];
                const uint8_t* from_ptr = ic.src_host ? m.store + gr.lo : weight_ptr(ic.src, gr.lo);
                if (!(c->fault_kind == FSW_FAULT_DROP_GROUP && c->fault_index == gi))  // fault injection (tests)
                    cudaMemcpyAsync(weight_ptr(ic.dst, gr.lo), from_ptr, gr.hi - gr.lo, cudaMemcpyDefault, sj);
                wv(sj, (CUdeviceptr)(g.progress + 32 * gr.stream), (cuuint32_t)(++cnt[gr.stream]), 0);
            }
            for (uint32_t j = 1; j < dp.streams; ++j) {
                cudaEventRecord(g.evd[j], g.sd[j]);
                cudaStreamWaitEvent(sc, g.evd[j], 0);
            }
        }
        cudaEventRecordWithFlags(g.evs1, sc, cudaEventRecordExternal);
        cudaEventRecord(g.evjoin, sc);
    }
    if (dma_cold) {
        cudaMemcpyAsync(g.dstage, g.hstage, kStageHdr, cudaMemcpyHostToDevice, sx);
        cudaMemsetAsync(g.ctl, 0, sizeof(DevCtl), sx);
    }
    cudaMemcpyAsync(g.dstage + kStageHdr, g.hstage + kStageHdr, m.input_bytes, cudaMemcpyHostToDevice, sx);
    if (ic.cold && !ic.striped) {
        if (ic.no_overlap) cudaStreamWaitEvent(sx, g.evjoin, 0);
        else if (engine_bytes_ready(ic.engine)) launch_gate(sx, g.ctl, ic.ctas + ic.tail_ctas);
    }
    const fsw_status lst = enqueue_layers(m, p, g, ic, sx);
    if (lst != FSW_OK) {
        cudaGraph_t dead = nullptr;
        cudaStreamEndCapture(sx, &dead);
        if (dead) cudaGraphDestroy(dead);
        cudaGetLastError();
        return lst;
    }
    if (ic.cold && !ic.striped && !ic.no_overlap) cudaStreamWaitEvent(sx, g.evjoin, 0);  // swap stamps final
    launch_finish(sx, g.ctl, g.ws + p.slot_off[m.output_slot], m.output_bytes, g.hout, g.hctl);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(sx, &graph);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(FSW_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
    }
    e = cudaGraphInstantiate(out, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(FSW_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
    return FSW_OK;
}

