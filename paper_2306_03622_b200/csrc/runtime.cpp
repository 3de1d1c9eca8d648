// runtime.cpp — libfsw host runtime behind include/fsw.h.
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
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "fsw.h"
#include "kernels.h"
#include "policy.h"

using namespace fsw;

// ==========================================================================================
// errors
// ==========================================================================================
static thread_local std::string g_err;

static fsw_status fail(fsw_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) return fail(FSW_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                                           __FILE__, __LINE__);                                    \
    } while (0)

extern "C" const char* fsw_last_error(void) { return g_err.c_str(); }
extern "C" const char* fsw_version(void) { return "fsw 0.1 (sm_100a)"; }

static inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
static double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// ==========================================================================================
// Arena: best-fit extent allocator with coalescing (the pre-allocated pool)
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
// model + plans
// ==========================================================================================
enum { LAYOUT_ROWMAJOR = 0, LAYOUT_TILED = 1 };

struct TensorInfo {
    fsw_tensor t;
    uint64_t st_off = 0, st_bytes = 0;
    uint32_t layout = LAYOUT_ROWMAJOR, rows = 0, cols = 0, rows_pad = 0, cols_pad = 0;
    int owner = -1;
    bool placed = false;
};

enum KernelKind { K_EMBED, K_LN, K_GEMV, K_GEMM, K_ATTN, K_IM2COL, K_MAXPOOL, K_AVGPOOL };

struct Launch {  // one kernel of the layer graph (addresses resolved for one GPU workspace)
    KernelKind kind;
    int layer;
    EmbedArgs embed;
    LnArgs ln;
    GemvArgs gemv;
    GemmArgs gemm;
    CUtensorMap tmap;
    AttnArgs attn;
    Im2colArgs im2col;
    PoolArgs pool;
};

struct Gpu;

struct GraphKey {
    int cold, flags, order, engine;
    uint64_t chunk;
    uint32_t seed, ctas, extra;
    uint64_t from = 0;   // first swapped store byte (partial caching: the cached prefix is skipped)
    int64_t pext = -1;   // DMA graphs: prefix extent offset (baked address)
    bool operator<(const GraphKey& o) const {
        return std::tie(cold, flags, order, engine, chunk, seed, ctas, extra, from, pext) <
               std::tie(o.cold, o.flags, o.order, o.engine, o.chunk, o.seed, o.ctas, o.extra, o.from, o.pext);
    }
};

// DMA engine plan: layer-aligned copy groups dealt round-robin to `streams` copy streams, and
// for every layer the per-stream group count that covers the layer's last byte.
struct DmaPlan {
    struct Group { uint64_t lo, hi; uint32_t stream; };
    std::vector<Group> groups;
    std::vector<std::array<uint32_t, kMaxWaitSrc>> target;  // [layer][stream]
    uint32_t streams = 1;
};

struct PieceSet {
    Piece* dev = nullptr;
    std::vector<Piece> host;
};

// Link-coded engines: the coded pieces one swap moves (store offsets >= from), with the DMA+decode
// engine's copy groups over the coded bytes [group lo, hi) and each piece's group index.
struct ZPieceSet {
    ZPiece* dev = nullptr;
    std::vector<ZPiece> host;
    std::vector<std::pair<uint64_t, uint64_t>> groups;  // DMAZ: coded-store byte ranges, in order
    uint64_t cfrom = 0, cend = 0;                        // coded bytes [cfrom, cend) cover the pieces
};

struct Plan {  // one model on one GPU
    bool built = false;
    std::vector<Launch> launches;
    std::vector<uint64_t> slot_off;      // workspace offset of each slot
    std::vector<int64_t> shadow_off;     // bf16 shadow of an f32 slot, or -1
    uint64_t ws_bytes = 0;
    std::map<GraphKey, cudaGraphExec_t> graphs;
    std::map<std::tuple<uint64_t, int, uint32_t, uint64_t>, PieceSet> pieces;  // (chunk, order, seed, from)
    std::map<std::tuple<uint64_t, uint32_t, uint64_t, uint64_t>, DmaPlan> dma;  // (group bytes, streams, from, split)
    // striped swap: source j of n gets every n-th piece; its table lives on the source's device
    std::map<std::tuple<uint64_t, uint32_t, uint32_t, int, uint64_t>, PieceSet> stripe;  // (chunk, n, j, device, from)
    // link-coded engines: (order, seed, from, DMAZ group bytes or 0 for SMZ) and striped (n, j, device, from)
    std::map<std::tuple<int, uint32_t, uint64_t, uint64_t>, ZPieceSet> zp;
    std::map<std::tuple<uint32_t, uint32_t, int, uint64_t>, ZPieceSet> zstripe;
};

struct Model {
    uint32_t id;
    std::string name;
    std::vector<TensorInfo> tensors;
    std::vector<uint32_t> refs;
    std::vector<fsw_slot> slots;
    std::vector<fsw_layer> layers;
    std::vector<uint64_t> region_off, region_bytes;
    int32_t input_slot, output_slot;
    uint64_t input_bytes = 0, output_bytes = 0, algorithmic_bytes = 0;
    uint32_t n_gemm = 0;
    uint8_t* store = nullptr;  // pinned, mapped host store (execution order)
    uint64_t store_bytes = 0, store_alloc = 0;
    bool store_wc = false;
    int numa_node = -1;        // node the store's pages were bound to (mbind before first touch), or -1
    // exponent-coded copy of the store (FSW_REG_LINK_CODE; kernels.h): pinned, mapped
    uint8_t* zstore = nullptr;
    uint64_t zbytes = 0, zalloc = 0;
    std::vector<ZPiece> zpieces;  // execution order, grp = 0
    // residency per GPU
    std::vector<int64_t> extent;       // pool offset of the model (split = 0) or of its suffix, or -1
    // partial-parameter caching: store bytes [0, split) — whole layers —
    // live in a separate prefix extent that pool evictions keep (valid once its bytes landed)
    uint64_t split = 0;
    std::vector<int64_t> pextent;      // prefix extent per GPU, or -1
    std::vector<uint8_t> pvalid;       // prefix bytes present
    std::vector<uint64_t> last_use;
    std::vector<std::unique_ptr<Plan>> plans;
    int inflight = 0;
    // heavy / light class for placement and eviction: 1, 0, or -1 auto
    int heavy = -1;
    double cold_ms_sum = 0, warm_ms_sum = 0;
    uint64_t n_cold_runs = 0, n_warm_runs = 0;
};

// A swap-kernel slot of a GPU acting as a striped-swap source for some target (its own ticket
// counter, stream and completion event).  A GPU can feed several targets' swaps at once.
struct SrcSlot {
    DevCtl* ctl = nullptr;
    cudaStream_t st = nullptr;
    cudaEvent_t done = nullptr;
    bool busy = false;
};
constexpr int kSrcSlots = 4;

struct Gpu {
    int dev = 0;
    SrcSlot src[kSrcSlots];
    cudaStream_t sx = nullptr, sc = nullptr;
    cudaStream_t sd[kMaxWaitSrc] = {};  // DMA copy streams (sd[0] == sc)
    cudaEvent_t evd[kMaxWaitSrc] = {};  // fork / join events of the DMA streams
    uint32_t* progress = nullptr;       // DMA: one group counter per copy stream, 128 B apart
    uint32_t* gemm_ctr = nullptr;       // split-K tile arrival counters (self-resetting)
    uint8_t* pool = nullptr;
    uint64_t pool_bytes = 0;
    fsw_arena* arena = nullptr;
    uint8_t* ws = nullptr;
    uint64_t ws_bytes = 0;
    uint32_t* ready = nullptr;
    uint32_t ready_cap = 0;
    DevCtl* ctl = nullptr;
    uint8_t* zstage = nullptr;   // DMAZ: device staging buffer for coded bytes (grown on demand)
    uint64_t zstage_cap = 0;
    uint32_t zstage_gen = 0;     // bumped on every reallocation (graphs bake the address)
    cudaStream_t sz = nullptr;   // DMAZ: decode-kernel stream
    uint8_t* dstage = nullptr;   // device: [DevDesc | pad | input]
    uint8_t* hstage = nullptr;   // pinned: same layout
    uint8_t* hout = nullptr;     // pinned, mapped: output (written by k_finish)
    DevCtl* hctl = nullptr;      // pinned, mapped: ctl copy (written by k_finish)
    uint64_t stage_cap = 0, out_cap = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs0 = nullptr, evs1 = nullptr, evfork = nullptr, evjoin = nullptr;
    bool busy = false;
    int loading = 0;  // 0, or 1 / 2 while a light / heavy model is being swapped in from the host
    uint64_t generation = 0;
    // stats
    uint64_t n_evictions = 0, bytes_swapped_total = 0, n_cold = 0, n_warm = 0;
};

constexpr uint64_t kStageHdr = 256;
constexpr uint32_t kGemmCtrs = 1u << 16;

// Tiling of one tcgen05 GEMM launch (gemm_tc.cu): tile width BN and split-K factor.
struct Tiling { int bn; uint32_t splits, kt_per; bool cluster; };
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

struct fsw_ctx {
    fsw_config cfg{};
    std::vector<Gpu> gpus;
    std::vector<std::unique_ptr<Model>> models;  // index = id (nullptr after unregister)
    std::mutex mu;
    std::condition_variable cv;
    uint64_t clock = 0;
    std::vector<std::vector<char>> peer;  // peer[i][j]: GPU i can store into GPU j's memory
    std::vector<int> neighbor;            // GPU sharing a PCIe switch (-1 none), fsw_config.pcie_neighbor
};

// ==========================================================================================
// init / shutdown
// ==========================================================================================
static fsw_status init_gpu(fsw_ctx* c, Gpu& g) {
    CU(cudaSetDevice(g.dev));
    CU(cudaFree(nullptr));  // create the context now (one shared runtime per GPU)
    init_gemm_attrs();
    init_ops_attrs();
    init_swap_attrs();
    CU(cudaStreamCreateWithFlags(&g.sx, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&g.sc, cudaStreamNonBlocking));
    g.sd[0] = g.sc;
    CU(cudaStreamCreateWithFlags(&g.sz, cudaStreamNonBlocking));
    for (int j = 1; j < kMaxWaitSrc; ++j) CU(cudaStreamCreateWithFlags(&g.sd[j], cudaStreamNonBlocking));
    for (int j = 0; j < kMaxWaitSrc; ++j) CU(cudaEventCreateWithFlags(&g.evd[j], cudaEventDisableTiming));
    CU(cudaMalloc(&g.progress, 128 * kMaxWaitSrc));
    CU(cudaMalloc(&g.gemm_ctr, sizeof(uint32_t) * kGemmCtrs));
    for (SrcSlot& sl : g.src) {
        CU(cudaMalloc(&sl.ctl, sizeof(DevCtl)));
        CU(cudaStreamCreateWithFlags(&sl.st, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    }
    CU(cudaMemset(g.gemm_ctr, 0, sizeof(uint32_t) * kGemmCtrs));
    CU(cudaMemset(g.progress, 0, 128 * kMaxWaitSrc));
    size_t free_b = 0, total_b = 0;
    CU(cudaMemGetInfo(&free_b, &total_b));
    uint64_t want = c->cfg.pool_bytes_per_gpu ? c->cfg.pool_bytes_per_gpu : (64ull << 30);
    want = std::min<uint64_t>(want, (uint64_t)(free_b * 0.6));
    g.pool_bytes = want / (64 << 10) * (64 << 10);
    CU(cudaMalloc(&g.pool, g.pool_bytes));
    g.arena = fsw_arena_create(g.pool_bytes, 64 << 10);
    g.ws_bytes = c->cfg.workspace_bytes_per_gpu ? c->cfg.workspace_bytes_per_gpu : (512ull << 20);
    CU(cudaMalloc(&g.ws, g.ws_bytes));
    g.ready_cap = 1u << 16;
    CU(cudaMalloc(&g.ready, sizeof(uint32_t) * g.ready_cap));
    CU(cudaMemset(g.ready, 0, sizeof(uint32_t) * g.ready_cap));
    CU(cudaMalloc(&g.ctl, sizeof(DevCtl)));
    CU(cudaMemset(g.ctl, 0, sizeof(DevCtl)));
    g.stage_cap = 16ull << 20;
    g.out_cap = 16ull << 20;
    CU(cudaMalloc(&g.dstage, g.stage_cap));
    CU(cudaHostAlloc(&g.hstage, g.stage_cap, cudaHostAllocPortable));
    CU(cudaHostAlloc(&g.hout, g.out_cap, cudaHostAllocPortable | cudaHostAllocMapped));
    CU(cudaHostAlloc(reinterpret_cast<void**>(&g.hctl), sizeof(DevCtl), cudaHostAllocPortable | cudaHostAllocMapped));
    memset(g.hstage, 0, kStageHdr);
    for (cudaEvent_t* e : {&g.ev0, &g.ev1, &g.evs0, &g.evs1}) CU(cudaEventCreate(e));
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
    if (c->cfg.copy_ctas == 0) c->cfg.copy_ctas = 16;
    if (c->cfg.copy_threads == 0) c->cfg.copy_threads = 256;
    if (c->cfg.chunk_bytes == 0) c->cfg.chunk_bytes = 16 << 10;
    if (c->cfg.stripe_min_bytes == 0) c->cfg.stripe_min_bytes = 256ull << 20;
    if (c->cfg.dma_min_bytes == 0) c->cfg.dma_min_bytes = 32ull << 20;
    if (c->cfg.dmaz_min_bytes == 0) c->cfg.dmaz_min_bytes = 128ull << 20;
    if (c->cfg.dma_group_bytes == 0) c->cfg.dma_group_bytes = 64ull << 20;
    if (c->cfg.dma_streams == 0) c->cfg.dma_streams = 1;
    if (c->cfg.engine > FSW_ENGINE_DMAZ || c->cfg.dma_streams > (uint32_t)kMaxWaitSrc || c->cfg.dma_group_bytes % 256)
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

static void free_plan(Gpu& g, Plan& p) {
    cudaSetDevice(g.dev);
    for (auto& kv : p.graphs) cudaGraphExecDestroy(kv.second);
    p.graphs.clear();
    for (auto& kv : p.pieces) cudaFree(kv.second.dev);
    p.pieces.clear();
    for (auto& kv : p.stripe) cudaFree(kv.second.dev);  // UVA: any current device
    p.stripe.clear();
    for (auto& kv : p.zp) cudaFree(kv.second.dev);
    p.zp.clear();
    for (auto& kv : p.zstripe) cudaFree(kv.second.dev);
    p.zstripe.clear();
}

static void free_store(Model& m, bool host_only) {
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
        cudaFree(g.ctl);
        cudaFree(g.dstage);
        cudaFree(g.zstage);
        cudaStreamDestroy(g.sz);
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
            cudaStreamDestroy(sl.st);
            cudaEventDestroy(sl.done);
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

// ==========================================================================================
// registration: validation + host store (execution order, GEMM weights tiled)
// ==========================================================================================
static uint64_t slot_numel(const fsw_slot& s) {
    uint64_t n = 1;
    for (uint32_t i = 0; i < s.rank; ++i) n *= s.shape[i];
    return n;
}
static uint32_t dt_size(uint32_t dt) { return dt == FSW_DT_BF16 ? 2 : 4; }
static uint64_t slot_bytes(const fsw_slot& s) { return slot_numel(s) * dt_size(s.dtype); }
static uint32_t slot_cols(const fsw_slot& s) { return s.rank ? s.shape[s.rank - 1] : 1; }
static uint64_t slot_rows(const fsw_slot& s) { return slot_numel(s) / std::max<uint32_t>(1, slot_cols(s)); }

// How a CONV2D layer runs (gemm_tc.cu): a 1x1/stride-1 conv is a plain GEMM over [P·Q][Cin];
// Cin % 64 == 0 convs are implicit GEMMs (4-D TMA gathers of the NHWC input); the rest (the
// ResNet stem, Cin = 3) go through an explicit im2col buffer.
enum ConvPath { CONV_DIRECT, CONV_IMPLICIT, CONV_IM2COL };
static uint32_t conv_rows_per_tile(uint32_t P, uint32_t Q) { return std::min<uint32_t>(128 / Q, P); }
static ConvPath conv_path(const fsw_tensor& W, const fsw_layer& L, const fsw_slot& si, const fsw_slot& so) {
    const uint32_t R = W.shape[1], Cin = W.shape[3], stride = (uint32_t)L.attr[1], Q = so.shape[1];
    if (R == 1 && W.shape[2] == 1 && stride == 1 && L.attr[2] == 0 && Cin % 64 == 0) return CONV_DIRECT;
    if (Cin % 64 == 0 && Q <= 128 && Q * stride <= 256 && conv_rows_per_tile(so.shape[0], Q) * stride <= 256 &&
        stride <= 8 && si.rank == 3)
        return CONV_IMPLICIT;
    return CONV_IM2COL;
}

// Rows of in0 a LINEAR layer reads.
static uint64_t linear_rows(const Model& m, const fsw_layer& L) {
    const uint64_t rin = slot_rows(m.slots[L.in0]);
    return L.attr[2] > 0 ? (uint64_t)L.attr[2] : rin;
}
static bool linear_is_gemm(const Model& m, const fsw_layer& L) { return linear_rows(m, L) > 8; }

// Tile order of a GEMM weight W[N][K]: 1024-B atoms of 8 rows x 64 bf16,
// atoms ordered k-tile-major; inside an atom row r is 128 B at r·128 and its 16-B chunk c
// sits at chunk position c ^ r (the UMMA/TMA SWIZZLE_128B pattern).  Padding is zero.
static inline uint64_t tiled_off(uint64_t n, uint64_t k, uint64_t n_pad) {
    return ((k / 64) * (n_pad / 8) + n / 8) * 1024 + (n % 8) * 128 + ((((k % 64) / 8) ^ (n % 8)) * 16) + (k % 8) * 2;
}

static fsw_status validate(const fsw_model_desc* d) {
    if (!d || !d->weights || !d->tensors || !d->slots || !d->layers || d->n_layers == 0)
        return fail(FSW_EINVAL, "register: incomplete description");
    for (uint32_t i = 0; i < d->n_tensors; ++i) {
        const fsw_tensor& t = d->tensors[i];
        if (t.dtype > FSW_DT_F32 || t.rank == 0 || t.rank > 4) return fail(FSW_EINVAL, "tensor %u: bad dtype/rank", i);
        uint64_t n = 1;
        for (uint32_t j = 0; j < t.rank; ++j) n *= t.shape[j];
        if (n * dt_size(t.dtype) != t.bytes) return fail(FSW_EINVAL, "tensor %u: bytes != numel*size", i);
        if (t.offset % 16) return fail(FSW_EINVAL, "tensor %u: offset not 16-B aligned", i);
        if (t.offset + t.bytes > d->weight_bytes) return fail(FSW_EINVAL, "tensor %u: beyond weight_bytes", i);
    }
    // overlap check
    std::vector<std::pair<uint64_t, uint64_t>> iv;
    for (uint32_t i = 0; i < d->n_tensors; ++i) iv.push_back({d->tensors[i].offset, d->tensors[i].offset + d->tensors[i].bytes});
    std::sort(iv.begin(), iv.end());
    for (size_t i = 1; i < iv.size(); ++i)
        if (iv[i].first < iv[i - 1].second) return fail(FSW_EINVAL, "tensors overlap in the weight blob");
    for (uint32_t i = 0; i < d->n_slots; ++i)
        if (d->slots[i].dtype > FSW_DT_I32 || d->slots[i].rank == 0 || d->slots[i].rank > 4)
            return fail(FSW_EINVAL, "slot %u: bad dtype/rank", i);
    if (d->input_slot < 0 || d->input_slot >= (int)d->n_slots || d->output_slot < 0 || d->output_slot >= (int)d->n_slots)
        return fail(FSW_EINVAL, "bad input/output slot");
    for (uint32_t i = 0; i < d->n_refs; ++i)
        if (d->refs[i] >= d->n_tensors) return fail(FSW_EINVAL, "ref %u out of range", i);
    for (uint32_t i = 0; i < d->n_layers; ++i) {
        const fsw_layer& L = d->layers[i];
        if (L.first_ref + L.n_refs > d->n_refs) return fail(FSW_EINVAL, "layer %u: refs out of range", i);
        auto bad_slot = [&](int s) { return s < -1 || s >= (int)d->n_slots; };
        if (bad_slot(L.in0) || bad_slot(L.in1) || L.out < 0 || L.out >= (int)d->n_slots || L.in0 < 0)
            return fail(FSW_EINVAL, "layer %u: bad slot index", i);
        if (L.out == L.in0 || L.out == L.in1) return fail(FSW_EINVAL, "layer %u: in-place layers are not allowed", i);
        if (L.out == d->input_slot) return fail(FSW_EINVAL, "layer %u: writes the input slot", i);
    }
    return FSW_OK;
}

// Per-op checks that depend on shapes and the kernels' supported dtypes.
static fsw_status check_layer(const Model& m, uint32_t li) {
    const fsw_layer& L = m.layers[li];
    const fsw_slot& si = m.slots[L.in0];
    const fsw_slot& so = m.slots[L.out];
    auto ref = [&](uint32_t j) -> const fsw_tensor& { return m.tensors[m.refs[L.first_ref + j]].t; };
    switch (L.op) {
        case FSW_OP_EMBED: {
            if (L.attr[0] < 1 || L.attr[0] > 4 || (uint32_t)L.attr[0] != L.n_refs) return fail(FSW_EINVAL, "layer %u: EMBED tables", li);
            if (si.dtype != FSW_DT_I32 || so.rank != 2 || so.dtype == FSW_DT_I32) return fail(FSW_EINVAL, "layer %u: EMBED slots", li);
            for (uint32_t j = 0; j < L.n_refs; ++j)
                if (ref(j).dtype != FSW_DT_BF16 || ref(j).rank != 2 || ref(j).shape[1] != so.shape[1])
                    return fail(FSW_EINVAL, "layer %u: EMBED table %u shape", li, j);
            if (slot_numel(si) != so.shape[0]) return fail(FSW_EINVAL, "layer %u: EMBED ids vs rows", li);
            break;
        }
        case FSW_OP_LAYERNORM:
            if (L.n_refs != 2 || si.dtype != FSW_DT_F32 || so.dtype == FSW_DT_I32 || slot_numel(si) != slot_numel(so))
                return fail(FSW_EINVAL, "layer %u: LAYERNORM needs f32 input, 2 refs", li);
            if (slot_cols(si) > 2048 || slot_cols(si) % 4 || ref(0).shape[0] != slot_cols(si)) return fail(FSW_EINVAL, "layer %u: LAYERNORM width", li);
            break;
        case FSW_OP_LINEAR: {
            if (L.n_refs < 1 || L.n_refs > 2) return fail(FSW_EINVAL, "layer %u: LINEAR refs", li);
            const fsw_tensor& W = ref(0);
            if (W.rank != 2 || W.dtype != FSW_DT_BF16 || W.shape[1] != slot_cols(si)) return fail(FSW_EINVAL, "layer %u: LINEAR W shape", li);
            if (W.shape[1] % 8) return fail(FSW_EINVAL, "layer %u: LINEAR K must be a multiple of 8", li);
            const uint64_t rows = linear_rows(m, L);
            if ((uint64_t)L.attr[1] + rows > slot_rows(si) || slot_numel(so) != rows * W.shape[0] || so.dtype == FSW_DT_I32)
                return fail(FSW_EINVAL, "layer %u: LINEAR rows/out shape", li);
            if (L.in1 >= 0 && (slot_numel(m.slots[L.in1]) != slot_numel(so) || m.slots[L.in1].dtype == FSW_DT_I32))
                return fail(FSW_EINVAL, "layer %u: LINEAR residual shape", li);
            if (rows > 8) {
                if (L.attr[1] != 0 || rows != slot_rows(si)) return fail(FSW_EINVAL, "layer %u: GEMM path needs all rows", li);
                if (slot_cols(si) % 8) return fail(FSW_EINVAL, "layer %u: GEMM K alignment", li);
            } else if (si.dtype == FSW_DT_I32 || slot_cols(si) * 4 > 200 * 1024 / (rows > 1 ? 8 : 1)) {
                return fail(FSW_EINVAL, "layer %u: GEMV input too wide", li);
            }
            if (L.n_refs == 2 && (ref(1).shape[0] != W.shape[0] || ref(1).dtype != FSW_DT_BF16))
                return fail(FSW_EINVAL, "layer %u: LINEAR bias", li);
            break;
        }
        case FSW_OP_ATTENTION: {
            const int H = L.attr[0], dh = L.attr[1];
            if (si.dtype != FSW_DT_BF16 || so.dtype != FSW_DT_BF16 || si.rank != 2 || H <= 0 || dh <= 0 || dh > 256 ||
                si.shape[1] != (uint32_t)(3 * H * dh) || so.shape[1] != (uint32_t)(H * dh) || so.shape[0] != si.shape[0] ||
                si.shape[0] > 256 || dh > 128 || dh % 8)
                return fail(FSW_EINVAL, "layer %u: ATTENTION shapes/dtypes (bf16 qkv [T][3Hdh], T<=256, dh<=128)", li);
            break;
        }
        case FSW_OP_CONV2D: {
            if (L.n_refs != 2 || si.rank != 3 || so.rank != 3 || si.dtype != FSW_DT_BF16 || so.dtype != FSW_DT_BF16)
                return fail(FSW_EINVAL, "layer %u: CONV2D needs bf16 NHWC slots and W, b", li);
            const fsw_tensor& W = ref(0);
            if (W.rank != 4 || W.shape[0] != so.shape[2] || W.shape[3] != si.shape[2] || W.shape[1] != W.shape[2])
                return fail(FSW_EINVAL, "layer %u: CONV2D weight shape", li);
            const int st = L.attr[1], pad = L.attr[2];
            if (st < 1 || pad < 0) return fail(FSW_EINVAL, "layer %u: CONV2D stride/pad", li);
            const uint32_t ho = (si.shape[0] + 2 * pad - W.shape[1]) / st + 1, wo = (si.shape[1] + 2 * pad - W.shape[2]) / st + 1;
            if (so.shape[0] != ho || so.shape[1] != wo) return fail(FSW_EINVAL, "layer %u: CONV2D output size", li);
            if (so.shape[2] % 8) return fail(FSW_EINVAL, "layer %u: CONV2D Cout must be a multiple of 8", li);
            if (L.in1 >= 0 && (m.slots[L.in1].dtype != FSW_DT_BF16 || slot_numel(m.slots[L.in1]) != slot_numel(so)))
                return fail(FSW_EINVAL, "layer %u: CONV2D residual", li);
            break;
        }
        case FSW_OP_MAXPOOL:
            if (si.rank != 3 || so.rank != 3 || si.dtype != FSW_DT_BF16 || so.dtype != FSW_DT_BF16 || si.shape[2] != so.shape[2])
                return fail(FSW_EINVAL, "layer %u: MAXPOOL", li);
            break;
        case FSW_OP_AVGPOOL:
            if (si.rank != 3 || si.dtype != FSW_DT_BF16 || so.dtype != FSW_DT_F32 || slot_numel(so) != si.shape[2])
                return fail(FSW_EINVAL, "layer %u: AVGPOOL", li);
            break;
        default:
            return fail(FSW_EINVAL, "layer %u: unknown op %u", li, L.op);
    }
    return FSW_OK;
}

// ---- NUMA placement of host stores ---------------------------------------------
// The NUMA node of a CUDA device, from sysfs (-1: unknown, or a single-node host).
static int gpu_numa_node(int dev) {
    char bus[64] = {};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, dev) != cudaSuccess) return -1;
    for (char* q = bus; *q; ++q) *q = (char)tolower(*q);
    char path[128];
    snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/numa_node", bus);
    FILE* f = fopen(path, "r");
    if (!f) return -1;
    int node = -1;
    if (fscanf(f, "%d", &node) != 1) node = -1;
    fclose(f);
    return node;
}
// Prefer `node` for the pages of [p, p + len) before their first touch (MPOL_PREFERRED: the
// allocation still succeeds when the node is full).  Returns the node bound, or -1.
static int bind_pages(void* p, size_t len, int node) {
    if (node < 0 || node >= 64) return -1;
    const unsigned long mask = 1ul << node;
    const long MPOL_PREFERRED_ = 1;
    return syscall(SYS_mbind, p, len, MPOL_PREFERRED_, &mask, 64ul, 0u) == 0 ? node : -1;
}

// ---- exponent-coded link format (kernels.h) -----------------------------------
// Header of a full block of 512 16-bit words: all zero -> kZZero; else h = the largest exponent and
// the code width b in 0..4 with the fewest bytes (words with h − e >= 2^b become exceptions), or raw
// when no width beats the 1024 raw bytes.
static uint32_t zheader(const uint16_t* w) {
    uint32_t emax = 0, any = 0;
    for (uint32_t i = 0; i < kZBlock / 2; ++i) {
        emax = std::max<uint32_t>(emax, (w[i] >> 7) & 0xffu);
        any |= w[i];
    }
    if (!any) return kZZero << 8;
    uint32_t hist[9] = {};  // hist[k] = words with h − e in [2^(k−1), 2^k) (k = 0: h − e = 0), k = 8: >= 128
    for (uint32_t i = 0; i < kZBlock / 2; ++i) {
        const uint32_t d = emax - ((w[i] >> 7) & 0xffu);
        hist[d ? std::min<uint32_t>(8, 32 - __builtin_clz(d)) : 0]++;
    }
    uint32_t best = kZRaw, best_bytes = kZBlock, best_n = 0, n = kZBlock / 2;
    for (uint32_t b = 0; b <= 4; ++b) {
        n -= hist[b];  // words with h − e >= 2^b
        const uint32_t bytes = zblock_bytes(emax | (b << 8) | (n << 16), kZBlock);
        if (bytes < best_bytes) {
            best = b;
            best_bytes = bytes;
            best_n = n;
        }
    }
    return best == kZRaw ? kZRaw << 8 : emax | (best << 8) | (best_n << 16);
}

// Coded block: 512 stream-A bytes at outa, zblock_b(hdr) stream-B bytes at outb (both zeroed).
static void zencode_block(const uint16_t* w, uint32_t hdr, uint8_t* outa, uint8_t* outb) {
    const uint32_t h = hdr & 0xffu, b = (hdr >> 8) & 0xffu;
    uint32_t k = 0;
    uint8_t* exc = outb + 64 * b;
    for (uint32_t i = 0; i < kZBlock / 2; ++i) {
        const uint32_t d = h - ((w[i] >> 7) & 0xffu);
        outa[i] = (uint8_t)(((w[i] >> 8) & 0x80u) | (w[i] & 0x7fu));
        if (d >> b) {  // exception: position and the whole word; code 0
            const uint32_t e = i | ((uint32_t)w[i] << 16);
            memcpy(exc + 4 * k++, &e, 4);
            continue;
        }
        for (uint32_t p = 0; p < b; ++p)
            if ((d >> p) & 1u) outb[64 * p + i / 8] |= (uint8_t)(1u << (i % 8));
    }
}

template <typename F>
static void parallel_for(size_t n, F f) {
    const size_t T = std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(), 32));
    if (n < 64 || T == 1) {
        for (size_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    std::atomic<size_t> next{0};
    for (size_t t = 0; t < T; ++t)
        th.emplace_back([&]() {
            for (size_t i; (i = next.fetch_add(256)) < n;)
                for (size_t j = i; j < std::min(n, i + 256); ++j) f(j);
        });
    for (auto& t : th) t.join();
}

// Build the coded copy of m.store: pieces of <= kZPiece bytes per layer region in execution order,
// headers first (parallel), then offsets, then the coded bytes (parallel) into a THP-backed mapping
// that is pinned and mapped for zero-copy reads like the store itself.
static fsw_status build_link_code(Model& m, bool host_only) {
    std::vector<ZPiece>& pcs = m.zpieces;
    pcs.clear();
    for (uint32_t li = 0; li < m.layers.size(); ++li)
        for (uint64_t o = 0; o < m.region_bytes[li]; o += kZPiece)
            pcs.push_back({m.region_off[li] + o, 0, (uint32_t)std::min<uint64_t>(kZPiece, m.region_bytes[li] - o), li, 0, 0, {}});
    const uint32_t bpp = kZPiece / kZBlock;
    std::vector<uint32_t> hdr(pcs.size() * bpp, 0);
    parallel_for(pcs.size(), [&](size_t i) {
        const ZPiece& pc = pcs[i];
        const uint32_t nfull = pc.bytes / kZBlock;
        for (uint32_t b = 0; b < nfull; ++b)
            hdr[i * bpp + b] = zheader(reinterpret_cast<const uint16_t*>(m.store + pc.off + (uint64_t)b * kZBlock));
        if (pc.bytes > nfull * kZBlock) hdr[i * bpp + nfull] = kZRaw << 8;  // partial tail block: raw
    });
    uint64_t cur = 0;
    for (size_t i = 0; i < pcs.size(); ++i) {
        ZPiece& pc = pcs[i];
        const uint32_t nb = (pc.bytes + kZBlock - 1) / kZBlock;
        uint32_t la = 0, lb = 0;  // stream A, stream B
        for (uint32_t b = 0; b < nb; ++b) {
            la += zblock_a(hdr[i * bpp + b], std::min(kZBlock, pc.bytes - b * kZBlock));
            lb += zblock_b(hdr[i * bpp + b]);
        }
        const uint32_t cb = (uint32_t)align_up(la, 128) + lb;
        pc.coff = cur;
        pc.cbytes = cb;
        memcpy(pc.hdr, &hdr[i * bpp], sizeof pc.hdr);
        cur = align_up(cur + cb, 128);
    }
    m.zbytes = cur;
    m.zalloc = align_up(std::max<uint64_t>(cur, 1), 2 << 20);
    void* p = mmap(nullptr, m.zalloc, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return fail(FSW_ENOMEM, "register: mmap of %llu coded bytes failed", (unsigned long long)m.zalloc);
    madvise(p, m.zalloc, MADV_HUGEPAGE);
    if (m.numa_node >= 0) bind_pages(p, m.zalloc, m.numa_node);
    m.zstore = static_cast<uint8_t*>(p);
    memset(m.zstore, 0, m.zalloc);  // alignment gaps stay zero
    parallel_for(pcs.size(), [&](size_t i) {
        const ZPiece& pc = pcs[i];
        uint8_t* out = m.zstore + pc.coff;
        const uint32_t nb = (pc.bytes + kZBlock - 1) / kZBlock;
        uint32_t la = 0;
        for (uint32_t b = 0; b < nb; ++b) la += zblock_a(hdr[i * bpp + b], std::min(kZBlock, pc.bytes - b * kZBlock));
        uint64_t oa = 0, ob = align_up(la, 128);
        for (uint32_t b = 0; b < nb; ++b) {
            const uint8_t* raw = m.store + pc.off + (uint64_t)b * kZBlock;
            const uint32_t hd = hdr[i * bpp + b], n = std::min(kZBlock, pc.bytes - b * kZBlock);
            const uint32_t kind = (hd >> 8) & 0xffu;
            if (kind == kZRaw) memcpy(out + oa, raw, n);
            else if (kind != kZZero) zencode_block(reinterpret_cast<const uint16_t*>(raw), hd, out + oa, out + ob);  // zeroed
            oa += zblock_a(hd, n);
            ob += zblock_b(hd);
        }
    });
    if (!host_only) {
        cudaError_t e = cudaHostRegister(m.zstore, m.zalloc, cudaHostRegisterPortable | cudaHostRegisterMapped);
        if (e != cudaSuccess) {
            munmap(m.zstore, m.zalloc);
            m.zstore = nullptr;
            return fail(FSW_ECUDA, "register: cudaHostRegister (coded store): %s", cudaGetErrorString(e));
        }
    }
    return FSW_OK;
}

extern "C" fsw_status fsw_register_model(fsw_ctx* c, const fsw_model_desc* d, uint32_t* model_id) {
    if (!c || !model_id) return fail(FSW_EINVAL, "register: NULL argument");
    fsw_status s = validate(d);
    if (s != FSW_OK) return s;
    auto m = std::make_unique<Model>();
    m->name = d->name ? d->name : "";
    m->tensors.resize(d->n_tensors);
    for (uint32_t i = 0; i < d->n_tensors; ++i) {
        m->tensors[i].t = d->tensors[i];
        m->algorithmic_bytes += d->tensors[i].bytes;
    }
    m->refs.assign(d->refs, d->refs + d->n_refs);
    m->slots.assign(d->slots, d->slots + d->n_slots);
    m->layers.assign(d->layers, d->layers + d->n_layers);
    m->input_slot = d->input_slot;
    m->output_slot = d->output_slot;
    m->input_bytes = slot_bytes(m->slots[d->input_slot]);
    m->output_bytes = slot_bytes(m->slots[d->output_slot]);
    for (uint32_t i = 0; i < d->n_layers; ++i)
        if ((s = check_layer(*m, i)) != FSW_OK) return s;

    // --- layouts: GEMM weights tiled, everything else row-major ---
    for (uint32_t li = 0; li < d->n_layers; ++li) {
        const fsw_layer& L = m->layers[li];
        const bool gemm = L.op == FSW_OP_CONV2D || (L.op == FSW_OP_LINEAR && linear_is_gemm(*m, L));
        if (gemm) m->n_gemm++;
        for (uint32_t j = 0; j < L.n_refs; ++j) {
            TensorInfo& ti = m->tensors[m->refs[L.first_ref + j]];
            const bool want_tiled = gemm && j == 0;
            if (ti.owner >= 0) {
                if ((ti.layout == LAYOUT_TILED) != want_tiled)
                    return fail(FSW_EINVAL, "layer %u: tensor shared between a GEMM and a non-GEMM use", li);
                continue;
            }
            ti.owner = (int)li;
            if (want_tiled) {
                ti.layout = LAYOUT_TILED;
                ti.rows = ti.t.shape[0];
                ti.cols = (uint32_t)(ti.t.bytes / 2 / ti.t.shape[0]);
                ti.rows_pad = (uint32_t)align_up(ti.rows, 16);
                ti.cols_pad = (uint32_t)align_up(ti.cols, 64);
                ti.st_bytes = (uint64_t)ti.rows_pad * ti.cols_pad * 2;
            } else {
                ti.layout = LAYOUT_ROWMAJOR;
                ti.st_bytes = ti.t.bytes;
            }
        }
    }
    // --- store offsets: layer regions in execution order, 256-B aligned ---
    m->region_off.assign(d->n_layers, 0);
    m->region_bytes.assign(d->n_layers, 0);
    uint64_t cur = 0;
    for (uint32_t li = 0; li < d->n_layers; ++li) {
        const fsw_layer& L = m->layers[li];
        m->region_off[li] = cur;
        for (uint32_t j = 0; j < L.n_refs; ++j) {
            TensorInfo& ti = m->tensors[m->refs[L.first_ref + j]];
            if (ti.owner != (int)li || ti.placed) continue;  // owned by an earlier layer / listed twice
            ti.placed = true;
            ti.st_off = cur;
            cur = align_up(cur + ti.st_bytes, 256);
        }
        m->region_bytes[li] = cur - m->region_off[li];
        if (m->region_bytes[li] >= (1ull << 32)) return fail(FSW_EINVAL, "layer %u: weights exceed 4 GiB", li);
    }
    // tensors not referenced by any layer are not swapped (not part of the access pattern)
    m->store_bytes = cur;
    if (m->store_bytes == 0) return fail(FSW_EINVAL, "register: model has no weights");

    // --- host store: pinned + mapped (cudaHostRegister of THP-backed mmap), or WC pinned ---
    const bool host_only = (c->cfg.flags & FSW_HOST_ONLY) != 0;
    const bool wc = !host_only && (c->cfg.flags & FSW_HOST_WC) != 0;
    m->store_alloc = align_up(m->store_bytes, 2 << 20);
    if (wc) {
        CU(cudaSetDevice(c->gpus[0].dev));
        void* p = nullptr;
        CU(cudaHostAlloc(&p, m->store_alloc, cudaHostAllocPortable | cudaHostAllocMapped | cudaHostAllocWriteCombined));
        m->store = static_cast<uint8_t*>(p);
        m->store_wc = true;
    } else {
        void* p = mmap(nullptr, m->store_alloc, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (p == MAP_FAILED) return fail(FSW_ENOMEM, "register: mmap of %llu bytes failed", (unsigned long long)m->store_alloc);
        madvise(p, m->store_alloc, MADV_HUGEPAGE);
        // the host link that reads the store is pool GPU 0's (striped swaps add the others)
        if (!host_only) m->numa_node = bind_pages(p, m->store_alloc, gpu_numa_node(c->gpus[0].dev));
        m->store = static_cast<uint8_t*>(p);
    }
    // pack (zero padding everywhere; first touch happens here)
    const uint8_t* src = static_cast<const uint8_t*>(d->weights);
    memset(m->store, 0, m->store_alloc);
    for (auto& ti : m->tensors) {
        if (ti.owner < 0) continue;
        if (ti.layout == LAYOUT_ROWMAJOR) {
            memcpy(m->store + ti.st_off, src + ti.t.offset, ti.t.bytes);
        } else {
            const uint16_t* w = reinterpret_cast<const uint16_t*>(src + ti.t.offset);
            for (uint64_t n = 0; n < ti.rows; ++n)
                for (uint64_t k = 0; k < ti.cols; ++k)
                    memcpy(m->store + ti.st_off + tiled_off(n, k, ti.rows_pad), &w[n * ti.cols + k], 2);
        }
    }
    if (!wc && !host_only) {
        CU(cudaSetDevice(c->gpus[0].dev));
        cudaError_t e = cudaHostRegister(m->store, m->store_alloc, cudaHostRegisterPortable | cudaHostRegisterMapped);
        if (e != cudaSuccess) {
            munmap(m->store, m->store_alloc);
            m->store = nullptr;
            return fail(FSW_ECUDA, "register: cudaHostRegister: %s", cudaGetErrorString(e));
        }
    }
    if (d->flags & FSW_REG_LINK_CODE) {
        if (!wc && !host_only) CU(cudaSetDevice(c->gpus[0].dev));
        s = build_link_code(*m, host_only);
        if (s != FSW_OK) {
            free_store(*m, host_only);
            return s;
        }
    }
    m->extent.assign(c->gpus.size(), -1);
    m->pextent.assign(c->gpus.size(), -1);
    m->pvalid.assign(c->gpus.size(), 0);
    m->last_use.assign(c->gpus.size(), 0);
    m->plans.resize(c->gpus.size());
    std::lock_guard<std::mutex> lk(c->mu);
    m->id = (uint32_t)c->models.size();
    *model_id = m->id;
    c->models.push_back(std::move(m));
    return FSW_OK;
}

static Model* find_model(fsw_ctx* c, uint32_t id) {
    if (!c || id >= c->models.size()) return nullptr;
    return c->models[id].get();
}

extern "C" fsw_status fsw_model_info_get(fsw_ctx* c, uint32_t id, fsw_model_info* out) {
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (!out) return fail(FSW_EINVAL, "NULL out");
    out->store_bytes = m->store_bytes;
    out->algorithmic_bytes = m->algorithmic_bytes;
    out->n_layers = (uint32_t)m->layers.size();
    out->n_tensors = (uint32_t)m->tensors.size();
    out->n_gemm_layers = m->n_gemm;
    out->input_bytes = m->input_bytes;
    out->output_bytes = m->output_bytes;
    out->output_dtype = m->slots[m->output_slot].dtype;
    out->coded_bytes = m->zstore ? m->zbytes : 0;
    out->numa_node = m->numa_node;
    return FSW_OK;
}

extern "C" fsw_status fsw_store_tensor_get(fsw_ctx* c, uint32_t id, uint32_t t, fsw_store_tensor* out) {
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (!out || t >= m->tensors.size()) return fail(FSW_EINVAL, "bad tensor index");
    const TensorInfo& ti = m->tensors[t];
    *out = {ti.st_off, ti.st_bytes, ti.layout, ti.rows, ti.cols, ti.rows_pad, ti.cols_pad, (uint32_t)ti.owner};
    return FSW_OK;
}

// ==========================================================================================
// plan: workspace layout + kernel list for one (model, GPU)
// ==========================================================================================
static fsw_status build_plan(fsw_ctx* c, Model& m, int gi) {
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
        const Tiling t = choose_tiling(m_tiles, a.n_pad, a.K / 64, a_kt_bytes, m_rows, &max_cl);
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
                    set_tiling(a, (a.M + 127) / 128, 128, 128 * 128);
                    const void* abase = si.dtype == FSW_DT_BF16 ? (const void*)sptr(L.in0) : (const void*)shadow(L.in0);
                    if (!make_tmap_act(&x.tmap, abase, a.M, slot_cols(si), slot_cols(si), 128 / a.mc))
                        return fail(FSW_ECUDA, "plan: cuTensorMapEncodeTiled failed (layer %u)", li);
                }
                break;
            }
            case FSW_OP_ATTENTION: {
                x.kind = K_ATTN;
                x.attn = {reinterpret_cast<const uint16_t*>(sptr(L.in0)), reinterpret_cast<uint16_t*>(sptr(L.out)),
                          si.shape[0], (uint32_t)L.attr[0], (uint32_t)L.attr[1], L.attr[2]};
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
    // split-K partials live after the activations and the im2col scratch
    const uint64_t part_off = align_up(off, 1024);
    p->ws_bytes = align_up(part_off + part_bytes, 1024);
    if (p->ws_bytes > g.ws_bytes)
        return fail(FSW_ENOMEM, "plan: workspace needs %llu bytes > %llu", (unsigned long long)p->ws_bytes, (unsigned long long)g.ws_bytes);
    for (Launch& x : p->launches)
        if (x.kind == K_GEMM) x.gemm.part = reinterpret_cast<float*>(g.ws + part_off);
    p->built = true;
    m.plans[gi] = std::move(p);
    return FSW_OK;
}

// Swap pieces for one chunk size / order: execution order, never straddling a layer region.
static fsw_status get_pieces(Model& m, Plan& p, Gpu& g, uint64_t chunk, int order, uint32_t seed, uint64_t from,
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

static const DmaPlan& get_dma_plan(Model& m, Plan& p, uint64_t grp, uint32_t streams, uint64_t from) {
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
// decode and compute that trail the last group are short; each piece records its group.
static fsw_status get_zpieces(Model& m, Plan& p, Gpu& g, int order, uint32_t seed, uint64_t from, uint64_t grp,
                              ZPieceSet** out) {
    const auto key = std::make_tuple(order, seed, from, grp);
    auto it = p.zp.find(key);
    if (it != p.zp.end()) {
        *out = &it->second;
        return FSW_OK;
    }
    ZPieceSet zs;
    for (const ZPiece& pc : m.zpieces)
        if (pc.off >= from) zs.host.push_back(pc);
    if (zs.host.empty()) return fail(FSW_EINVAL, "link-coded swap with nothing to move");
    zs.cfrom = zs.host.front().coff;
    zs.cend = align_up(zs.host.back().coff + zs.host.back().cbytes, 128);  // the coded store is 128-B padded
    if (grp) {
        // the DMA engine's plan (make_dma_plan) over coded bytes: tail taper inside layers, head ramp
        // at layer boundaries
        // head ramp on by default here (measured: DMAZ ResNet-50 0.890 -> 0.809 ms at ramp 4, BERT-base
        // neutral); off for the plain DMA engine, where it cost ResNet-50 2-5 %
        static const double ramp = getenv("FSW_DMAZ_RAMP") ? atof(getenv("FSW_DMAZ_RAMP")) : 4.0;
        const uint64_t tail_min = std::min<uint64_t>(grp, 1ull << 20);
        uint64_t lo = zs.cfrom;
        for (size_t i = 0; i < zs.host.size(); ++i) {
            ZPiece& pc = zs.host[i];
            pc.grp = (uint32_t)zs.groups.size();
            const bool last = i + 1 == zs.host.size();
            const uint64_t hi = last ? zs.cend : zs.host[i + 1].coff;
            const uint64_t want = std::min(grp, std::max(tail_min, (zs.cend - lo) / 2));
            const uint64_t want_close =
                ramp > 0 ? std::min(want, std::max(tail_min, (uint64_t)((double)(lo - zs.cfrom) * ramp))) : want;
            const bool boundary = last || zs.host[i + 1].layer != pc.layer;
            if (last || hi - lo >= want || (boundary && hi - lo >= want_close)) {
                zs.groups.push_back({lo, hi});
                lo = hi;
            }
        }
    }
    if (order == FSW_ORDER_REVERSE) std::reverse(zs.host.begin(), zs.host.end());
    if (order == FSW_ORDER_RANDOM) {
        std::mt19937_64 rng(seed);
        std::shuffle(zs.host.begin(), zs.host.end(), rng);
    }
    CU(cudaSetDevice(g.dev));
    CU(cudaMalloc(&zs.dev, sizeof(ZPiece) * zs.host.size()));
    CU(cudaMemcpy(zs.dev, zs.host.data(), sizeof(ZPiece) * zs.host.size(), cudaMemcpyHostToDevice));
    *out = &p.zp.emplace(key, std::move(zs)).first->second;
    return FSW_OK;
}

// Striped link-coded swap: runs of 16 consecutive coded pieces (256 KiB of store) dealt round-robin to
// n sources; source j's table lives on its device.
static fsw_status get_zstripe_pieces(Model& m, Plan& p, uint32_t n, uint32_t j, int dev, uint64_t from, ZPieceSet** out) {
    const auto key = std::make_tuple(n, j, dev, from);
    auto it = p.zstripe.find(key);
    if (it != p.zstripe.end()) {
        *out = &it->second;
        return FSW_OK;
    }
    ZPieceSet zs;
    uint64_t q = 0;
    for (const ZPiece& pc : m.zpieces) {
        if (pc.off < from) continue;
        if ((q++ / 16) % n == j) zs.host.push_back(pc);
    }
    CU(cudaSetDevice(dev));
    if (!zs.host.empty()) {
        CU(cudaMalloc(&zs.dev, sizeof(ZPiece) * zs.host.size()));
        CU(cudaMemcpy(zs.dev, zs.host.data(), sizeof(ZPiece) * zs.host.size(), cudaMemcpyHostToDevice));
    }
    *out = &p.zstripe.emplace(key, std::move(zs)).first->second;
    return FSW_OK;
}

static bool engine_coded(int e) { return e == FSW_ENGINE_SMZ || e == FSW_ENGINE_DMAZ; }
// Engines whose layer kernels wait on per-layer byte counters (released by a swap kernel).
static bool engine_bytes_ready(int e) { return e == FSW_ENGINE_SM || engine_coded(e); }

// Decoding swap CTAs (DMAZ and SMZ) unless the invoke sets copy_ctas: measured, 16 CTAs make the DMAZ
// decode the bottleneck (BERT-base 3.60 ms vs 2.94 with 32) and leave SMZ's TMA ring short of the link
// (ResNet-50 0.783 vs 0.739 ms) (profiles/r01/linkcode/).
constexpr uint32_t kDmazCtas = 32;

struct InvokeCfg {
    bool cold, no_overlap;
    int engine;  // FSW_ENGINE_SM / FSW_ENGINE_DMA (resolved)
    uint64_t chunk;
    int order;
    uint32_t seed, ctas;
    DevDesc dst;                 // the target's extents (DMA graphs bake these addresses)
    const DmaPlan* dma_plan;     // DMA engine only
    DevDesc src{};               // DMA: copy source extents (a peer GPU's), unless src_host
    bool src_host = true;        // DMA: copy from the pinned host store
    uint64_t from = 0;           // first swapped store byte (a cached prefix is skipped)
    bool striped = false;        // striped swap: sources launched outside the graph (fsw_invoke_ex)
    uint32_t local_ctas = 0;     // striped: swap CTAs running on the target GPU itself (gate)
    uint64_t zgrp = 0;           // DMAZ: copy-group bytes
};

// Striped swap: the execution-order piece list of the SM engine dealt round-robin to n sources
// (piece q goes to source q mod n), so every source streams a share of every layer and all of them
// advance through the model together; source j's table is allocated on source j's device.
static fsw_status get_stripe_pieces(Model& m, Plan& p, uint64_t chunk, uint32_t n, uint32_t j, int dev, uint64_t from,
                                    PieceSet** out) {
    const auto key = std::make_tuple(chunk, n, j, dev, from);
    auto it = p.stripe.find(key);
    if (it != p.stripe.end()) {
        *out = &it->second;
        return FSW_OK;
    }
    PieceSet ps;
    uint64_t q = 0;
    for (uint32_t li = 0; li < m.layers.size(); ++li)
        for (uint64_t o = 0; m.region_off[li] >= from && o < m.region_bytes[li]; o += chunk, ++q)
            if (q % n == j) ps.host.push_back({m.region_off[li] + o, (uint32_t)std::min<uint64_t>(chunk, m.region_bytes[li] - o), li});
    CU(cudaSetDevice(dev));
    if (!ps.host.empty()) {
        CU(cudaMalloc(&ps.dev, sizeof(Piece) * ps.host.size()));
        CU(cudaMemcpy(ps.dev, ps.host.data(), sizeof(Piece) * ps.host.size(), cudaMemcpyHostToDevice));
    }
    *out = &p.stripe.emplace(key, std::move(ps)).first->second;
    return FSW_OK;
}

static void enqueue_layers(Model& m, Plan& p, Gpu& g, const InvokeCfg& ic, cudaStream_t s) {
    const DevDesc* d = reinterpret_cast<const DevDesc*>(g.dstage);
    for (const Launch& x : p.launches) {
        Wait w{};
        w.ctl = g.ctl;
        w.layer = x.layer;
        if (ic.cold && m.region_bytes[x.layer] > 0 && m.region_off[x.layer] >= ic.from) {
            if (engine_bytes_ready(ic.engine)) {
                w.n = 1;
                w.ready[0] = g.ready + x.layer;
                w.target[0] = (uint32_t)m.region_bytes[x.layer];
                w.sys = ic.striped ? 1 : 0;
            } else {
                w.n = ic.dma_plan->streams;
                for (uint32_t j = 0; j < w.n; ++j) {
                    w.ready[j] = g.progress + 32 * j;
                    w.target[j] = ic.dma_plan->target[x.layer][j];
                }
            }
        }
        switch (x.kind) {
            case K_EMBED: launch_embed(s, d, w, x.embed); break;
            case K_LN: launch_layernorm(s, d, w, x.ln); break;
            case K_GEMV: launch_gemv(s, d, w, x.gemv); break;
            case K_GEMM: launch_gemm(s, d, w, &x.tmap, x.gemm); break;
            case K_ATTN: launch_attention(s, x.attn); break;
            case K_IM2COL: launch_im2col(s, x.im2col); break;
            case K_MAXPOOL: launch_maxpool(s, x.pool); break;
            case K_AVGPOOL: launch_avgpool(s, x.pool); break;
        }
    }
}

typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_writeValue32 get_write_value32() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess) return nullptr;
    return reinterpret_cast<PFN_writeValue32>(p);
}

// Capture the invoke graph of (model, GPU, cfg).  Root: H2D of [desc | input]; cold adds the
// ready/ctl reset, the swap kernel on its own stream (bracketed by external event nodes for
// timing) and the gate; then the flag-gated layer kernels; then D2H of output and ctl.
static fsw_status build_graph(fsw_ctx* c, Model& m, Plan& p, Gpu& g, const InvokeCfg& ic, cudaGraphExec_t* out) {
    PieceSet* ps = nullptr;
    ZPieceSet* zs = nullptr;
    if (ic.cold && ic.engine == FSW_ENGINE_SM && !ic.striped) {
        fsw_status s = get_pieces(m, p, g, ic.chunk, ic.order, ic.seed, ic.from, &ps);
        if (s != FSW_OK) return s;
    }
    if (ic.cold && engine_coded(ic.engine) && !ic.striped) {
        fsw_status s = get_zpieces(m, p, g, ic.order, ic.seed, ic.from, ic.engine == FSW_ENGINE_DMAZ ? ic.zgrp : 0, &zs);
        if (s != FSW_OK) return s;
        if (ic.engine == FSW_ENGINE_DMAZ && zs->cend - zs->cfrom > g.zstage_cap) return fail(FSW_EINVAL, "staging buffer too small");
    }
    if (ic.cold && (engine_bytes_ready(ic.engine) || ic.striped) && m.layers.size() > g.ready_cap)
        return fail(FSW_EINVAL, "too many layers");
    CU(cudaSetDevice(g.dev));
    cudaStream_t sx = g.sx, sc = g.sc;
    CU(cudaStreamBeginCapture(sx, cudaStreamCaptureModeThreadLocal));
    // The swap starts as early as possible: the DMA engine needs only its counters reset; the SM
    // engine also reads the invoke descriptor and the control block.  The input (up to 300 KB for
    // ResNet-50) is copied after the fork, overlapping the swap.
    const bool dma_cold = ic.cold && !ic.striped && ic.engine == FSW_ENGINE_DMA;
    if (dma_cold) cudaMemsetAsync(g.progress, 0, 128 * kMaxWaitSrc, sx);
    if (!dma_cold) cudaMemcpyAsync(g.dstage, g.hstage, kStageHdr, cudaMemcpyHostToDevice, sx);
    // striped: the counters and the control block are reset before the sources start (outside)
    if (!ic.striped && !dma_cold) cudaMemsetAsync(g.ctl, 0, sizeof(DevCtl), sx);
    if (ic.cold && ic.striped && !ic.no_overlap && ic.local_ctas) launch_gate(sx, g.ctl, ic.local_ctas);
    if (ic.cold && !ic.striped) {
        if (engine_bytes_ready(ic.engine)) cudaMemsetAsync(g.ready, 0, sizeof(uint32_t) * m.layers.size(), sx);
        if (ic.engine == FSW_ENGINE_DMAZ) cudaMemsetAsync(g.progress, 0, 128, sx);
        cudaEventRecord(g.evfork, sx);
        cudaStreamWaitEvent(sc, g.evfork, 0);
        cudaEventRecordWithFlags(g.evs0, sc, cudaEventRecordExternal);
        const DevDesc* desc = reinterpret_cast<const DevDesc*>(g.dstage);
        if (ic.engine == FSW_ENGINE_SM) {
            launch_swap(sc, (int)ic.ctas, (int)c->cfg.copy_threads, m.store, DevDesc{}, desc, ps->dev,
                        (uint32_t)ps->host.size(), g.ready, g.ctl, g.ctl, 0);
        } else if (ic.engine == FSW_ENGINE_SMZ) {
            // zero-copy decode: coded pieces straight from the mapped coded store over the host link
            launch_swapz(sc, (int)ic.ctas, (int)c->cfg.copy_threads, m.zstore, 0, DevDesc{}, desc, zs->dev,
                         (uint32_t)zs->host.size(), g.ready, g.ctl, g.ctl, 0, 0, nullptr);
        } else if (ic.engine == FSW_ENGINE_DMAZ) {
            // copy engine moves coded groups into the staging buffer (a fenced stream write of the group
            // count after each); the decode kernel, forked onto its own stream, waits per piece for its
            // group and decodes from HBM into the extent
            static PFN_writeValue32 wv = get_write_value32();
            if (!wv) return fail(FSW_ECUDA, "cuStreamWriteValue32 entry point unavailable");
            cudaEventRecord(g.evd[0], sc);
            cudaStreamWaitEvent(g.sz, g.evd[0], 0);
            launch_swapz(g.sz, (int)ic.ctas, (int)c->cfg.copy_threads, g.zstage, zs->cfrom, DevDesc{}, desc, zs->dev,
                         (uint32_t)zs->host.size(), g.ready, g.ctl, g.ctl, 0, 1, g.progress);
            uint32_t cnt = 0;
            for (const auto& gr : zs->groups) {
                cudaMemcpyAsync(g.zstage + (gr.first - zs->cfrom), m.zstore + gr.first, gr.second - gr.first,
                                cudaMemcpyHostToDevice, sc);
                wv(sc, (CUdeviceptr)g.progress, (cuuint32_t)(++cnt), 0);
            }
            cudaEventRecord(g.evd[1], g.sz);
            cudaStreamWaitEvent(sc, g.evd[1], 0);
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
            for (const auto& gr : dp.groups) {
                cudaStream_t sj = g.sd[gr.stream];
                const uint8_t* from_ptr = ic.src_host ? m.store + gr.lo : weight_ptr(ic.src, gr.lo);
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
        else if (engine_bytes_ready(ic.engine)) launch_gate(sx, g.ctl, ic.ctas);
    }
    enqueue_layers(m, p, g, ic, sx);
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

// ==========================================================================================
// pool residency
// ==========================================================================================
// Heavy / light: set by the caller, or measured — heavy iff pipelined swapping slows
// the inference down by more than 1.25x — and heavy while unmeasured.
static bool model_heavy(const Model& m) {
    if (m.heavy >= 0) return m.heavy != 0;
    if (!m.n_cold_runs || !m.n_warm_runs) return true;
    return (m.cold_ms_sum / m.n_cold_runs) > 1.25 * (m.warm_ms_sum / m.n_warm_runs);
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
    *heavy = model_heavy(*m) ? 1 : 0;
    return FSW_OK;
}

// Eviction invalidates, it never copies back.  The suffix (or whole model)
// extent goes; with keep_prefix a cached prefix stays (partial caching), else it goes too.
static void invalidate(fsw_ctx* c, Model& m, int gi, bool keep_prefix = false) {
    if (m.extent[gi] >= 0) {
        fsw_arena_free(c->gpus[gi].arena, (uint64_t)m.extent[gi]);
        m.extent[gi] = -1;
    }
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
            heavy.push_back(model_heavy(*o));
            uint32_t k = 0;
            for (int64_t e : o->extent) k += e >= 0;
            copies.push_back(k);
            last.push_back(o->last_use[gi]);
            in_use.push_back(o->inflight != 0);
        }
        const std::vector<uint32_t> order = eviction_order(heavy, copies, last, in_use);
        if (!order.empty()) {
            invalidate(c, *cand[order[0]], gi, /*keep_prefix=*/true);
            g.n_evictions++;
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

extern "C" fsw_status fsw_unregister_model(fsw_ctx* c, uint32_t id) {
    if (!c) return fail(FSW_EINVAL, "NULL ctx");
    std::unique_ptr<Model> m;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        Model* mp = find_model(c, id);
        if (!mp) return fail(FSW_ENOTFOUND, "model %u not found", id);
        if (mp->inflight) return fail(FSW_EBUSY, "model %u has an invoke in flight", id);
        for (size_t i = 0; i < c->gpus.size(); ++i) invalidate(c, *mp, (int)i);
        m = std::move(c->models[id]);
    }
    for (size_t i = 0; i < c->gpus.size(); ++i)
        if (m->plans[i]) free_plan(c->gpus[i], *m->plans[i]);
    free_store(*m, (c->cfg.flags & FSW_HOST_ONLY) != 0);
    return FSW_OK;
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
    out->bytes_swapped_total = g.bytes_swapped_total;
    out->n_invokes_cold = g.n_cold;
    out->n_invokes_warm = g.n_warm;
    return FSW_OK;
}

// ==========================================================================================
// invoke
// ==========================================================================================
// Algorithm 1 over the pool's live state; NVLink through NVSwitch is uniform.
static Decision pick_gpu(fsw_ctx* c, Model& m) {
    const size_t n = c->gpus.size();
    std::vector<uint8_t> avail(n), hosts(n), loading(n);
    for (size_t i = 0; i < n; ++i) {
        avail[i] = !c->gpus[i].busy;
        hosts[i] = m.extent[i] >= 0;
        loading[i] = (uint8_t)c->gpus[i].loading;
    }
    std::vector<float> link(n * n, 0.0f);
    for (size_t g = 0; g < n; ++g)
        for (size_t s = 0; s < n; ++s) link[g * n + s] = c->peer[g][s] ? 1.0f : 0.0f;
    return schedule(avail, hosts, c->neighbor, loading, link);
}

extern "C" fsw_status fsw_invoke_ex(fsw_ctx* c, uint32_t id, const fsw_invoke_opts* opts, const void* input,
                                    uint64_t input_bytes, void* output, uint64_t output_cap, fsw_invoke_stats* stats) {
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
            else if (m->extent[s] < 0) ss = fail(FSW_ESTATE, "invoke: model %u is not resident on gpu %d", id, s);
            else if (!c->peer[gi][s]) ss = fail(FSW_ETOPO, "invoke: gpu %d cannot read gpu %d", gi, s);
            else peer = s;
        } else if (cold && !o.n_stripe_src && !((o.flags | c->cfg.flags) & FSW_NO_PEER_SWAP)) {
            if (o.gpu < 0 && dec.kind == 2) peer = dec.src;  // Algorithm 1, line 11
            for (int s = 0; s < (int)c->gpus.size() && peer < 0; ++s)
                if (s != gi && m->extent[s] >= 0 && c->peer[gi][s]) peer = s;
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
        if (ss == FSW_OK && cold && peer < 0) g.loading = model_heavy(*m) ? 2 : 1;  // host link in use
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
    const uint32_t flags = o.flags | c->cfg.flags;
    const bool baseline = (flags & FSW_DMA_BASELINE) != 0;
    int engine = (int)(o.engine ? o.engine : c->cfg.engine);
    if (baseline) engine = FSW_ENGINE_DMA;
    const bool big = m->store_bytes >= c->cfg.dma_min_bytes;
    if (engine == FSW_ENGINE_AUTO)
        engine = m->zstore ? (m->store_bytes >= c->cfg.dmaz_min_bytes ? FSW_ENGINE_DMAZ : FSW_ENGINE_SMZ)
                           : (big ? FSW_ENGINE_DMA : FSW_ENGINE_SM);
    if (engine_coded(engine) && !m->zstore) return finish(fail(FSW_EINVAL, "invoke: model %u is not link-coded (FSW_REG_LINK_CODE)", id));
    // striped: sources store into the target with SM kernels (decoding ones for the coded engines)
    if (striped) engine = engine_coded(engine) ? FSW_ENGINE_SMZ : FSW_ENGINE_SM;
    if (peer >= 0) engine = FSW_ENGINE_DMA;  // NVLink copy-engine transfer from the peer's extent
    const uint64_t dgrp = baseline ? (2ull << 20) : o.dma_group_bytes ? o.dma_group_bytes : c->cfg.dma_group_bytes;
    const uint32_t dstr = baseline ? 1u : o.dma_streams ? o.dma_streams : c->cfg.dma_streams;
    if (engine > FSW_ENGINE_DMAZ || dgrp == 0 || dgrp % 256 || dstr == 0 || dstr > (uint32_t)kMaxWaitSrc)
        return finish(fail(FSW_EINVAL, "invoke: bad engine / dma_group_bytes / dma_streams"));
    auto extents = [&](int i) {  // the model's extents on pool GPU i
        return DevDesc{c->gpus[i].pool + (m->pextent[i] >= 0 ? m->pextent[i] : 0), c->gpus[i].pool + m->extent[i], m->split, 0};
    };
    InvokeCfg ic{cold, (flags & FSW_NO_OVERLAP) != 0, engine,
                 o.chunk_bytes ? o.chunk_bytes : c->cfg.chunk_bytes, (int)o.order, o.order_seed,
                 o.copy_ctas ? o.copy_ctas : engine_coded(engine) ? std::max(c->cfg.copy_ctas, kDmazCtas) : c->cfg.copy_ctas,
                 extents(gi), nullptr};
    ic.from = pcached ? m->split : 0;
    if (ic.chunk % 256 || ic.chunk == 0 || ic.chunk >= (1ull << 32)) return finish(fail(FSW_EINVAL, "invoke: bad chunk_bytes"));
    if (cold && engine == FSW_ENGINE_DMA) ic.dma_plan = &get_dma_plan(*m, p, dgrp, dstr, ic.from);
    ic.zgrp = dgrp;
    if (cold && engine == FSW_ENGINE_DMAZ && !striped && g.zstage_cap < m->zbytes) {
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
    for (size_t j = 0; j < srcs.size(); ++j) {
        if (engine == FSW_ENGINE_SMZ)
            st = get_zstripe_pieces(*m, p, (uint32_t)srcs.size(), (uint32_t)j, c->gpus[srcs[j]].dev, ic.from, &zps[j]);
        else
            st = get_stripe_pieces(*m, p, schunk, (uint32_t)srcs.size(), (uint32_t)j, c->gpus[srcs[j]].dev, ic.from, &sps[j]);
        if (st != FSW_OK) return finish(st);
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
    if (cold && engine == FSW_ENGINE_DMAZ && !striped) key.extra = g.zstage_gen;  // baked staging address
    if (cold && !sm) {  // DMA graphs bake addresses: the target extents and a peer source's extents
        key.extra = (uint32_t)((uint64_t)m->extent[gi] >> 16);
        key.pext = m->pextent[gi];
        if (peer >= 0) {
            key.order = peer + 1;
            key.seed = (uint32_t)((uint64_t)m->extent[peer] >> 16) ^ (uint32_t)((uint64_t)(m->pextent[peer] + 1) << 8);
        }
    }
    auto it = p.graphs.find(key);
    cudaGraphExec_t exec = nullptr;
    if (it == p.graphs.end()) {
        st = build_graph(c, *m, p, g, ic, &exec);
        if (st != FSW_OK) return finish(st);
        p.graphs[key] = exec;
    } else {
        exec = it->second;
    }
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
            if (engine == FSW_ENGINE_SMZ)
                launch_swapz(sl.st, (int)ic.ctas, (int)c->cfg.copy_threads, m->zstore, 0, ic.dst, nullptr, zps[j]->dev,
                             (uint32_t)zps[j]->host.size(), g.ready, sl.ctl, g.ctl, 1, 0, nullptr);
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
    if (e == cudaSuccess) e = cudaEventSynchronize(g.ev1);
    if (e != cudaSuccess) return finish(fail(FSW_ECUDA, "invoke: graph launch/sync: %s", cudaGetErrorString(e)));
    const DevCtl ctl = *g.hctl;
    if (ctl.err) {
        const char* what = ctl.err == 1 ? "ready-flag watchdog" : ctl.err == 2 ? "swap-gate watchdog" : "embedding id out of range";
        return finish(fail(ctl.err == 3 ? FSW_EINVAL : FSW_ETIMEOUT, "invoke: %s (layer %d)", what, ctl.err_layer));
    }
    memcpy(output, g.hout, m->output_bytes);
    if (stats) {
        memset(stats, 0, sizeof *stats);
        float ms = 0;
        cudaEventElapsedTime(&ms, g.ev0, g.ev1);
        stats->device_ms = ms;
        stats->gpu = gi;
        stats->n_sources = cold ? (striped ? (uint32_t)srcs.size() : 1) : 0;
        stats->swap_kind = cold ? (striped ? FSW_SWAP_STRIPED : peer >= 0 ? FSW_SWAP_PEER : FSW_SWAP_HOST) : FSW_SWAP_RESIDENT;
        stats->n_kernels = (uint32_t)p.launches.size() + 1 /*finish*/;
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
                for (size_t j = 0; j < srcs.size(); ++j) stats->n_copies += (uint32_t)(coded ? zps[j]->host.size() : sps[j]->host.size());
                if (coded) {
                    stats->wire_bytes = 0;
                    for (ZPieceSet* zs : zps)
                        for (const ZPiece& pc : zs->host) stats->wire_bytes += pc.cbytes;
                }
            } else if (coded) {
                if (ctl.t_last > ctl.t_first) stats->swap_span_ms = (ctl.t_last - ctl.t_first) * 1e-6;
                if (ctl.t_end > ctl.t_last) stats->compute_tail_ms = (ctl.t_end - ctl.t_last) * 1e-6;
                stats->n_kernels += ic.no_overlap ? 1 : 2;  // decoding swap kernel (+ gate)
                ZPieceSet* zs = nullptr;
                if (get_zpieces(*m, p, g, ic.order, ic.seed, ic.from, engine == FSW_ENGINE_DMAZ ? dgrp : 0, &zs) == FSW_OK) {
                    stats->n_copies = (uint32_t)(engine == FSW_ENGINE_DMAZ ? zs->groups.size() : zs->host.size());
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

extern "C" fsw_status fsw_invoke(fsw_ctx* c, uint32_t id, const void* input, uint64_t input_bytes, void* output,
                                 uint64_t output_cap, fsw_invoke_stats* stats) {
    return fsw_invoke_ex(c, id, nullptr, input, input_bytes, output, output_cap, stats);
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

extern "C" fsw_status fsw_debug_read_coded(fsw_ctx* c, uint32_t id, void* dst, uint64_t cap) {
    Model* m = find_model(c, id);
    if (!m) return fail(FSW_ENOTFOUND, "model %u not found", id);
    if (!m->zstore) return fail(FSW_ESTATE, "model %u is not link-coded", id);
    if (!dst || cap < m->zbytes) return fail(FSW_EINVAL, "read_coded: cap %llu < %llu", (unsigned long long)cap, (unsigned long long)m->zbytes);
    memcpy(dst, m->zstore, m->zbytes);
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
