// rt_internal.h — declarations shared by the translation units of libfsw's host runtime
// (runtime.cpp, store.cpp, plan.cpp, graph.cpp, invoke.cpp).  Not part of the C-ABI.
#pragma once
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

#include <nvtx3/nvToolsExt.h>  // header-only NVTX 3: ranges cost nothing unless a tool (nsys) is attached

#include "fsw.h"
#include "kernels.h"
#include "policy.h"

// A host range in an nsys timeline (domain "fsw"): placement, plan / graph build, staging, the graph launch
// and the wait for the output of every invoke, so its GPU work lines up with the call that issued it.
struct NvtxRange {
    explicit NvtxRange(const char* name) {
        static nvtxDomainHandle_t dom = nvtxDomainCreateA("fsw");
        nvtxEventAttributes_t a{};
        a.version = NVTX_VERSION;
        a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        a.messageType = NVTX_MESSAGE_TYPE_ASCII;
        a.message.ascii = name;
        nvtxDomainRangePushEx(dom, &a);
        d = dom;
    }
    ~NvtxRange() { nvtxDomainRangePop(d); }
    nvtxDomainHandle_t d;
};

using namespace fsw;

// errors (runtime.cpp): set the thread-local message for fsw_last_error and return s
fsw_status fail(fsw_status s, const char* fmt, ...);
#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) return fail(FSW_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                                           __FILE__, __LINE__);                                    \
    } while (0)


inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
inline double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// ==========================================================================================
// Arena: best-fit extent allocator with coalescing (the pre-allocated pool)
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
    const void* abase = nullptr;  // K_GEMM (linear): the bf16 activation matrix [M][a_cols] the A tiles come from
    uint32_t a_cols = 0;
    bool attn_tc = false;         // K_ATTN: the tcgen05 kernel (attn_tc.cu), tmap over the QKV activation
    int wait_layer2 = -1;         // K_GEMM with a folded LayerNorm: also wait for that layer's weights (its γ, β)
};

struct Gpu;

struct GraphKey {
    int cold, flags, order, engine;
    uint64_t chunk;
    uint32_t seed, ctas, extra;
    uint64_t from = 0;   // first swapped store byte (partial caching: the cached prefix is skipped)
    int64_t pext = -1;   // DMA graphs: prefix extent offset (baked address)
    int64_t ext = -1;    // DMA graphs: target extent offset (baked address)
    int64_t src_ext = -1, src_pext = -1;  // peer DMA graphs: the source GPU's extents (baked addresses)
    uint32_t fault = 0;  // debug fault injection generation (fsw_debug_set_fault)
    bool operator<(const GraphKey& o) const {
        return std::tie(cold, flags, order, engine, chunk, seed, ctas, extra, from, pext, ext, src_ext, src_pext, fault) <
               std::tie(o.cold, o.flags, o.order, o.engine, o.chunk, o.seed, o.ctas, o.extra, o.from, o.pext, o.ext,
                        o.src_ext, o.src_pext, o.fault);
    }
    bool baked() const { return ext >= 0; }  // addresses of one placement: bounded LRU cache
};

// An instantiated invoke graph and when it was last launched (graphs that bake one placement's
// addresses are destroyed least recently used first beyond kMaxBakedGraphs per plan).
struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    uint64_t last_use = 0;
    void* mk_ops = nullptr;  // the persistent kernel's op table of this graph (device memory), or null
};
constexpr size_t kMaxBakedGraphs = 8;

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
    struct Group { uint64_t lo, hi; uint32_t stream; };
    std::vector<Group> groups;                          // DMAZ: coded-store byte ranges, in order
    uint64_t cfrom = 0, cend = 0;                        // coded bytes [cfrom, cend) cover the pieces
    uint32_t n_body = 0;   // DMAZT: pieces [0, n_body) move by copy groups, [n_body, size) zero-copy (SMZ tail)
    uint8_t* htab = nullptr;  // the model's decode table on this set's device (entropy-coded pieces), or nullptr
};

// The persistent transformer kernel's plan (mega.cu): the op list without the per-invoke waits, one
// activation tensor map per GEMM op (device array), the per-op completion counters.
struct MegaPlan {
    bool on = false;
    std::vector<MkOp> ops;             // w filled per graph (cold / warm, engine)
    std::vector<int> launch_of;        // index into Plan::launches of each op
    CUtensorMap* tmaps = nullptr;      // device
    uint32_t* op_cnt = nullptr;        // device, zeroed by the graph before the kernel
    float* part = nullptr;             // split-K partials (workspace)
    int ctas = 148;
    unsigned long long* stamps = nullptr;  // FSW_MEGA_STAMPS: [n_ops][ctas][8] phase stamps (device)
};

struct Plan {  // one model on one GPU
    bool built = false;
    std::vector<Launch> launches;
    MegaPlan mega;
    void* last_mk_ops = nullptr;  // set by build_graph: the op table the new graph bakes
    std::vector<uint64_t> slot_off;      // workspace offset of each slot
    std::vector<int64_t> shadow_off;     // bf16 shadow of an f32 slot, or -1
    uint64_t ws_bytes = 0;
    std::map<GraphKey, GraphEntry> graphs;
    uint64_t graph_clock = 0;
    std::map<std::tuple<uint64_t, int, uint32_t, uint64_t>, PieceSet> pieces;  // (chunk, order, seed, from)
    std::map<std::tuple<uint64_t, uint32_t, uint64_t, uint64_t>, DmaPlan> dma;  // (group bytes, streams, from, split)
    // striped swap: source j of n gets every n-th piece; its table lives on the source's device
    std::map<std::tuple<uint64_t, uint64_t, uint32_t, int, uint64_t>, PieceSet> stripe;  // (chunk, sources' nodes, j, device, from)
    // link-coded engines: (order, seed, from, DMAZ group bytes or 0 for SMZ) and striped (n, j, device, from)
    std::map<std::tuple<int, uint32_t, uint64_t, uint64_t, uint32_t, uint32_t>, ZPieceSet> zp;  // + DMAZ copy streams, tail ‰
    std::map<std::tuple<uint64_t, uint32_t, int, uint64_t>, ZPieceSet> zstripe;  // (sources' nodes, j, device, from)
    // DMAZ striped: source j's runs of coded pieces (copy groups) and its pieces with coff = staging offset
    std::map<std::tuple<uint64_t, uint32_t, int, uint64_t, uint64_t>, ZPieceSet> zstripe_dma;  // + run bytes
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
    int numa_node = -1;        // node the store's pages were bound to (mbind before first touch), -1 none,
                               // -2 bound chunk-wise across the pool's nodes (store_node / zstore_node)
    std::vector<int> store_node, zstore_node;  // node of each 2-MiB chunk of the store / coded store (empty: one node)
    // exponent-coded copy of the store (FSW_REG_LINK_CODE; kernels.h): pinned, mapped
    uint8_t* zstore = nullptr;
    uint64_t zbytes = 0, zalloc = 0;
    std::vector<ZPiece> zpieces;  // execution order, grp = 0
    // entropy-coded pieces (v5, kernels.h kZHuff): the model's 16 canonical code lengths and the decoder's
    // 4096-entry table (empty when no piece is entropy-coded)
    uint8_t hlen[16] = {};
    std::vector<uint8_t> htab;
    // residency per GPU
    std::vector<int64_t> extent;       // pool offset of the model (split = 0) or of its suffix, or -1
    // partial-parameter caching: store bytes [0, split) — whole layers —
    // live in a separate prefix extent that pool evictions keep (valid once its bytes landed)
    uint64_t split = 0;
    std::vector<int64_t> pextent;      // prefix extent per GPU, or -1
    std::vector<uint8_t> pvalid;       // prefix bytes present
    // extent[i] holds every swapped byte: set under c->mu only after a cold invoke on GPU i succeeded.
    // A GPU->GPU swap reads only complete extents (an extent being swapped in is not a resident copy).
    std::vector<uint8_t> complete;
    std::vector<uint64_t> last_use;
    std::vector<std::unique_ptr<Plan>> plans;
    int inflight = 0;
    // heavy / light class for placement and eviction: 1, 0, or -1 auto
    int heavy = -1;
    double slo_ms = 0;  // tightest deadline of the functions serving this model (0 = none)
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
    // DMAZ striped source (copy engine over this GPU's own host link into `stage`, then a decode kernel
    // storing into the target): staging buffer, run counter, decode stream and its fork / join events
    uint8_t* stage = nullptr;
    uint64_t stage_cap = 0;
    uint32_t* progress = nullptr;
    cudaStream_t sdec = nullptr;
    cudaEvent_t evfork = nullptr, evjoin = nullptr;
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
    CUtensorMap wmap;            // the pool as 128-B rows: the 2-CTA GEMM's weight map (k_gemm2)
    bool wmap_ok = false;
    fsw_arena* arena = nullptr;
    uint8_t* ws = nullptr;
    uint64_t ws_bytes = 0;
    uint32_t* ready = nullptr;
    uint32_t ready_cap = 0;
    DevCtl* ctl = nullptr;
    DevCtl* ctl_tail = nullptr;  // DMAZT: the tail kernel's tickets and stamps
    uint8_t* zstage = nullptr;   // DMAZ: device staging buffer for coded bytes (grown on demand)
    uint64_t zstage_cap = 0;
    uint32_t zstage_gen = 0;     // bumped on every reallocation (graphs bake the address)
    cudaStream_t sz = nullptr;   // DMAZ: decode-kernel stream
    cudaEvent_t evz = nullptr;   // DMAZ: join of the decode stream
    cudaEvent_t evset = nullptr; // DMAZ: the layer stream's setup (descriptor, counters) is done
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
    uint64_t n_evictions_heavy = 0;  // evictions of a model in the heavy class at the time
    unsigned long long* trace = nullptr;  // device timeline (FSW_TRACE): kTraceStride u64 per layer
};

constexpr uint64_t kStageHdr = 256;
constexpr uint32_t kGemmCtrs = 1u << 16;

// Tiling of one tcgen05 GEMM launch (gemm_tc.cu): tile width BN, split-K factor, cluster reduction.
struct Tiling { int bn; uint32_t splits, kt_per; bool cluster; };

struct fsw_ctx {
    fsw_config cfg{};
    std::vector<Gpu> gpus;
    std::vector<std::unique_ptr<Model>> models;  // index = id (nullptr after unregister)
    std::mutex mu;
    std::condition_variable cv;
    uint64_t clock = 0;
    std::vector<std::vector<char>> peer;  // peer[i][j]: GPU i can store into GPU j's memory
    std::vector<int> neighbor;            // GPU sharing a PCIe switch (-1 none), fsw_config.pcie_neighbor
    // NUMA node of each pool GPU's PCIe root (sysfs; -1 unknown) and the distinct nodes.  With more than
    // one node the host stores are bound chunk-wise across them and striped swaps read node-locally.
    std::vector<int> gpu_node, nodes;
    bool fake_numa = false;               // FSW_FAKE_NUMA=k: pretend pool GPU i is on node i % k (no mbind)
    uint32_t fault_kind = 0, fault_index = 0, fault_gen = 0;  // fsw_debug_set_fault (tests)
    double heavy_theta = 0.05, queue_budget_ms = 0.0;          // heavy / light policy (fsw_set_heavy_policy)
};


// ---- slot, layer and tile helpers (registration and plans) ---------------------------------
inline uint64_t slot_numel(const fsw_slot& s) {
    uint64_t n = 1;
    for (uint32_t i = 0; i < s.rank; ++i) n *= s.shape[i];
    return n;
}
inline uint32_t dt_size(uint32_t dt) { return dt == FSW_DT_BF16 ? 2 : 4; }
inline uint64_t slot_bytes(const fsw_slot& s) { return slot_numel(s) * dt_size(s.dtype); }
inline uint32_t slot_cols(const fsw_slot& s) { return s.rank ? s.shape[s.rank - 1] : 1; }
inline uint64_t slot_rows(const fsw_slot& s) { return slot_numel(s) / std::max<uint32_t>(1, slot_cols(s)); }

// How a CONV2D layer runs (gemm_tc.cu): a 1x1/stride-1 conv is a plain GEMM over [P·Q][Cin];
// Cin % 64 == 0 convs are implicit GEMMs (4-D TMA gathers of the NHWC input); the rest (the
// ResNet stem, Cin = 3) go through an explicit im2col buffer.
enum ConvPath { CONV_DIRECT, CONV_IMPLICIT, CONV_IM2COL };
inline uint32_t conv_rows_per_tile(uint32_t P, uint32_t Q) { return std::min<uint32_t>(128 / Q, P); }
inline ConvPath conv_path(const fsw_tensor& W, const fsw_layer& L, const fsw_slot& si, const fsw_slot& so) {
    const uint32_t R = W.shape[1], Cin = W.shape[3], stride = (uint32_t)L.attr[1], Q = so.shape[1];
    if (R == 1 && W.shape[2] == 1 && stride == 1 && L.attr[2] == 0 && Cin % 64 == 0) return CONV_DIRECT;
    if (Cin % 64 == 0 && Q <= 128 && Q * stride <= 256 && conv_rows_per_tile(so.shape[0], Q) * stride <= 256 &&
        stride <= 8 && si.rank == 3)
        return CONV_IMPLICIT;
    return CONV_IM2COL;
}

// Rows of in0 a LINEAR layer reads.
inline uint64_t linear_rows(const Model& m, const fsw_layer& L) {
    const uint64_t rin = slot_rows(m.slots[L.in0]);
    return L.attr[2] > 0 ? (uint64_t)L.attr[2] : rin;
}
inline bool linear_is_gemm(const Model& m, const fsw_layer& L) { return linear_rows(m, L) > 8; }

// Tile order of a GEMM weight W[N][K]: 1024-B atoms of 8 rows x 64 bf16,
// atoms ordered k-tile-major; inside an atom row r is 128 B at r·128 and its 16-B chunk c
// sits at chunk position c ^ r (the UMMA/TMA SWIZZLE_128B pattern).  Padding is zero.
inline uint64_t tiled_off(uint64_t n, uint64_t k, uint64_t n_pad) {
    return ((k / 64) * (n_pad / 8) + n / 8) * 1024 + (n % 8) * 128 + ((((k % 64) / 8) ^ (n % 8)) * 16) + (k % 8) * 2;
}

// ---- swap engines ----------------------------------------------------------------------------
inline bool engine_coded(int e) { return e == FSW_ENGINE_SMZ || e == FSW_ENGINE_DMAZ || e == FSW_ENGINE_DMAZT; }
// Engines whose body moves by copy-engine groups into the DMAZ staging buffer.
inline bool engine_dmaz(int e) { return e == FSW_ENGINE_DMAZ || e == FSW_ENGINE_DMAZT; }
// Engines whose layer kernels wait on per-layer byte counters (released by a swap kernel).
inline bool engine_bytes_ready(int e) { return e == FSW_ENGINE_SM || engine_coded(e); }

// Decoding swap CTAs unless the invoke sets copy_ctas (profiles/r01/linkcode/).  SMZ: 16 CTAs leave
// the TMA ring short of the link (ResNet-50 0.783 vs 0.739 ms), 32 reach it.  DMAZ (register decoder,
// 256 threads): the two-tier codes of link format v4 decode at 117 GB/s of store bytes on 32 CTAs and
// 168 GB/s on 48 (measured alone, tools/dmaz_probe.py); beside the layer kernels 32 CTAs fall behind
// the copy engine (BERT-base 3.10 ms), 48 do not (2.82 ms, as 64 and 96).
constexpr uint32_t kSmzCtas = 32, kDmazCtas = 48;
// DMAZ decode CTAs (128-thread shared-memory decoder) for models with entropy-coded pieces (FSW_DMAZ_HUFF_CTAS)
inline uint32_t smz_huff_ctas() {  // SMZ decode CTAs for models with entropy-coded pieces (FSW_SMZ_HUFF_CTAS)
    static const uint32_t v = getenv("FSW_SMZ_HUFF_CTAS") ? (uint32_t)atoi(getenv("FSW_SMZ_HUFF_CTAS")) : 64u;
    return v;
}
inline uint32_t dmazt_huff_tail_ctas() {  // DMAZT zero-copy tail CTAs, entropy-coded pieces (FSW_DMAZT_HUFF_TAIL_CTAS)
    static const uint32_t v = getenv("FSW_DMAZT_HUFF_TAIL_CTAS") ? (uint32_t)atoi(getenv("FSW_DMAZT_HUFF_TAIL_CTAS")) : 64u;
    return v;
}
inline uint32_t dmaz_huff_ctas() {
    static const uint32_t v = getenv("FSW_DMAZ_HUFF_CTAS") ? (uint32_t)atoi(getenv("FSW_DMAZ_HUFF_CTAS")) : 128u;
    return v;
}

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
    uint32_t zstreams = 1;       // DMAZ: copy streams (groups dealt round-robin, one counter each)
    uint32_t tail_ctas = 0;      // DMAZT: CTAs of the zero-copy tail kernel
};

// ---- cross-unit functions ----------------------------------------------------------------
Model* find_model(fsw_ctx* c, uint32_t id);                                      // runtime.cpp
void free_plan(Gpu& g, Plan& p);                                                 // runtime.cpp
void free_store(Model& m, bool host_only);                                       // runtime.cpp
fsw_status build_link_code(fsw_ctx* c, Model& m, bool host_only);               // store.cpp
int gpu_numa_node(int dev);                                                      // store.cpp
constexpr uint64_t kNumaChunk = 2ull << 20;  // NUMA binding unit of the host stores (one THP page)
inline int chunk_node(const std::vector<int>& map, uint64_t off) { return map.empty() ? -1 : map[off / kNumaChunk]; }
fsw_status build_plan(fsw_ctx* c, Model& m, int gi);                             // plan.cpp
fsw_status build_mega(fsw_ctx* c, Model& m, Plan& p, Gpu& g);                   // plan.cpp
fsw_status get_pieces(Model& m, Plan& p, Gpu& g, uint64_t chunk, int order, uint32_t seed, uint64_t from,
                      PieceSet** out);                                           // graph.cpp
const DmaPlan& get_dma_plan(Model& m, Plan& p, uint64_t grp, uint32_t streams, uint64_t from);
fsw_status get_zpieces(Model& m, Plan& p, Gpu& g, int order, uint32_t seed, uint64_t from, uint64_t grp,
                       uint32_t streams, ZPieceSet** out, uint32_t tail_permille = 0);
uint32_t dmazt_tail_permille();                                                  // graph.cpp: FSW_DMAZT_TAIL
fsw_status get_zstripe_pieces(Model& m, Plan& p, const std::vector<int>& src_node, uint32_t j, int dev, uint64_t from,
                              ZPieceSet** out);
fsw_status get_stripe_pieces(Model& m, Plan& p, uint64_t chunk, const std::vector<int>& src_node, uint32_t j, int dev,
                             uint64_t from, PieceSet** out);
fsw_status get_zstripe_dma(Model& m, Plan& p, const std::vector<int>& src_node, uint32_t j, int dev, uint64_t from,
                           uint64_t run_bytes, ZPieceSet** out);
constexpr uint64_t kStripeRunBytes = 4ull << 20;  // DMAZ striped: coded bytes per copy run (>= ~8 us copy setup x 55 GB/s x 10)
fsw_status build_graph(fsw_ctx* c, Model& m, Plan& p, Gpu& g, const InvokeCfg& ic, cudaGraphExec_t* out);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_writeValue32 get_write_value32();                                           // graph.cpp: cuStreamWriteValue32
bool model_heavy(const fsw_ctx* c, const Model& m);                              // invoke.cpp
void invalidate(fsw_ctx* c, Model& m, int gi, bool keep_prefix = false);         // invoke.cpp
