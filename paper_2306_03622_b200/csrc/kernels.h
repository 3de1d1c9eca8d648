// kernels.h — launch interface between the host runtime (rt_internal.h and its units) and the sm_100a
// kernels (*.cu).  Plain C++ (no device code); included by both sides of libfsw.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fsw.h"

namespace fsw {

// Per-GPU device-side invoke descriptor, written by the first node of every invoke graph
// (one small H2D from pinned staging).  Kernels find the model's extent through it, so a
// graph built once per (model, GPU) stays valid whichever pool extent the model lands in.
// Partial-parameter caching splits a resident model at a layer boundary
// `split`: store bytes [0, split) live in a prefix extent that survives pool evictions, bytes
// [split, B) in the suffix extent.  split = 0: the whole model is the one extent at sbase.
struct DevDesc {
    uint8_t* wbase;       // prefix extent (store offsets [0, split))
    uint8_t* sbase;       // suffix extent (store offsets [split, B))
    uint64_t split;
    uint64_t generation;  // invoke counter (debug)
};
// HBM address of store offset `off` (tensors never straddle `split`).
__host__ __device__ __forceinline__ uint8_t* weight_ptr(const DevDesc& d, uint64_t off) {
    return off < d.split ? d.wbase + off : d.sbase + (off - d.split);
}

// Per-GPU device control block (zeroed at the root of each cold graph except `err`).
struct DevCtl {
    uint32_t ticket;          // next swap piece to claim
    uint32_t started;         // swap CTAs that have begun executing
    uint32_t pad0[2];
    unsigned long long t_first;  // %globaltimer when the first piece was claimed
    unsigned long long t_last;   // %globaltimer when the last piece was released
    unsigned long long t_end;    // %globaltimer when the last layer kernel finished
    int32_t err;                 // watchdog / protocol error word (sticky until cleared)
    int32_t err_layer;
};

// One swap piece: a byte range of one layer's region (pieces never straddle layers).
struct Piece {
    uint64_t off;     // offset in the host store == offset in the extent
    uint32_t bytes;   // multiple of 16
    uint32_t layer;   // ready counter to bump
};

// Readiness wait for a layer kernel: spin until ready[j][0] >= target[j] for every j < n.
//   SM engine : n = 1, the layer's byte counter, target = the layer's region bytes.
//   DMA engine: n = copy streams, each stream's group counter, target = groups of that stream
//               up to the group holding the layer's last byte.
constexpr int kMaxWaitSrc = 4;
struct Wait {
    const uint32_t* ready[kMaxWaitSrc];
    uint32_t target[kMaxWaitSrc];
    uint32_t n;  // 0 = no wait (warm invoke / no weights)
    uint32_t sys;  // 1: counters are bumped by other GPUs (striped swap) -> system-scope acquire
    DevCtl* ctl;
    int32_t layer;
    unsigned long long* trace;  // device timeline (FSW_TRACE) or nullptr
};

constexpr uint64_t kWatchdogNs = 20ull * 1000 * 1000 * 1000;  // 20 s

// ---- swap ---------------------------------------------------------------------------------
// SM swap engine.  Destinations: the extents of `dst` (by value), or of *desc when desc is not
// NULL (this GPU's invoke descriptor, written by the graph's first node); ready = the target's
// per-layer counters; own = this launch's ticket / stamps; gate = the target's control block
// whose `started` the target's gate kernel watches; sys = 1 when the target is another GPU
// (peer stores over NVLink, system-scope release).
void launch_swap(cudaStream_t s, int ctas, int threads, const uint8_t* host_mapped, DevDesc dst, const DevDesc* desc,
                 const Piece* pieces, uint32_t n_pieces, uint32_t* ready, DevCtl* own, DevCtl* gate, int sys);
void launch_gate(cudaStream_t s, DevCtl* ctl, uint32_t expected);
// ---- exponent-coded link format ---------------------------------------------
// A lossless recoding of the host store that moves ~30 % fewer bytes over the host link; the swap
// kernel decodes it on the fly, so the extent receives the store's bytes bit-exactly.  The store is
// cut into pieces of <= kZPiece raw bytes (never straddling a layer region); a piece is cut into
// blocks of kZBlock raw bytes = 512 16-bit words w_i, each described by a 32-bit header kept in the
// piece table (device memory): h = bits 0-7, b = bits 8-15, n = bits 16-31.  A coded piece (128-B
// aligned in the coded store) is two streams, so the bulk of every zero-copy load covers whole 128-B
// host read requests:
//   stream A, per block in order:  b == kZRaw  : the raw bytes (kZBlock, or the piece's tail bytes for
//                                                a partial last block);
//                                  b == kZZero : nothing (all 512 words are 0);
//                                  b in 0..4   : 512 bytes m_i = (w_i >> 8 & 0x80) | (w_i & 0x7f);
//   zero padding to a multiple of 128 bytes;
//   stream B, per coded block (b in 0..4) in order: b bit-planes of 64 bytes (bit i of plane p, byte i/8
//                                  bit i%8, = bit p of the code c_i), then n exceptions of 4 bytes
//                                  (position i in bits 0-15, the whole word w_i in bits 16-31),
//                                  zero-padded to a multiple of 16 bytes.
// A coded block decodes (patched frame of reference over the exponents e_i = w_i >> 7 & 0xff, h = max
// e_i) as w_i = (m_i & 0x80) << 8 | (h − c_i) << 7 | (m_i & 0x7f), then every exception overwrites its
// word.  A word is an exception iff h − e_i >= 2^b (its code is then 0).
// Two-tier blocks (b = kZTier + o, o in 0..3; v4) code d_i = h − e_i closer to its entropy: bits 16-25
// of the header are the escape count n_e, bits 26-31 the exception count n_x.  Stream B is two tier-1
// bit-planes of 64 bytes (2-bit codes t_i: t_i < 3 means d_i = o + t_i, t_i = 3 means escaped), then
// three tier-2 bit-planes of 4·ceil(n_e / 32) bytes each holding one 3-bit code s_j per escaped word
// in word order (bit j of plane q = bit q of s_j; d = s_j < o ? s_j : s_j + 3, so escapes cover
// d in [0, o) and [o + 3, 10]), then n_x exceptions as above (escaped words with d >= 11, s_j = 0),
// zero-padded to a multiple of 16 bytes.  The encoder picks per block the kind with the fewest bytes.
// Entropy-coded pieces (v5): every coded block of the piece is kind kZHuff (b = 0x20; raw and zero blocks
// may sit between them).  Header: h = bits 0-7, the block's escape count n_esc = bits 16-25.  The offset
// s_i = min(h − e_i, 15) of every word is a canonical Huffman code (MSB first) of the MODEL's 16 code lengths
// (<= kZHuffLmax bits; s = 15 = escape: the whole word is an exception).  Stream A as for coded blocks
// (512 sign|mantissa bytes); stream B of the piece = E = Σ n_esc exception words (16 bits, in (block,
// lane, i) order), zero-padded to 16 B, then 4·K 16-bit code words: word j belongs to sub-stream j mod 4
// (its (j / 4)-th word; K = the longest sub-stream, the others zero-padded), zero-padded to 16 B.
// Sub-stream q carries the piece's kZHuff blocks with index ≡ q (mod 4), in order.  Decoding a block of
// sub-stream q: for i = 0..15, every lane l (0..31) whose bit buffer does not hold its next whole code (the
// code its bits start, read with zeros after them, is longer than the bits held) first appends the
// sub-stream's next word (the needing lanes, in increasing l, take consecutive words), then every lane
// decodes one code from the top of its buffer: s for word 16·l + i.  Buffers start empty at the piece's start.  The decoded word is (m_i & 0x80) << 8 | ((h − s) & 0xff) << 7 | (m_i & 0x7f), or the
// next exception word when s = 15.  A piece is entropy-coded only when that is smaller than its v4 form
// and its coded bytes fit one SMZ ring slot (kZBuf): the decoder reads it from shared memory.
constexpr uint32_t kZPiece = 16384;
constexpr uint32_t kZBlock = 1024;
constexpr uint32_t kZRaw = 0xff, kZZero = 0xfe, kZTier = 0x10, kZHuff = 0x20;
constexpr uint32_t kZHuffLmax = 12, kZHuffEsc = 15;
constexpr uint32_t kZHuffTabBytes = 1u << kZHuffLmax;  // decode table: s | L << 4 for every 12-bit window
constexpr uint32_t kZBuf = 12288;  // SMZ ring slot: largest coded piece decoded from shared memory
__host__ __device__ __forceinline__ bool zhuff(uint32_t hdr) { return ((hdr >> 8) & 0xffu) == kZHuff; }
__host__ __device__ __forceinline__ uint32_t zhuff_nesc(uint32_t hdr) { return (hdr >> 16) & 0x3ffu; }
// stream-A and stream-B bytes of one block
__host__ __device__ __forceinline__ uint32_t zblock_a(uint32_t hdr, uint32_t raw_bytes) {
    const uint32_t b = (hdr >> 8) & 0xffu;
    return b == kZRaw ? raw_bytes : b == kZZero ? 0u : 512u;
}
__host__ __device__ __forceinline__ uint32_t zblock_b(uint32_t hdr) {
    const uint32_t b = (hdr >> 8) & 0xffu, n = hdr >> 16;
    if ((b & ~3u) == kZTier) return (128u + 12u * (((n & 0x3ffu) + 31u) / 32u) + 4u * (n >> 10) + 15u) & ~15u;
    return b <= 4 ? 64u * b + ((4u * n + 15u) & ~15u) : 0u;
}
// coded blocks (FOR or two-tier): tier-1 code planes, tier-2 plane bytes, exception count and offset
__host__ __device__ __forceinline__ bool ztier(uint32_t hdr) { return (((hdr >> 8) & 0xffu) & ~3u) == kZTier; }
__host__ __device__ __forceinline__ uint32_t zplanes(uint32_t hdr) { return ztier(hdr) ? 2u : (hdr >> 8) & 0xffu; }
__host__ __device__ __forceinline__ uint32_t zt2_bytes(uint32_t hdr) { return 4u * ((((hdr >> 16) & 0x3ffu) + 31u) / 32u); }
__host__ __device__ __forceinline__ uint32_t zexc_n(uint32_t hdr) { return ztier(hdr) ? hdr >> 26 : hdr >> 16; }
__host__ __device__ __forceinline__ uint32_t zexc_off(uint32_t hdr) {
    return ztier(hdr) ? 128u + 3u * zt2_bytes(hdr) : 64u * ((hdr >> 8) & 0xffu);
}
__host__ __device__ __forceinline__ uint32_t zblock_bytes(uint32_t hdr, uint32_t raw_bytes) {
    return zblock_a(hdr, raw_bytes) + zblock_b(hdr);
}
struct ZPiece {
    uint64_t off;     // raw store offset == extent offset
    uint64_t coff;    // offset of the coded piece in the coded store (multiple of 128)
    uint32_t bytes;   // raw bytes (multiple of 16, <= kZPiece)
    uint32_t layer;   // ready counter to bump
    uint32_t grp;     // DMA+decode engine: copy group carrying the piece (decode waits for progress > grp)
    uint32_t cbytes;  // coded bytes
    uint32_t hdr[16]; // block headers (0 for blocks past the piece's end)
};
// Decoding swap kernel.  src + (coff − src_base) is a coded piece: the mapped coded host store
// (stage = 0, zero-copy over the host link) or the device staging buffer the copy engine filled
// (stage = 1; each piece first waits until *progress > grp).  Destinations, ready counters, gate and
// sys as launch_swap.
// htab: the model's 4096-entry decode table of entropy-coded pieces (entry = s | len << 4 for every 12-bit
// prefix), or nullptr when the model has none; such models decode through the shared-memory (TMA ring)
// decoder on every path.
void launch_swapz(cudaStream_t s, int ctas, int threads, const uint8_t* src, uint64_t src_base, DevDesc dst,
                  const DevDesc* desc, const ZPiece* pieces, uint32_t n_pieces, uint32_t* ready, DevCtl* own,
                  DevCtl* gate, int sys, int stage, const uint32_t* progress, const uint8_t* htab);
// DMAZT tail: the zero-copy (SMZ) decoder over pieces of the mapped coded store, whose CTAs start their reads
// once *start_ctr >= start_after (the DMAZ body's last copy group published); its last releases are also
// stamped into the gate's t_last (the invoke's swap span).
void launch_swapz_after(cudaStream_t s, int ctas, const uint8_t* zstore, DevDesc dst, const DevDesc* desc, const ZPiece* pieces,
                        uint32_t n_pieces, uint32_t* ready, DevCtl* own, DevCtl* gate, const uint32_t* start_ctr,
                        uint32_t start_after, const uint8_t* htab);

void launch_finish(cudaStream_t s, DevCtl* ctl, const uint8_t* out, uint64_t bytes, uint8_t* host_out, DevCtl* host_ctl);

// ---- test mode (FSW_DEBUG_POISON, fsw_debug_set_fault, fsw_debug_litmus) ---------------------
void launch_poison(cudaStream_t s, void* p, uint64_t bytes, uint32_t pattern);
void set_drop_piece(uint32_t index);  // current device; ~0 = no fault
// One layer region of a litmus run: store offset, bytes, and the per-counter targets of its Wait.
struct LitmusLayer { uint64_t off; uint32_t bytes, layer; uint32_t target[kMaxWaitSrc]; };
// `ctas` consumer CTAs (layer regions round-robin); wbase.ready[j] = the counters (per_layer_counter:
// the base of the per-layer byte counters, indexed by LitmusLayer::layer), n, sys, ctl as a layer
// kernel's Wait.
void launch_litmus_check(cudaStream_t s, int ctas, DevDesc dst, const uint8_t* golden, const LitmusLayer* layers,
                         uint32_t n_layers, Wait wbase, int per_layer_counter, DevCtl* gate, uint32_t gate_expected,
                         unsigned long long* bad, unsigned long long* checked);

// ---- layer ops ----------------------------------------------------------------------------
struct EmbedArgs {
    const int32_t* ids; int n_tables; uint64_t table_off[4]; uint32_t table_rows[4]; int rule[4];
    uint32_t T, C; float* out; uint16_t* out_bf16;
};
void launch_embed(cudaStream_t s, const DevDesc* d, Wait w, const EmbedArgs& a);

struct LnArgs {
    const float* in; uint32_t rows, C; float eps; uint64_t g_off, b_off;
    float* out_f32; uint16_t* out_bf16;
};
void launch_layernorm(cudaStream_t s, const DevDesc* d, Wait w, const LnArgs& a);

struct GemvArgs {  // y[i][o] = act(x[r0+i]·W[o] + b[o] + res[i][o]),  W row-major [N][K] bf16
    const void* x; int x_bf16; uint32_t ldx, r0, rows, K, N;
    uint64_t w_off, b_off; int has_bias, act;
    const void* res; int res_bf16;
    void* out; int out_bf16; uint16_t* out2;
};
void launch_gemv(cudaStream_t s, const DevDesc* d, Wait w, const GemvArgs& a);

struct GemmArgs {  // out[m][n] = act(A[m]·W[n] + b[n] + res[m][n]); A via TMA, W tiled
    uint32_t M, N, K, n_pad;     // K = padded K (multiple of 64), n_pad = tiled rows
    uint64_t w_off, b_off; int has_bias, act;
    const void* res; int res_bf16; uint32_t ld_res;
    void* out; int out_bf16; uint32_t ld_out;
    uint16_t* out2;     // optional bf16 shadow of an f32 output (same ld)
    int bn;             // tile N: 16, 32, 64 or 128
    uint32_t m_rows;    // output rows per M tile: 128, or Hb·Q for an implicit-GEMM conv tile
    // split-K: gridDim.z = splits; split z covers 64-wide k tiles [z·kt_per, (z+1)·kt_per)
    uint32_t splits, kt_per;
    float* part;        // [m_tiles·n_tiles][splits][128][bn] fp32 partial tiles (splits > 1)
    uint32_t* ctr;      // [m_tiles·n_tiles] arrival counters, self-resetting (splits > 1)
    // implicit-GEMM convolution: A tile = Hb output rows x Q columns x 64 input channels of one
    // (r, s) tap, gathered by one 4-D TMA load (zero fill = padding, element stride = conv stride)
    int conv; uint32_t Q, stride, pad, S, Cin, Hb;
    // A multicast: CTAs of a (1, mc, 1) cluster share each A sub-tile, every CTA loading 128/mc rows
    // and broadcasting them (mc in {1, 2, 4, 8}; the A tensor map's box is 128/mc rows)
    uint32_t mc;
    // cluster split-K: the `splits` CTAs of one output tile form a (1, 1, cz) cluster (cz == splits <= 8)
    // and reduce their partial tiles over distributed shared memory instead of `part` / `ctr`
    uint32_t cz;
    // 2-CTA swap-AB GEMM (k_gemm2): pair_t = tokens per CTA pair (16, 32, 64 or 128), 0 = k_gemm.  The
    // A tensor map's box is then pair_t / 2 rows; weights come through the pool-wide map (wpool = the
    // GPU's pool base, the map's origin)
    uint32_t pair_t;
    const void* wpool;
    // weight-stationary swap-AB GEMM (k_gemm_ws, gemm_ws.cu): ws_tt = tokens per tile (16, 32, 64 or 128),
    // 0 = not used.  128 weight rows x ws_tt tokens per CTA; split-K over a (1, 1, splits) cluster (splits <= 8,
    // kt_per k sub-tiles each, all resident in shared memory); the A tensor map's box is ws_tt rows
    uint32_t ws_tt;
    uint32_t ws_stages;  // k_gemm_ws: 0 = the whole K range resident; else a ring of this many k sub-tile slots
    uint32_t trig_early;  // k_gemm_ws: 1 = release the successor's launch (PDL) at entry instead of after the MMAs
    // L2 prefetch (k_gemm / k_gemm_ws, resident invokes): the next GEMM's weights [pf_off, pf_off + pf_bytes) of
    // the store, dealt over this launch's CTAs; pf_bytes = 0: none
    uint64_t pf_off, pf_bytes;
    // LayerNorm folded into the k_gemm_ws launches around it (FSW_LN_FUSE; plan.cpp fuse_layernorms):
    //  * producer (st_out != null): the owner CTA of each (row tile, split) writes, per token, the (mean, M2) of
    //    its 128 / splits output columns to st_out[(tile · splits + split) · M + token];
    //  * A consumer (ln_x != null, stationary mode only): the operand tile is LN(ln_x) computed on load —
    //    (μ, rstd) merged from the ln_slots partials (ln_cnt values each, Chan's formula), γ / β from the
    //    store — written bf16 into the swizzled shared-memory tile instead of a TMA load; the launch with
    //    blockIdx.x = z = 0 stores (μ, rstd) per token to ln_musig;
    //  * residual consumer (res_musig != null): the residual is LN(res) = (res − μ)·rstd·γ + β recomputed from
    //    the pre-LN fp32 stream `res` and those (μ, rstd).
    float2* st_out;
    const float* ln_x; const float2* ln_st; uint32_t ln_slots, ln_cnt; uint64_t ln_g_off, ln_b_off; float ln_eps;
    float2* ln_musig;
    const float2* res_musig; uint64_t res_g_off, res_b_off;
};
void launch_gemm(cudaStream_t s, const DevDesc* d, Wait w, const CUtensorMap* tmA, const GemmArgs& a,
                 const CUtensorMap* tmW = nullptr);
bool make_tmap_pool(CUtensorMap* map, const void* pool, uint64_t bytes);
void launch_gemm_ws(cudaStream_t s, const DevDesc* d, Wait w, const CUtensorMap* tmX, const GemmArgs& a);
uint32_t gemm_ws_smem(uint32_t tt, uint32_t slots, uint32_t splits);  // dynamic shared memory of one CTA
int gemm_ws_max_active_clusters(uint32_t tt, uint32_t slots, int cz);  // clusters resident at once (this device)
void init_gemm_ws_attrs();

struct AttnArgs { const uint16_t* qkv; uint16_t* out; uint32_t T, H, dh; int causal; int32_t layer; unsigned long long* trace; };
void launch_attention(cudaStream_t s, const AttnArgs& a);
// tcgen05 attention (attn_tc.cu): T <= 128, dh = 64; tm = TMA map over the QKV activation [T][3·H·64], 64 x 128 boxes
bool attention_tc_ok(const AttnArgs& a);
void launch_attention_tc(cudaStream_t s, const CUtensorMap* tm, const AttnArgs& a);
void init_attn_tc_attrs();

struct Im2colArgs {
    const uint16_t* in; uint32_t H, W, C;
    uint16_t* out; uint32_t P, Q, R, S, stride, pad, K, Kpad;
    int32_t layer;
    unsigned long long* trace;
};
void launch_im2col(cudaStream_t s, const Im2colArgs& a);

struct PoolArgs {
    const uint16_t* in; uint32_t H, W, C; uint32_t P, Q, k, stride, pad;
    uint16_t* out; float* out_f32;
    int32_t layer;
    unsigned long long* trace;
};
void launch_maxpool(cudaStream_t s, const PoolArgs& a);
void launch_avgpool(cudaStream_t s, const PoolArgs& a);

// Device timeline (FSW_TRACE, fsw_debug_trace_read; DESIGN.md §5 "Overlap timeline"): per layer L,
// kTraceStride u64 at trace + L·kTraceStride: [0] ~(first kernel CTA entry), [1] last weight-wait done,
// [2] last kernel CTA exit, [3] ~(first piece of L released by a swap kernel), [4] last piece released.
// Min fields are stored complemented so that one memset to 0 resets every field (atomicMax for all).
constexpr uint32_t kTraceStride = 16;
void set_trace_swap(unsigned long long* t);  // current device; nullptr = off (swap.cu)
void set_trace_mega(unsigned long long* t);  // mega.cu
// ---- persistent transformer kernel (mega.cu; DESIGN.md §5 "k_mega") ---------------------------------
// One launch runs every layer of a transformer (EMBED, LAYERNORM, LINEAR, ATTENTION) on one CTA per SM.
// Op i is a list of n_tasks tasks; CTA c takes tasks c, c + grid, ... of every op in order.  A task of
// op i reads activations only after op `dep` (i − 1) has counted all its tasks done (release / acquire
// on a per-op counter); weights need only the layer's readiness (Wait), so a CTA's producer warp
// streams the next op's weight tiles while the previous op still runs.  GEMMs are swap-AB tcgen05
// tiles: 128 weight rows (UMMA M) x tt tokens (UMMA N) x a K range (split-K, partials reduced by the
// last split in split order).
enum MkKind : uint32_t { MK_GEMM = 1, MK_LN = 2, MK_ATTN = 3, MK_EMBED = 4, MK_GEMV = 5 };
struct MkOp {
    uint32_t kind, n_tasks;
    int32_t dep;                       // op whose completion the activations need (-1: none)
    int32_t layer;
    Wait w;                            // weights' readiness (n = 0: resident / no weights)
    uint32_t tt, n_rt, n_tt, splits, kt_per, tmap;  // GEMM tiling; tmap = index into the tensor-map array
    union {
        GemmArgs gemm;
        LnArgs ln;
        AttnArgs attn;
        EmbedArgs embed;
        GemvArgs gemv;
    };
};
constexpr uint32_t kMkTT = 64;  // largest token tile
// ops / counters / tensor maps in device memory; grid = one CTA per SM (ctas)
void launch_mega(cudaStream_t s, int ctas, const DevDesc* d, const MkOp* ops, uint32_t n_ops, uint32_t* op_cnt,
                 const CUtensorMap* tmaps, uint32_t* tile_ctr, float* part);
size_t mega_smem_bytes();
void set_mega_stamps(unsigned long long* p);  // current device; phase stamps [n_ops][ctas][8] or nullptr
void init_mega_attrs();

void init_gemm_attrs();
int gemm_max_active_clusters(int bn, int cz);  // clusters of cz GEMM CTAs resident at once (this device)
void init_swap_attrs();
void init_ops_attrs();

// Host helper: build the TMA descriptor of a row-major bf16 activation [rows][cols].
bool make_tmap_act(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                   uint32_t box_rows = 0 /* 0 = 128 */);
// Host helper: 4-D TMA descriptor of an NHWC bf16 input [H][W][C] for implicit-GEMM conv:
// box = 64 channels x Q output columns x Hb output rows, element strides = conv stride.
bool make_tmap_conv(CUtensorMap* map, const void* base, uint32_t H, uint32_t W, uint32_t C, uint32_t Q, uint32_t Hb,
                    uint32_t stride);

}  // namespace fsw
