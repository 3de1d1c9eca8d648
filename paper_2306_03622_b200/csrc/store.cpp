// store.cpp — model registration: table validation, the host store (execution order, GEMM weights
// in tensor-core tile order, THP-backed, NUMA-bound, pinned + mapped) and its link-coded copy
// (DESIGN.md §5b); model info; unregister.
#include "rt_internal.h"

// ==========================================================================================
// registration: validation + host store (execution order, GEMM weights tiled)
// ==========================================================================================
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
int gpu_numa_node(int dev) {
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
// the kind with the fewest bytes: a code width b in 0..4 (words with h − e >= 2^b become exceptions),
// a two-tier code with tier-1 offset o in 0..3 (at most 63 exceptions), or raw when nothing beats the
// 1024 raw bytes.
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
    uint32_t best = kZRaw << 8, best_bytes = kZBlock, n = kZBlock / 2;
    for (uint32_t b = 0; b <= 4; ++b) {
        n -= hist[b];  // words with h − e >= 2^b
        const uint32_t hd = emax | (b << 8) | (n << 16), bytes = zblock_bytes(hd, kZBlock);
        if (bytes < best_bytes) best = hd, best_bytes = bytes;
    }
    // two-tier kinds: tier 1 holds d in [o, o + 3), tier 2 d in [0, o) and [o + 3, 10], exceptions d >= 11
    uint32_t cnt[12] = {};  // cnt[d] for d <= 10, cnt[11] = words with d >= 11
    for (uint32_t i = 0; i < kZBlock / 2; ++i) cnt[std::min<uint32_t>(11, emax - ((w[i] >> 7) & 0xffu))]++;
    for (uint32_t o = 0; o < 4; ++o) {
        const uint32_t nx = cnt[11], ne = kZBlock / 2 - cnt[o] - cnt[o + 1] - cnt[o + 2];
        if (nx > 63) break;
        const uint32_t hd = emax | ((kZTier + o) << 8) | (ne << 16) | (nx << 26), bytes = zblock_bytes(hd, kZBlock);
        if (bytes < best_bytes) best = hd, best_bytes = bytes;
    }
    return best;
}

// Coded block: 512 stream-A bytes at outa, zblock_b(hdr) stream-B bytes at outb (both zeroed).
static void zencode_tier(const uint16_t* w, uint32_t hdr, uint8_t* outa, uint8_t* outb) {
    const uint32_t h = hdr & 0xffu, o = ((hdr >> 8) & 0xffu) - kZTier, ne = (hdr >> 16) & 0x3ffu;
    const uint32_t pw = 4 * ((ne + 31) / 32);  // bytes per tier-2 plane
    uint8_t* t2 = outb + 128;
    uint8_t* exc = t2 + 3 * pw;
    uint32_t j = 0, k = 0;
    for (uint32_t i = 0; i < kZBlock / 2; ++i) {
        const uint32_t d = h - ((w[i] >> 7) & 0xffu);
        outa[i] = (uint8_t)(((w[i] >> 8) & 0x80u) | (w[i] & 0x7fu));
        uint32_t t = 3;
        if (d >= o && d < o + 3) t = d - o;
        outb[(i >> 3)] |= (uint8_t)((t & 1u) << (i & 7));
        outb[64 + (i >> 3)] |= (uint8_t)((t >> 1) << (i & 7));
        if (t != 3) continue;
        uint32_t sj = d < o ? d : d - 3;  // escaped word j = this word's rank among the escapes
        if (d >= 11) {
            sj = 0;
            const uint32_t e = i | ((uint32_t)w[i] << 16);
            memcpy(exc + 4 * k++, &e, 4);
        }
        for (uint32_t q = 0; q < 3; ++q) t2[q * pw + (j >> 3)] |= (uint8_t)(((sj >> q) & 1u) << (j & 7));
        ++j;
    }
}

static void zencode_block(const uint16_t* w, uint32_t hdr, uint8_t* outa, uint8_t* outb) {
    if ((((hdr >> 8) & 0xffu) & ~3u) == kZTier) return zencode_tier(w, hdr, outa, outb);
    const uint32_t h = hdr & 0xffu, b = (hdr >> 8) & 0xffu;
    uint8_t code[kZBlock / 2];
    uint32_t k = 0;
    uint8_t* exc = outb + 64 * b;
    for (uint32_t i = 0; i < kZBlock / 2; ++i) {
        const uint32_t d = h - ((w[i] >> 7) & 0xffu);
        outa[i] = (uint8_t)(((w[i] >> 8) & 0x80u) | (w[i] & 0x7fu));
        const bool ex = (d >> b) != 0;  // exception: position and the whole word; code 0
        code[i] = ex ? 0 : (uint8_t)d;
        if (ex) {
            const uint32_t e = i | ((uint32_t)w[i] << 16);
            memcpy(exc + 4 * k++, &e, 4);
        }
    }
    for (uint32_t p = 0; p < b; ++p)  // plane p, 64 words per 64-bit lane word (bit i % 64 = word i)
        for (uint32_t q = 0; q < 8; ++q) {
            uint64_t v = 0;
            for (uint32_t i = 0; i < 64; ++i) v |= (uint64_t)((code[64 * q + i] >> p) & 1u) << i;
            memcpy(outb + 64 * p + 8 * q, &v, 8);
        }
}

// ---- entropy-coded pieces (format v5, kernels.h kZHuff) --------------------------------------------
// Canonical Huffman code over the word offsets s = min(h − e, 15) of the model's coded blocks, lengths
// limited to kZHuffLmax (the frequencies are flattened until the Huffman lengths fit).
struct HuffCode {
    uint8_t len[16] = {};
    uint16_t code[16] = {};
    bool ok = false;
};
static HuffCode huff_build(const uint64_t* freq_in) {
    HuffCode hc;
    uint64_t f[16];
    uint32_t used = 0;
    for (int s = 0; s < 16; ++s) used += (f[s] = freq_in[s]) != 0;
    if (used < 2) return hc;  // nothing to code (a one-symbol code would need 0-bit words)
    for (int round = 0; round < 64; ++round) {
        // Huffman lengths by repeated merging of the two lightest subtrees (16 symbols: O(n^2) is fine)
        std::vector<std::pair<uint64_t, std::vector<int>>> nodes;
        for (int s = 0; s < 16; ++s)
            if (f[s]) nodes.push_back({f[s], {s}});
        uint8_t len[16] = {};
        while (nodes.size() > 1) {
            std::sort(nodes.begin(), nodes.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
            auto a = nodes.back();
            nodes.pop_back();
            auto b = nodes.back();
            nodes.pop_back();
            for (int s : a.second) ++len[s];
            for (int s : b.second) ++len[s];
            a.second.insert(a.second.end(), b.second.begin(), b.second.end());
            nodes.push_back({a.first + b.first, a.second});
        }
        uint32_t mx = 0;
        for (int s = 0; s < 16; ++s) mx = std::max<uint32_t>(mx, len[s]);
        if (mx <= kZHuffLmax) {
            memcpy(hc.len, len, 16);
            break;
        }
        for (int s = 0; s < 16; ++s)
            if (f[s]) f[s] = f[s] / 2 + 1;
    }
    // canonical codes: by (length, symbol), MSB first
    uint32_t code = 0, prev = 0;
    for (uint32_t L = 1; L <= kZHuffLmax; ++L)
        for (int s = 0; s < 16; ++s)
            if (hc.len[s] == L) {
                code <<= (L - prev);
                prev = L;
                hc.code[s] = (uint16_t)code++;
            }
    hc.ok = true;
    return hc;
}

// Decoder table: for every 12-bit window, s | L << 4 of the code it starts with.
static void huff_table(const HuffCode& hc, std::vector<uint8_t>& tab) {
    tab.assign(kZHuffTabBytes, 0);
    for (int s = 0; s < 16; ++s) {
        const uint32_t L = hc.len[s];
        if (!L) continue;
        const uint32_t lo = (uint32_t)hc.code[s] << (kZHuffLmax - L), n = 1u << (kZHuffLmax - L);
        for (uint32_t k = 0; k < n; ++k) tab[lo + k] = (uint8_t)(s | (L << 4));
    }
}

// The entropy-coded form of one piece (raw bytes w, v4 block headers hdr4): its headers, exception words,
// the interleaved code words of stream B, and its coded size.  out == nullptr: size only.
struct HuffPiece {
    uint32_t hdr[16] = {};
    std::vector<uint16_t> exc, words;  // words: 4·K interleaved code words
    uint32_t la = 0, cbytes = 0;
};
static void huff_piece(const uint8_t* raw, uint32_t bytes, const uint32_t* hdr4, const HuffCode& hc, HuffPiece& hp) {
    const uint32_t nb = (bytes + kZBlock - 1) / kZBlock;
    std::vector<uint16_t> sub[4];
    for (uint32_t q = 0; q < 4; ++q) {
        // lane bit streams of sub-stream q: the codes of words 16 l + i of its blocks, in order
        std::vector<uint16_t> chunk[32];
        uint64_t acc[32] = {};
        uint32_t accb[32] = {};
        std::vector<uint32_t> blocks;
        for (uint32_t b = q; b < nb; b += 4) {
            const uint32_t k4 = (hdr4[b] >> 8) & 0xffu;
            if (k4 == kZRaw || k4 == kZZero) continue;
            blocks.push_back(b);
        }
        for (uint32_t b : blocks) {
            const uint16_t* w = reinterpret_cast<const uint16_t*>(raw + (uint64_t)b * kZBlock);
            const uint32_t h = hdr4[b] & 0xffu;
            for (uint32_t l = 0; l < 32; ++l)
                for (uint32_t i = 0; i < 16; ++i) {
                    const uint32_t d = h - ((w[16 * l + i] >> 7) & 0xffu), s = std::min(d, kZHuffEsc);
                    acc[l] = (acc[l] << hc.len[s]) | hc.code[s];
                    accb[l] += hc.len[s];
                    while (accb[l] >= 16) {
                        chunk[l].push_back((uint16_t)(acc[l] >> (accb[l] - 16)));
                        accb[l] -= 16;
                        acc[l] &= (1ull << accb[l]) - 1;
                    }
                }
        }
        for (uint32_t l = 0; l < 32; ++l)
            if (accb[l]) chunk[l].push_back((uint16_t)(acc[l] << (16 - accb[l])));
        // the decoder's refill order (kernels.h kZHuff): per word step, the lanes whose buffer lacks their next
        // whole code, in lane order
        uint32_t nbits[32] = {}, next[32] = {};
        for (uint32_t b : blocks) {
            const uint16_t* w = reinterpret_cast<const uint16_t*>(raw + (uint64_t)b * kZBlock);
            const uint32_t h = hdr4[b] & 0xffu;
            for (uint32_t i = 0; i < 16; ++i) {
                uint32_t need[32];
                for (uint32_t l = 0; l < 32; ++l) need[l] = hc.len[std::min(h - ((w[16 * l + i] >> 7) & 0xffu), kZHuffEsc)];
                for (uint32_t l = 0; l < 32; ++l)
                    if (need[l] > nbits[l]) {
                        sub[q].push_back(next[l] < chunk[l].size() ? chunk[l][next[l]] : 0);
                        ++next[l];
                        nbits[l] += 16;
                    }
                for (uint32_t l = 0; l < 32; ++l) nbits[l] -= need[l];
            }
        }
    }
    size_t K = 0;
    for (auto& v : sub) K = std::max(K, v.size());
    hp.words.assign(4 * K, 0);
    for (uint32_t q = 0; q < 4; ++q)
        for (size_t k = 0; k < sub[q].size(); ++k) hp.words[4 * k + q] = sub[q][k];
    hp.exc.clear();
    hp.la = 0;
    for (uint32_t b = 0; b < nb; ++b) {
        const uint32_t k4 = (hdr4[b] >> 8) & 0xffu, n = std::min(kZBlock, bytes - b * kZBlock);
        if (k4 == kZRaw || k4 == kZZero) {
            hp.hdr[b] = hdr4[b];
            hp.la += k4 == kZRaw ? n : 0;
            continue;
        }
        const uint16_t* w = reinterpret_cast<const uint16_t*>(raw + (uint64_t)b * kZBlock);
        const uint32_t h = hdr4[b] & 0xffu;
        uint32_t ne = 0;
        for (uint32_t i = 0; i < kZBlock / 2; ++i)
            if (h - ((w[i] >> 7) & 0xffu) >= kZHuffEsc) {
                hp.exc.push_back(w[i]);
                ++ne;
            }
        hp.hdr[b] = h | (kZHuff << 8) | (ne << 16);
        hp.la += 512;
    }
    hp.cbytes = (uint32_t)(align_up(hp.la, 128) + align_up(2 * hp.exc.size(), 16) + align_up(2 * hp.words.size(), 16));
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
// Bind [p, p + len) before first touch: to `node`, or — when the pool's GPUs span several NUMA nodes —
// 2-MiB chunk i to nodes[i % n] (striped swaps then deal each chunk's data to a source on its node).
// Returns the model's numa_node value and fills the chunk map.
static int bind_store(fsw_ctx* c, uint8_t* p, uint64_t len, int node, std::vector<int>& map) {
    map.clear();
    if (c->nodes.size() > 1) {
        for (uint64_t i = 0; i * kNumaChunk < len; ++i) {
            const int nd = c->nodes[i % c->nodes.size()];
            if (!c->fake_numa) bind_pages(p + i * kNumaChunk, std::min<uint64_t>(kNumaChunk, len - i * kNumaChunk), nd);
            map.push_back(nd);
        }
        return -2;
    }
    return bind_pages(p, len, node);
}

fsw_status build_link_code(fsw_ctx* c, Model& m, bool host_only) {
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
    // entropy-coded pieces (v5): one canonical code per model over the offsets of every coded block; a piece
    // takes it when that is smaller than its v4 form and fits a shared-memory ring slot (FSW_LINK_HUFF=0: off)
    // Entropy-coded pieces for stores >= 32 MiB: their decode is slower per word than v4's (a dependent
    // shared-memory round trip per code), which the larger models hide behind the link and the small ones
    // do not (measured: ResNet-50 SMZ 0.712 -> 0.700 ms, BERT-base DMAZT 2.779 -> 2.745 ms,
    // MLP 8 MB 0.156 -> 0.188 ms).  FSW_LINK_HUFF=0 never, =1 always (read per registration).
    const char* hv = getenv("FSW_LINK_HUFF");
    const bool huff_on = hv ? atoi(hv) != 0 : m.store_bytes >= (32ull << 20);
    HuffCode hc;
    if (huff_on) {
        std::vector<std::array<uint64_t, 16>> fr(pcs.size());
        parallel_for(pcs.size(), [&](size_t i) {
            fr[i].fill(0);
            const ZPiece& pc = pcs[i];
            for (uint32_t b = 0; b * kZBlock < pc.bytes; ++b) {
                const uint32_t hd = hdr[i * bpp + b], k4 = (hd >> 8) & 0xffu;
                if (k4 == kZRaw || k4 == kZZero) continue;
                const uint16_t* w = reinterpret_cast<const uint16_t*>(m.store + pc.off + (uint64_t)b * kZBlock);
                for (uint32_t j = 0; j < kZBlock / 2; ++j) fr[i][std::min((hd & 0xffu) - ((w[j] >> 7) & 0xffu), kZHuffEsc)]++;
            }
        });
        uint64_t freq[16] = {};
        for (auto& a : fr)
            for (int s = 0; s < 16; ++s) freq[s] += a[s];
        hc = huff_build(freq);
    }
    std::vector<uint8_t> is_huff(pcs.size(), 0);
    if (hc.ok) {
        parallel_for(pcs.size(), [&](size_t i) {
            const ZPiece& pc = pcs[i];
            const uint32_t nb = (pc.bytes + kZBlock - 1) / kZBlock;
            uint32_t la = 0, lb = 0;
            bool coded = false;
            for (uint32_t b = 0; b < nb; ++b) {
                const uint32_t hd = hdr[i * bpp + b], k4 = (hd >> 8) & 0xffu;
                la += zblock_a(hd, std::min(kZBlock, pc.bytes - b * kZBlock));
                lb += zblock_b(hd);
                coded |= k4 != kZRaw && k4 != kZZero;
            }
            if (!coded) return;
            HuffPiece hp;
            huff_piece(m.store + pc.off, pc.bytes, &hdr[i * bpp], hc, hp);
            if (hp.cbytes < align_up(la, 128) + lb && hp.cbytes <= kZBuf) {
                memcpy(&hdr[i * bpp], hp.hdr, sizeof hp.hdr);
                is_huff[i] = 1;
            }
        });
    }
    m.htab.clear();
    memset(m.hlen, 0, sizeof m.hlen);
    if (std::find(is_huff.begin(), is_huff.end(), 1) != is_huff.end()) {
        memcpy(m.hlen, hc.len, 16);
        huff_table(hc, m.htab);
    }
    // piece sizes (entropy-coded pieces: recomputed from their v4 headers, which hdr no longer holds)
    std::vector<uint32_t> hcb(pcs.size(), 0);
    parallel_for(pcs.size(), [&](size_t i) {
        if (!is_huff[i]) return;
        const ZPiece& pc = pcs[i];
        uint32_t h4[16];
        for (uint32_t b = 0; b < bpp; ++b) {
            const uint32_t hd = hdr[i * bpp + b];
            h4[b] = zhuff(hd) ? (hd & 0xffu) | (1u << 8) : hd;  // any coded v4 kind: huff_piece needs only h
        }
        HuffPiece hp;
        huff_piece(m.store + pc.off, pc.bytes, h4, hc, hp);
        hcb[i] = hp.cbytes;
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
        const uint32_t cb = is_huff[i] ? hcb[i] : (uint32_t)align_up(la, 128) + lb;
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
    if (!host_only) bind_store(c, static_cast<uint8_t*>(p), m.zalloc, m.numa_node, m.zstore_node);
    m.zstore = static_cast<uint8_t*>(p);
    parallel_for((m.zalloc + (2u << 20) - 1) / (2u << 20), [&](size_t i) {  // alignment gaps stay zero
        memset(m.zstore + i * (2u << 20), 0, std::min<uint64_t>(2u << 20, m.zalloc - i * (2u << 20)));
    });
    parallel_for(pcs.size(), [&](size_t i) {
        const ZPiece& pc = pcs[i];
        uint8_t* out = m.zstore + pc.coff;
        const uint32_t nb = (pc.bytes + kZBlock - 1) / kZBlock;
        uint32_t la = 0;
        for (uint32_t b = 0; b < nb; ++b) la += zblock_a(hdr[i * bpp + b], std::min(kZBlock, pc.bytes - b * kZBlock));
        uint64_t oa = 0, ob = align_up(la, 128);
        if (is_huff[i]) {  // v5: stream A, then the exception words, then the interleaved code words
            uint32_t h4[16];
            for (uint32_t b = 0; b < bpp; ++b) {
                const uint32_t hd = hdr[i * bpp + b];
                h4[b] = zhuff(hd) ? (hd & 0xffu) | (1u << 8) : hd;
            }
            HuffPiece hp;
            huff_piece(m.store + pc.off, pc.bytes, h4, hc, hp);
            for (uint32_t b = 0; b < nb; ++b) {
                const uint8_t* raw = m.store + pc.off + (uint64_t)b * kZBlock;
                const uint32_t hd = hdr[i * bpp + b], n = std::min(kZBlock, pc.bytes - b * kZBlock);
                const uint32_t kind = (hd >> 8) & 0xffu;
                if (kind == kZRaw) memcpy(out + oa, raw, n);
                else if (kind == kZHuff) {
                    const uint16_t* w = reinterpret_cast<const uint16_t*>(raw);
                    for (uint32_t j = 0; j < kZBlock / 2; ++j) out[oa + j] = (uint8_t)(((w[j] >> 8) & 0x80u) | (w[j] & 0x7fu));
                }
                oa += zblock_a(hd, n);
            }
            memcpy(out + ob, hp.exc.data(), 2 * hp.exc.size());
            ob += align_up(2 * hp.exc.size(), 16);
            memcpy(out + ob, hp.words.data(), 2 * hp.words.size());
            return;
        }
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
        if (!host_only)
            m->numa_node = bind_store(c, static_cast<uint8_t*>(p), m->store_alloc, gpu_numa_node(c->gpus[0].dev), m->store_node);
        m->store = static_cast<uint8_t*>(p);
    }
    // pack (zero padding everywhere; first touch happens here)
    const uint8_t* src = static_cast<const uint8_t*>(d->weights);
    // zero fill (first touch, 2-MiB chunks in parallel), then the tensors: row-major copies, and GEMM
    // weights re-laid in tile order one source row per task (16-bit stores; tiled_off keeps rows apart)
    const size_t kChunk = 2u << 20;
    parallel_for((m->store_alloc + kChunk - 1) / kChunk, [&](size_t i) {
        memset(m->store + i * kChunk, 0, std::min<uint64_t>(kChunk, m->store_alloc - i * kChunk));
    });
    for (auto& ti : m->tensors) {
        if (ti.owner < 0) continue;
        if (ti.layout == LAYOUT_ROWMAJOR) {
            memcpy(m->store + ti.st_off, src + ti.t.offset, ti.t.bytes);
        } else {
            const uint16_t* w = reinterpret_cast<const uint16_t*>(src + ti.t.offset);
            uint8_t* base = m->store + ti.st_off;
            parallel_for(ti.rows, [&](size_t n) {
                for (uint64_t k = 0; k < ti.cols; ++k)
                    *reinterpret_cast<uint16_t*>(base + tiled_off(n, k, ti.rows_pad)) = w[n * ti.cols + k];
            });
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
        s = build_link_code(c, *m, host_only);
        if (s != FSW_OK) {
            free_store(*m, host_only);
            return s;
        }
    }
    m->extent.assign(c->gpus.size(), -1);
    m->pextent.assign(c->gpus.size(), -1);
    m->pvalid.assign(c->gpus.size(), 0);
    m->complete.assign(c->gpus.size(), 0);
    m->last_use.assign(c->gpus.size(), 0);
    m->plans.resize(c->gpus.size());
    std::lock_guard<std::mutex> lk(c->mu);
    m->id = (uint32_t)c->models.size();
    *model_id = m->id;
    c->models.push_back(std::move(m));
    return FSW_OK;
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

