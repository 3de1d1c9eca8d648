// swap.cu — K1, the swap engine: host store (pinned, mapped) -> HBM extent, SM-driven.
//
// PAPER.md:579-583 moves models "from host to GPU through PCIe" with copy-engine DMA from
// pinned memory; PAPER.md:588-590 overlaps "the transmission of subsequent layers with the
// computation of previous layers".  Here the transfer is done by SMs instead of the copy
// engine: persistent warps claim pieces in execution order from a global ticket, stream
// them with 128-bit non-allocating loads from the mapped host store and 128-bit stores to
// HBM, and publish each finished piece with a release-add of its byte count on the layer's
// ready counter.  Layer kernels acquire that counter (device.cuh: wait_ready_*).
// The copy-engine DMA engine (runtime.cpp) publishes readiness with stream memory writes instead.
#include "device.cuh"

namespace fsw {

template <int U>
__global__ void __launch_bounds__(512) k_swap(const uint8_t* __restrict__ host, DevDesc dst, const DevDesc* __restrict__ desc,
                                              const Piece* __restrict__ pieces, uint32_t n_pieces,
                                              uint32_t* __restrict__ ready, DevCtl* __restrict__ own, DevCtl* gate, int sys) {
    if (threadIdx.x == 0) atomicAdd(&gate->started, 1u);
    const DevDesc dd = desc ? *desc : dst;
    const uint32_t lane = threadIdx.x & 31u;
    for (;;) {
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(&own->ticket, 1u);
        p = __shfl_sync(0xffffffffu, p, 0);
        if (p >= n_pieces) break;
        if (p == 0 && lane == 0) own->t_first = globaltimer();
        const Piece pc = pieces[p];
        const uint4* src = reinterpret_cast<const uint4*>(host + pc.off);
        uint4* out = reinterpret_cast<uint4*>(weight_ptr(dd, pc.off));
        const uint32_t n16 = pc.bytes >> 4;
        uint32_t i = lane;
        for (; i + (U - 1) * 32 < n16; i += U * 32) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = ld_stream_v4(src + i + u * 32);
#pragma unroll
            for (int u = 0; u < U; ++u) st_v4(out + i + u * 32, v[u]);
        }
        for (; i < n16; i += 32) st_v4(out + i, ld_stream_v4(src + i));
        if (sys) {
            // peer stores over NVLink: order them at system scope before the remote release
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            __syncwarp();
            if (lane == 0) red_release_sys_add(&ready[pc.layer], pc.bytes);
        } else {
            __threadfence();  // this lane's stores performed at gpu scope
            __syncwarp();
            if (lane == 0) red_release_gpu_add(&ready[pc.layer], pc.bytes);
        }
        if (lane == 0) atomicMax(&own->t_last, (unsigned long long)globaltimer());
    }
}

void launch_swap(cudaStream_t s, int ctas, int threads, const uint8_t* host_mapped, DevDesc dst, const DevDesc* desc,
                 const Piece* pieces, uint32_t n_pieces, uint32_t* ready, DevCtl* own, DevCtl* gate, int sys) {
    k_swap<8><<<ctas, threads, 0, s>>>(host_mapped, dst, desc, pieces, n_pieces, ready, own, gate, sys);
}

// ---- exponent-coded link format (kernels.h) -----------------------------------
// Loads of coded bytes: from the mapped host store they are read once, non-allocating; from the
// staging buffer (written by the copy engine, published by a fenced stream write) they are
// L2-coherent .cg loads ordered after the acquire of the group counter.
template <bool STAGE>
__device__ __forceinline__ uint4 zld4(const uint8_t* p) {
    uint4 r;
    if (STAGE)
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
    else
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
template <bool STAGE>
__device__ __forceinline__ uint2 zld2(const uint8_t* p) {
    uint2 r;
    if (STAGE)
        asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p) : "memory");
    else
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
template <bool STAGE>
__device__ __forceinline__ uint32_t zld16(const uint8_t* p) {
    uint16_t r;
    if (STAGE) asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(r) : "l"(p) : "memory");
    else asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
}
template <bool STAGE>
__device__ __forceinline__ uint32_t zld32(const uint8_t* p) {
    uint32_t r;
    if (STAGE) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    else asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// Lane l of a coded block: words 16l .. 16l+15 from its 16 stored bytes, its 16 bits of each code
// plane (plane p in the low half of pl[p]) and the block's base exponent h.
__device__ __forceinline__ void zdecode16(const uint4 sm, const uint32_t (&pl)[4], uint32_t h, uint4& o0, uint4& o1) {
    const uint32_t s[4] = {sm.x, sm.y, sm.z, sm.w};
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        uint32_t w2 = 0;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int i = 2 * k + half;  // word i of the lane's 16
            const uint32_t m = (s[i >> 2] >> (8 * (i & 3))) & 0xffu;
            const uint32_t c = ((pl[0] >> i) & 1u) | (((pl[1] >> i) & 1u) << 1) | (((pl[2] >> i) & 1u) << 2) |
                               (((pl[3] >> i) & 1u) << 3);
            w2 |= (((m & 0x80u) << 8) | ((h - c) << 7) | (m & 0x7fu)) << (16 * half);
        }
        o[k] = w2;
    }
    o0 = make_uint4(o[0], o[1], o[2], o[3]);
    o1 = make_uint4(o[4], o[5], o[6], o[7]);
}

// 32-bit word `wi` (0..3) of lane `src`'s uint4 v, for every lane (four shuffles and a select).
__device__ __forceinline__ uint32_t shfl_word(const uint4& v, uint32_t src, uint32_t wi) {
    const uint32_t x = __shfl_sync(0xffffffffu, v.x, src), y = __shfl_sync(0xffffffffu, v.y, src);
    const uint32_t z = __shfl_sync(0xffffffffu, v.z, src), w = __shfl_sync(0xffffffffu, v.w, src);
    return wi == 0 ? x : wi == 1 ? y : wi == 2 ? z : w;
}

__device__ __forceinline__ void wait_geq(const uint32_t* p, uint32_t v, DevCtl* ctl) {
    if (ld_acquire_gpu(p) >= v) return;
    const uint64_t t0 = globaltimer();
    uint32_t ns = 64;
    while (ld_acquire_gpu(p) < v) {
        __nanosleep(ns);
        if (ns < 512) ns <<= 1;
        if (globaltimer() - t0 > kWatchdogNs) {
            atomicExch(&ctl->err, 1);
            atomicExch(&ctl->err_layer, -1);
            return;
        }
    }
}

// Persistent warps claim coded pieces in the table's order (execution order), decode U blocks at a
// time (all loads of the U blocks issued before any store, so a warp keeps ~3 KB of host reads in
// flight), store 128-bit words into the extent, patch the exceptions and release the piece's raw bytes on its layer's
// counter — the same readiness protocol as k_swap, so layer kernels cannot tell the engines apart.
template <bool STAGE, int U>
__global__ void __maxnreg__(64) k_swapz(const uint8_t* __restrict__ src, uint64_t src_base, DevDesc dst,
                                               const DevDesc* __restrict__ desc, const ZPiece* __restrict__ pieces,
                                               uint32_t n_pieces, uint32_t* __restrict__ ready, DevCtl* __restrict__ own,
                                               DevCtl* gate, int sys, const uint32_t* progress) {
    if (threadIdx.x == 0) atomicAdd(&gate->started, 1u);
    const DevDesc dd = desc ? *desc : dst;
    const uint32_t lane = threadIdx.x & 31u;
    for (;;) {
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(&own->ticket, 1u);
        p = __shfl_sync(0xffffffffu, p, 0);
        if (p >= n_pieces) break;
        if (p == 0 && lane == 0) own->t_first = globaltimer();
        const ZPiece pc = pieces[p];
        if (STAGE) {
            if (lane == 0) wait_geq(progress, pc.grp + 1, own);
            __syncwarp();
        }
        const uint8_t* cp = src + (pc.coff - src_base);
        uint8_t* out = weight_ptr(dd, pc.off);
        const uint32_t nb = (pc.bytes + kZBlock - 1) / kZBlock;  // <= 16
        // header (from the device piece table) and coded offset of block `lane` (exclusive scan)
        const uint32_t hd = lane < nb ? __ldg(&pieces[p].hdr[lane]) : 0u;
        const uint32_t sz = lane < nb ? zblock_bytes(hd, min(kZBlock, pc.bytes - lane * kZBlock)) : 0u;
        uint32_t incl = sz;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += t;
        }
        const uint32_t boff = incl - sz;
        for (uint32_t b0 = 0; b0 < nb; b0 += U) {
            // all loads of U blocks first (memory-level parallelism over the host link), then stores
            uint4 q0[U], q1[U];
            uint32_t hh[U], ob[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t b = b0 + u;
                hh[u] = __shfl_sync(0xffffffffu, hd, b & 31u);
                ob[u] = __shfl_sync(0xffffffffu, boff, b & 31u);
                const uint32_t kind = (hh[u] >> 8) & 0xffu, n = hh[u] >> 16;
                const uint8_t* bp = cp + ob[u];
                if (b >= nb || kind == kZZero) continue;
                const bool full = b * kZBlock + kZBlock <= pc.bytes;
                if (kind == kZRaw) {
                    if (full) {
                        q0[u] = zld4<STAGE>(bp + lane * 16u);
                        q1[u] = zld4<STAGE>(bp + 512u + lane * 16u);
                    }
                    continue;
                }
                // stored bytes, then the planes + exceptions region as whole 16-B chunks (every load of
                // the block is a 16-B-per-lane load: whole 128-B host read requests)
                q0[u] = zld4<STAGE>(bp + lane * 16u);
                const uint32_t rb = 64u * kind + 4u * n;
                if (lane * 16u < rb) q1[u] = zld4<STAGE>(bp + 512u + lane * 16u);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t b = b0 + u;
                if (b >= nb) break;
                const uint32_t kind = (hh[u] >> 8) & 0xffu, n = hh[u] >> 16;
                uint8_t* bo = out + (uint64_t)b * kZBlock;
                uint4* o4 = reinterpret_cast<uint4*>(bo);
                if (kind == kZZero) {
                    st_v4(o4 + 2 * lane, make_uint4(0u, 0u, 0u, 0u));
                    st_v4(o4 + 2 * lane + 1, make_uint4(0u, 0u, 0u, 0u));
                } else if (kind == kZRaw) {
                    if (b * kZBlock + kZBlock <= pc.bytes) {
                        st_v4(o4 + lane, q0[u]);
                        st_v4(o4 + 32 + lane, q1[u]);
                    } else {  // the piece's partial tail (< 1 KiB, end of a layer region)
                        const uint32_t n16 = (pc.bytes - b * kZBlock) >> 4;
                        for (uint32_t i = lane; i < n16; i += 32) st_v4(o4 + i, zld4<STAGE>(cp + ob[u] + i * 16u));
                    }
                } else {
                    // lane l's 16 code bits of plane p: bytes 64p + 2l .. +1 of the region, i.e. half
                    // (l & 1) of word ((l & 7) >> 1) of chunk 4p + (l >> 3)
                    uint32_t pl[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (uint32_t pp = 0; pp < 4; ++pp)
                        if (pp < kind)
                            pl[pp] = (shfl_word(q1[u], 4u * pp + (lane >> 3), (lane & 7u) >> 1) >> (16u * (lane & 1u))) & 0xffffu;
                    // exception j (lane j < 32): word (j & 3) of chunk 4b + (j >> 2)
                    const uint32_t ex = n ? shfl_word(q1[u], (4u * kind + (lane >> 2)) & 31u, lane & 3u) : 0u;
                    uint4 o0, o1;
                    zdecode16(q0[u], pl, hh[u] & 0xffu, o0, o1);
                    st_v4(o4 + 2 * lane, o0);
                    st_v4(o4 + 2 * lane + 1, o1);
                    if (n) {
                        // exceptions overwrite their words after the warp's block stores (__syncwarp
                        // orders the warp's memory operations); those past the loaded 512-B region or
                        // past the 32nd are read directly (rare: the chooser keeps n small)
                        __syncwarp();
                        uint16_t* o16 = reinterpret_cast<uint16_t*>(bo);
                        const uint32_t in_reg = min(n, min(32u, (512u - 64u * kind) / 4u));
                        if (lane < in_reg) o16[ex & 0xffffu] = (uint16_t)(ex >> 16);
                        for (uint32_t j = in_reg + lane; j < n; j += 32) {
                            const uint32_t e = zld32<STAGE>(cp + ob[u] + 512u + 64u * kind + j * 4u);
                            o16[e & 0xffffu] = (uint16_t)(e >> 16);
                        }
                    }
                }
            }
        }
        if (sys) {
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            __syncwarp();
            if (lane == 0) red_release_sys_add(&ready[pc.layer], pc.bytes);
        } else {
            __threadfence();
            __syncwarp();
            if (lane == 0) red_release_gpu_add(&ready[pc.layer], pc.bytes);
        }
        if (lane == 0) atomicMax(&own->t_last, (unsigned long long)globaltimer());
    }
}

void launch_swapz(cudaStream_t s, int ctas, int threads, const uint8_t* src, uint64_t src_base, DevDesc dst,
                  const DevDesc* desc, const ZPiece* pieces, uint32_t n_pieces, uint32_t* ready, DevCtl* own,
                  DevCtl* gate, int sys, int stage, const uint32_t* progress) {
    if (stage)
        k_swapz<true, 2><<<ctas, threads, 0, s>>>(src, src_base, dst, desc, pieces, n_pieces, ready, own, gate, sys, progress);
    else
        k_swapz<false, 3><<<ctas, threads, 0, s>>>(src, src_base, dst, desc, pieces, n_pieces, ready, own, gate, sys, progress);
}

// Gate: the first node of the layer stream.  Holds the layer kernels back until every swap
// CTA is resident, so spinning layer CTAs can never occupy the SMs the swap needs
// (no deadlock whatever the block scheduler does).  One thread; costs one launch.
__global__ void k_gate(DevCtl* ctl, uint32_t expected) {
    const volatile uint32_t* st = &ctl->started;
    const uint64_t t0 = globaltimer();
    while (*st < expected) {
        __nanosleep(256);
        if (globaltimer() - t0 > kWatchdogNs) {
            atomicExch(&ctl->err, 2);
            break;
        }
    }
}

void launch_gate(cudaStream_t s, DevCtl* ctl, uint32_t expected) { k_gate<<<1, 1, 0, s>>>(ctl, expected); }

// Last node of every invoke graph: stamp the end, then write the output slot and the control
// block straight into mapped pinned host memory (zero-copy stores over PCIe), so the graph ends
// without device-to-host copy nodes; the host reads them after the graph's completion event.
__global__ void k_finish(DevCtl* ctl, const uint8_t* __restrict__ out, uint64_t bytes, uint8_t* host_out, DevCtl* host_ctl) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->t_end = globaltimer();
        *host_ctl = *ctl;
    }
    const uint64_t n16 = bytes >> 4, stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (uint64_t i = t0; i < n16; i += stride)
        reinterpret_cast<uint4*>(host_out)[i] = reinterpret_cast<const uint4*>(out)[i];
    for (uint64_t i = (n16 << 4) + t0; i < bytes; i += stride) host_out[i] = out[i];
}
void launch_finish(cudaStream_t s, DevCtl* ctl, const uint8_t* out, uint64_t bytes, uint8_t* host_out, DevCtl* host_ctl) {
    const uint64_t want = (bytes + 4095) / 4096;
    k_finish<<<(unsigned)(want < 1 ? 1 : want > 148 ? 148 : want), 256, 0, s>>>(ctl, out, bytes, host_out, host_ctl);
}

// No carveout preference for the swap kernels (measured: a max-shared carveout on every kernel made
// the SM engine slower, e.g. BERT-base 4.30 -> 4.76 ms, and did not shorten the layer kernels).
void init_swap_attrs() {}

}  // namespace fsw
