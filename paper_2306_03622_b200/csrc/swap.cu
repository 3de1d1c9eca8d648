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

}  // namespace fsw
