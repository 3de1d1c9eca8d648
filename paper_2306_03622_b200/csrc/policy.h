// policy.h — FaaSwap's node policies as pure host functions (no CUDA, no context state), shared by
// the runtime (placement and eviction inside fsw_invoke) and the request scheduler (sched.cpp),
// and exported through the C-ABI for tests (include/fsw.h, "Node policies").
#pragma once
#include <stdint.h>

#include <vector>

namespace fsw {

// RRC = (p·n − m) / (1 − p), from (m + RRC) / (n + RRC) = p.
double rrc(uint64_t n, uint64_t m, double p);

// sort by RRC (ascending; ties by index); the first k functions are high
// priority, k the largest integer with Σ_{j<=k} max(RRC_j, 0) <= α · Σ_i max(RRC_i, 0).
// Returns high[i] for every function.
std::vector<uint8_t> partition_high(const std::vector<double>& rrcs, double alpha);

// Algorithm 2: α·scalar (capped at 1) when the compliant ratio rose by more
// than |threshold|, α/scalar when it fell by more, else unchanged.
double alpha_config(double alpha, double last_ratio, double new_ratio, double scalar, double threshold);

// Algorithm 1.  Per GPU: available (idle), hosts (target model resident),
// neighbor (GPU sharing its PCIe switch, -1 = none), loading (0 none, 1 light model, 2 heavy model
// being swapped in from the host); link[g*n + s] = NVLink GB/s from s into g (empty = uniform).
// Ties: lowest GPU id, lowest (target, source) pair (SURVEY §8c reading 16).
struct Decision {
    int gpu = -1;   // -1: no GPU available (the request stays queued)
    int kind = 0;   // 0 run resident, 1 swap from the host, 2 swap from GPU `src`
    int src = -1;
};
Decision schedule(const std::vector<uint8_t>& available, const std::vector<uint8_t>& hosts,
                  const std::vector<int>& neighbor, const std::vector<uint8_t>& loading, const std::vector<float>& link);

// eviction order on one GPU.  Low-priority group first (light models, and heavy
// models with copies on >= 2 GPUs), then heavy sole copies; LRU inside each group; in-use models are
// never chosen.  Returns candidate indices in eviction order (the caller stops once it has room).
std::vector<uint32_t> eviction_order(const std::vector<uint8_t>& heavy, const std::vector<uint32_t>& copies,
                                     const std::vector<uint64_t>& last_use, const std::vector<uint8_t>& in_use);

// Heavy / light (a model is heavy when "model pipelining significantly slows down the
// inference", i.e. its swap is the bottleneck; used by Algorithm 1 and the eviction policy).
// Re-derived for B200: at batch 1 every model's swap is many times its
// sub-millisecond execution, so the paper's execution-relative test (cold / resident >
// 1.25) calls every model heavy.  With an SLO the test is against the request's latency budget instead:
//   slack = deadline − resident − queue_budget;  heavy  iff  slack <= 0  or  swap > theta · slack,
// swap = the swap's added latency (cold − resident).  Without an SLO (deadline <= 0) SPEC's rule:
// heavy iff resident + swap > 1.25 · resident (strict).  Monotone: more swap time never turns heavy light.
bool heavy_by_slo(double swap_ms, double resident_ms, double deadline_ms, double queue_budget_ms, double theta);

// Striped swap: deal units (pieces, or runs of coded pieces) in execution order to
// the sources so each unit is read by a source on the NUMA node holding its host pages: unit u goes to
// the sources whose node equals unit_node[u], round-robin among them (a counter per node); a unit whose
// node has no source (or is -1) goes round-robin over all sources.  Returns the source of every unit.
std::vector<uint32_t> stripe_deal(const std::vector<int>& unit_node, const std::vector<int>& src_node);

}  // namespace fsw
