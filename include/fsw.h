/*
 * fsw.h — C-ABI of libfsw: FaaSwap-style swap-in-and-execute of an inference model on B200.
 *
 * Paper: "FaaSwap: SLO-Aware, GPU-Efficient Serverless Inference via Model Swapping"
 * (arXiv 2306.03622).  Citations "PAPER.md:n" are lines of the paper's LaTeX source.
 *
 * The problem statement the calls follow:
 *   - functions publish models; requests invoke them
 *   - models are kept in host memory and bound to a GPU of the pool on each request
 *     ("late binding")               -> fsw_register_model / fsw_invoke
 *   - transfer of later layers overlaps computation of earlier layers, layer by layer
 *     ("Model swapping and pipeline execution") -> fsw_invoke (cold path)
 *   - a host copy is always kept; eviction only invalidates the GPU region
 *     ("Model eviction")                      -> fsw_evict
 *   - all GPU memory is pre-allocated and managed as blocks by the server
 *     ("Memory allocation and block management") -> fsw_pool_stats
 *   - one request per GPU at a time    -> invoke concurrency rule
 *   - no detailed model knowledge is needed; the paper records the
 *     parameter access pattern of the first run.  Here the access
 *     pattern is given explicitly as the layer table; its order IS the swap order.
 *
 * Conventions (all calls):
 *   - every function returns fsw_status; no C++ exception crosses the ABI;
 *     fsw_last_error() returns a thread-local message for the last failure.
 *   - all pointers are HOST pointers; device memory is library-owned and never exported
 *     (except the debug read-back copies below, which copy into caller host buffers).
 *   - sizes are bytes unless noted.  Failed calls leave no partial state.
 */
#ifndef FSW_H
#define FSW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FSW_OK = 0,
    FSW_EINVAL = 1,    /* malformed table, bad argument, output buffer too small          */
    FSW_ENOTFOUND = 2, /* unknown model id                                                 */
    FSW_ENOMEM = 3,    /* pool too small even after evicting every idle model; host OOM    */
    FSW_EBUSY = 4,     /* evict / unregister while an invoke of that model is in flight    */
    FSW_ESTATE = 5,    /* evict of a model not resident on that GPU                        */
    FSW_ECUDA = 6,     /* CUDA runtime failure (includes: no CUDA device)                  */
    FSW_ETIMEOUT = 7,  /* a layer kernel's ready-flag spin hit the watchdog                */
    FSW_ETOPO = 8      /* striping requested over GPUs that cannot reach the target        */
} fsw_status;

/* ---------------------------------------------------------------------------------------
 * Context
 * ------------------------------------------------------------------------------------- */
#define FSW_NO_OVERLAP   0x1u /* swap completes before the first layer kernel starts
                                 ("Non-pipeline" column of PAPER.md Table 4; also needed under
                                 ncu / compute-sanitizer, which serialise kernels)             */
#define FSW_DMA_BASELINE 0x2u /* the paper's transfer as a baseline: copy-engine DMA in ~2-MB
                                 groups, one copy stream; overrides the
                                 engine / group / stream settings                                */
#define FSW_HOST_WC      0x4u /* back host stores with write-combined pinned pages            */
#define FSW_NO_PEER_SWAP 0x10u /* never swap from another GPU's resident copy (Alg. 1 case 2 off)  */
#define FSW_HOST_ONLY    0x8u /* no GPU: registration / host-store / allocator logic only (tests);
                                 invoke returns FSW_ECUDA                                       */
#define FSW_TRACE        0x40u /* device timeline (also FSW_TRACE=1 in the environment at fsw_init): every
                                 kernel records per layer its first CTA entry, last weight-wait completion
                                 and last CTA exit, and the swap kernels the first / last release of the
                                 layer's pieces (%globaltimer ns); read with fsw_debug_trace_read.  A
                                 few atomics per CTA; off in the bench.                          */
#define FSW_DEBUG_POISON 0x20u /* test mode (also set by the environment variable FSW_DEBUG_POISON=1 at
                                 fsw_init): before every cold invoke, fill the extents the swap will
                                 write (prefix + suffix) and the DMAZ staging buffer with a per-invoke
                                 32-bit pattern, and before every invoke the model's activation
                                 workspace, so a byte the swap (or a layer kernel) fails to write can
                                 never pass as the stale correct byte of an earlier invoke.  Costs one
                                 HBM fill per invoke; off in the bench.                         */

typedef struct {
    uint32_t n_gpus;                  /* GPUs in the pool; 0 = all visible devices           */
    const int32_t* gpu_ids;           /* n_gpus CUDA device ordinals, or NULL = 0..n_gpus-1   */
    uint64_t pool_bytes_per_gpu;      /* weight pool per GPU, pre-allocated at init; 0 = 64 GiB
                                         (capped at 60% of free memory)                       */
    uint64_t workspace_bytes_per_gpu; /* activation workspace per GPU; 0 = 512 MiB            */
    uint32_t copy_ctas;               /* CTAs of the SM swap kernel; 0 = 16 (the link-coded engines'
                                         decode kernels use at least 32 (SMZ) / 48 (DMAZ))      */
    uint32_t copy_threads;            /* threads per swap CTA (multiple of 32); 0 = 256       */
    uint64_t chunk_bytes;             /* swap piece size (the paper's "group size",
                                         PAPER.md:600-604) of the SM engine; multiple of 256;
                                         0 = 16 KiB (small pieces keep the swap in layer order) */
    uint64_t stripe_min_bytes;        /* policy: stripe a cold host swap over every pool GPU with
                                         peer access to the target when the store has at least
                                         this many bytes; 0 = 256 MiB; UINT64_MAX = never         */
    uint32_t flags;                   /* FSW_NO_OVERLAP | FSW_DMA_BASELINE | FSW_HOST_WC       */
    uint32_t engine;                  /* FSW_ENGINE_*; 0 = AUTO                                */
    uint64_t dma_min_bytes;           /* AUTO picks DMA for models with at least this many store
                                         bytes, SM below; 0 = 32 MiB                           */
    uint64_t dma_group_bytes;         /* DMA / DMAZ engines: target bytes per copy group (whole layers
                                         are merged up to it, larger layers split, groups taper
                                         towards the end of the store); 0 = 64 MiB             */
    uint32_t dma_streams;             /* DMA / DMAZ engines: concurrent copy streams (1..4); 0 = 1
                                         (measured: more streams contend for the one host link)  */
    const int32_t* pcie_neighbor;     /* n_gpus entries: the pool GPU sharing each GPU's PCIe
                                         switch, −1 = none (Algorithm 1's "neighbor"); NULL = none
                                         (HGX B200: one switch per GPU)                          */
    uint64_t dmaz_min_bytes;          /* AUTO picks DMAZ for link-coded models with at least this
                                         many store bytes, SMZ below; 0 = 128 MiB (measured: SMZ
                                         wins on ResNet-50's 51 MB, DMAZ on BERT-base's 219 MB)  */
} fsw_config;

/* Swap engines.  All move the host store into the extent in execution order and
 * publish readiness in device memory that the layer kernels acquire:
 *   SM : persistent CTAs stream pieces with 128-bit loads from mapped host memory; one release-add
 *        of the piece's bytes on its layer's counter per piece (fine-grained, no per-copy setup);
 *   DMA: copy-engine cudaMemcpyAsync of layer-aligned groups on `dma_streams` streams; after each
 *        group a stream memory write (no SM) bumps that stream's group counter.               */
enum { FSW_ENGINE_AUTO = 0, FSW_ENGINE_SM = 1, FSW_ENGINE_DMA = 2, FSW_ENGINE_SMZ = 3, FSW_ENGINE_DMAZ = 4, FSW_ENGINE_DMAZT = 5 };
/* Link-coded engines (models registered with FSW_REG_LINK_CODE).  The host link carries
 * the model's exponent-coded store (lossless; on the synthetic weights 0.68 of the bytes with the per-block codes, 0.66 with
 * the entropy-coded pieces of stores >= 32 MiB, see fsw_debug_coded_code) and a kernel decodes it into the
 * extent, releasing each decoded piece's bytes on its layer's counter (the SM protocol):
 *   SMZ : persistent CTAs stream coded pieces zero-copy from the mapped coded store with TMA bulk copies
 *         into a shared-memory ring and decode them from there;
 *   DMAZ: copy-engine DMA of layer-ordered, tapered groups of coded pieces into a device staging
 *         buffer, each followed by a stream write of the group count; persistent decode CTAs wait for
 *         their piece's group, then decode from HBM.
 *   DMAZT: DMAZ for the body of the coded store and SMZ for its tail (the last 7 MB of coded bytes, at most a
 *         quarter; FSW_DMAZT_TAIL_MB overrides): the copy engine's larger PCIe reads for most of the bytes, and
 *         no copy-group latency at the end, where a group's decode and the last layers' compute would trail it.
 *         The tail's CTAs are resident from the start (the gate counts them) and begin reading the host
 *         store once the last body group has landed, so the link carries one transfer at a time.
 * AUTO picks, for link-coded models, DMAZT at >= dmaz_min_bytes, SMZ below; DMA / SM (by dma_min_bytes)
 * otherwise. */

typedef struct fsw_ctx fsw_ctx; /* opaque; one per process */

/* Create the per-GPU runtime: one shared CUDA context per GPU with all kernels preloaded
 * (PAPER.md:551-555), the pre-allocated weight pool, workspace and streams.
 * cfg may be NULL (defaults).  Returns FSW_ECUDA when no CUDA device is present, unless
 * cfg->flags has FSW_HOST_ONLY (then no GPU is touched and n_gpus is 0).                   */
fsw_status fsw_init(const fsw_config* cfg, fsw_ctx** out);
void fsw_shutdown(fsw_ctx* ctx);
const char* fsw_last_error(void);
const char* fsw_version(void);

/* ---------------------------------------------------------------------------------------
 * Model description (layer table)
 * ------------------------------------------------------------------------------------- */
enum { FSW_DT_BF16 = 0, FSW_DT_F32 = 1, FSW_DT_I32 = 2 };

enum {
    FSW_OP_EMBED = 1,     /* out[t] = Σ_j table_j[row_j(t)]                  refs: tables
                             attr[0] = n tables, attr[1+j] = FSW_RULE_* of table j          */
    FSW_OP_LAYERNORM = 2, /* out = (x−μ)/√(σ²+eps)·γ + β over the last dim    refs: γ, β
                             attr[0] = eps as IEEE float bits                               */
    FSW_OP_LINEAR = 3,    /* out[i] = act(x[r0+i]·Wᵀ + b + in1[i]),  W [N][K] refs: W [, b]
                             attr[0] = FSW_ACT_*, attr[1] = r0, attr[2] = rows (0 = all)    */
    FSW_OP_ATTENTION = 4, /* in0 row t = [q | k | v] (H·dh each); out = softmax(qkᵀ/√dh)·v
                             attr[0] = H, attr[1] = dh, attr[2] = causal                     */
    FSW_OP_CONV2D = 5,    /* NHWC, W [Cout][R][S][Cin];  out = act(conv + b + in1)  refs: W, b
                             attr[0] = FSW_ACT_*, attr[1] = stride, attr[2] = pad            */
    FSW_OP_MAXPOOL = 6,   /* attr[0] = k, attr[1] = stride, attr[2] = pad (pad = −∞)         */
    FSW_OP_AVGPOOL = 7    /* global average over H·W: [H][W][C] -> [1][C]                    */
};
enum { FSW_ACT_NONE = 0, FSW_ACT_RELU = 1, FSW_ACT_GELU_ERF = 2, FSW_ACT_GELU_TANH = 3, FSW_ACT_TANH = 4 };
enum { FSW_RULE_IDS = 0, FSW_RULE_POSITION = 1, FSW_RULE_ZERO = 2 };

/* A weight tensor inside the caller's blob: row-major, `bytes` = numel · sizeof(dtype),
 * offset 16-B aligned.  Tensors may be referenced by several layers (tied weights).       */
typedef struct { uint64_t offset, bytes; uint32_t dtype, rank; uint32_t shape[4]; } fsw_tensor;
/* An activation slot (a named buffer in the per-GPU workspace); dtype = storage dtype.   */
typedef struct { uint32_t dtype, rank; uint32_t shape[4]; } fsw_slot;
/* A layer: op, its weight tensors refs[first_ref .. first_ref+n_refs), activation slots
 * in0 / in1 (−1 = none) and out (must differ from in0 and in1).                           */
typedef struct { uint32_t op, first_ref, n_refs; int32_t in0, in1, out; int32_t attr[8]; } fsw_layer;

#define FSW_REG_ADOPT 0x1u /* reserved: pin the caller's buffer in place (not yet supported) */
#define FSW_REG_LINK_CODE 0x2u /* also build the exponent-coded copy of the store (pinned, mapped) that
                                  the SMZ / DMAZ engines move over the host link (format
                                  at fsw_coded_piece below).  Lossless: the extent receives the store's
                                  bytes bit-exactly.  Costs ~0.66-0.68x the store in extra host memory;
                                  entropy-coded pieces (format v5) are built for stores >= 32 MiB
                                  (environment FSW_LINK_HUFF=0 / 1: never / always).             */

typedef struct {
    const char* name;
    const void* weights; uint64_t weight_bytes;        /* caller-owned; copied (FSW_REG_COPY)  */
    const fsw_tensor* tensors; uint32_t n_tensors;
    const uint32_t* refs; uint32_t n_refs;
    const fsw_slot* slots; uint32_t n_slots;
    const fsw_layer* layers; uint32_t n_layers;        /* execution order == swap order        */
    int32_t input_slot, output_slot;
    uint32_t flags;
} fsw_model_desc;

/* Validate the table, lay the weights out in the library's pinned, mapped, THP-backed host store
 * (pages bound to pool GPU 0's NUMA node before first touch) in execution order (each layer's
 * tensors contiguous, 256-B aligned; GEMM weights re-laid in the tensor-core tile order described
 * in DESIGN.md §4), and register it for zero-copy device access.  Untimed, one-time (the paper's model repository).
 * The caller may free `weights` on return.  Errors: EINVAL (bad table), ENOMEM, ECUDA.   */
fsw_status fsw_register_model(fsw_ctx* ctx, const fsw_model_desc* desc, uint32_t* model_id);
/* EBUSY while an invoke of the model is in flight; evicts it from every GPU first.        */
fsw_status fsw_unregister_model(fsw_ctx* ctx, uint32_t model_id);

typedef struct {
    uint64_t store_bytes;      /* host-store bytes (= bytes moved by one cold swap)         */
    uint64_t algorithmic_bytes;/* Σ tensor bytes (excludes alignment / tile padding)        */
    uint32_t n_layers, n_tensors, n_gemm_layers;
    uint64_t input_bytes, output_bytes;
    uint32_t output_dtype;
    uint64_t coded_bytes;      /* bytes of the exponent-coded store (FSW_REG_LINK_CODE), else 0 */
    int32_t numa_node;         /* NUMA node the host store's pages prefer (that of pool GPU 0's PCIe
                                  root, from sysfs; bound before first touch), −1 if unknown / none,
                                  −2 when the pool spans several nodes: 2-MiB chunks are then bound
                                  round-robin across the pool's nodes and striped swaps deal each
                                  chunk's data to a source on its node (fsw_policy_stripe_deal)  */
} fsw_model_info;
fsw_status fsw_model_info_get(fsw_ctx* ctx, uint32_t model_id, fsw_model_info* out);

/* Where tensor `tensor` sits in the host store (and in HBM when resident, same offsets).
 * layout 0 = row-major copy of the caller bytes; 1 = tensor-core tiles
 * with rows padded to rows_pad and columns (K) padded to cols_pad.                      */
typedef struct { uint64_t offset, bytes; uint32_t layout, rows, cols, rows_pad, cols_pad, owner_layer; } fsw_store_tensor;
fsw_status fsw_store_tensor_get(fsw_ctx* ctx, uint32_t model_id, uint32_t tensor, fsw_store_tensor* out);

/* ---------------------------------------------------------------------------------------
 * Invoke
 * ------------------------------------------------------------------------------------- */
enum { FSW_SWAP_RESIDENT = 0, FSW_SWAP_HOST = 1, FSW_SWAP_PEER = 2, FSW_SWAP_STRIPED = 3 };

typedef struct {
    double total_ms;        /* host wall clock: call entry -> output in the caller buffer   */
    double device_ms;       /* CUDA events around the invoke graph on the launching stream  */
    double swap_ms;         /* CUDA events around the swap kernel on its own stream         */
    double swap_span_ms;    /* SM: %globaltimer first piece claimed -> last released; DMA: = swap_ms */
    double compute_tail_ms; /* last weight byte landed -> last layer finished (SM: %globaltimer;
                               DMA: CUDA events, includes the output D2H)                     */
    uint64_t bytes_swapped;
    double link_gbps;       /* bytes_swapped / swap_ms                                       */
    int32_t gpu;
    uint32_t swap_kind;     /* FSW_SWAP_*                                                     */
    uint32_t n_sources;
    uint32_t n_kernels;     /* kernels launched by this invoke (incl. the swap kernel)       */
    uint32_t engine;        /* FSW_ENGINE_SM / FSW_ENGINE_DMA for a cold invoke, else 0        */
    uint32_t n_copies;      /* swap pieces (SM) or copy-engine groups (DMA) of this invoke      */
    uint64_t wire_bytes;    /* bytes that crossed the host / peer link (= bytes_swapped, except the
                               link-coded engines, which move coded bytes)                      */
    double host_setup_ms;   /* host: call entry -> graph launched (placement, extent, staging)   */
    double host_wait_ms;    /* host: graph launched -> output in the caller buffer              */
} fsw_invoke_stats;

/* Run one request: pick a GPU (resident and idle first, then the lowest idle id,
 * PAPER.md:845-850 / SPEC tie-break), allocate a pool extent (evicting LRU idle models),
 * swap in pipelined with execution (cold) or run resident (warm), return the output.
 * input_bytes must equal the input slot size; output_cap ≥ the output slot size.
 * Blocks while every GPU is busy (one request per GPU).                     */
fsw_status fsw_invoke(fsw_ctx* ctx, uint32_t model_id, const void* input, uint64_t input_bytes,
                      void* output, uint64_t output_cap, fsw_invoke_stats* stats /* nullable */);

enum { FSW_ORDER_EXEC = 0, FSW_ORDER_REVERSE = 1, FSW_ORDER_RANDOM = 2 };
typedef struct {
    int32_t gpu;          /* −1 = scheduler's choice                                           */
    uint32_t n_stripe_src;/* striped swap: 0 = ctx policy (stripe_min_bytes);
                             else the number of entries of stripe_src                          */
    uint64_t chunk_bytes; /* 0 = ctx default                                                   */
    uint32_t order;       /* FSW_ORDER_* : order in which swap pieces are claimed (tests)      */
    uint32_t order_seed;
    uint32_t copy_ctas;   /* 0 = ctx default                                                   */
    uint32_t flags;       /* FSW_NO_OVERLAP | FSW_DMA_BASELINE, OR-ed with the ctx flags       */
    uint32_t engine;      /* FSW_ENGINE_*; 0 = ctx default                                     */
    uint64_t dma_group_bytes; /* 0 = ctx default                                               */
    uint32_t dma_streams;     /* 0 = ctx default                                               */
    const int32_t* stripe_src; /* n_stripe_src pool GPU indices that each load a round-robin share of
                             every layer's pieces from the host store over their own host link and
                             store it into the target's extent (peer stores over NVLink for remote
                             sources).  Duplicates are allowed: every entry runs its own swap kernel
                             (single-GPU tests list the target several times).  A single entry equal
                             to the target means "no striping".  ETOPO if a source has no peer
                             access to the target.                                             */
    uint32_t peer_src;    /* GPU->GPU swap (Alg. 1 case 2): 0 = policy (a cold
                             invoke copies from another pool GPU that holds the model, over
                             NVLink, before falling back to the host link; FSW_NO_PEER_SWAP turns
                             it off); k > 0 = copy from pool GPU k-1 (ESTATE if not resident there,
                             ETOPO without peer access)                                        */
} fsw_invoke_opts;
fsw_status fsw_invoke_ex(fsw_ctx* ctx, uint32_t model_id, const fsw_invoke_opts* opts,
                         const void* input, uint64_t input_bytes, void* output, uint64_t output_cap,
                         fsw_invoke_stats* stats);

/* Invalidate the model's extent on `gpu` (−1 = every GPU).  No device→host copy
 * (PAPER.md:611-614).  ESTATE if not resident there, EBUSY if an invoke is in flight.    */
fsw_status fsw_evict(fsw_ctx* ctx, uint32_t model_id, int32_t gpu);
#define FSW_EVICT_KEEP_PREFIX 0x1u /* invalidate only the part beyond the model's cached prefix     */
fsw_status fsw_evict_ex(fsw_ctx* ctx, uint32_t model_id, int32_t gpu, uint32_t flags);

/* Partial-parameter caching (future work in PAPER.md:1209-1211): keep the
 * first `bytes` of the host store (rounded down to a layer boundary, leaving at least one layer to
 * swap) resident in a separate pool extent that survives the pool's evictions (and
 * fsw_evict_ex(FSW_EVICT_KEEP_PREFIX)), so a cold invoke swaps only the rest: its layer kernels
 * for cached layers start without waiting.  0 = no caching.  ESTATE while the model is resident
 * anywhere (evict it first).  *actual = the prefix bytes chosen.                            */
fsw_status fsw_model_set_cache_prefix(fsw_ctx* ctx, uint32_t model_id, uint64_t bytes, uint64_t* actual);

typedef struct {
    uint64_t capacity, used, largest_free;
    uint32_t n_resident, n_extents;
    uint64_t n_evictions, bytes_swapped_total, n_invokes_cold, n_invokes_warm;
    uint64_t prefix_bytes_cached;     /* valid cached prefixes held on this GPU (NEXT #4)     */
    uint64_t n_evictions_heavy;       /* of n_evictions: models in the heavy class when evicted */
} fsw_pool_stats;
fsw_status fsw_pool_stats_get(fsw_ctx* ctx, int32_t gpu, fsw_pool_stats* out);
fsw_status fsw_n_gpus(fsw_ctx* ctx, uint32_t* n);

/* Fault injection (tests: negative controls of the bit-exact and litmus checks).  kind:
 *   FSW_FAULT_NONE       : clear;
 *   FSW_FAULT_DROP_PIECE : the swap kernels (SM, SMZ, DMAZ decode; every source of a striped swap)
 *                          skip the stores of the piece they claim as number `index` but still
 *                          release its bytes on the layer counter;
 *   FSW_FAULT_DROP_GROUP : the copy-engine engines (DMA, DMAZ) skip copy group `index` but still
 *                          publish its completion.
 * Process-wide on the device side (every pool GPU); cached invoke graphs are rebuilt.  EINVAL on
 * an unknown kind.                                                                            */
enum { FSW_FAULT_NONE = 0, FSW_FAULT_DROP_PIECE = 1, FSW_FAULT_DROP_GROUP = 2 };
fsw_status fsw_debug_set_fault(fsw_ctx* ctx, uint32_t kind, uint32_t index);

/* Readiness-protocol litmus test (DESIGN.md §5 "Memory ordering"; the correctness claim of
 * PAPER.md:519 under the layer overlap of PAPER.md:588-590).  Runs `iters` iterations on pool GPU
 * `gpu` of: poison a scratch extent (and the DMAZ staging buffer), reset the counters, then run the
 * swap engine `engine` (FSW_ENGINE_SM / DMA / SMZ / DMAZ; `ctas` swap CTAs for the kernel engines)
 * as the producer of model `model_id`'s store into that extent, CONCURRENTLY with `ctas` consumer
 * CTAs that take the layers round-robin and, per layer, do exactly what a layer kernel does before
 * reading weights — one thread acquires the layer's counter(s) (wait_ready), executes
 * fence.proxy.async.global and issues cp.async.bulk copies of the layer region into shared memory —
 * and compare every 16-byte word with the store.  *bad_words = words that differed (summed over all
 * iterations), *checked_bytes = bytes compared (= iters x store bytes when nothing timed out).
 * The model must have no invoke in flight (EBUSY); ENOMEM if the pool has no room for the scratch
 * extent; ETIMEOUT if a consumer's spin hit the watchdog; EINVAL for a bad engine / ctas (1..1024)
 * or a coded engine on a model that is not link-coded.                                          */
fsw_status fsw_debug_litmus(fsw_ctx* ctx, uint32_t model_id, int32_t gpu, uint32_t engine, uint32_t ctas, uint32_t iters,
                            uint64_t* bad_words, uint64_t* checked_bytes);

/* The device timeline of the last invoke of `model_id` on `gpu` (FSW_TRACE): out[16·L + i] for every layer
 * L of the model = %globaltimer ns of i = 0 the first kernel CTA entry, 1 the last weight-wait completion,
 * 2 the last CTA exit, 3 the first and 4 the last release of one of the layer's swap pieces (kernel
 * engines; the copy engine records nothing), and for GEMM layers 5 the last return from the wait on the
 * predecessor kernel (griddepcontrol.wait), 6 the last MMA completion, 7 the last epilogue start, 8-15
 * kernel-specific epilogue phases; 0 = no event.  t_invoke (nullable, 3 entries): the
 * invoke's first piece claimed, last piece released, graph end.  ESTATE without FSW_TRACE; EINVAL if
 * cap_layers < the model's layers.                                                                   */
fsw_status fsw_debug_trace_read(fsw_ctx* ctx, uint32_t model_id, int32_t gpu, uint64_t* out, uint32_t cap_layers,
                                uint64_t* t_invoke);

/* Phase stamps of the persistent transformer kernel's last run on `gpu` (environment FSW_MEGA_STAMPS=1 at plan
 * time; tools/mega_phases.py): out = [n_ops][ctas][8] %globaltimer ns (producer dependency resolved, MMA first
 * stage full, last commit, epilogue accumulator ready, epilogue stored, task done, compute task dependency
 * resolved, compute body done; 0 = none), ops_out (nullable) = [n_ops][4] (kind, n_tasks, tt, splits).  ESTATE
 * without the persistent-kernel plan or stamps; EINVAL if cap < n_ops·ctas·8 (*n_ops, *ctas still set). */
fsw_status fsw_debug_mega_stamps(fsw_ctx* ctx, uint32_t model_id, int32_t gpu, uint64_t* out, uint32_t* ops_out, uint64_t cap,
                                 uint32_t* n_ops, uint32_t* ctas);

/* Debug / test read-back (copies into caller host memory). */
fsw_status fsw_debug_read_resident(fsw_ctx* ctx, uint32_t model_id, int32_t gpu, void* dst, uint64_t cap);
fsw_status fsw_debug_read_store(fsw_ctx* ctx, uint32_t model_id, void* dst, uint64_t cap);
/* Link-coded store (FSW_REG_LINK_CODE): the coded bytes, and the piece table in execution order.
 * Piece i covers store bytes [off, off + bytes) of layer `layer` (bytes <= 16 KiB, a multiple of 16)
 * and is coded at [coff, coff + cbytes) of the coded store (coff a multiple of 128; gaps are zero).
 * Its nb = ceil(bytes / 1024) blocks of 512 16-bit words w_i have 32-bit headers hdr[0..nb) (the rest
 * 0): h = bits 0-7, b = bits 8-15, n = bits 16-31.  The coded piece is stream A, zero padding to a
 * multiple of 128 bytes, then stream B:
 *   stream A, per block:  b = 0xff : the raw bytes (1024, or bytes − 1024 (nb − 1) for a partial last
 *                                    block);  b = 0xfe : nothing (512 zero words);
 *                         b = 0..4 : 512 bytes m_i = (w_i >> 8 & 0x80) | (w_i & 0x7f);
 *                         b = 0x10..0x13 : the same 512 bytes m_i;
 *   stream B, per block with b = 0..4: b bit-planes of 64 bytes (bit i of plane p, byte i/8 bit i%8,
 *                         = bit p of code c_i); n exceptions of 4 bytes (position in bits 0-15, the
 *                         whole word in bits 16-31), zero-padded to a multiple of 16 bytes;
 *             per block with b = 0x10 + o (two-tier, o = 0..3; n = n_e | n_x << 10): 2 tier-1 planes
 *                         of 64 bytes (2-bit t_i), 3 tier-2 planes of 4·ceil(n_e / 32) bytes (3-bit s_j of
 *                         the j-th word with t_i = 3, bit j of plane q = bit q of s_j), n_x exceptions,
 *                         zero-padded to a multiple of 16 bytes.
 * A coded block decodes as w_i = (m_i & 0x80) << 8 | (h − c_i) << 7 | (m_i & 0x7f), then each
 * exception's word replaces w_position.  c_i = the b-bit code (b = 0..4), or (two-tier) o + t_i when
 * t_i < 3, else s_j < o ? s_j : s_j + 3.
 * ENOTFOUND / ESTATE (model not link-coded) / EINVAL (cap too small; *n is still set).              */
typedef struct { uint64_t off, coff; uint32_t bytes, cbytes, layer, pad; uint32_t hdr[16]; } fsw_coded_piece;
/* Entropy-coded pieces (format v5, b = 0x20): a piece either keeps the per-block codes above
 * or has every coded block of kind 0x20 (raw and zero blocks may remain).  Header of a 0x20 block: h = bits
 * 0-7, n_esc = bits 16-25.  Each word's offset s_i = min(h − e_i, 15) is coded with the model's canonical
 * Huffman code (lengths_out below: length L_s of symbol s, 0 = unused, all <= 12; codes assigned in order of
 * (L_s, s), MSB first); s = 15 marks an exception.  Stream A: 512 bytes m_i per 0x20 block (as above).
 * Stream B: the E = Σ n_esc exception words (16 bits each, whole words, in order of (block, l, i)), zero-
 * padded to a multiple of 16 bytes; then 4·K 16-bit code words, word j being word j / 4 of sub-stream
 * j mod 4 (K = the longest sub-stream; shorter ones zero-padded), zero-padded to a multiple of 16 bytes.
 * Sub-stream q carries the 0x20 blocks whose index in the piece is ≡ q (mod 4), in increasing order; 32
 * lanes l each keep a bit buffer (empty at the piece's start).  For each of its blocks and i = 0..15: every
 * lane whose buffer does not hold its next whole code (the code its bits start, read with zeros after them,
 * is longer than the bits held) appends the sub-stream's next word (MSB first; the lanes that need one take
 * consecutive words in increasing l), then every lane removes one code from the front of its buffer: s of
 * word 16·l + i.  w = (m & 0x80) << 8 | ((h − s) & 0xff) << 7 | (m & 0x7f) for s < 15, else the next
 * exception word.  lengths_out: 16 bytes, all 0 when the model has no entropy-coded piece.            */
fsw_status fsw_debug_coded_code(fsw_ctx* ctx, uint32_t model_id, uint8_t* lengths_out);
fsw_status fsw_debug_read_coded(fsw_ctx* ctx, uint32_t model_id, void* dst, uint64_t cap);
fsw_status fsw_debug_coded_pieces(fsw_ctx* ctx, uint32_t model_id, fsw_coded_piece* out, uint32_t cap, uint32_t* n);
/* Activation slot of the last invoke of `model_id` on `gpu` (valid until the next invoke). */
fsw_status fsw_debug_read_slot(fsw_ctx* ctx, uint32_t model_id, int32_t gpu, int32_t slot, void* dst, uint64_t cap);

/* ---------------------------------------------------------------------------------------
 * Node policies (§5).  Pure host functions, no context: the
 * runtime's placement (fsw_invoke) and eviction (weight pool) call the same code.
 * ------------------------------------------------------------------------------------- */
/* Required request count: (p·n − m)/(1 − p).  EINVAL unless 0 < p < 1, m <= n. */
fsw_status fsw_policy_rrc(uint64_t n, uint64_t m, double p, double* out);
/* α partition: with functions sorted by RRC (ties by index), high[i] = 1 for
 * the first k, k the largest with Σ_{j<=k} max(RRC_j,0) <= α·Σ_i max(RRC_i,0).  EINVAL if α ∉ [0,1]. */
fsw_status fsw_policy_partition(const double* rrc, uint32_t n, double alpha, uint8_t* high);
/* Algorithm 2.  EINVAL unless scalar > 1. */
fsw_status fsw_policy_alpha(double alpha, double last_ratio, double new_ratio, double scalar, double threshold,
                            double* out);
/* Algorithm 1.  Per GPU i of n: available[i] (idle), hosts[i] (target model
 * resident), neighbor[i] (GPU sharing its PCIe switch, −1 none; NULL = none), loading[i] (0 none,
 * 1 light, 2 heavy model being swapped in from the host; NULL = none), link[g·n+s] (NVLink GB/s
 * from s into g, 0 = no link; NULL = uniform, as on NVSwitch).  kind: 0 run resident, 1 swap from
 * the host, 2 swap from GPU src.  Ties: lowest GPU id / (target, source).  EBUSY: no GPU available. */
typedef struct { int32_t gpu; uint32_t kind; int32_t src; } fsw_decision;
fsw_status fsw_policy_schedule(uint32_t n, const uint8_t* available, const uint8_t* hosts, const int32_t* neighbor,
                               const uint8_t* loading, const float* link, fsw_decision* out);
/* Heaviness-aware LRU: eviction order of n resident models on one GPU — light
 * models and heavy models with >= 2 copies first, then sole-copy heavy models, LRU within each;
 * in-use models are skipped.  order has n entries; n_order = how many were emitted.            */
fsw_status fsw_policy_eviction_order(uint32_t n, const uint8_t* heavy, const uint32_t* copies, const uint64_t* last_use,
                                     const uint8_t* in_use, uint32_t* order, uint32_t* n_order);
/* Striped swap: the source of each of n_units units (pieces, or runs of coded
 * pieces, in execution order) — a unit goes to the sources whose NUMA node equals unit_node[u],
 * round-robin among them; a unit whose node has no source (or is −1) goes round-robin over all n_src
 * sources.  The runtime deals its striped swaps with this function.  EINVAL on NULL / n_src == 0. */
fsw_status fsw_policy_stripe_deal(uint32_t n_units, const int32_t* unit_node, uint32_t n_src, const int32_t* src_node,
                                  uint32_t* out);
/* Heavy / light (heavy when "model pipelining significantly slows down the inference
 * execution"; the class drives Algorithm 1's neighbour test and the eviction groups).
 * Re-derived for B200: with swap = the swap's added latency (cold − resident), the
 * model's SLO deadline and a queueing budget,
 *     slack = deadline − resident − queue_budget;   heavy  iff  slack <= 0  or  swap > theta · slack;
 * without a deadline (deadline <= 0) SPEC S:43-51's execution-relative rule: heavy iff
 * resident + swap > 1.25 · resident.  EINVAL on a negative time, theta <= 0.                   */
fsw_status fsw_policy_heavy(double swap_ms, double resident_ms, double deadline_ms, double queue_budget_ms, double theta,
                            int32_t* heavy);
/* A model's class: 1 heavy, 0 light, −1 auto = fsw_policy_heavy on its measured mean cold and resident
 * device latencies (before both are measured: swap ≈ link bytes / 55 GB/s, resident 0), its tightest
 * SLO (fsw_model_set_slo; fsw_function_register sets it) and the context's theta / queue budget
 * (fsw_set_heavy_policy; defaults 0.05 and 0 ms).                                              */
fsw_status fsw_model_set_heavy(fsw_ctx* ctx, uint32_t model_id, int32_t heavy);
fsw_status fsw_model_is_heavy(fsw_ctx* ctx, uint32_t model_id, int32_t* heavy);
/* Record a deadline of a function served by the model (the tightest one is kept).  EINVAL if <= 0. */
fsw_status fsw_model_set_slo(fsw_ctx* ctx, uint32_t model_id, double deadline_ms);
fsw_status fsw_set_heavy_policy(fsw_ctx* ctx, double theta, double queue_budget_ms);

/* ---------------------------------------------------------------------------------------
 * Request scheduler: functions = (model, deadline, tail percentile p);
 * requests queue in two priority classes by RRC and are dispatched onto the pool's GPUs
 * through fsw_invoke (placement by Algorithm 1, at most max_inflight at once).  Input/output
 * buffers of a submitted request stay caller-owned and must stay valid until fsw_wait.
 * ------------------------------------------------------------------------------------- */
typedef struct fsw_sched fsw_sched;
typedef struct {
    double alpha0;        /* initial α; 0 = 0.5                                               */
    double scalar;        /* Algorithm 2 scale factor; 0 = 2                  */
    double threshold;     /* Algorithm 2 threshold; 0 = 0.04                  */
    double period_ms;     /* α re-configuration period; 0 = 10 000 ms                         */
    uint32_t max_inflight;/* concurrent invokes; 0 = n_gpus (one request per GPU)      */
} fsw_sched_config;
fsw_status fsw_sched_create(fsw_ctx* ctx, const fsw_sched_config* cfg, fsw_sched** out);
void fsw_sched_destroy(fsw_sched* s);  /* serves every queued request, then stops            */
fsw_status fsw_function_register(fsw_sched* s, uint32_t model_id, double deadline_ms, double p, uint32_t* fid);
fsw_status fsw_submit(fsw_sched* s, uint32_t fid, const void* input, uint64_t input_bytes, void* output,
                      uint64_t output_cap, uint64_t* ticket);
typedef struct {
    double queue_ms, total_ms, device_ms; /* submit -> dispatch, submit -> output, invoke graph */
    int32_t met_deadline, gpu;
    uint32_t swap_kind;                   /* FSW_SWAP_*                                          */
    fsw_status status;
} fsw_request_stats;
fsw_status fsw_wait(fsw_sched* s, uint64_t ticket, fsw_request_stats* out); /* returns its status */
typedef struct {
    uint64_t n, m;                        /* completed requests / within the deadline            */
    double rrc, rrc_normalized, avg_latency_ms;
    uint32_t high, queued;
} fsw_function_stats;
fsw_status fsw_function_stats_get(fsw_sched* s, uint32_t fid, fsw_function_stats* out);
typedef struct {
    double alpha;
    uint32_t n_functions, n_high, active_functions, slo_compliant_functions;
    uint64_t completed, met_deadline, n_resident, n_host_swaps, n_peer_swaps, n_striped_swaps;
} fsw_sched_stats;
fsw_status fsw_sched_stats_get(fsw_sched* s, fsw_sched_stats* out);

/* The DMA engine's copy plan for (group_bytes, streams), host logic only (usable with
 * FSW_HOST_ONLY): n_groups copy groups [lo, hi) of the host store in execution order, each
 * dealt to copy stream group_stream[i] = i mod streams; for every layer L, layer_targets[4L+j]
 * = the number of stream-j groups that must have landed before L's weights are complete.
 * group_lo_hi has 2·cap_groups entries; n_groups is set even when cap_groups is too small
 * (then EINVAL).  Any output pointer may be NULL.                                          */
fsw_status fsw_debug_dma_plan(fsw_ctx* ctx, uint32_t model_id, uint64_t group_bytes, uint32_t streams,
                              uint64_t* group_lo_hi, uint32_t* group_stream, uint32_t cap_groups,
                              uint32_t* n_groups, uint32_t* layer_targets);

/* The DMAZ engine's copy plan of a link-coded model (host logic only, usable with FSW_HOST_ONLY):
 * n_groups copy groups [lo, hi) of the coded store, in order, tiling it; group i goes to copy
 * stream group_stream[i] = i mod streams; piece_group[p] (one entry per coded piece, see
 * fsw_debug_coded_pieces) = (stream << 24) | (index of the piece's group among its stream's groups).
 * ESTATE if the model is not link-coded; EINVAL for a bad argument or cap_groups too small (n_groups
 * is still set).  Any output pointer except n_groups may be NULL.                              */
fsw_status fsw_debug_dmaz_plan(fsw_ctx* ctx, uint32_t model_id, uint64_t group_bytes, uint32_t streams,
                               uint64_t* group_lo_hi, uint32_t* group_stream, uint32_t cap_groups,
                               uint32_t* n_groups, uint32_t* piece_group);

/* ---------------------------------------------------------------------------------------
 * Extent allocator of the weight pool (pure host logic, usable without a GPU; tests).
 * Best-fit over a free list of [offset, size) extents with coalescing on free.
 * ------------------------------------------------------------------------------------- */
typedef struct fsw_arena fsw_arena;
fsw_arena* fsw_arena_create(uint64_t capacity, uint64_t align);
void fsw_arena_destroy(fsw_arena* a);
fsw_status fsw_arena_alloc(fsw_arena* a, uint64_t bytes, uint64_t* offset); /* ENOMEM if no fit */
fsw_status fsw_arena_free(fsw_arena* a, uint64_t offset);                   /* EINVAL if unknown */
void fsw_arena_stats(const fsw_arena* a, uint64_t* used, uint64_t* largest_free, uint32_t* n_allocated);

#ifdef __cplusplus
}
#endif
#endif /* FSW_H */
