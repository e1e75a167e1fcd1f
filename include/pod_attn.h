/*
 * pod_attn.h -- C ABI of the B200-native POD-Attention hot path.
 *
 * One launch computes the prefill-chunk attention and the batched paged-KV
 * decode attention of a hybrid batch concurrently (SM-aware CTA scheduling),
 * followed by a split-KV LSE merge.  The reference (arxiv/paper_2410_18038,
 * `attnsim`, header-only C++20) has no ABI: its path is the C++ templates
 * listed per entry point below (paths relative to /root/reference/proj/).
 * Reference C++ exceptions map to pod_status codes; nothing throws across
 * this boundary.
 *
 * Plain C types only; CUDA streams are passed as `void*` (a cudaStream_t).
 * All device pointers are caller-owned; pod_attn_run* allocate nothing, so a
 * (plan, workspace) pair can be captured in a CUDA graph.  One (plan,
 * workspace) pair must not run on two streams at once; one plan may be run from
 * several host threads with distinct workspaces (its tensor-map cache is locked).
 * Launches go to the calling thread's current CUDA device.
 */
#ifndef POD_ATTN_H_
#define POD_ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POD_ATTN_ABI_VERSION 2

/* Mirrors the exception classes of the reference (include/attnsim/types.hpp:12-15,
 * attention.hpp:113-116,155-163,249,304; work_decomp.hpp:33-47,151-152). */
typedef enum pod_status {
    POD_OK = 0,
    POD_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument                 */
    POD_ERR_LOGIC = 2,            /* std::logic_error (cache too short ...) */
    POD_ERR_DOMAIN = 3,           /* std::domain_error (empty cache ...)    */
    POD_ERR_OUT_OF_RANGE = 4,     /* std::out_of_range (bad head index)     */
    POD_ERR_CONFIG = 5,           /* attnsim::ConfigError (infeasible smem) */
    POD_ERR_CUDA = 6,             /* a CUDA runtime/driver call failed      */
    POD_ERR_UNSUPPORTED = 7       /* shape the sm_100a kernels do not cover */
} pod_status;

/* ModelShape (include/attnsim/types.hpp:60-76).  `scale` is the softmax
 * DIVISOR: scores are (q.k)/scale (attention.hpp:124,193,206). */
typedef struct pod_shape {
    int32_t num_q_heads;
    int32_t num_kv_heads;
    int32_t head_dim;     /* kernels: 8..128 in steps of 8 (below 128 run zero-padded); others plan
                             fine but pod_attn_run* report POD_ERR_UNSUPPORTED */
    double scale;
} pod_shape;

/* PrefillSpec (include/attnsim/work_decomp.hpp:18-22). */
typedef struct pod_prefill_spec {
    int64_t chunk_size;      /* tokens in this chunk            */
    int64_t context_len;     /* full prompt length              */
    int64_t position_offset; /* tokens before this chunk        */
} pod_prefill_spec;

enum { POD_KV_HND = 0, POD_KV_NHD = 1 };
enum { POD_DTYPE_BF16 = 0, POD_DTYPE_FP16 = 1 };

/* HybridBatchSpec (work_decomp.hpp:28-48) plus the paged-KV description the
 * GPU adds (the reference has no paging).
 * Request numbering for page_indptr: request 0 is the prefill (if any), then
 * the decodes in order.  The prefill request's pages must hold at least
 * position_offset + chunk_size tokens (attention.hpp:159-160); decode i's pages
 * hold decode_context_len[i] tokens (its own new token included, :269). */
typedef struct pod_batch {
    int32_t has_prefill;
    pod_prefill_spec prefill;
    int64_t num_decodes;
    const int64_t* decode_context_len; /* host array [num_decodes]          */
    int32_t page_size;                 /* tokens per page (default 16)      */
    int32_t kv_layout;                 /* POD_KV_HND (default) / POD_KV_NHD */
    int32_t dtype;                     /* POD_DTYPE_BF16 / POD_DTYPE_FP16   */
} pod_batch;

/* GpuSpec (include/attnsim/gpu.hpp:12-37); only num_sms and the rates feed
 * select_tile_config / limit_prefill_splits (work_decomp.hpp:88-155). */
typedef struct pod_device {
    int32_t num_sms;
    double compute_rate_per_sm;
    double mem_bandwidth_total;
    double mem_bandwidth_per_sm;
    double mem_interference;
    int32_t max_ctas_per_sm;
    double shared_mem_per_sm;
} pod_device;

/* TileConfig (work_decomp.hpp:50-60). */
typedef struct pod_tile_config {
    int64_t prefill_tile_q;
    int64_t decode_tile_q;
    int64_t tile_kv;
    int32_t warps_per_cta;
    int32_t ctas_per_sm;
    double shared_mem_per_cta;
    int32_t virtual_decode;
    int32_t split_wave_cap;
} pod_tile_config;

/* CtaTask (work_decomp.hpp:62-73).  op: 0 prefill, 1 decode (OpKind, types.hpp:17). */
typedef struct pod_task {
    int32_t op;
    int32_t request_id;
    int32_t kv_head;
    int32_t q_tile;
    int64_t kv_begin;
    int64_t kv_end;
    int32_t is_virtual;
    int32_t slot_quanta;
    int64_t barrier_segments;
    double compute_work;
    double memory_work;
} pod_task;

enum {
    POD_POLICY_FIFTY_FIFTY = 0,  /* SmPolicy::FiftyFifty (gpu_sim.hpp:97-99)          */
    POD_POLICY_PROPORTIONAL = 1, /* SmPolicy::Proportional, gcd of PHYSICAL CTAs (:100-105) */
    POD_POLICY_CLAMPED = 2,      /* proportional, rounded to the per-SM slot count     */
    POD_POLICY_COMPLEMENT = 3,   /* bind from the roles resident on the SM:
                                    prefill while < prefill_ratio prefill CTAs run there */
    /* 4-6 retired (two-block slot engine, greedy balance, spatial partition): all
       measured slower than COMPLEMENT / WARPSPEC; pod_attn_plan rejects them */
    POD_POLICY_WARPSPEC = 7,     /* one CTA per SM hosting a prefill engine (two 128-row
                                    M-blocks, Q/S/P/O in TMEM) and a decode warp group side
                                    by side; each binds items from its pool at runtime */
    POD_POLICY_AUTO = 8          /* default: WARPSPEC for hybrid batches whose decode share
                                    of the serial time (algorithmic work at measured B200
                                    rates) is >= 0.1 and whose decode contexts average >= 2K,
                                    else COMPLEMENT; inside WARPSPEC the pair engine runs
                                    64-key tiles below a decode share of 0.57, 32-key tiles
                                    above (the plan records the resolved policy and width) */
};

enum {
    POD_TILE_REFERENCE = 0, /* select_tile_config / make_tile_config (work_decomp.hpp:119-145) */
    POD_TILE_B200 = 1       /* prefill_tile_q = 128/group (one tcgen05 M-block per CTA)       */
};

typedef struct pod_options {
    int32_t policy;          /* POD_POLICY_*                                        */
    int32_t tile_mode;       /* POD_TILE_*                                          */
    int32_t ctas_per_sm;     /* 0 = from tile selection; else 2 or 4 (make_tile_config) */
    int32_t virtual_decode;  /* -1 = keep the tile config's flag, 0 = off, 1 = on    */
    int32_t split_wave_cap;  /* 0 = keep the tile config's value (2)                */
    int32_t decode_splits;   /* 0 = auto (fill the machine), else splits per (request, kv head) */
    const pod_tile_config* tile_override; /* non-NULL: use this TileConfig verbatim */
    int32_t precision;       /* POD_PRECISION_* for the prefill P operand            */
    int32_t out_dtype;       /* POD_OUT_*: element type of o_prefill / o_decode (LSE stays fp32) */
    int32_t prefill_tile_keys; /* warp-specialised pair engine: 0 = by decode share, 32 or 64 forces */
    int32_t prefill_s_buffers; /* 64-key pair engine: 0 = by decode share, 1 = one S buffer per block (Q in
                                  TMEM), 2 = two S buffers per block (Q in smem, 2-stage decode rings) */
} pod_options;

enum {
    POD_OUT_F32 = 0,  /* fp32 outputs (default; the reference's AttentionPartial.o, attention.hpp:86-93) */
    POD_OUT_BF16 = 1, /* bf16 outputs, RNE of the fp32 result: half the HBM / PCIe / all-gather bytes */
    POD_OUT_F16 = 2   /* fp16 outputs, RNE of the fp32 result */
};

enum {
    POD_PRECISION_SPLIT = 0, /* P = bf16 hi + bf16 lo (two PV MMAs): ~16-bit P, any V     */
    POD_PRECISION_FAST = 1,  /* P rounded to one bf16 (FlashAttention-style): error ~2e-3,
                                at the north-star bar itself at 16K keys                  */
    POD_PRECISION_F16PV = 2  /* default: P rounded to fp16 (11-bit), V tiles converted
                                bf16 -> fp16 in shared memory, one fp16 PV MMA: error
                                ~3e-4 of the output scale; exact V for |V| <= 65504 (larger
                                V saturates: use SPLIT); fp16 pools: P fp16, no conversion */
};

/* What the plan decided, for benches and tests. */
typedef struct pod_plan_info {
    pod_tile_config config;
    int64_t prefill_splits;     /* limit_prefill_splits() result (work_decomp.hpp:147-155) */
    int64_t num_prefill_tasks;  /* == decompose_prefill().size()                          */
    int64_t num_decode_tasks;   /* == decompose_decode().size() (virtual tasks if enabled) */
    int64_t num_prefill_ctas;   /* physical CTAs of the prefill role                       */
    int64_t num_decode_ctas;    /* physical CTAs of the decode role                        */
    int64_t decode_splits;      /* KV splits per (request, kv head) on the GPU             */
    int64_t prefill_ratio;      /* scheduler ratio (make_scheduler_state, gpu_sim.hpp:91)  */
    int64_t decode_ratio;
    int64_t smem_bytes;         /* dynamic smem per CTA of the fused kernel                */
    int64_t workspace_bytes;
    int32_t num_merge_rows_prefill; /* (row, q head) pairs needing a split merge */
    int32_t num_merge_rows_decode;
    int32_t policy;             /* the POD_POLICY_* the plan runs (POD_POLICY_AUTO resolved) */
    int32_t prefill_tile_keys;  /* keys per prefill K/V tile of the warp-specialised pair engine (32 or 64; 0 otherwise) */
    int32_t prefill_s_buffers;  /* S buffers per block of that engine (32 keys: 2; 64 keys: 1 or 2; 0 otherwise) */
} pod_plan_info;

typedef struct pod_plan pod_plan;

/* Fills a pod_device for CUDA device `device` (num_sms from
 * cudaDevAttrMultiProcessorCount, smem from cudaDevAttrMaxSharedMemoryPerMultiprocessor)
 * with rates calibrated to B200 measured peaks. */
pod_status pod_device_query(int device, pod_device* out);
/* The reference's default A100-like GpuSpec (gpu.hpp:12-37), for parity tests. */
void pod_device_reference_default(pod_device* out);
void pod_options_default(pod_options* out);

/* Host-only, pure and reentrant.  Replaces decompose_hybrid()
 * (work_decomp.hpp:249-261) + select_tile_config() (:139-145) +
 * make_scheduler_state() (gpu_sim.hpp:91-107). */
pod_status pod_attn_plan(const pod_shape* shape, const pod_batch* batch, const pod_device* dev,
                         const pod_options* opts, pod_plan** out);
void pod_attn_plan_destroy(pod_plan* plan);
pod_status pod_attn_plan_get_info(const pod_plan* plan, pod_plan_info* out);
/* Task tables with decompose_prefill / decompose_decode semantics
 * (work_decomp.hpp:157-247).  On input *n_* are capacities (pass NULL arrays to
 * query counts); on output the counts. */
pod_status pod_attn_plan_tasks(const pod_plan* plan, pod_task* prefill, int64_t* n_prefill,
                               pod_task* decode, int64_t* n_decode);
size_t pod_attn_workspace_bytes(const pod_plan* plan);
/* Uploads the plan's CTA tables into `workspace` and zeroes the scheduler
 * counters (stream-ordered).  Required once per (plan, workspace) pair; the
 * fused kernel re-zeroes its counters itself at the end of every launch. */
pod_status pod_attn_workspace_init(const pod_plan* plan, void* workspace, void* stream);

/* The fused hybrid-batch launch: SM-aware role binding,
 * prefill role = tcgen05 causal tile (attention.hpp:148-222 semantics),
 * decode role = split-KV paged decode with virtual warps (attention.hpp:240-292),
 * then the LSE merge (attention.hpp:294-326).
 *   q_prefill  [chunk][Hq][d]                         (attention.hpp:45-69)
 *   q_decode   [num_decodes][Hq][d]                   (attention.hpp:71-84)
 *   k_pool, v_pool  HND [num_pages][Hkv][page_size][d] or NHD [num_pages][page_size][Hkv][d]
 *   page_indptr [num_requests + 1], page_indices [...] (int32, device)
 *   o_prefill  [chunk][Hq][d] fp32 (or bf16/fp16 per options.out_dtype), lse_prefill [chunk][Hq] fp32 (natural log)
 *   o_decode   [num_decodes][Hq][d] (same element type), lse_decode [num_decodes][Hq] fp32
 * Unused outputs may be NULL when the batch has no such part. */
pod_status pod_attn_run(const pod_plan* plan, const void* q_prefill, const void* q_decode,
                        const void* k_pool, const void* v_pool, int64_t num_pages,
                        const int32_t* page_indptr, const int32_t* page_indices, void* o_prefill,
                        float* lse_prefill, void* o_decode, float* lse_decode, void* workspace,
                        void* stream);
/* Serial comparator (gpu_sim.hpp:496-506): the same prefill and decode device
 * code as two back-to-back launches on one stream, then the merge. */
pod_status pod_attn_run_serial(const pod_plan* plan, const void* q_prefill, const void* q_decode,
                               const void* k_pool, const void* v_pool, int64_t num_pages,
                               const int32_t* page_indptr, const int32_t* page_indices,
                               void* o_prefill, float* lse_prefill, void* o_decode,
                               float* lse_decode, void* workspace, void* stream);
/* Standalone halves (prefill-alone / decode-alone timings and unit tests).
 * which: 0 = prefill only, 1 = decode only.  Includes that part's merge. */
pod_status pod_attn_run_part(const pod_plan* plan, int which, const void* q_prefill,
                             const void* q_decode, const void* k_pool, const void* v_pool,
                             int64_t num_pages, const int32_t* page_indptr,
                             const int32_t* page_indices, void* o_prefill, float* lse_prefill,
                             void* o_decode, float* lse_decode, void* workspace, void* stream);

/* Optional device-side role log of the fused kernel (the GPU analogue of
 * SmAssignment, gpu_sim.hpp:141-148): when set (non-NULL, device memory of
 * 8 int32 per fused CTA), every CTA writes {smid, ticket, op, cta_id,
 * arrival order, t_start_lo, t_end_lo, blockIdx}. */
pod_status pod_attn_set_role_log(pod_plan* plan, int32_t* device_log);

/* Device gather probe: copies logical token rows of request `req` through the
 * page table into out [ctx][Hkv][d] (raw 16-bit words) -- checks the paged
 * indexing bit-exactly against the CPU gather. */
pod_status pod_attn_gather_probe(const pod_plan* plan, const void* kv_pool, int64_t num_pages,
                                 const int32_t* page_indptr, const int32_t* page_indices,
                                 int32_t req, int64_t ctx, uint16_t* out, void* stream);

/* o_proj consumer of the attention output (the reference has no
 * projection, its hot path ends at the attention output): Y += O W with O [tokens][K]
 * bf16 (this rank's q heads, K = Hq/T x d: the o_prefill / o_decode rows as bf16,
 * POD_OUT_BF16), W [K][N] bf16 (the W_o rows of those heads), fp32 accumulate.
 * Under KV-head-group TP the projection is row-parallel, so no all-gather of O is
 * needed: with accumulate = 1 every 128 x 128 output tile is reduced into the row
 * owner's fp32 Y (y_parts[t] holds rows [t*rows_per_rank, (t+1)*rows_per_rank), mapped
 * peer memory for t != this rank) while the GEMM runs -- a GEMM with a fused
 * reduce-scatter.  accumulate = 0 (world = 1) stores instead.  Y must be zeroed before
 * the reducing launches.  K % 64 == 0, N % 128 == 0.  Stream-ordered. */
pod_status pod_oproj_run(const void* o, const void* w, int64_t tokens, int64_t k, int64_t n,
                         void* const* y_parts, int32_t world, int64_t rows_per_rank,
                         int32_t accumulate, void* stream);

/* Benchmark utility: overwrites `bytes` of device memory (a buffer larger than the
 * 126 MB L2) with zeros, evicting the L2 between timed layers.  The kernel prefers
 * the max-shared-memory L1 carve-out, the one the POD kernels use, so the flush does
 * not leave the SMs in a configuration the next POD launch must switch back from
 * (a generic memset costs the following launch ~7-10 us of reconfiguration).
 * Stream-ordered. */
pod_status pod_attn_l2_flush(void* buf, int64_t bytes, void* stream);

/* KV append (the step before attention in a layer): scatters the
 * batch's new K/V tokens into the paged pools through the block table.  The prefill
 * chunk's tokens take positions [position_offset, position_offset + chunk_size) of
 * request 0, decode b's single token takes position context_len_b - 1 of request b+1
 * (the newest key each query attends to).  Token t of request r lands in page
 * page_indices[page_indptr[r] + t / page_size], slot t % page_size, for every KV head
 * (HND or NHD as planned).  Inputs: k_new / v_new rows [chunk][Hkv][d] (prefill) and
 * [B][Hkv][d] (decode), the pool dtype.  A pure copy: bit-exact.  Stream-ordered;
 * run it before pod_attn_run on the same stream.  (No reference counterpart: the
 * reference keeps contiguous caches.)  `workspace` is the plan's
 * (pod_attn_workspace_init'ed): it holds the decode positions. */
pod_status pod_attn_append_kv(const pod_plan* plan, const void* k_new_prefill, const void* v_new_prefill,
                              const void* k_new_decode, const void* v_new_decode, void* k_pool, void* v_pool,
                              int64_t num_pages, const int32_t* page_indptr, const int32_t* page_indices,
                              void* workspace, void* stream);

/* Resident CTAs per SM the driver allows for the fused / prefill-only /
 * decode-only kernels of this plan's instantiation (cudaOccupancyMaxActiveBlocksPerMultiprocessor). */
pod_status pod_attn_occupancy(const pod_plan* plan, int32_t* fused, int32_t* prefill, int32_t* decode);

const char* pod_status_string(pod_status s);
/* Last CUDA error string seen by this thread's most recent failing call. */
const char* pod_last_error(void);
int pod_attn_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* POD_ATTN_H_ */
