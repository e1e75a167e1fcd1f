// pod_internal.h -- plan object and device-side CTA descriptors shared by the
// host planner (pod_plan.cpp) and the kernels (pod_attn.cu).
#pragma once

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pod_attn.h"

namespace pod {

// Fixed by the sm_100a kernels.
constexpr int kHeadDim = 128;       // the compiled head dim (all BASELINE configs); d < 128 runs zero-padded
constexpr int kMBlock = 128;        // tcgen05 M: packed (row, q-head) rows per prefill block
constexpr int kKvTile = 64;         // prefill keys per tcgen05 N tile (4 pages of 16)
constexpr int kDecodeWarps = 4;     // virtual decode CTAs per physical CTA
#ifndef POD_SM_DEC_WARPS
#define POD_SM_DEC_WARPS 6
#endif
constexpr int kSmDecodeWarps = POD_SM_DEC_WARPS;   // decode warps of the warp-specialised kernel (pod_sm.cuh)
constexpr int kPrefillWarps = 4;    // softmax warps (one TMEM lane quadrant each)
constexpr int kThreads = 192;       // 4 softmax warps + 1 TMA-producer warp + 1 MMA warp
constexpr int kMaxSms = 1024;       // sm counter slots (sized for %nsmid, not %smid density)

// One physical prefill CTA = one CtaTask of decompose_prefill (work_decomp.hpp:204-247):
// chunk rows [row_begin, row_begin+rows) x the `group` q heads of kv_head, keys [kv_begin, kv_end).
struct PrefillCta {
    int32_t row_begin;
    int32_t rows;
    int32_t kv_head;
    int32_t kv_begin;
    int32_t kv_end;
    int32_t split;     // index of this split within its q tile
    int32_t n_splits;  // eff_splits of the tile (work_decomp.hpp:223)
    int32_t q_tile;
};

// One physical decode CTA = one (request, kv head, kv split) parent; its 4 warps are
// the virtual decode CTAs over split_ranges(kv_end - kv_begin, 4) (work_decomp.hpp:179-197).
struct DecodeCta {
    int32_t request;   // decode index (0-based among decodes)
    int32_t kv_head;
    int32_t kv_begin;
    int32_t kv_end;
    int32_t split;
    int32_t n_splits;
    int32_t ctx;
    int32_t page_row;  // row of page_indptr holding this request's pages
};

// Scheduler counters at the head of the workspace (gpu_sim.hpp:82-89).
struct SchedCounters {
    uint32_t sm_ctr[kMaxSms];
    uint32_t cta_assign[2];
    uint32_t done;
    uint32_t arrival;
    uint32_t running_prefill[kMaxSms];  // POD_POLICY_COMPLEMENT: prefill CTAs resident per SM
};

struct WorkspaceLayout {
    size_t off_counters = 0;
    size_t off_pctas = 0;
    size_t off_dctas = 0;
    size_t off_tile_splits = 0;   // int32 per prefill q tile: eff_splits
    size_t off_ppart_o = 0;       // [max_splits][chunk][Hq][d] fp32 (only if splits > 1)
    size_t off_ppart_lse = 0;     // [max_splits][chunk][Hq]
    size_t off_dpart_o = 0;       // [num_decodes][splits][Hq][d]
    size_t off_dpart_lse = 0;     // [num_decodes][splits][Hq]
    size_t off_dec_pos = 0;       // int32 per decode: position of its new token (context_len - 1)
    size_t off_dec_nsplit = 0;    // int32 per decode: its KV split count (the merge reads it)
    size_t off_vshadow = 0;       // fp16 copy of the prefill request's V, [logical page][Hkv][16][d] (vs_pages)
    size_t total = 0;
};

}  // namespace pod

struct pod_plan {
    pod_shape shape{};
    pod_batch batch{};
    std::vector<int64_t> decode_ctx;
    pod_device dev{};
    pod_options opts{};
    pod_tile_config cfg{};
    int64_t prefill_splits = 1;
    int64_t prefill_q_tiles = 0;
    std::vector<pod_task> prefill_tasks;
    std::vector<pod_task> decode_tasks;
    std::vector<pod::PrefillCta> pctas;
    std::vector<pod::DecodeCta> dctas;
    std::vector<int32_t> tile_splits;
    std::vector<int32_t> dec_pos;  // context_len - 1 per decode (KV append)
    std::vector<int32_t> dec_nsplit;  // KV splits per decode request (min(splits, ctx))
    bool pf_tn64 = false;          // warp-specialised: 64-key pair engine (see pod_plan.cpp)
    bool pf_db = false;            // ... with two S buffers per block (prefill_item_db, kernel instance 1)
    int64_t decode_splits = 1;     // largest split count (partials' stride)
    int32_t vs_pages = 0;          // > 0: prefill V read from an fp16 shadow of these many pages (pod_plan.cpp)
    int64_t dec_split_base = 1;    // splits of requests [0, dec_tail_start)
    int64_t dec_tail_start = 0;    // first request with decode_splits splits
    int64_t prefill_ratio = 1;
    int64_t decode_ratio = 1;
    int32_t max_prefill_splits = 1;
    int32_t merge_rows_prefill = 0;
    int32_t merge_rows_decode = 0;
    int64_t smem_bytes = 0;
    pod::WorkspaceLayout ws;
    int32_t* role_log = nullptr;
    // Tensor maps of the last run (5 x CUtensorMap, 128 B each), re-encoded only when
    // the Q / K / V pointers or the pool size change: host launch cost per run.
    // Guarded by map_mu (concurrent pod_attn_run calls on one plan).
    std::mutex map_mu;
    const void* map_key[4] = {nullptr, nullptr, nullptr, nullptr};  // q, k, v, workspace
    int64_t map_pages = -1;
    alignas(64) unsigned char map_blob[6 * 128];
};

namespace pod {
// Dynamic shared memory of the fused / prefill kernel (defined in pod_attn.cu).
int64_t fused_smem_bytes();
// Dynamic shared memory of the warp-specialised one-CTA-per-SM kernel.
int64_t sm_smem_bytes(bool db);
void set_last_error(const std::string& s);
}  // namespace pod
