// pod_plan.cpp -- host planner behind pod_attn_plan (include/pod_attn.h).
//
// Restates the reference's hybrid-batch planning so the task table matches
// decompose_hybrid() field by field (tests/test_plan.py checks it against the
// reference compiled in oracle/_ref):
//   HybridBatchSpec::validate      work_decomp.hpp:33-47
//   estimate_*_serial              work_decomp.hpp:88-112
//   make_tile_config               work_decomp.hpp:119-136
//   select_tile_config             work_decomp.hpp:139-145
//   limit_prefill_splits           work_decomp.hpp:147-155
//   decompose_decode               work_decomp.hpp:157-202
//   decompose_prefill              work_decomp.hpp:204-247
//   make_scheduler_state           gpu_sim.hpp:91-107
// and then lowers the tasks to the physical CTA tables the sm_100a kernels
// consume, plus the workspace layout.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <stdexcept>

#include "pod_internal.h"

#ifndef POD_WHOLE_WAVES
#define POD_WHOLE_WAVES 1  // warp-specialised decode items rounded up to whole waves
#endif

namespace {

struct Status : std::exception {
    pod_status code;
    std::string msg;
    Status(pod_status c, std::string m) : code(c), msg(std::move(m)) {}
};

[[noreturn]] void fail(pod_status c, const char* m) { throw Status(c, m); }

template <typename L, typename R>
constexpr L ceil_div(L x, R y) {
    return (x + static_cast<L>(y) - 1) / static_cast<L>(y);
}

// ModelShape::validate (types.hpp:68-75).
void validate_shape(const pod_shape& s) {
    if (s.num_q_heads < 1 || s.num_kv_heads < 1 || s.head_dim < 1)
        fail(POD_ERR_INVALID_ARGUMENT, "ModelShape: head counts and head_dim must be >= 1");
    if (s.num_q_heads % s.num_kv_heads != 0)
        fail(POD_ERR_INVALID_ARGUMENT, "ModelShape: num_q_heads must be divisible by num_kv_heads");
    if (!(s.scale > 0.0)) fail(POD_ERR_INVALID_ARGUMENT, "ModelShape: scale must be positive");
}

// HybridBatchSpec::validate (work_decomp.hpp:33-47).
void validate_batch(const pod_plan& p) {
    validate_shape(p.shape);
    if (!p.batch.has_prefill && p.decode_ctx.empty())
        fail(POD_ERR_INVALID_ARGUMENT, "HybridBatchSpec: batch is empty");
    if (p.batch.has_prefill) {
        const auto& pf = p.batch.prefill;
        if (pf.chunk_size < 1) fail(POD_ERR_INVALID_ARGUMENT, "HybridBatchSpec: chunk_size must be >= 1");
        if (pf.position_offset < 0 || pf.position_offset + pf.chunk_size > pf.context_len)
            fail(POD_ERR_INVALID_ARGUMENT, "HybridBatchSpec: chunk exceeds prompt");
    }
    for (int64_t c : p.decode_ctx)
        if (c < 1) fail(POD_ERR_INVALID_ARGUMENT, "HybridBatchSpec: decode context must be >= 1");
}

double aggregate_compute_rate(const pod_device& g) { return g.compute_rate_per_sm * g.num_sms; }

// detail::estimate_prefill_serial (work_decomp.hpp:88-102).
double estimate_prefill_serial(const pod_plan& p) {
    if (!p.batch.has_prefill) return 0.0;
    const auto& pf = p.batch.prefill;
    const pod_shape& s = p.shape;
    const long probe_tile = 128;
    double compute = 0, memory = 0;
    for (long t0 = 0; t0 < pf.chunk_size; t0 += probe_tile) {
        const long rows = std::min<long>(probe_tile, pf.chunk_size - t0);
        const long span = pf.position_offset + t0 + rows;
        compute += static_cast<double>(probe_tile) * s.num_q_heads * span;
        memory += 2.0 * span * s.head_dim * s.num_kv_heads +
                  static_cast<double>(rows) * s.num_q_heads * s.head_dim;
    }
    return std::max(compute / aggregate_compute_rate(p.dev), memory / p.dev.mem_bandwidth_total);
}

// detail::estimate_decode_serial (work_decomp.hpp:104-112).
double estimate_decode_serial(const pod_plan& p) {
    const pod_shape& s = p.shape;
    double compute = 0, memory = 0;
    for (int64_t ctx : p.decode_ctx) {
        compute += 16.0 * ctx * s.num_kv_heads;
        memory += 2.0 * ctx * s.head_dim * s.num_kv_heads;
    }
    return std::max(compute / aggregate_compute_rate(p.dev), memory / p.dev.mem_bandwidth_total);
}

// make_tile_config (work_decomp.hpp:119-136).
pod_tile_config make_tile_config(int ctas_per_sm) {
    pod_tile_config c{};
    c.prefill_tile_q = 128;
    c.decode_tile_q = 16;
    c.tile_kv = 64;
    c.warps_per_cta = 4;
    c.ctas_per_sm = 2;
    c.shared_mem_per_cta = 65536.0;
    c.virtual_decode = 0;
    c.split_wave_cap = 2;
    if (ctas_per_sm == 2) {
        c.ctas_per_sm = 2;
        c.prefill_tile_q = 128;
        c.tile_kv = 64;
        c.shared_mem_per_cta = 65536.0;
    } else if (ctas_per_sm == 4) {
        c.ctas_per_sm = 4;
        c.prefill_tile_q = 64;
        c.tile_kv = 32;
        c.shared_mem_per_cta = 32768.0;
    } else {
        fail(POD_ERR_INVALID_ARGUMENT, "make_tile_config: ctas_per_sm must be 2 or 4");
    }
    c.decode_tile_q = 16;
    return c;
}

// limit_prefill_splits (work_decomp.hpp:147-155).
long limit_prefill_splits(long natural, const pod_device& g, const pod_tile_config& c) {
    if (natural < 1) fail(POD_ERR_INVALID_ARGUMENT, "limit_prefill_splits: parallelism must be >= 1");
    const long cap = static_cast<long>(c.split_wave_cap) * g.num_sms;
    return std::max<long>(1, cap / natural);
}

// decompose_decode (work_decomp.hpp:157-202).
void decompose_decode(pod_plan& p) {
    const pod_shape& s = p.shape;
    const pod_tile_config& config = p.cfg;
    p.decode_tasks.clear();
    for (size_t r = 0; r < p.decode_ctx.size(); ++r) {
        const long ctx = p.decode_ctx[r];
        for (int h = 0; h < s.num_kv_heads; ++h) {
            if (!config.virtual_decode) {
                pod_task t{};
                t.op = 1;
                t.request_id = static_cast<int>(r);
                t.kv_head = h;
                t.kv_begin = 0;
                t.kv_end = ctx;
                t.compute_work = static_cast<double>(config.decode_tile_q) * ctx;
                t.memory_work = 2.0 * ctx * s.head_dim;
                t.barrier_segments = std::max<long>(1, ceil_div(ctx, config.tile_kv));
                t.slot_quanta = config.warps_per_cta;
                p.decode_tasks.push_back(t);
            } else {
                const long base = ctx / config.warps_per_cta;
                const long rem = ctx % config.warps_per_cta;
                long pos = 0;
                for (int w = 0; w < config.warps_per_cta; ++w) {
                    const long len = base + (w < rem ? 1 : 0);
                    pod_task t{};
                    t.op = 1;
                    t.request_id = static_cast<int>(r);
                    t.kv_head = h;
                    t.kv_begin = pos;
                    t.kv_end = pos + len;
                    t.is_virtual = 1;
                    t.compute_work = static_cast<double>(config.decode_tile_q) * len;
                    t.memory_work = 2.0 * len * s.head_dim;
                    t.barrier_segments = std::max<long>(1, ceil_div(len, config.tile_kv));
                    t.slot_quanta = 1;
                    p.decode_tasks.push_back(t);
                    pos += len;
                }
            }
        }
    }
}

// decompose_prefill (work_decomp.hpp:204-247).
void decompose_prefill(pod_plan& p) {
    const auto& pf = p.batch.prefill;
    const pod_shape& s = p.shape;
    const pod_tile_config& config = p.cfg;
    const int group = s.num_q_heads / s.num_kv_heads;
    const long q_tiles = ceil_div(pf.chunk_size, config.prefill_tile_q);
    const long natural = q_tiles * s.num_kv_heads;
    const long splits = limit_prefill_splits(natural, p.dev, config);
    p.prefill_splits = splits;
    p.prefill_q_tiles = q_tiles;
    p.prefill_tasks.clear();
    p.tile_splits.assign(q_tiles, 1);
    for (long tile = 0; tile < q_tiles; ++tile) {
        const long rows = std::min<long>(config.prefill_tile_q, pf.chunk_size - tile * config.prefill_tile_q);
        const long kv_count = pf.position_offset + tile * config.prefill_tile_q + rows;
        const long eff_splits = std::min<long>(splits, ceil_div(kv_count, config.tile_kv));
        p.tile_splits[tile] = static_cast<int32_t>(eff_splits);
        const long base = kv_count / eff_splits;
        const long rem = kv_count % eff_splits;
        for (int h = 0; h < s.num_kv_heads; ++h) {
            long pos = 0;
            for (long sp = 0; sp < eff_splits; ++sp) {
                const long len = base + (sp < rem ? 1 : 0);
                pod_task t{};
                t.op = 0;
                t.request_id = 0;
                t.kv_head = h;
                t.q_tile = static_cast<int>(tile);
                t.kv_begin = pos;
                t.kv_end = pos + len;
                t.compute_work = static_cast<double>(config.prefill_tile_q) * group * len;
                t.memory_work = 2.0 * len * s.head_dim + static_cast<double>(rows) * group * s.head_dim;
                t.barrier_segments = std::max<long>(1, ceil_div(len, config.tile_kv));
                t.slot_quanta = config.warps_per_cta;
                p.prefill_tasks.push_back(t);
                pos += len;
            }
        }
    }
}

// Lower tasks to the kernels' physical CTA tables.
double decode_share(const pod_plan& p);

void lower(pod_plan& p) {
    const pod_shape& s = p.shape;
    p.pctas.clear();
    p.dctas.clear();
    p.max_prefill_splits = 1;
    if (p.batch.has_prefill) {
        for (const pod_task& t : p.prefill_tasks) {
            pod::PrefillCta c{};
            c.q_tile = t.q_tile;
            c.row_begin = static_cast<int32_t>(t.q_tile * p.cfg.prefill_tile_q);
            c.rows = static_cast<int32_t>(
                std::min<int64_t>(p.cfg.prefill_tile_q, p.batch.prefill.chunk_size - c.row_begin));
            c.kv_head = t.kv_head;
            c.kv_begin = static_cast<int32_t>(t.kv_begin);
            c.kv_end = static_cast<int32_t>(t.kv_end);
            c.n_splits = p.tile_splits[t.q_tile];
            p.max_prefill_splits = std::max(p.max_prefill_splits, c.n_splits);
            p.pctas.push_back(c);
        }
        // split index within (tile, head): tasks are ordered tile, head, split.
        for (size_t i = 0; i < p.pctas.size();) {
            const int n = p.pctas[i].n_splits;
            for (int sp = 0; sp < n; ++sp) p.pctas[i + sp].split = sp;
            i += n;
        }
    }
    // Decode: one physical CTA per (request, kv head, split); its warps are the
    // virtual CTAs.  decode_splits = 1 reproduces the reference's virtual tasks
    // exactly (4 warps x split_ranges(ctx, 4)).
    const int64_t parents = static_cast<int64_t>(p.decode_ctx.size()) * s.num_kv_heads;
    int64_t splits = p.opts.decode_splits;
    const bool warpspec = p.opts.policy == POD_POLICY_WARPSPEC;
    if (splits <= 0) {
        if (warpspec) {
            // one decode group per SM: items of <= ~4 MB of K/V (the per-item latency
            // stays a small share) and at least 1.5 items per SM (a short tail);
            // measured sweep: C2 B=64 / B=32 / B=16 -> 2, C3 TP4 rank -> 2,
            // C3 TP8 rank -> 4 (2 x nsm / parents gave 3 and 5: 2-7 % slower)
            int64_t max_ctx = 0;
            for (int64_t c : p.decode_ctx) max_ctx = std::max(max_ctx, c);
            const int64_t parent_bytes = max_ctx * 4 * s.head_dim;  // bf16 K + V of one KV head
            const int64_t by_size = ceil_div(parent_bytes, int64_t(4) << 20);
            const int64_t by_count = parents == 0 ? 1 : ceil_div(3 * static_cast<int64_t>(p.dev.num_sms), 2 * parents);
            splits = std::max<int64_t>(1, std::max(by_size, by_count));
        } else {
            const int64_t slots = static_cast<int64_t>(p.dev.num_sms) * 2;
            splits = parents >= slots || parents == 0 ? 1 : ceil_div(slots, parents);
        }
    }
    int64_t min_ctx = INT64_MAX;
    for (int64_t c : p.decode_ctx) min_ctx = std::min(min_ctx, c);
    if (!p.decode_ctx.empty()) {
        // each warp keeps at least one page of keys
        const int warps = warpspec ? pod::kSmDecodeWarps : pod::kDecodeWarps;
        const int64_t cap = std::max<int64_t>(1, min_ctx / (warps * 16));
        if (p.opts.decode_splits <= 0) splits = std::min(splits, cap);
    }
    p.decode_splits = std::max<int64_t>(1, splits);
    // Pair-engine tile width (warp-specialised kernel): 64-key tiles with one S buffer
    // per block issue a third fewer MMAs and half the barrier hops per key (prefill
    // -6 %, fused -5..11 % up to a decode share of 0.52 in the C5 sweep) but slow the
    // decode-dominant fused batches (+2..9 % from a share of 0.62, C2 B=64 among them),
    // so they serve batches with a decode share below 0.57.
    {
        const int32_t keys = p.opts.prefill_tile_keys;
        p.pf_tn64 = warpspec && p.batch.has_prefill && (keys == 64 || (keys == 0 && decode_share(p) < 0.57));
        // two S buffers per block (Q in smem, the decode group at 2 ring stages per warp): fused C2
        // B=8 (decode share 0.17) 356 -> 332 us, B=16 (0.29) 357 -> 351, but C1 (0.32) 56.3 -> 58.4
        // and B=32 (0.45) 436 -> 555 -- the smaller decode rings cost more than the prefill gains
        const int32_t sb = p.opts.prefill_s_buffers;
        p.pf_db = p.pf_tn64 && (sb == 2 || (sb == 0 && decode_share(p) < 0.30));
    }
    // Whole waves (warp-specialised kernel): the decode items are claimed in id order
    // (request-major) by one decode group per SM, so a count that is not a multiple of
    // the SM count leaves SMs idle for the last item's duration.  The last requests get
    // one split more, lifting the item count to the next multiple of num_sms (the items
    // claimed last are the smaller ones).  decode_splits becomes the largest count (the
    // partials' stride); dec_split_base is the count of requests below dec_tail_start.
    p.dec_split_base = p.decode_splits;
    p.dec_tail_start = static_cast<int64_t>(p.decode_ctx.size());
    // (decode-dominant batches only: when the prefill role is the longer one the decode
    // balance does not set the makespan and the extra merge rows cost ~1 %, C2 B=16)
    if (warpspec && p.opts.decode_splits <= 0 && !p.decode_ctx.empty() && POD_WHOLE_WAVES &&
        decode_share(p) >= 0.5) {
        int64_t min_ctx = INT64_MAX;
        for (int64_t c : p.decode_ctx) min_ctx = std::min(min_ctx, c);
        const int64_t cap = std::max<int64_t>(1, min_ctx / (pod::kSmDecodeWarps * 16));
        const int64_t nb = static_cast<int64_t>(p.decode_ctx.size());
        const int64_t items = parents * p.decode_splits, nsm = p.dev.num_sms;
        const int64_t extra = ceil_div(items, nsm) * nsm - items;   // parents needing one more split
        const int64_t ntail = std::min<int64_t>(nb, extra / s.num_kv_heads);
        if (ntail > 0 && p.decode_splits + 1 <= cap) {
            p.dec_tail_start = nb - ntail;
            p.decode_splits += 1;
        }
    }
    auto splits_of = [&](size_t r) {
        return static_cast<int64_t>(r) >= p.dec_tail_start ? p.decode_splits : p.dec_split_base;
    };
    const int page_row0 = p.batch.has_prefill ? 1 : 0;
    p.dec_nsplit.clear();
    for (size_t r = 0; r < p.decode_ctx.size(); ++r) {
        const long ctx = p.decode_ctx[r];
        const long sp_n = std::min<long>(splits_of(r), ctx);
        p.dec_nsplit.push_back(static_cast<int32_t>(sp_n));
        const long base = ctx / sp_n, rem = ctx % sp_n;
        for (int h = 0; h < s.num_kv_heads; ++h) {
            long pos = 0;
            for (long sp = 0; sp < sp_n; ++sp) {
                const long len = base + (sp < rem ? 1 : 0);
                pod::DecodeCta c{};
                c.request = static_cast<int32_t>(r);
                c.kv_head = h;
                c.kv_begin = static_cast<int32_t>(pos);
                c.kv_end = static_cast<int32_t>(pos + len);
                c.split = static_cast<int32_t>(sp);
                c.n_splits = static_cast<int32_t>(sp_n);
                c.ctx = static_cast<int32_t>(ctx);
                c.page_row = page_row0 + static_cast<int32_t>(r);
                p.dctas.push_back(c);
                pos += len;
            }
        }
    }
    p.merge_rows_prefill = 0;
    if (p.batch.has_prefill)
        for (long tile = 0; tile < p.prefill_q_tiles; ++tile)
            if (p.tile_splits[tile] > 1) {
                const long rows = std::min<long>(p.cfg.prefill_tile_q,
                                                 p.batch.prefill.chunk_size - tile * p.cfg.prefill_tile_q);
                p.merge_rows_prefill += static_cast<int32_t>(rows * s.num_q_heads);
            }
    p.merge_rows_decode = 0;
    for (size_t r = 0; r < p.decode_ctx.size(); ++r)
        if (std::min<int64_t>(splits_of(r), p.decode_ctx[r]) > 1)
            p.merge_rows_decode += s.num_q_heads;
}

// make_scheduler_state (gpu_sim.hpp:91-107) over PHYSICAL CTA counts.
void scheduler_ratio(pod_plan& p) {
    const long P = static_cast<long>(p.pctas.size());
    const long D = static_cast<long>(p.dctas.size());
    if (p.opts.policy == POD_POLICY_FIFTY_FIFTY) {
        p.prefill_ratio = 1;
        p.decode_ratio = 1;
    } else if (p.opts.policy == POD_POLICY_PROPORTIONAL) {
        const long g = std::gcd(P, D);
        p.prefill_ratio = g > 0 ? P / g : (P > 0 ? 1 : 0);
        p.decode_ratio = g > 0 ? D / g : (D > 0 ? 1 : 0);
        if (p.prefill_ratio == 0 && p.decode_ratio == 0) p.prefill_ratio = 1;
    } else if (p.opts.policy == POD_POLICY_COMPLEMENT) {
        // one prefill CTA per SM (2 slots): the other slot streams decode
        p.prefill_ratio = P > 0 ? 1 : 0;
        p.decode_ratio = 1;
    } else if (p.opts.policy == POD_POLICY_WARPSPEC) {
        // both roles on every SM for as long as both pools have work
        p.prefill_ratio = P > 0 ? 1 : 0;
        p.decode_ratio = D > 0 ? 1 : 0;
        if (P == 0 && D == 0) p.prefill_ratio = 1;
    } else {
        // proportional share rounded to the per-SM slot count, never starving an op
        const int slots = std::max(2, p.cfg.ctas_per_sm);
        if (P == 0 || D == 0) {
            p.prefill_ratio = P > 0 ? 1 : 0;
            p.decode_ratio = D > 0 ? 1 : 0;
            if (P == 0 && D == 0) p.prefill_ratio = 1;
        } else {
            long pr = std::lround(static_cast<double>(slots) * P / static_cast<double>(P + D));
            pr = std::clamp<long>(pr, 1, slots - 1);
            p.prefill_ratio = pr;
            p.decode_ratio = slots - pr;
        }
    }
}

void layout_workspace(pod_plan& p) {
    auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
    const pod_shape& s = p.shape;
    size_t off = 0;
    p.ws.off_counters = off;
    off = align(off + sizeof(pod::SchedCounters));
    p.ws.off_pctas = off;
    off = align(off + p.pctas.size() * sizeof(pod::PrefillCta));
    p.ws.off_dctas = off;
    off = align(off + p.dctas.size() * sizeof(pod::DecodeCta));
    p.ws.off_tile_splits = off;
    off = align(off + p.tile_splits.size() * sizeof(int32_t));
    const int64_t chunk = p.batch.has_prefill ? p.batch.prefill.chunk_size : 0;
    const size_t pp = p.max_prefill_splits > 1 ? static_cast<size_t>(p.max_prefill_splits) * chunk * s.num_q_heads : 0;
    p.ws.off_ppart_o = off;
    off = align(off + pp * s.head_dim * sizeof(float));
    p.ws.off_ppart_lse = off;
    off = align(off + pp * sizeof(float));
    const size_t dp = p.decode_splits > 1 ? static_cast<size_t>(p.decode_ctx.size()) * p.decode_splits * s.num_q_heads : 0;
    p.ws.off_dpart_o = off;
    off = align(off + dp * s.head_dim * sizeof(float));
    p.ws.off_dpart_lse = off;
    off = align(off + dp * sizeof(float));
    p.ws.off_dec_pos = off;
    off = align(off + p.decode_ctx.size() * sizeof(int32_t));
    p.ws.off_dec_nsplit = off;
    off = align(off + p.decode_ctx.size() * sizeof(int32_t));
    p.ws.off_vshadow = off;
    off = align(off + static_cast<size_t>(p.vs_pages) * s.num_kv_heads * p.batch.page_size * s.head_dim * 2);
    p.ws.total = off;
    p.dec_pos.clear();
    for (int64_t c : p.decode_ctx) p.dec_pos.push_back(static_cast<int32_t>(c - 1));
}

pod_tile_config b200_tile_config(const pod_plan& p) {
    // One tcgen05 M-block (128 packed (row, q-head) rows) per prefill CTA; the
    // kernel's KV tile is 64 keys.  Two CTAs per SM (smem ~112 KB each).
    pod_tile_config c = make_tile_config(2);
    const int group = p.shape.num_q_heads / p.shape.num_kv_heads;
    // warp-specialised kernel: two 128-row M-blocks per prefill item (pair engine)
    const bool two_blocks = p.opts.policy == POD_POLICY_WARPSPEC;
    const int rows = (two_blocks ? 2 : 1) * pod::kMBlock;
    c.prefill_tile_q = std::max(1, rows / group);
    c.tile_kv = pod::kKvTile;
    c.shared_mem_per_cta = static_cast<double>(p.opts.policy == POD_POLICY_WARPSPEC ? pod::sm_smem_bytes(false)
                                                                                   : pod::fused_smem_bytes());
    c.virtual_decode = 1;
    return c;
}

// Decode share of the serial time from algorithmic work at measured B200 rates
// (prefill ~0.68 PFLOP/s with the hi+lo P split, paged decode ~6.6 TB/s).
double decode_share(const pod_plan& p) {
    if (!p.batch.has_prefill) return 1.0;
    if (p.decode_ctx.empty()) return 0.0;
    const auto& pf = p.batch.prefill;
    const double C = static_cast<double>(pf.chunk_size), off = static_cast<double>(pf.position_offset);
    const double flops = 4.0 * p.shape.head_dim * p.shape.num_q_heads * (C * off + C * (C + 1) / 2.0);
    double bytes = 0;
    for (int64_t c : p.decode_ctx) bytes += 4.0 * c * p.shape.num_kv_heads * p.shape.head_dim;
    const double t_p = flops / 0.68e15, t_d = bytes / 6.6e12;
    return t_d / (t_p + t_d);
}

void build(pod_plan& p) {
    validate_batch(p);
    if (p.opts.policy == POD_POLICY_AUTO) {
        // measured on B200: the one-CTA-per-SM kernel wins unless the
        // prefill dominates almost entirely (decode share < 0.1: chunks >= 2K next to a
        // few decodes, e.g. 2048@16K + 8 x 16K: 835 vs 783 us, 4096@4K + 8 x 4K: 302 vs
        // 280 us); with the 64-key pair engine it wins C2 B = 8 (462 vs 493 us) and
        // 512@4K + 8 x 4K (106 vs 147 us)
        // Decode-only and short-context batches keep the two-CTA kernel: more decode
        // groups per SM amortise the per-item latency (64 x 2K decode-only: 107 vs
        // 126 us; 512@1536 + 64 x 1K: 93 vs 106 us).
        double avg_ctx = 0;
        for (int64_t c : p.decode_ctx) avg_ctx += static_cast<double>(c);
        avg_ctx = p.decode_ctx.empty() ? 0 : avg_ctx / static_cast<double>(p.decode_ctx.size());
        // (the warp-specialised pair engine needs the B200 tile config's 256-row items)
        const bool b200_tiles = p.opts.tile_mode == POD_TILE_B200 && !p.opts.tile_override;
        p.opts.policy = (b200_tiles && p.batch.has_prefill && decode_share(p) >= 0.1 && avg_ctx >= 2048)
                            ? POD_POLICY_WARPSPEC
                            : POD_POLICY_COMPLEMENT;
    }
    if (p.opts.tile_override) {
        p.cfg = *p.opts.tile_override;
        if (p.cfg.prefill_tile_q < 1 || p.cfg.tile_kv < 1 || p.cfg.warps_per_cta < 1)
            fail(POD_ERR_INVALID_ARGUMENT, "TileConfig: tiles must be >= 1");
    } else if (p.opts.tile_mode == POD_TILE_B200) {
        p.cfg = b200_tile_config(p);
        if (p.opts.ctas_per_sm == 4) fail(POD_ERR_UNSUPPORTED, "B200 tile mode: 4 CTAs/SM not built yet");
        // Split selection per batch shape: prefill items must be fine enough to
        // fill the slots the decode leaves behind.  Decode share of the serial
        // time from algorithmic work at measured B200 rates (prefill ~0.68 PFLOP/s,
        // paged decode ~6.6 TB/s): > 0.55 -> 2 waves (reference rule), > 0.4 -> 4, else 8.
        if (p.opts.split_wave_cap <= 0 && p.batch.has_prefill && !p.decode_ctx.empty()) {
            const double share = decode_share(p);
            if (p.opts.policy == POD_POLICY_WARPSPEC)
                // one prefill engine per SM keeps working while the decode runs;
                // KV splits only pay their merge (measured: cap 1 best for C1, C2)
                p.cfg.split_wave_cap = 1;
            else
                p.cfg.split_wave_cap = share > 0.55 ? 2 : (share > 0.4 ? 4 : 8);
        }
    } else {
        if (p.opts.ctas_per_sm != 0) {
            p.cfg = make_tile_config(p.opts.ctas_per_sm);
        } else {
            // select_tile_config (work_decomp.hpp:139-145)
            const bool prefill_dominant =
                estimate_prefill_serial(p) >= estimate_decode_serial(p) && p.batch.has_prefill;
            p.cfg = make_tile_config(prefill_dominant ? 2 : 4);
        }
    }
    // the warp-specialised pair engine runs at most two 128-row M-blocks per item
    if (p.opts.policy == POD_POLICY_WARPSPEC && p.batch.has_prefill &&
        p.cfg.prefill_tile_q * (p.shape.num_q_heads / p.shape.num_kv_heads) > 2 * pod::kMBlock)
        fail(POD_ERR_UNSUPPORTED, "POD_POLICY_WARPSPEC: prefill_tile_q x group must be <= 256 (use POD_TILE_B200)");
    // -1 keeps the config's flag (reference configs: off; B200 config: on)
    if (p.opts.virtual_decode == 0) p.cfg.virtual_decode = 0;
    if (p.opts.virtual_decode == 1) p.cfg.virtual_decode = 1;
    if (p.opts.split_wave_cap > 0) p.cfg.split_wave_cap = p.opts.split_wave_cap;
    if (p.batch.has_prefill) decompose_prefill(p);
    if (!p.decode_ctx.empty()) decompose_decode(p);
    lower(p);
    scheduler_ratio(p);
    p.smem_bytes = p.opts.policy == POD_POLICY_WARPSPEC ? pod::sm_smem_bytes(p.pf_db) : pod::fused_smem_bytes();
    // POD_PRECISION_F16PV on bf16 data needs V in fp16.  The two-CTA kernel's prefill CTA
    // converting every V tile it streams sits on its softmax warps' critical path (S is
    // double-buffered there): prefill-alone at C2 is 327 us with it, 256 us without (bf16 P,
    // same MMA count).  Its plans convert the prefill request's V once per launch into a
    // dense fp16 shadow in the workspace instead (pod_attn.cu, v_shadow_kernel; the POD
    // kernel is its programmatic dependent and waits at its first V load).  The pair engines
    // hide most of the conversion behind their single-buffered S: the shadow pays on the
    // prefill-dominant 64-key plans (fused C2 B=8 365 -> 354 us, B=16 388 -> 370) and not
    // on the decode-dominant 32-key ones (C2 B=64 686 -> 693: one more HBM pass).
    p.vs_pages = 0;
    if (p.batch.has_prefill && p.batch.dtype == POD_DTYPE_BF16 && p.opts.precision == POD_PRECISION_F16PV &&
        (p.opts.policy == POD_POLICY_COMPLEMENT || (p.opts.policy == POD_POLICY_WARPSPEC && p.pf_tn64)))
        p.vs_pages = static_cast<int32_t>(
            ceil_div(p.batch.prefill.position_offset + p.batch.prefill.chunk_size, int64_t(p.batch.page_size)));
    layout_workspace(p);
}

}  // namespace

extern "C" {

void pod_device_reference_default(pod_device* out) {
    // GpuSpec defaults (gpu.hpp:12-37).
    out->num_sms = 108;
    out->compute_rate_per_sm = 0.25;
    out->mem_bandwidth_total = 108.0;
    out->mem_bandwidth_per_sm = 1.2;
    out->mem_interference = 0.25;
    out->max_ctas_per_sm = 4;
    out->shared_mem_per_sm = 167936.0;
}

void pod_options_default(pod_options* out) {
    std::memset(out, 0, sizeof(*out));
    out->policy = POD_POLICY_AUTO;
    out->tile_mode = POD_TILE_B200;
    out->ctas_per_sm = 0;
    out->virtual_decode = -1;
    out->split_wave_cap = 0;
    out->decode_splits = 0;
    out->tile_override = nullptr;
    out->precision = POD_PRECISION_F16PV;
    out->out_dtype = POD_OUT_F32;
    out->prefill_tile_keys = 0;
    out->prefill_s_buffers = 0;
}

pod_status pod_attn_plan(const pod_shape* shape, const pod_batch* batch, const pod_device* dev,
                         const pod_options* opts, pod_plan** out) {
    if (!shape || !batch || !dev || !out) return POD_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    pod_plan* p = new pod_plan();
    try {
        p->shape = *shape;
        p->batch = *batch;
        if (batch->num_decodes < 0 || (batch->num_decodes > 0 && !batch->decode_context_len))
            fail(POD_ERR_INVALID_ARGUMENT, "pod_batch: decode_context_len missing");
        p->decode_ctx.assign(batch->decode_context_len, batch->decode_context_len + batch->num_decodes);
        p->batch.decode_context_len = nullptr;
        if (p->batch.page_size <= 0) p->batch.page_size = 16;
        p->dev = *dev;
        if (p->dev.num_sms < 1 || p->dev.num_sms > pod::kMaxSms)
            fail(POD_ERR_INVALID_ARGUMENT, "pod_device: num_sms out of range");
        if (opts)
            p->opts = *opts;
        else
            pod_options_default(&p->opts);
        {
            const int32_t pol = p->opts.policy;
            if (!(pol == POD_POLICY_FIFTY_FIFTY || pol == POD_POLICY_PROPORTIONAL || pol == POD_POLICY_CLAMPED ||
                  pol == POD_POLICY_COMPLEMENT || pol == POD_POLICY_WARPSPEC || pol == POD_POLICY_AUTO))
                fail(POD_ERR_INVALID_ARGUMENT, "pod_options: policy must be a POD_POLICY_* value (4-6 are retired)");
        }
        if (p->opts.precision < POD_PRECISION_SPLIT || p->opts.precision > POD_PRECISION_F16PV)
            fail(POD_ERR_INVALID_ARGUMENT, "pod_options: precision must be a POD_PRECISION_* value");
        if (p->opts.out_dtype < POD_OUT_F32 || p->opts.out_dtype > POD_OUT_F16)
            fail(POD_ERR_INVALID_ARGUMENT, "pod_options: out_dtype must be a POD_OUT_* value");
        if (p->opts.prefill_s_buffers < 0 || p->opts.prefill_s_buffers > 2)
            fail(POD_ERR_INVALID_ARGUMENT, "pod_options: prefill_s_buffers must be 0, 1 or 2");
        if (p->opts.prefill_tile_keys != 0 && p->opts.prefill_tile_keys != 32 && p->opts.prefill_tile_keys != 64)
            fail(POD_ERR_INVALID_ARGUMENT, "pod_options: prefill_tile_keys must be 0, 32 or 64");
        build(*p);
        p->opts.tile_override = nullptr;  // do not keep caller pointers
        *out = p;
        return POD_OK;
    } catch (const Status& s) {
        pod::set_last_error(s.msg);
        delete p;
        return s.code;
    } catch (const std::exception& e) {
        pod::set_last_error(e.what());
        delete p;
        return POD_ERR_INVALID_ARGUMENT;
    }
}

void pod_attn_plan_destroy(pod_plan* plan) { delete plan; }

pod_status pod_attn_plan_get_info(const pod_plan* p, pod_plan_info* out) {
    if (!p || !out) return POD_ERR_INVALID_ARGUMENT;
    std::memset(out, 0, sizeof(*out));
    out->config = p->cfg;
    out->prefill_splits = p->batch.has_prefill ? p->prefill_splits : 0;
    out->num_prefill_tasks = static_cast<int64_t>(p->prefill_tasks.size());
    out->num_decode_tasks = static_cast<int64_t>(p->decode_tasks.size());
    out->num_prefill_ctas = static_cast<int64_t>(p->pctas.size());
    out->num_decode_ctas = static_cast<int64_t>(p->dctas.size());
    out->decode_splits = p->decode_splits;
    out->prefill_ratio = p->prefill_ratio;
    out->decode_ratio = p->decode_ratio;
    out->smem_bytes = p->smem_bytes;
    out->workspace_bytes = static_cast<int64_t>(p->ws.total);
    out->num_merge_rows_prefill = p->merge_rows_prefill;
    out->num_merge_rows_decode = p->merge_rows_decode;
    out->policy = p->opts.policy;
    out->prefill_tile_keys = p->opts.policy == POD_POLICY_WARPSPEC && p->batch.has_prefill ? (p->pf_tn64 ? 64 : 32) : 0;
    out->prefill_s_buffers = out->prefill_tile_keys == 0 ? 0 : (!p->pf_tn64 || p->pf_db) ? 2 : 1;
    return POD_OK;
}

pod_status pod_attn_plan_tasks(const pod_plan* p, pod_task* prefill, int64_t* n_prefill,
                               pod_task* decode, int64_t* n_decode) {
    if (!p || !n_prefill || !n_decode) return POD_ERR_INVALID_ARGUMENT;
    const int64_t np = static_cast<int64_t>(p->prefill_tasks.size());
    const int64_t nd = static_cast<int64_t>(p->decode_tasks.size());
    if (prefill) {
        if (*n_prefill < np) return POD_ERR_INVALID_ARGUMENT;
        std::copy(p->prefill_tasks.begin(), p->prefill_tasks.end(), prefill);
    }
    if (decode) {
        if (*n_decode < nd) return POD_ERR_INVALID_ARGUMENT;
        std::copy(p->decode_tasks.begin(), p->decode_tasks.end(), decode);
    }
    *n_prefill = np;
    *n_decode = nd;
    return POD_OK;
}

size_t pod_attn_workspace_bytes(const pod_plan* p) { return p ? p->ws.total : 0; }

pod_status pod_attn_set_role_log(pod_plan* p, int32_t* device_log) {
    if (!p) return POD_ERR_INVALID_ARGUMENT;
    p->role_log = device_log;
    return POD_OK;
}

const char* pod_status_string(pod_status s) {
    switch (s) {
        case POD_OK: return "ok";
        case POD_ERR_INVALID_ARGUMENT: return "invalid_argument";
        case POD_ERR_LOGIC: return "logic_error";
        case POD_ERR_DOMAIN: return "domain_error";
        case POD_ERR_OUT_OF_RANGE: return "out_of_range";
        case POD_ERR_CONFIG: return "config_error";
        case POD_ERR_CUDA: return "cuda_error";
        case POD_ERR_UNSUPPORTED: return "unsupported";
    }
    return "unknown";
}

int pod_attn_abi_version(void) { return POD_ATTN_ABI_VERSION; }

}  // extern "C"
