// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper that compiles the REFERENCE's own headers
// (/root/reference/proj/include/attnsim/*.hpp, included in place via -I; no
// reference source is copied into this repo) into oracle/_ref/libattnsim_ref.so
// (see oracle/Makefile).  It is used to
//   * pin the C restatement (oracle/pod_oracle.c) and generate tests/golden/,
//   * check the product planner field-by-field against decompose_hybrid,
//   * time the reference CPU path for bench.py's cpu_baseline / --impl reference.
// Exceptions are mapped to the status codes of include/pod_attn.h.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <vector>

#include "attnsim/attention.hpp"
#include "attnsim/csv.hpp"  // parallel_for (csv.hpp:57-73)
#include "attnsim/gpu.hpp"
#include "attnsim/gpu_sim.hpp"
#include "attnsim/rng.hpp"
#include "attnsim/serving.hpp"
#include "attnsim/types.hpp"
#include "attnsim/work_decomp.hpp"

using namespace attnsim;

namespace {

enum : int {
    kOk = 0,
    kInvalid = 1,
    kLogic = 2,
    kDomain = 3,
    kOutOfRange = 4,
    kConfig = 5,
    kOther = 9,
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const ConfigError&) {
        return kConfig;
    } catch (const std::out_of_range&) {
        return kOutOfRange;
    } catch (const std::invalid_argument&) {
        return kInvalid;
    } catch (const std::domain_error&) {
        return kDomain;
    } catch (const std::logic_error&) {
        return kLogic;
    } catch (...) {
        return kOther;
    }
}

ModelShape make_shape(int hq, int hkv, int d, double scale) {
    ModelShape s;
    s.num_q_heads = hq;
    s.num_kv_heads = hkv;
    s.head_dim = d;
    s.scale = scale;
    return s;
}

KVCache make_cache(const double* k, const double* v, long ctx, int hkv, int d) {
    KVCache c(ctx, hkv, d);
    const size_t n = static_cast<size_t>(ctx) * hkv * d;
    if (n) {
        std::memcpy(c.k.data(), k, n * sizeof(double));
        std::memcpy(c.v.data(), v, n * sizeof(double));
    }
    return c;
}

}  // namespace

extern "C" {

// Same layout as pod_task in include/pod_attn.h.
struct ref_task {
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
};

struct ref_tile_config {
    int64_t prefill_tile_q;
    int64_t decode_tile_q;
    int64_t tile_kv;
    int32_t warps_per_cta;
    int32_t ctas_per_sm;
    double shared_mem_per_cta;
    int32_t virtual_decode;
    int32_t split_wave_cap;
};

struct ref_gpu_spec {
    int32_t num_sms;
    double compute_rate_per_sm;
    double mem_bandwidth_total;
    double mem_bandwidth_per_sm;
    double mem_interference;
    int32_t max_ctas_per_sm;
    double shared_mem_per_sm;
};

// Rng (rng.hpp:11-47): n draws of next_double().
void ref_rng_doubles(uint64_t seed, int64_t n, double* out) {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.next_double();
}

void ref_rng_longs(uint64_t seed, int64_t n, int64_t lo, int64_t hi, int64_t* out) {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.next_long(lo, hi);
}

int ref_gqa_kv_head(int q_head, int hq, int hkv, int* out) {
    return guarded([&] { *out = gqa_kv_head(q_head, make_shape(hq, hkv, 1, 1.0)); });
}

void ref_split_ranges(int64_t n, int64_t splits, int64_t* begin, int64_t* end) {
    auto r = split_ranges(n, splits);
    for (size_t i = 0; i < r.size(); ++i) {
        begin[i] = r[i].begin;
        end[i] = r[i].end;
    }
}

int ref_naive_attention(const double* q, int64_t m, const double* k, const double* v, int64_t n,
                        int64_t d, double scale, int has_causal, int64_t causal_offset,
                        double* out) {
    return guarded([&] {
        Matd Q(m, d), K(n, d), V(n, d);
        if (m * d) std::memcpy(Q.data.data(), q, sizeof(double) * m * d);
        if (n * d) {
            std::memcpy(K.data.data(), k, sizeof(double) * n * d);
            std::memcpy(V.data.data(), v, sizeof(double) * n * d);
        }
        Matd o = has_causal ? naive_attention(Q, K, V, scale, std::optional<long>(causal_offset))
                            : naive_attention(Q, K, V, scale);
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
    });
}

int ref_tiled_prefill(const double* q, int64_t chunk, int64_t offset, const double* k,
                      const double* v, int64_t ctx, int hq, int hkv, int d, double scale,
                      int64_t tile_q, int64_t tile_kv, double* out) {
    return guarded([&] {
        QueryChunk qc(chunk, hq, d, offset);
        if (qc.q.size()) std::memcpy(qc.q.data(), q, sizeof(double) * qc.q.size());
        KVCache cache = make_cache(k, v, ctx, hkv, d);
        Matd o = tiled_prefill_attention(qc, cache, make_shape(hq, hkv, d, scale), tile_q, tile_kv);
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
    });
}

int ref_decode_splitk(const double* q, const double* k, const double* v, int64_t ctx, int hq,
                      int hkv, int d, double scale, int64_t num_splits, double* o_parts,
                      double* lse_parts, int64_t* ranges, int64_t* n_parts) {
    return guarded([&] {
        DecodeQuery dq(hq, d);
        std::memcpy(dq.q.data(), q, sizeof(double) * dq.q.size());
        KVCache cache = make_cache(k, v, ctx, hkv, d);
        auto parts = decode_attention_splitk(dq, cache, make_shape(hq, hkv, d, scale), num_splits);
        for (size_t s = 0; s < parts.size(); ++s) {
            std::memcpy(o_parts + s * hq * d, parts[s].o.data.data(), sizeof(double) * hq * d);
            std::memcpy(lse_parts + s * hq, parts[s].lse.data(), sizeof(double) * hq);
            ranges[2 * s] = parts[s].kv_range.begin;
            ranges[2 * s + 1] = parts[s].kv_range.end;
        }
        *n_parts = static_cast<int64_t>(parts.size());
    });
}

int ref_merge_partials(const double* o_parts, const double* lse_parts, const int64_t* ranges,
                       int64_t n, int64_t rows, int64_t d, double* out) {
    return guarded([&] {
        std::vector<AttentionPartial> parts(n);
        for (int64_t i = 0; i < n; ++i) {
            parts[i].o = Matd(rows, d);
            std::memcpy(parts[i].o.data.data(), o_parts + i * rows * d, sizeof(double) * rows * d);
            parts[i].lse.assign(lse_parts + i * rows, lse_parts + (i + 1) * rows);
            parts[i].kv_range = Interval{ranges[2 * i], ranges[2 * i + 1]};
        }
        Matd o = merge_partials(parts);
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
    });
}

int ref_decode_attention(const double* q, const double* k, const double* v, int64_t ctx, int hq,
                         int hkv, int d, double scale, double* out) {
    return guarded([&] {
        DecodeQuery dq(hq, d);
        std::memcpy(dq.q.data(), q, sizeof(double) * dq.q.size());
        KVCache cache = make_cache(k, v, ctx, hkv, d);
        Matd o = decode_attention(dq, cache, make_shape(hq, hkv, d, scale));
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
    });
}

// ---------------------------------------------------------------- planner --

static GpuSpec to_gpu(const ref_gpu_spec* g) {
    GpuSpec s;
    s.num_sms = g->num_sms;
    s.compute_rate_per_sm = g->compute_rate_per_sm;
    s.mem_bandwidth_total = g->mem_bandwidth_total;
    s.mem_bandwidth_per_sm = g->mem_bandwidth_per_sm;
    s.mem_interference = g->mem_interference;
    s.max_ctas_per_sm = g->max_ctas_per_sm;
    s.shared_mem_per_sm = g->shared_mem_per_sm;
    return s;
}

static TileConfig to_cfg(const ref_tile_config* c) {
    TileConfig t;
    t.prefill_tile_q = c->prefill_tile_q;
    t.decode_tile_q = c->decode_tile_q;
    t.tile_kv = c->tile_kv;
    t.warps_per_cta = c->warps_per_cta;
    t.ctas_per_sm = c->ctas_per_sm;
    t.shared_mem_per_cta = c->shared_mem_per_cta;
    t.virtual_decode = c->virtual_decode != 0;
    t.split_wave_cap = c->split_wave_cap;
    return t;
}

static void from_cfg(const TileConfig& t, ref_tile_config* c) {
    c->prefill_tile_q = t.prefill_tile_q;
    c->decode_tile_q = t.decode_tile_q;
    c->tile_kv = t.tile_kv;
    c->warps_per_cta = t.warps_per_cta;
    c->ctas_per_sm = t.ctas_per_sm;
    c->shared_mem_per_cta = t.shared_mem_per_cta;
    c->virtual_decode = t.virtual_decode ? 1 : 0;
    c->split_wave_cap = t.split_wave_cap;
}

static HybridBatchSpec make_batch(int hq, int hkv, int d, double scale, int has_prefill,
                                  int64_t chunk, int64_t prompt, int64_t offset, int64_t n_dec,
                                  const int64_t* dec_ctx) {
    HybridBatchSpec b;
    b.shape = make_shape(hq, hkv, d, scale);
    if (has_prefill) b.prefill = PrefillSpec{chunk, prompt, offset};
    for (int64_t i = 0; i < n_dec; ++i) b.decodes.push_back(DecodeSpec{dec_ctx[i]});
    return b;
}

static void to_task(const CtaTask& t, ref_task* o) {
    o->op = static_cast<int32_t>(t.op);
    o->request_id = t.request_id;
    o->kv_head = t.kv_head;
    o->q_tile = t.q_tile;
    o->kv_begin = t.kv_split.begin;
    o->kv_end = t.kv_split.end;
    o->is_virtual = t.is_virtual ? 1 : 0;
    o->slot_quanta = t.slot_quanta;
    o->barrier_segments = t.barrier_segments;
    o->compute_work = t.compute_work;
    o->memory_work = t.memory_work;
}

int ref_make_tile_config(int ctas_per_sm, ref_tile_config* out) {
    return guarded([&] { from_cfg(make_tile_config(ctas_per_sm), out); });
}

int ref_select_tile_config(int hq, int hkv, int d, double scale, int has_prefill, int64_t chunk,
                           int64_t prompt, int64_t offset, int64_t n_dec, const int64_t* dec_ctx,
                           const ref_gpu_spec* gpu, ref_tile_config* out) {
    return guarded([&] {
        auto b = make_batch(hq, hkv, d, scale, has_prefill, chunk, prompt, offset, n_dec, dec_ctx);
        from_cfg(select_tile_config(b, to_gpu(gpu)), out);
    });
}

int ref_limit_prefill_splits(int64_t natural, const ref_gpu_spec* gpu, const ref_tile_config* cfg,
                             int64_t* out) {
    return guarded([&] { *out = limit_prefill_splits(natural, to_gpu(gpu), to_cfg(cfg)); });
}

// decompose_hybrid (work_decomp.hpp:249-261).  cfg == nullptr selects the
// config with select_tile_config; the chosen config is written to cfg_out.
// Task arrays must hold at least *n_prefill / *n_decode entries on input
// (capacities); on output they hold the counts.
int ref_decompose_hybrid(int hq, int hkv, int d, double scale, int has_prefill, int64_t chunk,
                         int64_t prompt, int64_t offset, int64_t n_dec, const int64_t* dec_ctx,
                         const ref_gpu_spec* gpu, const ref_tile_config* cfg,
                         ref_tile_config* cfg_out, ref_task* prefill_tasks, int64_t* n_prefill,
                         ref_task* decode_tasks, int64_t* n_decode) {
    return guarded([&] {
        auto b = make_batch(hq, hkv, d, scale, has_prefill, chunk, prompt, offset, n_dec, dec_ctx);
        GpuSpec g = to_gpu(gpu);
        WorkDecomposition wd = cfg ? decompose_hybrid(b, g, to_cfg(cfg)) : decompose_hybrid(b, g);
        from_cfg(wd.config, cfg_out);
        if ((int64_t)wd.prefill_tasks.size() > *n_prefill ||
            (int64_t)wd.decode_tasks.size() > *n_decode)
            throw std::length_error("ref_decompose_hybrid: task capacity");
        for (size_t i = 0; i < wd.prefill_tasks.size(); ++i)
            to_task(wd.prefill_tasks[i], prefill_tasks + i);
        for (size_t i = 0; i < wd.decode_tasks.size(); ++i)
            to_task(wd.decode_tasks[i], decode_tasks + i);
        *n_prefill = (int64_t)wd.prefill_tasks.size();
        *n_decode = (int64_t)wd.decode_tasks.size();
    });
}

// make_scheduler_state + sm_aware_assign (gpu_sim.hpp:91-131) replayed over
// a sequence of CTA arrivals.
void ref_sched_replay(int proportional, int64_t p_total, int64_t d_total, int num_sms,
                      const int* sm_ids, int64_t n, int64_t* pr, int64_t* dr, int* op_out,
                      int64_t* id_out) {
    auto st = make_scheduler_state(proportional ? SmPolicy::Proportional : SmPolicy::FiftyFifty,
                                   p_total, d_total, num_sms);
    *pr = st.prefill_ratio;
    *dr = st.decode_ratio;
    for (int64_t i = 0; i < n; ++i) {
        auto pick = sm_aware_assign(sm_ids[i], st);
        if (!pick) {
            op_out[i] = -1;
            id_out[i] = -1;
        } else {
            op_out[i] = static_cast<int>(pick->op);
            id_out[i] = pick->cta_id;
        }
    }
}

// ------------------------------------------------------- CPU baseline path --
//
// Runs the reference's own hot-path functions over a list of shards with the
// reference's parallel_for (csv.hpp:59-73) and returns elapsed seconds.
//   prefill shard = tiled_prefill_attention on QueryChunk(rows, group, d,
//     offset + r0) against a one-KV-head cache (ModelShape{group, 1, d}) --
//     an exact restriction by GQA consistency (test_attention.cpp:252-270)
//     and row independence (attention.hpp:183-212);
//   decode shard  = decode_attention(DecodeQuery(group, d), one-KV-head cache).
struct ref_shard {
    int32_t kind;        // 0 prefill, 1 decode
    int32_t group;       // q heads served by the KV head
    int64_t rows;        // prefill rows (1 for decode)
    int64_t offset;      // absolute position of the first prefill row
    int64_t ctx;         // keys in k/v
    const double* q;     // [rows][group][d] or [group][d]
    const double* k;     // [ctx][1][d]
    const double* v;     // [ctx][1][d]
    double* out;         // [rows][group*d] or [group][d]
};

double ref_run_shards(const ref_shard* shards, int64_t n, int d, double scale, int64_t tile_q,
                      int64_t tile_kv, int threads, int* status) {
    std::vector<int> st(n, 0);
    auto t0 = std::chrono::steady_clock::now();
    parallel_for((size_t)n, threads, [&](size_t i) {
        const ref_shard& s = shards[i];
        st[i] = guarded([&] {
            ModelShape shape = make_shape(s.group, 1, d, scale);
            KVCache cache = make_cache(s.k, s.v, s.ctx, 1, d);
            if (s.kind == 0) {
                QueryChunk qc(s.rows, s.group, d, s.offset);
                std::memcpy(qc.q.data(), s.q, sizeof(double) * qc.q.size());
                Matd o = tiled_prefill_attention(qc, cache, shape, tile_q, tile_kv);
                std::memcpy(s.out, o.data.data(), sizeof(double) * o.data.size());
            } else {
                DecodeQuery dq(s.group, d);
                std::memcpy(dq.q.data(), s.q, sizeof(double) * dq.q.size());
                Matd o = decode_attention(dq, cache, shape);
                std::memcpy(s.out, o.data.data(), sizeof(double) * o.data.size());
            }
        });
    });
    auto t1 = std::chrono::steady_clock::now();
    *status = 0;
    for (int x : st)
        if (x) *status = x;
    return std::chrono::duration<double>(t1 - t0).count();
}

// Serving simulator (serving.hpp): trace generation and the iteration loop with a
// linear cost c0 + c1 * tokens (the cost the reference's own serving tests use), for
// pinning the Python serving-loop port (paper_2410_18038_b200/serving.py).
static TokenDist make_dist(int kind, double a, double b) {
    TokenDist t;
    t.kind = kind == 0 ? TokenDist::Kind::Fixed : kind == 1 ? TokenDist::Kind::Uniform : TokenDist::Kind::LogNormal;
    t.a = a;
    t.b = b;
    return t;
}

int ref_generate_trace(double qps, int64_t n, int pk, double pa, double pb, int dk, double da, double db,
                       uint64_t seed, double* arrival, int64_t* ptok, int64_t* dtok) {
    return guarded([&] {
        auto tr = generate_trace(qps, n, make_dist(pk, pa, pb), make_dist(dk, da, db), seed);
        for (int64_t i = 0; i < n; ++i) {
            arrival[i] = tr[i].arrival_time;
            ptok[i] = tr[i].prefill_tokens;
            dtok[i] = tr[i].decode_tokens;
        }
    });
}

// metrics: ttft50, ttft99, tbt50, tbt99, lat50, lat99, throughput, stall@200, stall@500
int ref_run_serving_linear(int64_t n, const double* arrival, const int64_t* ptok, const int64_t* dtok,
                           int policy_kind, int64_t chunk, int64_t max_batch, int64_t token_budget, double c0,
                           double c1, int64_t max_iters, double* it_t0, double* it_t1, int64_t* it_preq,
                           int64_t* it_ptok, int64_t* it_ndec, int64_t* n_iters, double* ttft, double* latency,
                           double* metrics) {
    return guarded([&] {
        std::vector<Request> tr(n);
        for (int64_t i = 0; i < n; ++i) tr[i] = Request{arrival[i], ptok[i], dtok[i]};
        SchedulerPolicy pol = policy_kind == 0 ? SchedulerPolicy::prefill_prioritized()
                                               : SchedulerPolicy::chunked_hybrid(chunk, max_batch, token_budget);
        auto cost = [&](const HybridBatchSpec& b, bool) {
            long tokens = b.prefill ? b.prefill->chunk_size : 0;
            return c0 + c1 * (tokens + (double)b.decodes.size());
        };
        ModelShape shape{16, 4, 128, 11.3137};
        auto r = run_serving(tr, pol, cost, false, shape, {200.0, 500.0});
        *n_iters = (int64_t)r.iterations.size();
        for (size_t i = 0; i < r.iterations.size() && (int64_t)i < max_iters; ++i) {
            it_t0[i] = r.iterations[i].t_start;
            it_t1[i] = r.iterations[i].t_end;
            it_preq[i] = r.iterations[i].prefill_request;
            it_ptok[i] = r.iterations[i].prefill_tokens;
            it_ndec[i] = r.iterations[i].decode_requests;
        }
        for (int64_t i = 0; i < n; ++i) {
            ttft[i] = r.ttft[i];
            latency[i] = r.latency[i];
        }
        const Metrics& m = r.metrics;
        double v[9] = {m.ttft_p50, m.ttft_p99, m.tbt_p50, m.tbt_p99, m.latency_p50, m.latency_p99, m.throughput,
                       m.stall_pct_at[0].second, m.stall_pct_at[1].second};
        std::memcpy(metrics, v, sizeof(v));
    });
}

// ------------------------------------------------- DES predictor (N3) --

// The reference's discrete-event model of one hybrid batch on `gpu`
// (gpu_sim.hpp:781-816, work_decomp.hpp:139-145,249-261), for cross-validation
// against measured B200 times.  out[8] =
//   {serial makespan (select_tile_config decomposition, Strategy::Serial),
//    best fused makespan (best_fused_makespan: {2,4} CTAs/SM x {5050, prop}),
//    oracle_runtime (combined roofline of the same tasks),
//    prefill-alone makespan, decode-alone makespan (Serial, same config),
//    selected ctas_per_sm, streams makespan, fused makespan at the selected config (5050)}
int ref_des_predict(int hq, int hkv, int d, double scale, int has_prefill, int64_t chunk,
                    int64_t prompt, int64_t offset, int64_t n_dec, const int64_t* dec_ctx,
                    const ref_gpu_spec* gpu, double* out) {
    return guarded([&] {
        auto b = make_batch(hq, hkv, d, scale, has_prefill, chunk, prompt, offset, n_dec, dec_ctx);
        const GpuSpec g = to_gpu(gpu);
        SimOptions opt;
        opt.record_trace = false;
        const TileConfig cfg = select_tile_config(b, g);
        const auto launches = make_attention_launches(decompose_hybrid(b, g, cfg));
        out[0] = simulate(g, launches, ExecutionStrategy::serial(), 0, opt).makespan;
        out[1] = best_fused_makespan(g, b, 0);
        out[2] = oracle_runtime(g, launches);
        out[3] = out[4] = 0;
        for (size_t i = 0; i < launches.size(); ++i) {
            const double t = simulate(g, {launches[i]}, ExecutionStrategy::serial(), 0, opt).makespan;
            out[launches[i].stream_id == 0 ? 3 : 4] = t;
        }
        out[5] = cfg.ctas_per_sm;
        out[6] = simulate(g, launches, ExecutionStrategy::streams(), 0, opt).makespan;
        out[7] = simulate(g, launches, ExecutionStrategy::sm_aware(SmPolicy::FiftyFifty), 0, opt).makespan;
    });
}

}  // extern "C"
