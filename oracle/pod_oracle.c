/*
 * pod_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C, double-precision restatement of the reference's attention
 * numerics (arxiv/paper_2410_18038, `attnsim`), used by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg to check the
 * CUDA path.  Nothing under paper_2410_18038_b200/ links or loads this file.
 *
 * Parity status: PINNED.  Every function here is checked (tests/test_oracle.py)
 * against (a) the golden vectors in tests/golden/ that were produced by the
 * reference's own headers compiled into oracle/_ref/ (oracle/Makefile), and
 * (b) the reference test expectations of proj/tests/test_attention.cpp.
 *
 * Citations are `file:line` relative to /root/reference/proj/include/attnsim/.
 *
 * Layouts follow the reference:
 *   q chunk   [chunk][Hq][d]          (attention.hpp:45-69, q_at :229-231)
 *   kv cache  [ctx][Hkv][d]           (attention.hpp:20-43, index :202-204)
 *   decode q  [Hq][d]                 (attention.hpp:71-84)
 *   partial   o [rows][d], lse [rows] (attention.hpp:86-93)
 *
 * Errors mirror the reference's exception classes as status codes
 * (same numbering as include/pod_attn.h's pod_status).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum {
    ORC_OK = 0,
    ORC_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    ORC_LOGIC = 2,            /* std::logic_error       */
    ORC_DOMAIN = 3,           /* std::domain_error      */
    ORC_OUT_OF_RANGE = 4,     /* std::out_of_range      */
};

/* ModelShape::validate (types.hpp:68-75). */
static int shape_ok(int hq, int hkv, int d, double scale) {
    if (hq < 1 || hkv < 1 || d < 1) return 0;
    if (hq % hkv != 0) return 0;
    if (!(scale > 0.0)) return 0;
    return 1;
}

/* gqa_kv_head (attention.hpp:100-106): q_head / group_size. */
int orc_gqa_kv_head(int q_head, int hq, int hkv, int* out) {
    if (q_head < 0 || q_head >= hq) return ORC_OUT_OF_RANGE;
    *out = q_head / (hq / hkv);
    return ORC_OK;
}

/* split_ranges (attention.hpp:224-238): lengths n/s, +1 for the first n%s. */
void orc_split_ranges(long n, long splits, long* begin, long* end) {
    const long base = n / splits, rem = n % splits;
    long pos = 0;
    for (long s = 0; s < splits; ++s) {
        const long len = base + (s < rem ? 1 : 0);
        begin[s] = pos;
        end[s] = pos + len;
        pos += len;
    }
}

/* naive_attention (attention.hpp:108-146): dense two-pass softmax, optional
 * causal offset (has_causal != 0): row i sees keys <= offset + i. */
int orc_naive_attention(const double* q, long m, const double* k, const double* v, long n, long d,
                        double scale, int has_causal, long causal_offset, double* out) {
    if (m < 1 || n < 1) return ORC_INVALID_ARGUMENT;
    if (!(scale > 0.0)) return ORC_INVALID_ARGUMENT;
    double* scores = (double*)malloc(sizeof(double) * (size_t)n);
    memset(out, 0, sizeof(double) * (size_t)(m * d));
    for (long i = 0; i < m; ++i) {
        long visible = n;
        if (has_causal) {
            visible = causal_offset + i + 1;
            if (visible > n) visible = n;
        }
        if (visible <= 0) {
            free(scores);
            return ORC_DOMAIN;
        }
        for (long j = 0; j < n; ++j) {
            double acc = 0;
            for (long c = 0; c < d; ++c) acc += q[i * d + c] * k[j * d + c];
            scores[j] = acc / scale;
        }
        double row_max = -INFINITY;
        for (long j = 0; j < visible; ++j) row_max = fmax(row_max, scores[j]);
        double denom = 0;
        for (long j = 0; j < visible; ++j) {
            scores[j] = exp(scores[j] - row_max);
            denom += scores[j];
        }
        for (long j = 0; j < visible; ++j) {
            const double w = scores[j] / denom;
            for (long c = 0; c < d; ++c) out[i * d + c] += w * v[j * d + c];
        }
    }
    free(scores);
    return ORC_OK;
}

/* tiled_prefill_attention (attention.hpp:148-222).  For every q head, q tile
 * and kv tile: per row, a max pass over the tile's visible keys (:189-194),
 * rescale of the running denominator/accumulator (:195-201), then an exp/PV
 * pass (:202-210); the tile's kv walk is bounded by the last row's visibility
 * (:180).  out is [chunk][hq*d]. */
int orc_tiled_prefill(const double* q, long chunk, long offset, const double* k, const double* v,
                      long ctx, int hq, int hkv, int d, double scale, long tile_q, long tile_kv,
                      double* out) {
    if (tile_q < 1 || tile_kv < 1) return ORC_INVALID_ARGUMENT;
    if (offset < 0) return ORC_INVALID_ARGUMENT;
    if (ctx < offset + chunk) return ORC_LOGIC;
    if (!shape_ok(hq, hkv, d, scale)) return ORC_INVALID_ARGUMENT;
    const int group = hq / hkv;
    double* row_max = (double*)malloc(sizeof(double) * (size_t)tile_q);
    double* denom = (double*)malloc(sizeof(double) * (size_t)tile_q);
    double* acc = (double*)malloc(sizeof(double) * (size_t)tile_q * (size_t)d);
    for (int h = 0; h < hq; ++h) {
        const int kvh = h / group;
        for (long t0 = 0; t0 < chunk; t0 += tile_q) {
            const long t1 = (chunk < t0 + tile_q) ? chunk : t0 + tile_q;
            const long rows = t1 - t0;
            for (long r = 0; r < rows; ++r) {
                row_max[r] = -INFINITY;
                denom[r] = 0;
            }
            memset(acc, 0, sizeof(double) * (size_t)rows * (size_t)d);
            const long kv_limit = offset + t1;
            for (long k0 = 0; k0 < kv_limit; k0 += tile_kv) {
                const long k1 = (kv_limit < k0 + tile_kv) ? kv_limit : k0 + tile_kv;
                for (long r = 0; r < rows; ++r) {
                    const long visible = offset + t0 + r + 1;
                    const long jend = (k1 < visible) ? k1 : visible;
                    if (jend <= k0) continue;
                    const double* qrow = q + ((t0 + r) * hq + h) * (long)d;
                    double tile_max = -INFINITY;
                    for (long j = k0; j < jend; ++j) {
                        const double* krow = k + (j * hkv + kvh) * (long)d;
                        double s = 0;
                        for (int c = 0; c < d; ++c) s += qrow[c] * krow[c];
                        tile_max = fmax(tile_max, s / scale);
                    }
                    const double new_max = fmax(row_max[r], tile_max);
                    const double rescale = row_max[r] == -INFINITY ? 0.0 : exp(row_max[r] - new_max);
                    denom[r] *= rescale;
                    double* arow = acc + r * (long)d;
                    for (int c = 0; c < d; ++c) arow[c] *= rescale;
                    for (long j = k0; j < jend; ++j) {
                        const double* krow = k + (j * hkv + kvh) * (long)d;
                        double s = 0;
                        for (int c = 0; c < d; ++c) s += qrow[c] * krow[c];
                        const double w = exp(s / scale - new_max);
                        denom[r] += w;
                        const double* vrow = v + (j * hkv + kvh) * (long)d;
                        for (int c = 0; c < d; ++c) arow[c] += w * vrow[c];
                    }
                    row_max[r] = new_max;
                }
            }
            for (long r = 0; r < rows; ++r) {
                double* orow = out + (t0 + r) * (long)hq * d + (long)h * d;
                for (int c = 0; c < d; ++c) orow[c] = acc[r * (long)d + c] / denom[r];
            }
        }
    }
    free(row_max);
    free(denom);
    free(acc);
    return ORC_OK;
}

/* decode_attention_splitk (attention.hpp:240-292) for one decode query.
 * Writes up to min(num_splits, ctx) partials: o_parts [splits][hq][d],
 * lse_parts [splits][hq] (natural log, :287), ranges [splits][2].
 * *n_parts receives the clamped split count (:254). */
int orc_decode_splitk(const double* q, const double* k, const double* v, long ctx, int hq, int hkv,
                      int d, double scale, long num_splits, double* o_parts, double* lse_parts,
                      long* ranges, long* n_parts) {
    if (num_splits < 1) return ORC_INVALID_ARGUMENT;
    if (ctx < 1) return ORC_DOMAIN;
    if (!shape_ok(hq, hkv, d, scale)) return ORC_INVALID_ARGUMENT;
    const long splits = num_splits < ctx ? num_splits : ctx;
    const int group = hq / hkv;
    long* b = (long*)malloc(sizeof(long) * (size_t)splits);
    long* e = (long*)malloc(sizeof(long) * (size_t)splits);
    orc_split_ranges(ctx, splits, b, e);
    for (long s = 0; s < splits; ++s) {
        ranges[2 * s] = b[s];
        ranges[2 * s + 1] = e[s];
        for (int h = 0; h < hq; ++h) {
            const int kvh = h / group;
            const double* qrow = q + (long)h * d;
            double m = -INFINITY;
            for (long j = b[s]; j < e[s]; ++j) {
                const double* krow = k + (j * hkv + kvh) * (long)d;
                double acc = 0;
                for (int c = 0; c < d; ++c) acc += qrow[c] * krow[c];
                m = fmax(m, acc / scale);
            }
            double denom = 0;
            double* orow = o_parts + (s * hq + h) * (long)d;
            for (int c = 0; c < d; ++c) orow[c] = 0;
            for (long j = b[s]; j < e[s]; ++j) {
                const double* krow = k + (j * hkv + kvh) * (long)d;
                double acc = 0;
                for (int c = 0; c < d; ++c) acc += qrow[c] * krow[c];
                const double w = exp(acc / scale - m);
                denom += w;
                const double* vrow = v + (j * hkv + kvh) * (long)d;
                for (int c = 0; c < d; ++c) orow[c] += w * vrow[c];
            }
            for (int c = 0; c < d; ++c) orow[c] /= denom;
            lse_parts[s * hq + h] = m + log(denom);
        }
    }
    *n_parts = splits;
    free(b);
    free(e);
    return ORC_OK;
}

/* merge_partials (attention.hpp:294-326): stable sort by range begin (:300-301),
 * reject overlaps (:302-307), lse_total = m + log(sum exp(lse_i - m))
 * (:313-317), O = sum exp(lse_i - lse_total) * O_i in range order (:318-323).
 * o_parts [n][rows][d], lse_parts [n][rows], ranges [n][2].
 * lse_out (may be NULL) receives lse_total, which the reference computes
 * internally but does not return. */
int orc_merge_partials(const double* o_parts, const double* lse_parts, const long* ranges, long n,
                       long rows, long d, double* out, double* lse_out) {
    if (n < 1) return ORC_INVALID_ARGUMENT;
    long* order = (long*)malloc(sizeof(long) * (size_t)n);
    for (long i = 0; i < n; ++i) order[i] = i;
    /* insertion sort: stable, like the reference's comparison on begin only */
    for (long i = 1; i < n; ++i) {
        long x = order[i], j = i - 1;
        while (j >= 0 && ranges[2 * order[j]] > ranges[2 * x]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = x;
    }
    for (long i = 1; i < n; ++i) {
        if (ranges[2 * order[i]] < ranges[2 * order[i - 1] + 1]) {
            free(order);
            return ORC_LOGIC;
        }
    }
    memset(out, 0, sizeof(double) * (size_t)(rows * d));
    for (long r = 0; r < rows; ++r) {
        double m = -INFINITY;
        for (long i = 0; i < n; ++i) m = fmax(m, lse_parts[order[i] * rows + r]);
        double total = 0;
        for (long i = 0; i < n; ++i) total += exp(lse_parts[order[i] * rows + r] - m);
        const double lse_total = m + log(total);
        if (lse_out) lse_out[r] = lse_total;
        for (long i = 0; i < n; ++i) {
            const long p = order[i];
            const double w = exp(lse_parts[p * rows + r] - lse_total);
            const double* prow = o_parts + (p * rows + r) * d;
            for (long c = 0; c < d; ++c) out[r * d + c] += w * prow[c];
        }
    }
    free(order);
    return ORC_OK;
}

/* decode_attention (attention.hpp:328-333) = merge(splitk(., 1)), plus the
 * natural-log LSE of the full range.  out [hq][d], lse [hq]. */
int orc_decode_attention(const double* q, const double* k, const double* v, long ctx, int hq,
                         int hkv, int d, double scale, double* out, double* lse) {
    long rng[2], n = 0;
    double* lse_p = (double*)malloc(sizeof(double) * (size_t)hq);
    int st = orc_decode_splitk(q, k, v, ctx, hq, hkv, d, scale, 1, out, lse_p, rng, &n);
    if (st == ORC_OK && lse) memcpy(lse, lse_p, sizeof(double) * (size_t)hq);
    free(lse_p);
    return st;
}

/* Prefill LSE, which tiled_prefill_attention does not emit: row r of the chunk
 * sees keys [0, offset + r] (attention.hpp:184-186), so its LSE is the
 * single-split decode LSE of that row against the prefix-truncated cache
 * (attention.hpp:243-292) -- SURVEY.md 8(c).  lse [chunk][hq]. */
int orc_prefill_lse(const double* q, long chunk, long offset, const double* k, long ctx, int hq,
                    int hkv, int d, double scale, double* lse) {
    if (offset < 0) return ORC_INVALID_ARGUMENT;
    if (ctx < offset + chunk) return ORC_LOGIC;
    if (!shape_ok(hq, hkv, d, scale)) return ORC_INVALID_ARGUMENT;
    const int group = hq / hkv;
    for (long r = 0; r < chunk; ++r) {
        const long visible = offset + r + 1;
        for (int h = 0; h < hq; ++h) {
            const int kvh = h / group;
            const double* qrow = q + (r * hq + h) * (long)d;
            double m = -INFINITY;
            for (long j = 0; j < visible; ++j) {
                const double* krow = k + (j * hkv + kvh) * (long)d;
                double acc = 0;
                for (int c = 0; c < d; ++c) acc += qrow[c] * krow[c];
                m = fmax(m, acc / scale);
            }
            double denom = 0;
            for (long j = 0; j < visible; ++j) {
                const double* krow = k + (j * hkv + kvh) * (long)d;
                double acc = 0;
                for (int c = 0; c < d; ++c) acc += qrow[c] * krow[c];
                denom += exp(acc / scale - m);
            }
            lse[r * hq + h] = m + log(denom);
        }
    }
    return ORC_OK;
}

/* Paged-KV gather: rebuild the reference's contiguous per-request cache
 * [ctx][hkv][d] (attention.hpp:36-38) from a bf16 page pool.  This is the one
 * piece of integer arithmetic the GPU adds (SPEC.md:113 rules paging out of
 * the simulator): logical token t of request `req` lives in physical page
 * page_indices[page_indptr[req] + t / page_size] at slot t % page_size.
 *   layout 0 (HND): pool [num_pages][hkv][page_size][d]
 *   layout 1 (NHD): pool [num_pages][page_size][hkv][d]
 * Values are widened bf16 -> double exactly (bit-exact by construction). */
static double bf16_to_double(uint16_t x) {
    union {
        uint32_t u;
        float f;
    } c;
    c.u = ((uint32_t)x) << 16;
    return (double)c.f;
}

int orc_gather_pages(const uint16_t* pool, int layout, long num_pages, int hkv, int page_size,
                     int d, const int32_t* page_indptr, const int32_t* page_indices, int req,
                     long ctx, double* k_out_or_v_out) {
    const long npages = page_indptr[req + 1] - page_indptr[req];
    if ((ctx + page_size - 1) / page_size > npages) return ORC_LOGIC;
    for (long t = 0; t < ctx; ++t) {
        const long page = page_indices[page_indptr[req] + t / page_size];
        const long slot = t % page_size;
        if (page < 0 || page >= num_pages) return ORC_OUT_OF_RANGE;
        for (int h = 0; h < hkv; ++h) {
            size_t base;
            if (layout == 0)
                base = (((size_t)page * hkv + h) * page_size + slot) * d;
            else
                base = (((size_t)page * page_size + slot) * hkv + h) * d;
            double* dst = k_out_or_v_out + ((size_t)t * hkv + h) * d;
            for (int c = 0; c < d; ++c) dst[c] = bf16_to_double(pool[base + c]);
        }
    }
    return ORC_OK;
}

/* KV append (SURVEY.md 8(f) N2 -- the write step before attention; the reference
 * keeps contiguous caches, so this restates the paged-layout contract
 * of orc_gather_pages in the other direction): rows [ntok][hkv][d] (16-bit words)
 * land at positions pos0 .. pos0+ntok-1 of request `req`.  A pure copy. */
int orc_append_kv(uint16_t* pool, int layout, long num_pages, int hkv, int page_size, int d,
                  const int32_t* page_indptr, const int32_t* page_indices, int req, long pos0, long ntok,
                  const uint16_t* rows) {
    const long npages = page_indptr[req + 1] - page_indptr[req];
    if (pos0 < 0 || (pos0 + ntok + page_size - 1) / page_size > npages) return ORC_LOGIC;
    for (long i = 0; i < ntok; ++i) {
        const long t = pos0 + i;
        const long page = page_indices[page_indptr[req] + t / page_size];
        const long slot = t % page_size;
        if (page < 0 || page >= num_pages) return ORC_OUT_OF_RANGE;
        for (int h = 0; h < hkv; ++h) {
            size_t base;
            if (layout == 0)
                base = (((size_t)page * hkv + h) * page_size + slot) * d;
            else
                base = (((size_t)page * page_size + slot) * hkv + h) * d;
            const uint16_t* src = rows + ((size_t)i * hkv + h) * d;
            for (int c = 0; c < d; ++c) pool[base + c] = src[c];
        }
    }
    return ORC_OK;
}

/* SM-aware CTA scheduler semantics (gpu_sim.hpp:80-131),
 * restated for checking the device role log.  Proportional ratio is the
 * gcd-reduced P:D (gpu_sim.hpp:100-105). */
static long gcd_l(long a, long b) {
    while (b) {
        long t = a % b;
        a = b;
        b = t;
    }
    return a;
}

void orc_sched_ratio(int proportional, long p, long dd, long* pr, long* dr) {
    if (!proportional) {
        *pr = 1;
        *dr = 1;
        return;
    }
    const long g = gcd_l(p, dd);
    *pr = g > 0 ? p / g : (p > 0 ? 1 : 0);
    *dr = g > 0 ? dd / g : (dd > 0 ? 1 : 0);
    if (*pr == 0 && *dr == 0) *pr = 1;
}

/* Replays sm_aware_assign for a sequence of CTA arrivals (sm_ids[i]).
 * op_out[i] = 0 prefill / 1 decode / -1 nullopt, id_out[i] = claimed id. */
void orc_sm_aware_replay(long pr, long dr, long p_total, long d_total, int num_sms,
                         const int* sm_ids, long n, int* op_out, long* id_out) {
    long* sm_ctr = (long*)calloc((size_t)num_sms, sizeof(long));
    long assign[2] = {0, 0};
    const long ratio = pr + dr;
    for (long i = 0; i < n; ++i) {
        const long ticket = sm_ctr[sm_ids[i]]++ % ratio;
        int op = ticket < pr ? 0 : 1;
        long cta = assign[op]++;
        if (cta >= (op == 0 ? p_total : d_total)) {
            op = 1 - op;
            cta = assign[op]++;
            if (cta >= (op == 0 ? p_total : d_total)) {
                op_out[i] = -1;
                id_out[i] = -1;
                continue;
            }
        }
        op_out[i] = op;
        id_out[i] = cta;
    }
    free(sm_ctr);
}
