// pod_attn.cu -- sm_100a kernels of the POD-Attention hot path and the C ABI
// run entry points (include/pod_attn.h).
//
//   prefill role : causal chunked-prefill tile; QK^T and PV on tcgen05 with
//                  TMEM accumulators, K/V/Q staged by TMA (128B swizzle);
//                  semantics of tiled_prefill_attention (attention.hpp:148-222)
//                  restricted to the CTA's kv split, emitting O and LSE.
//   decode role  : split-KV paged decode on CUDA cores, one warp per virtual
//                  decode CTA (work_decomp.hpp:179-197),
//                  online softmax + warp-shuffle reductions, in-CTA LSE merge
//                  of the 4 virtual CTAs; semantics of decode_attention_splitk
//                  (attention.hpp:240-292).
//   merge        : LSE merge of split partials (merge_partials, attention.hpp:294-326).
//   fused kernel : SM-aware runtime role binding (PAPER.md:387-423,
//                  gpu_sim.hpp:114-131) over P + D CTAs, counters self-reset.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <string>
#include <vector>

#include "pod_internal.h"

// timing experiments only (tools/micro/build_variant.sh); both 0 in the product
#ifndef POD_EXP_FAKE
#define POD_EXP_FAKE 0
#endif
#ifndef POD_SOFTMAX_SKIP
#define POD_SOFTMAX_SKIP 0
#endif
#ifndef POD_UNIFORM_WARP
#define POD_UNIFORM_WARP 1  // two-CTA kernel: see uniform_warp()
#endif
#ifndef POD_SM_NOLOAD
#define POD_SM_NOLOAD 0
#endif
#ifndef POD_SM_NOMMA
#define POD_SM_NOMMA 0
#endif
#include "sm100_ptx.cuh"

namespace pod {

namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& s) { g_last_error = s; }

// ------------------------------------------------------------ smem plan --
// Prefill role (offsets from the 1024-aligned dynamic smem base):
constexpr uint32_t kQBytes = kMBlock * kHeadDim * 2;        // 32 KB: 2 swizzle columns of 128 x 128B
constexpr uint32_t kKvStageBytes = kKvTile * kHeadDim * 2;  // 16 KB
constexpr uint32_t kOffQ = 0;
constexpr uint32_t kOffK = kOffQ + kQBytes;                 // 2 stages
constexpr uint32_t kOffV = kOffK + 2 * kKvStageBytes;       // 2 stages
// Decode role: per-warp TMA rings of K+V head-pages below the barrier block.
#ifndef POD_DEC_STAGES
#define POD_DEC_STAGES 3
#endif
#ifndef POD_DEC_WARPS
#define POD_DEC_WARPS 4
#endif
#ifndef POD_DEC_SLEEP
#define POD_DEC_SLEEP 0  // decode page waits: spin (0) or __nanosleep back-off
#endif
// Warps that stream one decode item (the planner's 4 virtual decode CTAs,
// kDecodeWarps, are the item's logical split; the kernel may use more warps).
constexpr int kDecWarpsK = POD_DEC_WARPS;
static_assert(kDecWarpsK <= kThreads / 32, "decode warps");
constexpr int kDecStages = POD_DEC_STAGES;             // pages in flight per warp
constexpr uint32_t kDecPageBytes = 16 * kHeadDim * 2;  // one head-page of K (or V): 4 KB
constexpr uint32_t kDecStageBytes = 2 * kDecPageBytes; // K + V
constexpr uint32_t kDecWarpBytes = kDecStages * kDecStageBytes;
constexpr uint32_t kPrefillBytes = kOffV + 2 * kKvStageBytes;
constexpr uint32_t kOffBar = kPrefillBytes > kDecWarpsK * kDecWarpBytes ? kPrefillBytes
                                                                          : kDecWarpsK * kDecWarpBytes;  // 16 mbarriers
constexpr uint32_t kOffTmemSlot = kOffBar + 128;
constexpr uint32_t kOffDecBar = kOffBar + 160;              // 4 warps x kDecStages decode mbarriers
constexpr uint32_t kOffRole = kOffTmemSlot + 16;          // role[0..3]
constexpr uint32_t kSmemBytes = kOffDecBar + kDecWarpsK * kDecStages * 8 + 32;  // 98560 B -> 2 CTAs / SM
static_assert(kOffRole + 16 <= kOffDecBar, "role slots");
static_assert(POD_DEC_STAGES != 3 || kSmemBytes * 2 + 2048 <= 233472, "two CTAs must fit one SM");
constexpr uint32_t kTmemCols = 256;                         // S0 | S1 | O(128)
constexpr uint32_t kTmemS0 = 0, kTmemO = 128;

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct RunParams {
    const void* q_prefill;
    const void* q_decode;
    const void* k_pool;
    const void* v_pool;
    const int32_t* page_indptr;
    const int32_t* page_indices;
    void* o_prefill;
    float* lse_prefill;
    void* o_decode;
    int out_fmt;  // POD_OUT_*: element type of o_prefill / o_decode
    float* lse_decode;
    float* ppart_o;
    float* ppart_lse;
    float* dpart_o;
    float* dpart_lse;
    const PrefillCta* pctas;
    const DecodeCta* dctas;
    SchedCounters* ctr;
    int32_t* role_log;
    int32_t num_pctas;
    int32_t num_dctas;
    int32_t prefill_ratio;
    int32_t decode_ratio;
    int32_t hq;
    int32_t hd;  // head dim of the tensors (8..128, multiple of 8); the kernels compute at 128, zero-padded
    int32_t hkv;
    int32_t group;
    int32_t chunk;
    int32_t offset;
    int32_t kv_layout;
    int32_t decode_splits;   // largest split count = partials' stride
    int32_t dec_split_base;  // splits of requests below dec_tail_start
    int32_t dec_tail_start;
    int32_t policy;
    int32_t p_split;  // prefill P as bf16 hi + lo (two PV MMAs)
    int32_t p_f16;    // POD_PRECISION_F16PV: P as fp16, V stages converted to fp16 in smem (bf16 data)
    int32_t pf_tn64;  // warp-specialised kernel: 64-key pair engine (prefill-dominant plans)
    int32_t pf_db;    // ... with two S buffers per block: kernel instance 1 (prefill_item_db)
    const int32_t* dec_nsplit;  // KV splits of each decode request (min(splits, ctx), pod_plan.cpp)
    int32_t vs_pages;  // > 0: prefill V tiles from the fp16 shadow (logical pages, already converted)
    int32_t trace;         // debug builds (POD_TRACE_STAMPS): per-tile cycle stamps after the role log
    int32_t trace_mode;    // debug builds: 2 = serialise MMA issue with completion (execution latency probe)
    int64_t num_pages;
    float sl2;  // log2(e) / scale  (scale is the reference's divisor)
};

// Packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
          "l"(*reinterpret_cast<uint64_t*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(d)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
    return *reinterpret_cast<float2*>(&d);
}

// 2^x on the FMA pipe for a pair (FA4-style MUFU offload): x = j + f with j = round(x)
// (the 1.5 * 2^23 magic add), f in [-0.5, 0.5], 2^f by a degree-4 minimax polynomial
// (max rel. error 2.6e-6, far below fp16 P's 2^-12), 2^j added into the exponent field.
// x is clamped at -126 (masked scores, x = -inf, give 2^-126: 0 once P is rounded to
// 16 bits; their share of the fp32 row sum is < 1e-37 relative).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    x = make_float2(fmaxf(x.x, -126.f), fmaxf(x.y, -126.f));
    const float2 magic = make_float2(12582912.f, 12582912.f);
    const float2 t = fadd2(x, magic);
    const float2 r = fadd2(t, make_float2(-12582912.f, -12582912.f));  // round(x)
    const float2 f = ffma2(r, make_float2(-1.f, -1.f), x);                // x - round(x)
    float2 q = ffma2(make_float2(0.009570068679749966f, 0.009570068679749966f), f,
                     make_float2(0.055917806923389435f, 0.055917806923389435f));
    q = ffma2(q, f, make_float2(0.240247443318367f, 0.240247443318367f));
    q = ffma2(q, f, make_float2(0.6931218504905701f, 0.6931218504905701f));
    q = ffma2(q, f, make_float2(0.9999992847442627f, 0.9999992847442627f));
    return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23)),
                       __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23)));
}
#ifndef POD_EXP_POLY
#define POD_EXP_POLY 0  // default pairs per 8 whose exp2 runs on the FMA pipe (0 = all on MUFU; the
                        // double-S pair engine passes 1 explicitly)
#endif

template <int kFmt>
__device__ __forceinline__ uint32_t pack2(float x, float y) {
    if constexpr (kFmt == 1) {
        __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
        return *reinterpret_cast<uint32_t*>(&h);
    } else {
        __half2 h = __floats2half2_rn(x, y);
        return *reinterpret_cast<uint32_t*>(&h);
    }
}
template <int kFmt>
__device__ __forceinline__ float2 unpack2(uint32_t w) {
    if constexpr (kFmt == 1) {
        return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
    } else {
        return __half22float2(*reinterpret_cast<const __half2*>(&w));
    }
}
// ============================================================ prefill ===
template <int kFmt>
__device__ __forceinline__ void prefill_issue_qk(uint32_t tmem_s, uint32_t sQ, uint32_t sK) {
    constexpr uint32_t idesc = ptx::idesc_f16(kFmt, kMBlock, kKvTile, 0);
#pragma unroll
    for (int kk = 0; kk < kHeadDim / 16; ++kk) {
        const uint32_t koff = (kk & 3) * 32u;  // 16 elements = 32 B inside the 128 B swizzle row
        const uint64_t a = ptx::sw128_desc(sQ + (kk >> 2) * (kMBlock * 128) + koff, 16, 1024);
        const uint64_t b = ptx::sw128_desc(sK + (kk >> 2) * (kKvTile * 128) + koff, 16, 1024);
        ptx::umma_f16_ss_elect(tmem_s, a, b, idesc, kk > 0 ? 1u : 0u);
    }
}

// O (+)= P V with P (bf16, 128 x 64) read from TMEM (2 values per 32-bit column,
// 8 columns per K=16 step) and V (64 keys x 128 d, MN-major SW128) from smem in the
// page-major image of prefill_load_v_pages: K-step kk = head-page kk (4 KB), the two
// 64-d halves 2 KB apart (LBO).
template <int kFmt>
__device__ __forceinline__ void prefill_issue_pv(uint32_t tmem_o, uint32_t tmem_p, uint32_t sV,
                                                 bool accumulate, bool split) {
    constexpr uint32_t idesc = ptx::idesc_f16(kFmt, kMBlock, kHeadDim, 1);  // kFmt: P and V format
#pragma unroll
    for (int kk = 0; kk < kKvTile / 16; ++kk) {
        const uint64_t b = ptx::sw128_desc(sV + kk * 4096, 2048, 1024);
        ptx::umma_f16_ts_elect(tmem_o, tmem_p + kk * 8, b, idesc, (accumulate || kk > 0) ? 1u : 0u);
        if (split) ptx::umma_f16_ts_elect(tmem_o, tmem_p + 32 + kk * 8, b, idesc, 1u);  // + P_lo V
    }
}

// One softmax row of a 64-key tile: p = 2^(s * sl2 - m) (one FFMA2 per pair, one
// MUFU per score), P written over the row's S columns in TMEM as the A operand of
// the TS MMA.  Returns the row sum of p (fp32).
//   kMode 0: one P, rounded to nearest (columns [0,32))
//   kMode 1: bf16 hi + lo by truncation (integer byte permutes, no conversion unit):
//            hi = top 16 bits of p, lo = p - hi (exact in fp32) truncated; hi in
//            [0,32), lo in [32,64); hi + lo keeps ~15 mantissa bits
//   kMode 2: hi + lo rounded to nearest (fp16 inputs)
//   kMode 3: one P rounded to fp16 (POD_PRECISION_F16PV), columns [0, kN/2)
template <int kFmt, int kMode, int kN = kKvTile, int kPoly = POD_EXP_POLY>
__device__ __forceinline__ float softmax_p_row(const float (&s)[kN], float sl2, float neg_m, uint32_t s_addr) {
    const float2 sl2v = make_float2(sl2, sl2), nm2 = make_float2(neg_m, neg_m);
    float2 lsum2 = make_float2(0.f, 0.f), lsum2b = make_float2(0.f, 0.f);  // two chains
#pragma unroll
    for (int hf = 0; hf < kN / 32; ++hf) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
            const float2 x = ffma2(make_float2(s[32 * hf + c], s[32 * hf + c + 1]), sl2v, nm2);
#if POD_EXP_FAKE  // timing experiment only: exp2 replaced by one FMA-pipe op
            const float p0 = x.x * 0.5f, p1 = x.y * 0.5f;
#else
            float p0, p1;
            if (kPoly > 0 && (c / 2) % 8 >= 8 - kPoly) {  // kPoly of every 8 pairs on the FMA pipe
                const float2 e = ex2_poly2(x);
                p0 = e.x;
                p1 = e.y;
            } else {
                p0 = ptx::ex2(x.x);
                p1 = ptx::ex2(x.y);
            }
#endif
            if (c & 2)
                lsum2b = fadd2(lsum2b, make_float2(p0, p1));
            else
                lsum2 = fadd2(lsum2, make_float2(p0, p1));
            if constexpr (kMode == 1) {
                const uint32_t u0 = __float_as_uint(p0), u1 = __float_as_uint(p1);
                hi[c / 2] = __byte_perm(u0, u1, 0x7632);
                const float2 lv = fadd2(make_float2(p0, p1), make_float2(-__uint_as_float(u0 & 0xffff0000u),
                                                                         -__uint_as_float(u1 & 0xffff0000u)));
                lo[c / 2] = __byte_perm(__float_as_uint(lv.x), __float_as_uint(lv.y), 0x7632);
            } else if constexpr (kMode == 3) {
                hi[c / 2] = pack2<0>(p0, p1);
            } else {
                hi[c / 2] = pack2<kFmt>(p0, p1);
                if constexpr (kMode == 2) {
                    const float2 hv = unpack2<kFmt>(hi[c / 2]);
                    lo[c / 2] = pack2<kFmt>(p0 - hv.x, p1 - hv.y);
                }
            }
        }
        ptx::tmem_st16(s_addr + 16 * hf, hi);
        if constexpr (kMode == 1 || kMode == 2) ptx::tmem_st16(s_addr + kN / 2 + 16 * hf, lo);
    }
    return (lsum2.x + lsum2.y) + (lsum2b.x + lsum2b.y);
}

// Row max of kN scores as a tree (depth log3 kN of FMNMX3 instead of a kN/2-long chain).
template <int kN>
__device__ __forceinline__ float row_max(const float (&s)[kN]) {
    float m[kN / 2];
#pragma unroll
    for (int c = 0; c < kN / 2; ++c) m[c] = fmaxf(s[2 * c], s[2 * c + 1]);
#pragma unroll
    for (int w = kN / 4; w >= 1; w /= 2) {
#pragma unroll
        for (int c = 0; c < w; ++c) m[c] = fmaxf(m[c], m[c + w]);
    }
    return m[0];
}

// POD_PRECISION_F16PV: one V stage converted bf16 -> fp16 in place in shared memory.
// The conversion is elementwise, so the SW128 image stays the B operand layout of
// the PV MMA, which then runs fp16 x fp16 with P rounded to fp16 (11-bit significand:
// ~8x less P rounding error than bf16, one PV MMA instead of the hi + lo pair).
// Exact for |v| in [2^-14, 65504] (bf16's 8-bit significand fits fp16's 11); smaller
// magnitudes become fp16 subnormals (abs error <= 2^-25), larger ones saturate.
// kThr threads (tid in [0, kThr)) share the stage; the generic -> async proxy fence
// makes the stores visible to the tensor core once the caller's mbarrier arrival
// (the P-full hand-off) is observed by the MMA issuer.
__device__ __forceinline__ uint32_t bf16x2_to_f16x2(uint32_t w) {
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;"
        : "=r"(r)
        : "f"(__uint_as_float(w & 0xffff0000u)), "f"(__uint_as_float(w << 16)));
    return r;
}
template <uint32_t kBytes, int kThr>
__device__ __forceinline__ void v_stage_to_f16(uint32_t stage, int tid) {
    static_assert(kBytes % (16u * kThr) == 0, "whole 16-byte chunks per thread");
#pragma unroll
    for (uint32_t i = 0; i < kBytes / (16u * kThr); ++i) {
        const uint32_t a = stage + (i * kThr + static_cast<uint32_t>(tid)) * 16u;
        uint32_t w0, w1, w2, w3;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(a));
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(bf16x2_to_f16x2(w0)),
                     "r"(bf16x2_to_f16x2(w1)), "r"(bf16x2_to_f16x2(w2)), "r"(bf16x2_to_f16x2(w3))
                     : "memory");
    }
    ptx::fence_proxy_async_smem();
}

struct BlockRange {
    int r0;      // first chunk row of the block
    int nrows;   // chunk rows in the block
    int kt0;     // first key of tile 0 (page aligned)
    int nt;      // kv tiles
};

__device__ __forceinline__ BlockRange prefill_block(const RunParams& p, const PrefillCta& job,
                                                    int b) {
    const int rpb = kMBlock / p.group;
    BlockRange br;
    br.r0 = job.row_begin + b * rpb;
    br.nrows = min(rpb, job.rows - b * rpb);
    const int r_last = br.r0 + br.nrows - 1;
    const int kv_hi = min(job.kv_end, p.offset + r_last + 1);
    br.kt0 = (job.kv_begin / 16) * 16;
    br.nt = kv_hi > job.kv_begin ? (kv_hi - br.kt0 + kKvTile - 1) / kKvTile : 0;
    return br;
}

// Page ids of one block-table row.  (A per-lane shuffle cache of the ids measured
// slower than these direct L1-resident loads in the producer warp: 483 vs 405 us
// prefill-alone, C2 -- so the lookup stays a plain __ldg.)
struct PageIds {
    const int32_t* row;
    int n;  // pages in the row
    __device__ __forceinline__ void init(const int32_t* r, int npages, int /*first*/) {
        row = r;
        n = npages;
    }
    __device__ __forceinline__ int get(int j) const { return __ldg(row + j); }
};

// Issue the 8 TMA boxes (4 pages x 2 swizzle columns) of one 64-key tile
// (warp-uniform call; page ids from the warp's cache).
__device__ __forceinline__ void prefill_load_kv_tile(const RunParams& p, const CUtensorMap* tm,
                                                     uint32_t dst, uint32_t bar, int kt, int kv_head,
                                                     PageIds& ids) {
    int phys_pg[kKvTile / 16];
#pragma unroll
    for (int pg = 0; pg < kKvTile / 16; ++pg) phys_pg[pg] = ids.get(min(kt / 16 + pg, ids.n - 1));
#pragma unroll
    for (int pg = 0; pg < kKvTile / 16; ++pg) {
        const int phys = phys_pg[pg];
#pragma unroll
        for (int dh = 0; dh < 2; ++dh) {
            const uint32_t d = dst + dh * (kKvTile * 128) + pg * 2048;
            if (p.kv_layout == POD_KV_HND)
                ptx::tma_load_4d_elect(d, tm, bar, dh * 64, 0, kv_head, phys);
            else
                ptx::tma_load_4d_elect(d, tm, bar, dh * 64, kv_head, 0, phys);
        }
    }
}

// V of one prefill tile as one 4 KB TMA box per head-page (the decode role's 5-D
// view: (64 d, 16 slots, 2 d-halves, head, page)): smem [page][d-half][16 keys][64 d],
// SW128.  Half the TMA issues of the K layout ([d-half][keys][64 d], two boxes per
// page), which the QK MMA needs for a uniform 8-key group stride along N; the PV MMA
// reads V with K = keys, one head-page per K=16 step (LBO = 2 KB between the d-halves,
// K-steps 4 KB apart), so the page-major image serves it directly.
template <int kPages>
__device__ __forceinline__ void prefill_load_v_pages(const CUtensorMap* tdv, uint32_t dst, uint32_t bar, int kt,
                                                     int kv_head, const PageIds& ids, int vs_pages = 0) {
    int phys[kPages];  // the fp16 shadow (vs_pages > 0) is indexed by logical page
#pragma unroll
    for (int pg = 0; pg < kPages; ++pg)
        phys[pg] = vs_pages ? min(kt / 16 + pg, vs_pages - 1) : ids.get(min(kt / 16 + pg, ids.n - 1));
#pragma unroll
    for (int pg = 0; pg < kPages; ++pg) ptx::tma_load_5d_elect(dst + pg * 4096, tdv, bar, 0, 0, 0, kv_head, phys[pg]);
}

// Prefill role: one CTA = one CtaTask of decompose_prefill (q tile x kv head x kv
// split), processed as M-blocks of 128 packed (row, q-head) rows.  Warp roles:
//   warps 0-3  softmax: TMEM lane quadrant w, one M row per thread
//   warp 4     TMA producer (Q, K and V boxes through the page table)
//   warp 5     MMA issuer (one thread): S = Q K^T (SS), O += P V (TS, P in TMEM)
// S tiles are double-buffered in TMEM; each softmax thread overwrites its S row
// with its bf16 P row, so P is double-buffered for free and never touches smem.
// All hand-offs are mbarriers (no CTA-wide barrier inside the KV loop).
// Pipeline counters that persist across the work items a resident CTA runs:
// mbarrier phases continue from item to item, so barriers are initialised once.
struct PrefillState {
    int g = 0;   // KV tiles issued so far (stage = g & 1, phase = (g >> 1) & 1)
    int qb = 0;  // Q blocks loaded so far
    int items = 0;
};

// Debug trace (RunParams::trace): CTA 0, first prefill item, first 256 tiles.
#ifndef POD_TRACE_STAMPS
#define POD_TRACE_STAMPS 0  // debug builds: -DPOD_TRACE_STAMPS=1 enables the per-tile cycle stamps
#endif
// Final-output rows: fp32, or 16-bit (POD_OUT_BF16 / POD_OUT_F16) = RNE of the same
// fp32 value, so a 16-bit run equals the rounded fp32 run bit for bit.  Split
// partials always stay fp32 (fmt 0).
struct ORow {
    char* ptr;
    int fmt;
};
__device__ __forceinline__ ORow out_row(void* base, size_t elem, int fmt) {
    return {static_cast<char*>(base) + elem * (fmt ? 2u : 4u), fmt};
}
__device__ __forceinline__ uint32_t pack16(int fmt, float a, float b) {
    if (fmt == 1) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<const uint32_t*>(&h);
    }
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void store4(const ORow& o, int c, float4 v) {
    if (o.fmt == 0)
        *reinterpret_cast<float4*>(o.ptr + 4 * c) = v;
    else
        *reinterpret_cast<uint2*>(o.ptr + 2 * c) = make_uint2(pack16(o.fmt, v.x, v.y), pack16(o.fmt, v.z, v.w));
}
__device__ __forceinline__ void store1(const ORow& o, int c, float v) {
    if (o.fmt == 0)
        reinterpret_cast<float*>(o.ptr)[c] = v;
    else if (o.fmt == 1)
        reinterpret_cast<__nv_bfloat16*>(o.ptr)[c] = __float2bfloat16_rn(v);
    else
        reinterpret_cast<__half*>(o.ptr)[c] = __float2half_rn(v);
}

// Warp index broadcast from lane 0, so the compiler treats it (and the role loops
// derived from it) as warp-uniform and keeps MMA / TMA operands on the uniform datapath.
__device__ __forceinline__ int uniform_warp() {
    return POD_UNIFORM_WARP ? __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0)
                            : static_cast<int>(threadIdx.x >> 5);
}

__device__ __forceinline__ void trace_stamp(const RunParams& p, int items, int t, int k) {
    if (POD_TRACE_STAMPS && p.trace && blockIdx.x == 0 && items == 0 && t < 768 && p.role_log) {
        int32_t* tr = p.role_log + p.trace;
        tr[t * 8 + k] = static_cast<int32_t>(clock64());
    }
}

template <int kFmt>
__device__ void prefill_item(const RunParams& p, const CUtensorMap* tmq, const CUtensorMap* tmk,
                             const CUtensorMap* tmv, int cta_id, uint8_t* smem, uint32_t tmem,
                             PrefillState& ps) {
    const PrefillCta job = p.pctas[cta_id];
    const int tid = threadIdx.x;
    const int warp = uniform_warp(), lane = tid & 31;
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t sQ = sbase + kOffQ, sK = sbase + kOffK, sV = sbase + kOffV;
    const uint32_t bar0 = sbase + kOffBar;
    const uint32_t b_qfull = bar0 + 0, b_qempty = bar0 + 8;
    const uint32_t b_kfull = bar0 + 16, b_kempty = bar0 + 32;  // [2] each, 8 B apart
    const uint32_t b_vfull = bar0 + 48, b_vempty = bar0 + 64;
    const uint32_t b_sfull = bar0 + 80;                        // [2]
    const uint32_t b_pfull = bar0 + 96;                        // [2], 4 arrivals (one per softmax warp)
    const uint32_t b_pv = bar0 + 112;                          // [2]

    const int G = p.group;
    const int rpb = kMBlock / G;
    const int nblocks = (job.rows + rpb - 1) / rpb;
    const int pbeg = p.page_indptr[0];
    const int npages = p.page_indptr[1] - pbeg;
    // every thread advances the shared counters identically (broadcast from lane 0: the
    // compiler then keeps the stage / phase arithmetic on the uniform datapath)
    int g0 = __shfl_sync(0xffffffffu, ps.g, 0), qb0 = __shfl_sync(0xffffffffu, ps.qb, 0);
    for (int b = 0; b < nblocks; ++b) {
        const int nt = prefill_block(p, job, b).nt;
        if (nt > 0) {
            ps.g += nt;
            ps.qb += 1;
        }
    }
    ps.items += 1;

    if (warp == 4) {
        // ------------------------------------------------ TMA producer --
        // (warp-uniform loop; single-thread instructions are elect-predicated)
        {
            PageIds pk, pvi;
            pk.init(p.page_indices + pbeg, npages, (job.kv_begin / 16));
            pvi.init(p.page_indices + pbeg, npages, (job.kv_begin / 16));
            int g = g0, qb = qb0;
            for (int b = 0; b < nblocks; ++b) {
                const BlockRange br = prefill_block(p, job, b);
                if (br.nt == 0) continue;
                if (b > 0) {  // every block restarts at the item's first key
                    pk.init(p.page_indices + pbeg, npages, br.kt0 / 16);
                    pvi.init(p.page_indices + pbeg, npages, br.kt0 / 16);
                }
                if (qb > 0) ptx::mbar_wait_relaxed<>(b_qempty, (qb - 1) & 1);
                ptx::mbar_arrive_expect_tx_elect(b_qfull, kQBytes);
                ptx::tma_load_3d_elect(sQ, tmq, b_qfull, 0, job.kv_head * G, br.r0);
                ptx::tma_load_3d_elect(sQ + kMBlock * 128, tmq, b_qfull, 64, job.kv_head * G, br.r0);
                ++qb;
                for (int t = 0; t <= br.nt; ++t) {
                    if (t < br.nt) {  // K of tile t
                        const int gg = g + t, st = gg & 1;
                        if (gg >= 2) ptx::mbar_wait_relaxed<>(b_kempty + 8 * st, ((gg >> 1) - 1) & 1);
                        trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), 256 + t, 4);
                        ptx::mbar_arrive_expect_tx_elect(b_kfull + 8 * st, kKvStageBytes);
                        prefill_load_kv_tile(p, tmk, sK + st * kKvStageBytes, b_kfull + 8 * st,
                                             br.kt0 + t * kKvTile, job.kv_head, pk);
                        trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), 256 + t, 5);
                    }
                    if (t > 0) {  // V of tile t-1
                        const int gg = g + t - 1, st = gg & 1;
                        // the fp16 V shadow is written by the kernel launched just before this
                        // one (programmatic dependent launch): wait for it at the first V load
                        if (p.vs_pages && t == 1) ptx::griddep_wait();
                        if (gg >= 2) ptx::mbar_wait_relaxed<>(b_vempty + 8 * st, ((gg >> 1) - 1) & 1);
                        trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), 256 + t - 1, 6);
                        ptx::mbar_arrive_expect_tx_elect(b_vfull + 8 * st, kKvStageBytes);
                        prefill_load_v_pages<kKvTile / 16>(tmv, sV + st * kKvStageBytes, b_vfull + 8 * st,
                                                           br.kt0 + (t - 1) * kKvTile, job.kv_head, pvi, p.vs_pages);
                        trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), 256 + t - 1, 7);
                    }
                }
                g += br.nt;
            }
        }
    } else if (warp == 5) {
        // -------------------------------------------------- MMA issuer --
        {
            int g = g0, qb = qb0;
            for (int b = 0; b < nblocks; ++b) {
                const BlockRange br = prefill_block(p, job, b);
                if (br.nt == 0) continue;
                ptx::mbar_wait(b_qfull, qb & 1);
                for (int j = 0; j < 2 && j < br.nt; ++j) {
                    const int gg = g + j, st = gg & 1;
                    ptx::mbar_wait(b_kfull + 8 * st, (gg >> 1) & 1);
                    ptx::tc_fence_after();
                    prefill_issue_qk<kFmt>(tmem + kTmemS0 + st * kKvTile, sQ, sK + st * kKvStageBytes);
                    ptx::umma_commit_elect(b_sfull + 8 * st);
                    ptx::umma_commit_elect(b_kempty + 8 * st);
                    if (j == br.nt - 1) ptx::umma_commit_elect(b_qempty);
                }
                for (int t = 0; t < br.nt; ++t) {
                    const int gg = g + t, st = gg & 1;
                    ptx::mbar_wait(b_pfull + 8 * st, (gg >> 1) & 1);
                    trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), t, 3);
                    ptx::mbar_wait(b_vfull + 8 * st, (gg >> 1) & 1);
                    trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), t, 4);
                    ptx::tc_fence_after();
                    if (kFmt == 1 && p.p_f16)  // fp16 P x fp16 V (converted by the softmax warps)
                        prefill_issue_pv<0>(tmem + kTmemO, tmem + kTmemS0 + st * kKvTile, sV + st * kKvStageBytes,
                                            t > 0, false);
                    else
                        prefill_issue_pv<kFmt>(tmem + kTmemO, tmem + kTmemS0 + st * kKvTile,
                                               sV + st * kKvStageBytes, t > 0, p.p_split != 0);
                    ptx::umma_commit_elect(b_pv + 8 * st);
                    ptx::umma_commit_elect(b_vempty + 8 * st);
                    trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), t, 7);
                    if (p.trace_mode == 2 && blockIdx.x == 0 && ps.items == 1 && b == 0) {
                        ptx::mbar_wait(b_pv + 8 * st, (gg >> 1) & 1);  // debug: PV execution latency
                        trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), 512 + t, 0);
                    }
                    if (t + 2 < br.nt) {
                        const int g2 = gg + 2;
                        ptx::mbar_wait(b_kfull + 8 * st, (g2 >> 1) & 1);
                        trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), t, 5);
                        ptx::tc_fence_after();
                        prefill_issue_qk<kFmt>(tmem + kTmemS0 + st * kKvTile, sQ, sK + st * kKvStageBytes);
                        ptx::umma_commit_elect(b_sfull + 8 * st);
                        ptx::umma_commit_elect(b_kempty + 8 * st);
                        if (t + 2 == br.nt - 1) ptx::umma_commit_elect(b_qempty);
                        trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), 512 + t, 1);
                        if (p.trace_mode == 2 && blockIdx.x == 0 && ps.items == 1 && b == 0) {
                            ptx::mbar_wait(b_sfull + 8 * st, (g2 >> 1) & 1);  // debug: QK execution latency
                            trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), 512 + t, 2);
                        }
                    }
                }
                g += br.nt;
                ++qb;
            }
        }
    } else {
        // ------------------------------------------ softmax (128 threads) --
        const int m = tid;  // TMEM lane == M row
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
        int g = g0;
        for (int b = 0; b < nblocks; ++b) {
            const BlockRange br = prefill_block(p, job, b);
            const int my_r = br.r0 + m / G;
            const int my_g = m % G;
            const bool row_ok = (m / G) < br.nrows;
            const int vis = p.offset + my_r;  // last visible key (inclusive)
            const int qhead = job.kv_head * G + my_g;
            ORow orow;
            float* lrow;
            if (job.n_splits == 1) {
                orow = out_row(p.o_prefill, (static_cast<size_t>(my_r) * p.hq + qhead) * p.hd, p.out_fmt);
                lrow = p.lse_prefill + static_cast<size_t>(my_r) * p.hq + qhead;
            } else {
                const size_t row = (static_cast<size_t>(job.split) * p.chunk + my_r) * p.hq + qhead;
                orow = out_row(p.ppart_o, row * p.hd, 0);
                lrow = p.ppart_lse + row;
            }
            if (br.nt == 0) {
                if (row_ok) {
                    for (int c = 0; c < p.hd; c += 4) store4(orow, c, make_float4(0.f, 0.f, 0.f, 0.f));
                    *lrow = -INFINITY;
                }
                continue;
            }
            float m_run = -INFINITY, l_run = 0.f;
            for (int t = 0; t < br.nt; ++t) {
                const int gg = g + t, st = gg & 1;
                const uint32_t s_addr = lane_base + kTmemS0 + st * kKvTile;
                if (tid == 0) trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), t, 0);
                ptx::mbar_wait(b_sfull + 8 * st, (gg >> 1) & 1);
                if (tid == 0) trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), t, 1);
                ptx::tc_fence_after();
                float s[kKvTile];
                ptx::tmem_ld32(s_addr, *reinterpret_cast<float(*)[32]>(&s[0]));
                ptx::tmem_ld32(s_addr + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
                ptx::tmem_wait_ld();
                const int kb = br.kt0 + t * kKvTile;
                // valid keys of this row inside the tile: [lo, hi)
                const int lo = max(job.kv_begin - kb, 0);
                const int hi = row_ok ? min(min(job.kv_end, vis + 1) - kb, kKvTile) : 0;
                // interior tiles (every row of the warp sees every key) skip masking
                if (!__all_sync(0xffffffffu, lo == 0 && hi == kKvTile)) {
#pragma unroll
                    for (int c = 0; c < kKvTile; ++c)
                        if (c < lo || c >= hi) s[c] = -INFINITY;
                }
                const float tmax = row_max<kKvTile>(s);
                const float m_new = fmaxf(m_run, tmax * p.sl2);
                // lazy rescale (only when the max grows by > 2^8): exact algebra,
                // the stale reference max bounds p by 256.
                const bool need = m_new > m_run + 8.f;
                const float m_use = need ? m_new : m_run;
                const float factor = need ? ptx::ex2(m_run - m_new) : 1.f;
                l_run *= factor;
                m_run = m_use;
                // P -> TMEM over the consumed S row (A operand of the TS MMA), in two
                // 32-key halves of hi parts in columns [0,32); with p_split the lo
                // parts (p - hi) go to [32,64), so hi + lo carries ~15 mantissa bits.
                // A row with nothing visible yet has m = -inf and all scores -inf:
                // offset 0 keeps ex2(-inf) = 0 without a predicate per score.
                const float neg_m = m_use == -INFINITY ? 0.f : -m_use;
                float lsum;
                if (kFmt == 1 && p.p_f16)
                    lsum = softmax_p_row<kFmt, 3>(s, p.sl2, neg_m, s_addr);
                else if (kFmt == 1 && p.p_split)
                    lsum = softmax_p_row<kFmt, 1>(s, p.sl2, neg_m, s_addr);
                else if (p.p_split)
                    lsum = softmax_p_row<kFmt, 2>(s, p.sl2, neg_m, s_addr);
                else
                    lsum = softmax_p_row<kFmt, 0>(s, p.sl2, neg_m, s_addr);
                l_run += lsum;
                if (kFmt == 1 && p.p_f16 && !p.vs_pages) {  // V(t) -> fp16 before P(t) goes to the MMA issuer
                    ptx::mbar_wait(b_vfull + 8 * st, (gg >> 1) & 1);
                    v_stage_to_f16<kKvStageBytes, 128>(sV + st * kKvStageBytes, tid);
                }
                if (tid == 0) trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), t, 2);
                // O is rescaled only when the reference max moved (rare, lazy): only
                // then wait for PV_{t-1}, the newest MMA that writes O (PV_t cannot be
                // issued before this warp arrives, so the parity wait is unambiguous).
                if (t > 0 && __any_sync(0xffffffffu, need)) {
                    ptx::mbar_wait(b_pv + 8 * ((gg - 1) & 1), ((gg - 1) >> 1) & 1);
                    if (tid == 0) trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), t, 6);
                    ptx::tc_fence_after();
#pragma unroll 1
                    for (int ch = 0; ch < kHeadDim / 32; ++ch) {
                        float o[32];
                        ptx::tmem_ld32(lane_base + kTmemO + ch * 32, o);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int c = 0; c < 32; ++c) o[c] *= factor;
                        ptx::tmem_st32(lane_base + kTmemO + ch * 32, o);
                    }
                }
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) trace_stamp(p, ps.items - 1 + (b > 0 ? 1 : 0), 256 + t, warp);
                if (lane == 0) ptx::mbar_arrive(b_pfull + 8 * st);
            }
            // ------------------------------------------------- epilogue --
            {
                const int gl = g + br.nt - 1;
                ptx::mbar_wait(b_pv + 8 * (gl & 1), (gl >> 1) & 1);
            }
            ptx::tc_fence_after();
            const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll 1
            for (int ch = 0; ch < kHeadDim / 32; ++ch) {
                float o[32];
                ptx::tmem_ld32(lane_base + kTmemO + ch * 32, o);
                ptx::tmem_wait_ld();
                if (row_ok) {
#pragma unroll
                    for (int c = 0; c < 32; c += 4)
                        if (ch * 32 + c < p.hd)
                            store4(orow, ch * 32 + c,
                                   make_float4(o[c] * inv, o[c + 1] * inv, o[c + 2] * inv, o[c + 3] * inv));
                }
            }
            if (row_ok) *lrow = l_run > 0.f ? (m_run + ptx::lg2(l_run)) * kLn2 : -INFINITY;
            ptx::tc_fence_before();
            g += br.nt;
        }
    }
}

// ============================================================= decode ===
static_assert(kDecWarpsK * kDecWarpBytes <= kOffBar, "decode rings must fit below the barrier block");

// Decode inner products on the warp-level tensor path (mma.sync m16n8k16,
// fp32 accumulate): the G query heads of a KV head are the M rows (padded to
// 16), 8 keys are an N tile, so a 16-key page costs 16 MMAs for Q K^T and 32
// for P V (P split into bf16 hi + lo parts, which keeps P at ~16 mantissa bits).
// K/V pages land in shared memory through TMA with the 128-byte swizzle, read
// back with ldmatrix (.trans for V) without bank conflicts.
template <int kFmt>
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
    if constexpr (kFmt == 1)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
    else
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// Byte offset of (row, 16-byte chunk c in 0..15) of a 16 x 128 page stored as two
// 128B-swizzled column halves of 2 KB (TMA SWIZZLE_128B boxes of 64 elements).
__device__ __forceinline__ uint32_t page_off(int row, int c) {
    return static_cast<uint32_t>((c >> 3) * 2048 + row * 128 + (((c & 7) ^ (row & 7)) << 4));
}

__device__ __forceinline__ void decode_issue_page(const RunParams& p, const CUtensorMap* tk,
                                                  const CUtensorMap* tv, uint32_t dst, uint32_t bar,
                                                  int h, int phys) {
    ptx::mbar_arrive_expect_tx_elect(bar, kDecStageBytes);
    ptx::tma_load_5d_elect(dst, tk, bar, 0, 0, 0, h, phys);
    ptx::tma_load_5d_elect(dst + kDecPageBytes, tv, bar, 0, 0, 0, h, phys);
}

__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
// A-operand mma: D (16 x 8) += A (16 x 16, four regs) * B (16 x 8).
template <int kFmt>
__device__ __forceinline__ void mma16816a(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    if constexpr (kFmt == 1)
        asm(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    else
        asm(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One physical decode CTA: 4 warps = 4 virtual decode CTAs over
// split_ranges(kv_end - kv_begin, 4) (work_decomp.hpp:179-197, semantics of
// decode_attention_splitk, attention.hpp:240-292).  Each warp streams its pages
// (K and V head-pages, 4 KB each) through its own 3-stage TMA ring and computes
// in the transposed form  S^T = K Q^T  and  O^T += V^T P^T  (mma.sync m16n8k16):
// the 16 keys of a page are the M rows and the G <= 8 query heads the N columns,
// so a page costs 8 MMAs for the scores and 16 for P V (P split into bf16 hi + lo).
// Lane (g, t) = (lane / 4, lane % 4) holds scores of keys g, g + 8 for heads
// 2t, 2t + 1; per-head max / sum are shuffle reductions over g.  The 4 warp
// partials are LSE-merged through shared memory at the end.
// Decode group geometry: kW warps, each with a kS-stage ring of K+V head-pages.
// `ring0` / `bars0`: shared addresses of warp 0's ring and barriers; `red` aliases
// the ring region for the in-group merge; `bar_id` names the group's barrier.
template <int G, int kFmt, int kW, int kS>
__device__ void decode_item(const RunParams& p, const CUtensorMap* tk, const CUtensorMap* tv, int cta_id,
                            int warp, uint32_t ring0, uint32_t bars0, float* red, int bar_id, int& dpos) {
    static_assert(G <= 8, "decode: G query heads of one KV head are the N = 8 MMA columns");
    constexpr int kDecStages = kS;
    const int lane = threadIdx.x & 31;
    const int tid = warp * 32 + lane;
    const DecodeCta job = p.dctas[cta_id];
    const int len = job.kv_end - job.kv_begin;
    const int base = len / kW, rem = len % kW;
    const int wb = job.kv_begin + warp * base + min(warp, rem);
    const int we = wb + base + (warp < rem ? 1 : 0);
    const int h = job.kv_head;
    const int gq = lane >> 2, tq = lane & 3;
    const uint32_t ring = ring0 + warp * (kS * kDecStageBytes);
    const uint32_t bars = bars0 + warp * (kS * 8);
    const bool h0ok = 2 * tq < G, h1ok = 2 * tq + 1 < G;  // this lane's two head columns exist
    // G = 2, 4: P lo is packed into the free head columns (lane t ^ G/2)
    constexpr bool kPack = G == 2 || G == 4;
    constexpr int kPackXor = G / 2;
    const bool lo_lane = kPack && tq >= G / 2;

    // B fragments of Q^T (N = heads): head gq, d = 16 ks + 2t (+8); zero for heads >= G
    using elem_t = uint16_t;
    uint32_t qb[8][2];
    {
        const elem_t* q = static_cast<const elem_t*>(p.q_decode) +
                          (static_cast<size_t>(job.request) * p.hq + h * G + gq) * p.hd;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {  // d past hd: zero (the K pages read zeros there too)
            qb[ks][0] = gq < G && 16 * ks + 2 * tq < p.hd ? *reinterpret_cast<const uint32_t*>(q + 16 * ks + 2 * tq) : 0u;
            qb[ks][1] = gq < G && 16 * ks + 8 + 2 * tq < p.hd ? *reinterpret_cast<const uint32_t*>(q + 16 * ks + 8 + 2 * tq)
                                                               : 0u;
        }
    }
    float m0 = -INFINITY, m1 = -INFINITY;  // running max of heads 2t, 2t+1 (log2 domain)
    float l0 = 0.f, l1 = 0.f;              // this lane's partial sums (keys g, g+8)
    float o[8][4];                         // O^T fragments: d-tile md, rows d = 16md + g (+8), cols heads 2t, 2t+1
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;

    const int32_t* pidx = p.page_indices + p.page_indptr[job.page_row];
    const int pg0 = wb >> 4;
    const int npg = we > wb ? ((we - 1) >> 4) - pg0 + 1 : 0;
    // page ids: two 32-entry windows [cache_base, +32) and [+32, +64), one id per lane
    // (the second window is loaded one window ahead, off the critical path)
    int cache_base = 0;
    int cached = (lane < npg) ? __ldg(pidx + pg0 + lane) : 0;
    int cached2 = (32 + lane < npg) ? __ldg(pidx + pg0 + 32 + lane) : 0;
#pragma unroll
    for (int j = 0; j < kDecStages; ++j) {
        const int phys = __shfl_sync(0xffffffffu, cached, j);
        const int st = (dpos + j) % kDecStages;
        if (j < npg) decode_issue_page(p, tk, tv, ring + st * kDecStageBytes, bars + 8 * st, h, phys);
    }
    __syncwarp();
    const int lm = lane >> 3, lr = lane & 7;  // ldmatrix: matrix lm, row lr
    // S^T (16 keys x 8 heads) = K Q^T of one page: 8 k-steps as two independent
    // MMA chains (even / odd k-steps) to halve the dependent-latency chain.
    auto scores = [&](uint32_t kst, float (&sc)[4]) {
        float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < 8; ks += 2) {
            uint32_t a[4], b[4];  // keys 0-7 / 8-15 x d 16ks..+7 / +8..+15
            ldsm_x4(kst + page_off((lm & 1) * 8 + lr, 2 * ks + (lm >> 1)), a[0], a[1], a[2], a[3]);
            ldsm_x4(kst + page_off((lm & 1) * 8 + lr, 2 * ks + 2 + (lm >> 1)), b[0], b[1], b[2], b[3]);
            mma16816a<kFmt>(sa, a, qb[ks][0], qb[ks][1]);
            mma16816a<kFmt>(sb, b, qb[ks + 1][0], qb[ks + 1][1]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) sc[c] = sa[c] + sb[c];
    };
    // Software pipeline over pages: the score MMAs of page i+1 are issued before the
    // softmax and P V of page i, so their latency overlaps the dependent chain of i.
    float sc[4] = {0.f, 0.f, 0.f, 0.f};
    // debug trace (POD_TRACE): CTA 0, items by claim order, rows 512 + k
    int32_t* dtr = nullptr;
    if (p.trace && blockIdx.x == 0 && p.role_log) {
        int32_t* cnt = p.role_log + p.trace + 767 * 8 + 7;  // item counter (last row)
        const int k = __shfl_sync(0xffffffffu, (warp == 0 && lane == 0) ? atomicAdd(cnt, 0) : 0, 0);
        if (k < 200) dtr = p.role_log + p.trace + (512 + k) * 8;
        if (dtr && lane == 0) dtr[warp == 0 ? 0 : 7] = static_cast<int32_t>(clock64());
    }
    if (npg > 0) {
        const int st = dpos % kDecStages;
        ptx::mbar_wait(bars + 8 * st, (dpos / kDecStages) & 1);
        if (dtr && lane == 0 && warp == 0) dtr[1] = static_cast<int32_t>(clock64());
        scores(ring + st * kDecStageBytes, sc);
    }
    for (int i = 0; i < npg; ++i) {
        const int n = dpos + i;
        const int st = n % kDecStages;
        const uint32_t vst = ring + st * kDecStageBytes + kDecPageBytes;
        float scn[4] = {0.f, 0.f, 0.f, 0.f};
        if (i + 1 < npg) {
            const int st1 = (n + 1) % kDecStages;
#if POD_DEC_SLEEP > 0
            ptx::mbar_wait_relaxed<POD_DEC_SLEEP>(bars + 8 * st1, ((n + 1) / kDecStages) & 1);
#else
            ptx::mbar_wait(bars + 8 * st1, ((n + 1) / kDecStages) & 1);
#endif
            scores(ring + st1 * kDecStageBytes, scn);
        }
        // sc: (key g, head 2t), (key g, head 2t+1), (key g+8, head 2t), (key g+8, head 2t+1)
        float x[4] = {sc[0] * p.sl2, sc[1] * p.sl2, sc[2] * p.sl2, sc[3] * p.sl2};
        const int kfirst = (pg0 + i) * 16;
        if (kfirst < wb || kfirst + 16 > we) {
            const int k0 = kfirst + gq, k1 = kfirst + gq + 8;
            if (k0 < wb || k0 >= we) x[0] = x[1] = -INFINITY;
            if (k1 < wb || k1 >= we) x[2] = x[3] = -INFINITY;
        }
        float mx0 = fmaxf(x[0], x[2]), mx1 = fmaxf(x[1], x[3]);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
        const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
        const float f0 = ptx::ex2(m0 - n0), f1 = ptx::ex2(m1 - n1);  // m = -inf -> 0
        m0 = n0;
        m1 = n1;
        const float p00 = h0ok ? ptx::ex2(x[0] - n0) : 0.f, p01 = h1ok ? ptx::ex2(x[1] - n1) : 0.f;
        const float p10 = h0ok ? ptx::ex2(x[2] - n0) : 0.f, p11 = h1ok ? ptx::ex2(x[3] - n1) : 0.f;
        l0 = l0 * f0 + (p00 + p10);
        l1 = l1 * f1 + (p01 + p11);
        // P^T as the B operand: transpose the two 8x8 (key x head) blocks; hi + lo parts
        const uint32_t h0 = pack2<kFmt>(p00, p01), h1 = pack2<kFmt>(p10, p11);
        const float2 u0 = unpack2<kFmt>(h0), u1 = unpack2<kFmt>(h1);
        const uint32_t q0 = pack2<kFmt>(p00 - u0.x, p01 - u0.y), q1 = pack2<kFmt>(p10 - u1.x, p11 - u1.y);
        if constexpr (kPack) {
            // G <= 4: the lo parts ride in the unused head columns [G, 2G) (lanes
            // t ^ G/2), so one MMA per d-tile accumulates O_hi and O_lo side by side
            const float f0s = __shfl_xor_sync(0xffffffffu, f0, kPackXor), f1s = __shfl_xor_sync(0xffffffffu, f1, kPackXor);
            const uint32_t q0s = __shfl_xor_sync(0xffffffffu, q0, kPackXor), q1s = __shfl_xor_sync(0xffffffffu, q1, kPackXor);
            const float rf0 = lo_lane ? f0s : f0, rf1 = lo_lane ? f1s : f1;
            if (!__all_sync(0xffffffffu, rf0 == 1.f && rf1 == 1.f)) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    o[j][0] *= rf0;
                    o[j][1] *= rf1;
                    o[j][2] *= rf0;
                    o[j][3] *= rf1;
                }
            }
            const uint32_t b0 = movmatrix_t(lo_lane ? q0s : h0), b1 = movmatrix_t(lo_lane ? q1s : h1);
            // ---- O^T (128 d x [hi heads | lo heads]) += V^T P^T: one MMA per 16-d tile
#pragma unroll
            for (int md = 0; md < 8; ++md) {
                uint32_t a[4];  // A = V^T: rows d 16md..+7 / +8..+15, cols keys 0-7 / 8-15
                ldsm_x4_t(vst + page_off((lm >> 1) * 8 + lr, 2 * md + (lm & 1)), a[0], a[1], a[2], a[3]);
                mma16816a<kFmt>(o[md], a, b0, b1);
            }
        } else {
            if (!__all_sync(0xffffffffu, f0 == 1.f && f1 == 1.f)) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    o[j][0] *= f0;
                    o[j][1] *= f1;
                    o[j][2] *= f0;
                    o[j][3] *= f1;
                }
            }
            const uint32_t bh0 = movmatrix_t(h0), bh1 = movmatrix_t(h1);
            const uint32_t bl0 = movmatrix_t(q0), bl1 = movmatrix_t(q1);
            // ---- O^T (128 d x 8 heads) += V^T P^T: one MMA per 16-d tile (x2 for hi/lo)
#pragma unroll
            for (int md = 0; md < 8; ++md) {
                uint32_t a[4];  // A = V^T: rows d 16md..+7 / +8..+15, cols keys 0-7 / 8-15
                ldsm_x4_t(vst + page_off((lm >> 1) * 8 + lr, 2 * md + (lm & 1)), a[0], a[1], a[2], a[3]);
                mma16816a<kFmt>(o[md], a, bh0, bh1);
                mma16816a<kFmt>(o[md], a, bl0, bl1);
            }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) sc[c] = scn[c];
        // ---- refill this stage (K consumed last iteration, V just now) with page i + kDecStages
        const int nxt = i + kDecStages;
        if (nxt < npg) {
            if (nxt - cache_base >= 32) {
                cache_base += 32;
                cached = cached2;
                cached2 = (cache_base + 32 + lane < npg) ? __ldg(pidx + pg0 + cache_base + 32 + lane) : 0;
            }
            const int phys = __shfl_sync(0xffffffffu, cached, nxt - cache_base);
            __syncwarp();
            decode_issue_page(p, tk, tv, ring + st * kDecStageBytes, bars + 8 * st, h, phys);
        }
    }
    dpos += npg;
    if (dtr && lane == 0) atomicMax(&dtr[2 + (warp == 0 ? 0 : 1)], static_cast<int32_t>(clock64()));
    if constexpr (kPack) {  // O = O_hi + O_lo (hi lanes keep the sum)
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) o[j][c] += __shfl_xor_sync(0xffffffffu, o[j][c], kPackXor);
    }
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, off);
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    // in-group merge of the warps' ranges (LSE merge, attention.hpp:294-326);
    // reuses the ring region (every warp is past its last TMA wait).
    constexpr int kStride = kHeadDim + 4;
    static_assert(kW * 8 * (kHeadDim + 4) * 4 <= kW * kS * kDecStageBytes, "merge scratch fits the rings");
    ptx::named_bar_sync(bar_id, kW * 32);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
        const int head = 2 * tq + hh;
        if (head < G) {
            float* dst = red + (warp * G + head) * kStride;
#pragma unroll
            for (int md = 0; md < 8; ++md) {
                dst[16 * md + gq] = o[md][hh];
                dst[16 * md + gq + 8] = o[md][2 + hh];
            }
            if (gq == 0) {
                dst[kHeadDim] = hh ? m1 : m0;
                dst[kHeadDim + 1] = hh ? l1 : l0;
            }
        }
    }
    ptx::named_bar_sync(bar_id, kW * 32);
    for (int idx = tid; idx < G * p.hd; idx += kW * 32) {  // the tensor's d columns (hd <= 128)
        const int g = idx / p.hd, d = idx % p.hd;
        float mw[kW], M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kW; ++w) {
            mw[w] = red[(w * G + g) * kStride + kHeadDim];
            M = fmaxf(M, mw[w]);
        }
        float L = 0.f, acc = 0.f;
#pragma unroll
        for (int w = 0; w < kW; ++w) {
            const float wt = ptx::ex2(mw[w] - M);  // empty warp: m = -inf -> 0
            L += red[(w * G + g) * kStride + kHeadDim + 1] * wt;
            acc += red[(w * G + g) * kStride + d] * wt;
        }
        const int qhead = h * G + g;
        if (dtr && idx == tid && tid == 0) dtr[4] = static_cast<int32_t>(clock64());
        const float out = acc / L;
        const float lse = (M + ptx::lg2(L)) * kLn2;
        if (job.n_splits == 1) {
            store1(out_row(p.o_decode, (static_cast<size_t>(job.request) * p.hq + qhead) * p.hd, p.out_fmt), d,
                   out);
            if (d == 0) p.lse_decode[static_cast<size_t>(job.request) * p.hq + qhead] = lse;
        } else {
            const size_t row = (static_cast<size_t>(job.request) * p.decode_splits + job.split) * p.hq + qhead;
            p.dpart_o[row * p.hd + d] = out;
            if (d == 0) p.dpart_lse[row] = lse;
        }
    }
    if (dtr && tid == 0) {
        dtr[5] = static_cast<int32_t>(clock64());
        atomicAdd(p.role_log + p.trace + 767 * 8 + 7, 1);
    }
}

// ============================================================== merge ===
// merge_partials (attention.hpp:294-326) for one output row, one warp: lse_tot = m +
// log sum exp(lse_i - m), O = sum_i exp(lse_i - lse_tot) O_i in split (= kv-range)
// order.  Partials are read through L2 (ld.global.cg): they were written by other
// SMs during this launch (in-kernel merge) or the previous one.
__device__ __forceinline__ void merge_row(const float* po, const float* pl, size_t stride_o, size_t stride_l, int n,
                                          const ORow& out_o, float* out_l, int lane, int hd) {
    float M = -INFINITY;
    for (int i = 0; i < n; ++i) M = fmaxf(M, __ldcg(pl + i * stride_l));
    float tot = 0.f;
    for (int i = 0; i < n; ++i) tot += ptx::ex2((__ldcg(pl + i * stride_l) - M) * kLog2e);
    const float lse_tot = M + ptx::lg2(tot) * kLn2;
    if (lane == 0) *out_l = lse_tot;
    if (lane * 4 >= hd) return;  // columns past the head dim
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = 0; i < n; ++i) {
        const float w = ptx::ex2((__ldcg(pl + i * stride_l) - lse_tot) * kLog2e);
        const float4 v = __ldcg(reinterpret_cast<const float4*>(po + i * stride_o + lane * 4));
        acc.x += w * v.x;
        acc.y += w * v.y;
        acc.z += w * v.z;
        acc.w += w * v.w;
    }
    store4(out_o, lane * 4, acc);
}


// One warp per output (row, q head): O = sum_i exp(lse_i - lse_tot) O_i in
// split order (= kv-range order), lse_tot = m + log(sum exp(lse_i - m)).
// mode 0: prefill rows r in [0, chunk); partials [split][chunk][Hq][d].
// mode 1: decode requests; partials [req][splits][Hq][d].
// One launch merges both kinds: warps [0, prefill_rows) the prefill rows (mode 0),
// the next decode_rows warps the decode rows (mode 1).
__global__ void __launch_bounds__(256) merge_kernel(RunParams p, const int32_t* tile_splits,
                                                    int tile_q, int prefill_rows, int decode_rows) {
    // launched as a programmatic dependent of the POD kernel (its launch latency overlaps
    // the kernel's tail); every partial it reads is visible once this returns
    ptx::griddep_wait();
    int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    int mode = 0;
    if (warp_global >= prefill_rows) {
        warp_global -= prefill_rows;
        mode = 1;
        if (warp_global >= decode_rows) return;
    }
    const int r = warp_global / p.hq, qh = warp_global % p.hq;
    int n;
    const float* po;
    const float* pl;
    size_t stride_o, stride_l;
    ORow out_o;
    float* out_l;
    if (mode == 0) {
        n = tile_splits[r / tile_q];
        if (n <= 1) return;
        const size_t row = static_cast<size_t>(r) * p.hq + qh;
        po = p.ppart_o + row * p.hd;
        pl = p.ppart_lse + row;
        stride_l = static_cast<size_t>(p.chunk) * p.hq;
        stride_o = stride_l * p.hd;
        out_o = out_row(p.o_prefill, row * p.hd, p.out_fmt);
        out_l = p.lse_prefill + row;
    } else {
        n = p.dec_nsplit[r];  // this request's own split count (min(splits, ctx), whole waves)
        if (n <= 1) return;
        const size_t row = static_cast<size_t>(r) * p.decode_splits * p.hq + qh;
        po = p.dpart_o + row * p.hd;
        pl = p.dpart_lse + row;
        stride_l = p.hq;
        stride_o = stride_l * p.hd;
        out_o = out_row(p.o_decode, (static_cast<size_t>(r) * p.hq + qh) * p.hd, p.out_fmt);
        out_l = p.lse_decode + static_cast<size_t>(r) * p.hq + qh;
    }
    merge_row(po, pl, stride_o, stride_l, n, out_o, out_l, lane, p.hd);
}

// ============================================================ kernels ===
// Picks the next work item for this resident CTA: SM-aware runtime role binding
// (gpu_sim.hpp:114-131).  Returns op (0 prefill, 1 decode,
// -1 both pools exhausted) and the claimed dense per-op id.
__device__ __forceinline__ int2 claim_item(const RunParams& p, uint32_t sm, int32_t* log_slot_out) {
    const int ratio = p.prefill_ratio + p.decode_ratio;
    const uint32_t raw = atomicAdd(&p.ctr->sm_ctr[sm], 1u);
    int op;
    if (p.policy == POD_POLICY_COMPLEMENT) {
        // bind from what is resident on this SM: prefill while fewer than
        // prefill_ratio prefill items run here, decode otherwise
        const uint32_t resident = atomicAdd(&p.ctr->running_prefill[sm], 1u);
        op = resident < static_cast<uint32_t>(p.prefill_ratio) ? 0 : 1;
        if (op == 1) atomicSub(&p.ctr->running_prefill[sm], 1u);
    } else {
        const int ticket = static_cast<int>(raw % static_cast<uint32_t>(ratio));
        op = ticket < p.prefill_ratio ? 0 : 1;
    }
    int id = static_cast<int>(atomicAdd(&p.ctr->cta_assign[op], 1u));
    if (id >= (op == 0 ? p.num_pctas : p.num_dctas)) {
        if (p.policy == POD_POLICY_COMPLEMENT && op == 0) atomicSub(&p.ctr->running_prefill[sm], 1u);
        op ^= 1;
        id = static_cast<int>(atomicAdd(&p.ctr->cta_assign[op], 1u));
        if (id >= (op == 0 ? p.num_pctas : p.num_dctas))
            op = -1;
        else if (p.policy == POD_POLICY_COMPLEMENT && op == 0)
            atomicAdd(&p.ctr->running_prefill[sm], 1u);
    }
    *log_slot_out = -1;
    if (p.role_log && op >= 0) {
        const uint32_t slot = atomicAdd(&p.ctr->arrival, 1u);
        int32_t* rec = p.role_log + 8 * slot;
        rec[0] = static_cast<int32_t>(sm);
        rec[1] = static_cast<int32_t>(raw);
        rec[2] = op;
        rec[3] = id;
        rec[4] = static_cast<int32_t>(slot);
        rec[5] = static_cast<int32_t>(ptx::globaltimer() & 0x7fffffff);
        rec[7] = static_cast<int32_t>(blockIdx.x);
        *log_slot_out = static_cast<int32_t>(slot);
    }
    return make_int2(op, id);
}

// The POD kernel: a persistent grid of 2 CTAs per SM (every CTA holds 256 TMEM
// columns, two fill the SM's 512).  Each CTA repeatedly binds a role for its
// next work item -- a prefill CtaTask or a decode (request, kv head, split)
// parent with 4 virtual warps -- until both pools are drained.  Launched with
// num_dctas = 0 (or num_pctas = 0) it is the standalone prefill (decode) kernel
// of the serial comparator.  Persistence matters on sm_100: kernels that use
// tcgen05 get one new CTA dispatched only into an idle SM, so a classic
// CTA-per-task grid would lose the second slot after the first wave.
template <int G, int kFmt>
__global__ void __launch_bounds__(kThreads, 2)
    pod_fused_kernel(const __grid_constant__ RunParams p, const __grid_constant__ CUtensorMap tmq,
                     const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                     const __grid_constant__ CUtensorMap tdk, const __grid_constant__ CUtensorMap tdv) {
    extern __shared__ __align__(1024) uint8_t smem[];
    int* role = reinterpret_cast<int*>(smem + kOffRole);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmemSlot);
    const int tid = threadIdx.x, warp = uniform_warp(), lane = tid & 31;
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t sm = ptx::smid();
    if (tid == 0) {
        if (sbase & 1023u) __trap();  // SW128 atoms need a 1024-aligned base
        // p_full (12, 13) get one arrival per softmax warp; q_full (0) is filled by TMA
        // (expect_tx, one arrival)
        for (int i = 0; i < 16; ++i) ptx::mbar_init(sbase + kOffBar + 8 * i, (i == 12 || i == 13) ? kPrefillWarps : 1);
        for (int i = 0; i < kDecWarpsK * kDecStages; ++i) ptx::mbar_init(sbase + kOffDecBar + 8 * i, 1);
        ptx::fence_mbar_init();
    }
    // TMEM: every CTA holds 256 columns.  Every CTA that allocates relinquishes its
    // permit at once: on sm_100 a second CTA of a tcgen05 kernel is only co-scheduled
    // on an SM after the resident one has relinquished.
    const uint32_t ncols = kTmemCols;
    if (warp == 0) {
        ptx::tmem_alloc(ptx::smem_u32(tmem_slot), ncols);
        ptx::tmem_relinquish();
    }
    if (warp == 4 && lane == 0) {
        if (p.num_pctas > 0) ptx::prefetch_tmap(&tmq);
        ptx::prefetch_tmap(&tmk);
        ptx::prefetch_tmap(&tmv);
        ptx::prefetch_tmap(&tdk);
        ptx::prefetch_tmap(&tdv);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    PrefillState ps;
    int dpos = 0;
    while (true) {
        if (tid == 0) {
            int32_t slot = -1;
            const int2 w = claim_item(p, sm, &slot);
            role[0] = w.x;
            role[1] = w.y;
            role[2] = slot;
        }
        __syncthreads();
        const int op = __shfl_sync(0xffffffffu, role[0], 0), id = __shfl_sync(0xffffffffu, role[1], 0),
                  slot = role[2];
        __syncthreads();  // role[] is rewritten by the next claim
        if (op < 0) break;
        if (op == 0) {
            prefill_item<kFmt>(p, &tmq, &tmk, p.vs_pages ? &tmv : &tdv, id, smem, tmem, ps);
        } else {
            if (warp < kDecWarpsK)
                decode_item<G, kFmt, kDecWarpsK, kDecStages>(p, &tdk, &tdv, id, warp, sbase, sbase + kOffDecBar,
                                                             reinterpret_cast<float*>(smem), 2, dpos);
        }
        ptx::tc_fence_before();
        __syncthreads();
        ptx::tc_fence_after();
        if (tid == 0) {
            if (p.policy == POD_POLICY_COMPLEMENT && op == 0) atomicSub(&p.ctr->running_prefill[sm], 1u);
            if (slot >= 0) p.role_log[8 * slot + 6] = static_cast<int32_t>(ptx::globaltimer() & 0x7fffffff);
        }
    }
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, ncols);
    }
    ptx::griddep_launch_dependents();  // the split merge may start launching (it waits for completion)
    if (tid == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(&p.ctr->done, 1u);
        if (prev == gridDim.x - 1) {
            // last CTA out: re-arm the counters for the next launch (graph friendly)
            const uint32_t n = min(ptx::nsmid(), static_cast<uint32_t>(kMaxSms));
            for (uint32_t i = 0; i < n; ++i) {
                p.ctr->sm_ctr[i] = 0;
                p.ctr->running_prefill[i] = 0;
            }
            p.ctr->cta_assign[0] = 0;
            p.ctr->cta_assign[1] = 0;
            p.ctr->arrival = 0;
            p.ctr->done = 0;
            __threadfence();
        }
    }
}

#include "pod_sm.cuh"
#include "pod_oproj.cuh"

__global__ void __launch_bounds__(256) l2_flush_kernel(uint4* __restrict__ buf, size_t n16) {
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        buf[i] = z;
}

__global__ void gather_probe_kernel(const uint16_t* pool, int layout, int hkv, const int32_t* indptr,
                                    const int32_t* indices, int req, int ctx, int hd, uint16_t* out) {
    const int nc = hd / 8;  // 16-byte chunks per row
    const size_t n = static_cast<size_t>(ctx) * hkv * nc;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int chunk = static_cast<int>(i % nc);
        const int h = static_cast<int>((i / nc) % hkv);
        const int t = static_cast<int>(i / nc / hkv);
        const int phys = indices[indptr[req] + t / 16];
        const int slot = t % 16;
        size_t src;
        if (layout == POD_KV_HND)
            src = ((static_cast<size_t>(phys) * hkv + h) * 16 + slot) * hd;
        else
            src = ((static_cast<size_t>(phys) * 16 + slot) * hkv + h) * hd;
        const uint4 v = *reinterpret_cast<const uint4*>(pool + src + chunk * 8);
        *reinterpret_cast<uint4*>(out + (static_cast<size_t>(t) * hkv + h) * hd + chunk * 8) = v;
    }
}

// ========================================================== KV append ===
// One warp per (new token, KV head): 16 lanes x 16 B move the K row, the other 16
// the V row (256 B each at d = 128), from the dense new-token rows into the token's
// page slot.  HBM-bound copy: 2 x 256 B read + 2 x 256 B written per (token, head).
__global__ void __launch_bounds__(256) append_kv_kernel(const uint4* __restrict__ kp, const uint4* __restrict__ vp,
                                                        const uint4* __restrict__ kd, const uint4* __restrict__ vd,
                                                        uint4* k_pool, uint4* v_pool, const int32_t* indptr,
                                                        const int32_t* indices, const int32_t* dec_pos, int chunk,
                                                        int offset, int ndec, int hkv, int layout, int kVecs) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int rows = (chunk + ndec) * hkv;
    if (warp >= rows) return;
    const int tok = warp / hkv, h = warp % hkv;
    const bool is_pf = tok < chunk;
    const int req = is_pf ? 0 : (chunk > 0 ? 1 : 0) + (tok - chunk);
    const int pos = is_pf ? offset + tok : __ldg(dec_pos + (tok - chunk));
    const int phys = __ldg(indices + __ldg(indptr + req) + pos / 16);
    const int slot = pos % 16;
    // kVecs: 16-byte vectors per row (16 at d = 128)
    const size_t src = (static_cast<size_t>(is_pf ? tok : tok - chunk) * hkv + h) * kVecs;
    const size_t dst = (layout == POD_KV_HND ? ((static_cast<size_t>(phys) * hkv + h) * 16 + slot)
                                             : ((static_cast<size_t>(phys) * 16 + slot) * hkv + h)) * kVecs;
    const int c = lane & 15;
    if (c >= kVecs) return;
    const uint4* in = lane < 16 ? (is_pf ? kp : kd) : (is_pf ? vp : vd);
    uint4* out = lane < 16 ? k_pool : v_pool;
    out[dst + c] = __ldg(in + src + c);
}

// POD_PRECISION_F16PV, plans with vs_pages (pod_plan.cpp): the prefill request's V
// converted bf16 -> fp16 once per launch into a dense shadow [logical page][Hkv][16][d]
// (the decode role's 5-D page view with logical page ids), so the prefill CTAs stream V
// tiles that are already the PV MMA's fp16 B operand.  HBM-bound: 2 B read + 2 B written
// per element, grid-stride over 16-byte vectors.
__global__ void __launch_bounds__(256) v_shadow_kernel(const uint4* __restrict__ v_pool, uint4* __restrict__ shadow,
                                                       const int32_t* __restrict__ indptr,
                                                       const int32_t* __restrict__ indices, int pages, int hkv,
                                                       int vecs /* 16-byte vectors per row: d / 8 */, int layout) {
    const size_t per_page = static_cast<size_t>(hkv) * 16 * vecs;
    const size_t n = static_cast<size_t>(pages) * per_page;
    ptx::griddep_launch_dependents();  // the POD kernel may launch now (its prefill waits for us)
    const int32_t* row = indices + __ldg(indptr);  // request 0 = the prefill
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int lp = static_cast<int>(i / per_page);
        const size_t rem = i % per_page;
        const int h = static_cast<int>(rem / (16 * vecs));
        const int slot = static_cast<int>((rem / vecs) % 16), c = static_cast<int>(rem % vecs);
        const size_t phys = static_cast<size_t>(__ldg(row + lp));
        const size_t src = (layout == POD_KV_HND ? ((phys * hkv + h) * 16 + slot) : ((phys * 16 + slot) * hkv + h)) *
                               vecs + c;
        const uint4 w = __ldg(v_pool + src);
        shadow[i] = make_uint4(bf16x2_to_f16x2(w.x), bf16x2_to_f16x2(w.y), bf16x2_to_f16x2(w.z),
                               bf16x2_to_f16x2(w.w));
    }
}

// ================================================================ host ===
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    });
    return fn;
}

pod_status cuda_fail(cudaError_t e, const char* where) {
    set_last_error(std::string(where) + ": " + cudaGetErrorString(e));
    return POD_ERR_CUDA;
}

int64_t fused_smem_bytes() { return kSmemBytes; }
int64_t sm_smem_bytes(bool db) { return db ? SmLay<1>::kSmem : SmLay<0>::kSmem; }

struct Maps {
    CUtensorMap q, k, v;  // prefill role: SW128 boxes of 64 d x 16 tokens, Q boxes of 64 d x 128 rows
    CUtensorMap dk, dv;   // decode role: one whole head-page per box (5D view, SW128 halves)
    CUtensorMap vs;       // the fp16 V shadow (plans with vs_pages): dv's view over logical pages
};

pod_status make_maps(const pod_plan* plan, const void* q_prefill, const void* k_pool, const void* v_pool,
                     int64_t num_pages, void* workspace, Maps* m) {
    std::memset(m, 0, sizeof(*m));
    EncodeTiledFn enc = encode_fn();
    if (!enc) {
        set_last_error("cuTensorMapEncodeTiled unavailable");
        return POD_ERR_CUDA;
    }
    const CUtensorMapDataType dt = plan->batch.dtype == POD_DTYPE_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                                       : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const int hkv = plan->shape.num_kv_heads, hq = plan->shape.num_q_heads;
    const int G = hq / hkv;
    const cuuint64_t hd = static_cast<cuuint64_t>(plan->shape.head_dim);  // boxes past hd read zeros
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    {
        cuuint64_t dims[4], strides[3];
        cuuint32_t box[4];
        if (plan->batch.kv_layout == POD_KV_HND) {
            dims[0] = hd; dims[1] = 16; dims[2] = hkv; dims[3] = num_pages;
            strides[0] = hd * 2; strides[1] = 16ull * hd * 2; strides[2] = 16ull * hkv * hd * 2;
            box[0] = 64; box[1] = 16; box[2] = 1; box[3] = 1;
        } else {
            dims[0] = hd; dims[1] = hkv; dims[2] = 16; dims[3] = num_pages;
            strides[0] = hd * 2; strides[1] = static_cast<cuuint64_t>(hkv) * hd * 2;
            strides[2] = 16ull * hkv * hd * 2;
            box[0] = 64; box[1] = 1; box[2] = 16; box[3] = 1;
        }
        for (int which = 0; which < 2; ++which) {
            CUresult r = enc(which == 0 ? &m->k : &m->v, dt, 4, const_cast<void*>(which == 0 ? k_pool : v_pool),
                             dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) {
                set_last_error("cuTensorMapEncodeTiled(kv) failed: " + std::to_string(static_cast<int>(r)));
                return POD_ERR_CUDA;
            }
            // Decode role: one 4 KB box per head-page.  The page is viewed as
            // (64 d, 16 slots, 2 d-halves, head, page) so a single TMA op lands it
            // as two 128B-swizzled 2 KB halves ([half][slot][64 d]), the same smem
            // image as two SW128 boxes (TMA issue rate, not bytes, bounds small boxes).
            cuuint64_t d5[5], s5[4];
            const cuuint32_t box5[5] = {64, 16, 2, 1, 1}, estr5[5] = {1, 1, 1, 1, 1};
            d5[0] = hd < 64 ? hd : 64; d5[1] = 16; d5[2] = (hd + 63) / 64; d5[3] = hkv; d5[4] = num_pages;
            if (plan->batch.kv_layout == POD_KV_HND) {
                s5[0] = hd * 2; s5[1] = 128; s5[2] = 16ull * hd * 2; s5[3] = 16ull * hkv * hd * 2;
            } else {
                s5[0] = static_cast<cuuint64_t>(hkv) * hd * 2; s5[1] = 128; s5[2] = hd * 2;
                s5[3] = 16ull * hkv * hd * 2;
            }
            r = enc(which == 0 ? &m->dk : &m->dv, dt, 5, const_cast<void*>(which == 0 ? k_pool : v_pool), d5, s5,
                    box5, estr5, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) {
                set_last_error("cuTensorMapEncodeTiled(decode kv) failed: " + std::to_string(static_cast<int>(r)));
                return POD_ERR_CUDA;
            }
        }
    }
    if (plan->batch.has_prefill) {
        cuuint64_t dims[3] = {hd, static_cast<cuuint64_t>(hq), static_cast<cuuint64_t>(plan->batch.prefill.chunk_size)};
        cuuint64_t strides[2] = {hd * 2, static_cast<cuuint64_t>(hq) * hd * 2};
        cuuint32_t box[3] = {64, static_cast<cuuint32_t>(G), static_cast<cuuint32_t>(kMBlock / G)};
        CUresult r = enc(&m->q, dt, 3, const_cast<void*>(q_prefill), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_last_error("cuTensorMapEncodeTiled(q) failed: " + std::to_string(static_cast<int>(r)));
            return POD_ERR_CUDA;
        }
    }
    if (plan->vs_pages > 0) {  // the fp16 V shadow: dense [logical page][Hkv][16][d], dv's 5-D view
        cuuint64_t d5[5], s5[4];
        const cuuint32_t box5[5] = {64, 16, 2, 1, 1}, estr5[5] = {1, 1, 1, 1, 1};
        d5[0] = hd < 64 ? hd : 64; d5[1] = 16; d5[2] = (hd + 63) / 64; d5[3] = hkv; d5[4] = plan->vs_pages;
        s5[0] = hd * 2; s5[1] = 128; s5[2] = 16ull * hd * 2; s5[3] = 16ull * hkv * hd * 2;
        CUresult r = enc(&m->vs, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5,
                         static_cast<uint8_t*>(workspace) + plan->ws.off_vshadow, d5, s5, box5, estr5,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_last_error("cuTensorMapEncodeTiled(v shadow) failed: " + std::to_string(static_cast<int>(r)));
            return POD_ERR_CUDA;
        }
    } else {
        m->vs = m->v;  // (unused)
    }
    return POD_OK;
}

RunParams make_params(const pod_plan* plan, const void* q_prefill, const void* q_decode, const void* k_pool, const void* v_pool,
                      int64_t num_pages, const int32_t* indptr, const int32_t* indices, void* o_prefill,
                      float* lse_prefill, void* o_decode, float* lse_decode, void* workspace) {
    RunParams p{};
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    p.q_prefill = q_prefill;
    p.q_decode = q_decode;
    p.k_pool = k_pool;
    p.v_pool = v_pool;
    p.page_indptr = indptr;
    p.page_indices = indices;
    p.o_prefill = o_prefill;
    p.lse_prefill = lse_prefill;
    p.o_decode = o_decode;
    p.lse_decode = lse_decode;
    p.ppart_o = reinterpret_cast<float*>(ws + plan->ws.off_ppart_o);
    p.ppart_lse = reinterpret_cast<float*>(ws + plan->ws.off_ppart_lse);
    p.dpart_o = reinterpret_cast<float*>(ws + plan->ws.off_dpart_o);
    p.dpart_lse = reinterpret_cast<float*>(ws + plan->ws.off_dpart_lse);
    p.pctas = reinterpret_cast<const PrefillCta*>(ws + plan->ws.off_pctas);
    p.dctas = reinterpret_cast<const DecodeCta*>(ws + plan->ws.off_dctas);
    p.ctr = reinterpret_cast<SchedCounters*>(ws + plan->ws.off_counters);
    p.role_log = plan->role_log;
    p.num_pctas = static_cast<int32_t>(plan->pctas.size());
    p.num_dctas = static_cast<int32_t>(plan->dctas.size());
    p.prefill_ratio = static_cast<int32_t>(plan->prefill_ratio);
    p.decode_ratio = static_cast<int32_t>(plan->decode_ratio);
    p.hq = plan->shape.num_q_heads;
    p.hd = plan->shape.head_dim;
    p.hkv = plan->shape.num_kv_heads;
    p.group = p.hq / p.hkv;
    p.chunk = plan->batch.has_prefill ? static_cast<int32_t>(plan->batch.prefill.chunk_size) : 0;
    p.offset = plan->batch.has_prefill ? static_cast<int32_t>(plan->batch.prefill.position_offset) : 0;
    p.kv_layout = plan->batch.kv_layout;
    p.decode_splits = static_cast<int32_t>(plan->decode_splits);
    p.dec_split_base = static_cast<int32_t>(plan->dec_split_base);
    p.dec_tail_start = static_cast<int32_t>(plan->dec_tail_start);
    p.policy = plan->opts.policy;
    p.p_split = plan->opts.precision == POD_PRECISION_SPLIT ? 1 : 0;
    p.p_f16 = plan->opts.precision == POD_PRECISION_F16PV ? 1 : 0;
    p.pf_tn64 = plan->pf_tn64 ? 1 : 0;
    p.pf_db = plan->pf_db ? 1 : 0;
    p.out_fmt = plan->opts.out_dtype;
    p.dec_nsplit = reinterpret_cast<const int32_t*>(ws + plan->ws.off_dec_nsplit);
    p.vs_pages = plan->vs_pages;
#if POD_TRACE_STAMPS
    {  // debug builds only: POD_TRACE=1 (stamps) / 2 (serialised MMA issue) after the role log
        static const char* trace_env = std::getenv("POD_TRACE");
        const int t = trace_env ? std::atoi(trace_env) : 0;
        p.trace = t ? static_cast<int32_t>(8 * (plan->pctas.size() + plan->dctas.size())) : 0;
        p.trace_mode = t;
    }
#endif
    p.num_pages = num_pages;
    p.sl2 = static_cast<float>(1.4426950408889634 / plan->shape.scale);
    return p;
}

// head dims below 128 run through the d = 128 kernels zero-padded: TMA boxes past the
// tensor's d are zero-filled (K, V, and the two-CTA kernel's Q), Q rows loaded by threads
// are zero past d, and only d columns of O are stored.  16-byte TMA strides need d % 8 == 0.
bool head_dim_ok(int d) { return d >= 8 && d <= kHeadDim && d % 8 == 0; }

pod_status check_supported(const pod_plan* plan) {
    if (!head_dim_ok(plan->shape.head_dim)) {
        set_last_error("head_dim must be a multiple of 8 in [8, 128]");
        return POD_ERR_UNSUPPORTED;
    }
    const int G = plan->shape.num_q_heads / plan->shape.num_kv_heads;
    if (G != 1 && G != 2 && G != 4 && G != 8) {
        set_last_error("GQA group must be 1, 2, 4 or 8");
        return POD_ERR_UNSUPPORTED;
    }
    if (plan->batch.page_size != 16) {
        set_last_error("only page_size 16 is compiled");
        return POD_ERR_UNSUPPORTED;
    }
    return POD_OK;
}

// cudaFuncSetAttribute is per device context: set the large dynamic-smem limits once
// per (kernel instantiation, device), thread-safely, and report a failure.
template <int G, int kFmt>
pod_status set_kernel_attributes() {
    constexpr int kMaxDev = 64;
    static std::once_flag once[kMaxDev];
    static cudaError_t err[kMaxDev];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev < 0 || dev >= kMaxDev) {
        set_last_error("device ordinal out of range");
        return POD_ERR_CUDA;
    }
    std::call_once(once[dev], [&] {
        cudaError_t r = cudaFuncSetAttribute(pod_fused_kernel<G, kFmt>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kSmemBytes);
        // the merges run right after a max-shared-memory POD kernel: keep the SM's
        // L1 / shared split (no carve-out reconfiguration between the launches)
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(pod_sm_kernel<G, kFmt, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SmLay<0>::kSmem);
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(pod_sm_kernel<G, kFmt, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SmLay<1>::kSmem);
        err[dev] = r;
    });
    if (err[dev] != cudaSuccess) return cuda_fail(err[dev], "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
    return POD_OK;
}

template <int G, int kFmt>
pod_status launch_all(const pod_plan* plan, int mode, const RunParams& p, const Maps& maps, cudaStream_t s) {
    // mode 0 fused, 1 serial, 2 prefill only, 3 decode only
    pod_status st = set_kernel_attributes<G, kFmt>();
    if (st != POD_OK) return st;
    const int nsm = plan->dev.num_sms;
    const bool shadow = p.vs_pages > 0 && mode != 3;
    if (shadow) {
        const uint8_t* ws = reinterpret_cast<const uint8_t*>(p.ctr) - plan->ws.off_counters;
        const size_t n = static_cast<size_t>(p.vs_pages) * p.hkv * 16 * (p.hd / 8);
        v_shadow_kernel<<<static_cast<int>(std::min<size_t>((n + 255) / 256, 8 * nsm)), 256, 0, s>>>(
            static_cast<const uint4*>(p.v_pool), reinterpret_cast<uint4*>(const_cast<uint8_t*>(ws) + plan->ws.off_vshadow),
            p.page_indptr, p.page_indices, p.vs_pages, p.hkv, p.hd / 8, p.kv_layout);
    }
    const CUtensorMap& pf_v = shadow ? maps.vs : maps.v;  // the prefill role's V map argument
    bool pdl = shadow;  // only the launch right after v_shadow_kernel is its programmatic dependent
    auto launch = [&](const RunParams& q) {
        const int items = q.num_pctas + q.num_dctas;
        if (items <= 0) return;
        const bool dep = pdl;
        pdl = false;
        if (q.policy == POD_POLICY_WARPSPEC) {
            if (dep) {  // a programmatic dependent of v_shadow_kernel (prefill waits at its first V load)
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(nsm);
                cfg.blockDim = dim3(sm3::kThreads);
                cfg.dynamicSmemBytes = q.pf_db ? SmLay<1>::kSmem : SmLay<0>::kSmem;
                cfg.stream = s;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                if (q.pf_db)
                    cudaLaunchKernelEx(&cfg, pod_sm_kernel<G, kFmt, 1>, q, maps.k, pf_v, maps.dk, maps.dv);
                else
                    cudaLaunchKernelEx(&cfg, pod_sm_kernel<G, kFmt, 0>, q, maps.k, pf_v, maps.dk, maps.dv);
            } else {
                if (q.pf_db)
                    pod_sm_kernel<G, kFmt, 1><<<nsm, sm3::kThreads, SmLay<1>::kSmem, s>>>(q, maps.k, pf_v, maps.dk,
                                                                                         maps.dv);
                else
                    pod_sm_kernel<G, kFmt, 0><<<nsm, sm3::kThreads, SmLay<0>::kSmem, s>>>(q, maps.k, pf_v, maps.dk,
                                                                                         maps.dv);
            }
        } else {
            const int grid = std::min(items, 2 * nsm);  // persistent: 2 resident CTAs per SM
            if (dep) {  // a programmatic dependent of v_shadow_kernel (prefill waits at its first V load)
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(kThreads);
                cfg.dynamicSmemBytes = kSmemBytes;
                cfg.stream = s;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, pod_fused_kernel<G, kFmt>, q, maps.q, maps.k, pf_v, maps.dk, maps.dv);
            } else {
                pod_fused_kernel<G, kFmt><<<grid, kThreads, kSmemBytes, s>>>(q, maps.q, maps.k, pf_v, maps.dk, maps.dv);
            }
        }
    };
    if (mode == 0) {
        launch(p);
    } else {
        if (mode == 1 || mode == 2) {
            RunParams q = p;
            q.num_dctas = 0;
            launch(q);
        }
        if (mode == 1 || mode == 3) {
            RunParams q = p;
            q.num_pctas = 0;
            launch(q);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "pod kernel launch");
    // split merges
    // (an in-kernel merge -- each finished split releases its parent with red.release, a
    // drained engine merges complete parents -- measured slower than this one launch:
    // C1 fused 86 vs 63 us, TP8 rank 233 vs 131 us: the merges then run in the launch's
    // tail on the few warps of drained engines instead of the whole machine)
    const bool do_p = (mode != 3) && plan->merge_rows_prefill > 0;
    // (an in-kernel merge by the group finishing a parent's last split measured ~8 us
    // slower at C2 B=64 than this 5 us launch: per-item fences + barriers)
    const bool do_d = (mode != 2) && plan->merge_rows_decode > 0;
    const uint8_t* ws = reinterpret_cast<const uint8_t*>(p.ctr);
    const int32_t* tile_splits = reinterpret_cast<const int32_t*>(ws - plan->ws.off_counters + plan->ws.off_tile_splits);
    // the merges are ONE programmatic dependent launch: it overlaps the POD kernel's tail
    auto merge = [&](int tq, int prows, int drows) {
        const int rows = prows + drows;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((rows + 7) / 8);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, merge_kernel, p, tile_splits, tq, prows, drows);
    };
    if (do_p || do_d) {
        e = merge(static_cast<int>(plan->cfg.prefill_tile_q), do_p ? p.chunk * p.hq : 0,
                  do_d ? static_cast<int>(plan->decode_ctx.size()) * p.hq : 0);
        if (e != cudaSuccess) return cuda_fail(e, "pod merge launch");
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "pod merge launch");
    return POD_OK;
}

template <int kFmt>
pod_status dispatch_g(const pod_plan* plan, int mode, const RunParams& p, const Maps& maps, cudaStream_t s) {
    switch (p.group) {
        case 1: return launch_all<1, kFmt>(plan, mode, p, maps, s);
        case 2: return launch_all<2, kFmt>(plan, mode, p, maps, s);
        case 4: return launch_all<4, kFmt>(plan, mode, p, maps, s);
        case 8: return launch_all<8, kFmt>(plan, mode, p, maps, s);
    }
    return POD_ERR_UNSUPPORTED;
}

pod_status run_mode(const pod_plan* plan, int mode, const void* q_prefill, const void* q_decode,
                    const void* k_pool, const void* v_pool, int64_t num_pages, const int32_t* indptr,
                    const int32_t* indices, void* o_prefill, float* lse_prefill, void* o_decode,
                    float* lse_decode, void* workspace, void* stream) {
    if (!plan || !k_pool || !v_pool || !indptr || !indices || !workspace) return POD_ERR_INVALID_ARGUMENT;
    pod_status st = check_supported(plan);
    if (st != POD_OK) return st;
    const bool need_p = plan->batch.has_prefill && mode != 3;
    const bool need_d = !plan->decode_ctx.empty() && mode != 2;
    if (need_p && (!q_prefill || !o_prefill || !lse_prefill)) return POD_ERR_INVALID_ARGUMENT;
    if (need_d && (!q_decode || !o_decode || !lse_decode)) return POD_ERR_INVALID_ARGUMENT;
    Maps maps;
    static_assert(sizeof(Maps) == sizeof(plan->map_blob), "map cache size");
    {
        // Tensor-map cache (host launch cost): the plan is const for callers, the cache
        // is not part of its semantics; a mutex keeps concurrent runs of one plan safe.
        pod_plan* mp = const_cast<pod_plan*>(plan);
        std::lock_guard<std::mutex> lock(mp->map_mu);
        if (mp->map_key[0] == q_prefill && mp->map_key[1] == k_pool && mp->map_key[2] == v_pool &&
            mp->map_key[3] == workspace && mp->map_pages == num_pages) {
            std::memcpy(&maps, mp->map_blob, sizeof(Maps));
        } else {
            st = make_maps(plan, q_prefill, k_pool, v_pool, num_pages, workspace, &maps);
            if (st != POD_OK) return st;
            std::memcpy(mp->map_blob, &maps, sizeof(Maps));
            mp->map_key[0] = q_prefill;
            mp->map_key[1] = k_pool;
            mp->map_key[2] = v_pool;
            mp->map_key[3] = workspace;
            mp->map_pages = num_pages;
        }
    }
    RunParams p = make_params(plan, q_prefill, q_decode, k_pool, v_pool, num_pages, indptr, indices, o_prefill,
                              lse_prefill, o_decode, lse_decode, workspace);
    if (mode == 2) p.num_dctas = 0;
    if (mode == 3) p.num_pctas = 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (plan->batch.dtype == POD_DTYPE_FP16) return dispatch_g<0>(plan, mode, p, maps, s);
    return dispatch_g<1>(plan, mode, p, maps, s);
}

}  // namespace pod

using namespace pod;

extern "C" {

pod_status pod_device_query(int device, pod_device* out) {
    if (!out) return POD_ERR_INVALID_ARGUMENT;
    int sms = 0, smem = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    e = cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    // B200 calibration: 1 compute unit = one (row, key)
    // pair at d = 128 = 4*128 FLOP; 1 memory unit = one bf16 element; 1 time unit = 1 us.
    const double tf = 1665.7e12, hbm = 6538.9e9;
    out->num_sms = sms;
    out->compute_rate_per_sm = tf / (4.0 * kHeadDim) / 1e6 / sms;
    out->mem_bandwidth_total = hbm / 2.0 / 1e6;
    out->mem_bandwidth_per_sm = 1.2 * out->mem_bandwidth_total / sms;
    out->mem_interference = 0.25;
    out->max_ctas_per_sm = 4;
    out->shared_mem_per_sm = smem;
    return POD_OK;
}

pod_status pod_attn_workspace_init(const pod_plan* plan, void* workspace, void* stream) {
    if (!plan || !workspace) return POD_ERR_INVALID_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    cudaError_t e = cudaMemsetAsync(ws + plan->ws.off_counters, 0, sizeof(SchedCounters), s);
    if (e == cudaSuccess && !plan->pctas.empty())
        e = cudaMemcpyAsync(ws + plan->ws.off_pctas, plan->pctas.data(), plan->pctas.size() * sizeof(PrefillCta),
                            cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && !plan->dctas.empty())
        e = cudaMemcpyAsync(ws + plan->ws.off_dctas, plan->dctas.data(), plan->dctas.size() * sizeof(DecodeCta),
                            cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && !plan->dec_pos.empty())
        e = cudaMemcpyAsync(ws + plan->ws.off_dec_pos, plan->dec_pos.data(), plan->dec_pos.size() * sizeof(int32_t),
                            cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && !plan->dec_nsplit.empty())
        e = cudaMemcpyAsync(ws + plan->ws.off_dec_nsplit, plan->dec_nsplit.data(),
                            plan->dec_nsplit.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && !plan->tile_splits.empty())
        e = cudaMemcpyAsync(ws + plan->ws.off_tile_splits, plan->tile_splits.data(),
                            plan->tile_splits.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "pod_attn_workspace_init");
    return POD_OK;
}

pod_status pod_attn_run(const pod_plan* plan, const void* q_prefill, const void* q_decode, const void* k_pool,
                        const void* v_pool, int64_t num_pages, const int32_t* page_indptr,
                        const int32_t* page_indices, void* o_prefill, float* lse_prefill, void* o_decode,
                        float* lse_decode, void* workspace, void* stream) {
    return run_mode(plan, 0, q_prefill, q_decode, k_pool, v_pool, num_pages, page_indptr, page_indices, o_prefill,
                    lse_prefill, o_decode, lse_decode, workspace, stream);
}

pod_status pod_attn_run_serial(const pod_plan* plan, const void* q_prefill, const void* q_decode,
                               const void* k_pool, const void* v_pool, int64_t num_pages,
                               const int32_t* page_indptr, const int32_t* page_indices, void* o_prefill,
                               float* lse_prefill, void* o_decode, float* lse_decode, void* workspace,
                               void* stream) {
    return run_mode(plan, 1, q_prefill, q_decode, k_pool, v_pool, num_pages, page_indptr, page_indices, o_prefill,
                    lse_prefill, o_decode, lse_decode, workspace, stream);
}

pod_status pod_attn_run_part(const pod_plan* plan, int which, const void* q_prefill, const void* q_decode,
                             const void* k_pool, const void* v_pool, int64_t num_pages,
                             const int32_t* page_indptr, const int32_t* page_indices, void* o_prefill,
                             float* lse_prefill, void* o_decode, float* lse_decode, void* workspace,
                             void* stream) {
    if (which != 0 && which != 1) return POD_ERR_INVALID_ARGUMENT;
    return run_mode(plan, which == 0 ? 2 : 3, q_prefill, q_decode, k_pool, v_pool, num_pages, page_indptr,
                    page_indices, o_prefill, lse_prefill, o_decode, lse_decode, workspace, stream);
}

pod_status pod_attn_l2_flush(void* buf, int64_t bytes, void* stream) {
    if (!buf || bytes < 16) return POD_ERR_INVALID_ARGUMENT;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(l2_flush_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        cudaSharedmemCarveoutMaxShared);
    });
    if (attr_err != cudaSuccess) return cuda_fail(attr_err, "l2_flush attributes");
    l2_flush_kernel<<<4 * 148, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint4*>(buf),
                                                                           static_cast<size_t>(bytes) / 16);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "l2_flush");
    return POD_OK;
}

pod_status pod_attn_gather_probe(const pod_plan* plan, const void* kv_pool, int64_t num_pages,
                                 const int32_t* page_indptr, const int32_t* page_indices, int32_t req,
                                 int64_t ctx, uint16_t* out, void* stream) {
    (void)num_pages;
    if (!plan || !kv_pool || !page_indptr || !page_indices || !out || ctx < 1) return POD_ERR_INVALID_ARGUMENT;
    if (!head_dim_ok(plan->shape.head_dim) || plan->batch.page_size != 16) return POD_ERR_UNSUPPORTED;
    gather_probe_kernel<<<148, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint16_t*>(kv_pool), plan->batch.kv_layout, plan->shape.num_kv_heads, page_indptr,
        page_indices, req, static_cast<int>(ctx), plan->shape.head_dim, out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "gather_probe");
    return POD_OK;
}

pod_status pod_attn_append_kv(const pod_plan* plan, const void* k_new_prefill, const void* v_new_prefill,
                              const void* k_new_decode, const void* v_new_decode, void* k_pool, void* v_pool,
                              int64_t num_pages, const int32_t* page_indptr, const int32_t* page_indices,
                              void* workspace, void* stream) {
    (void)num_pages;
    if (!plan || !k_pool || !v_pool || !page_indptr || !page_indices || !workspace) return POD_ERR_INVALID_ARGUMENT;
    if (!head_dim_ok(plan->shape.head_dim) || plan->batch.page_size != 16) {
        set_last_error("append_kv: head_dim must be a multiple of 8 in [8, 128], page_size 16");
        return POD_ERR_UNSUPPORTED;
    }
    const int chunk = plan->batch.has_prefill ? static_cast<int>(plan->batch.prefill.chunk_size) : 0;
    const int ndec = static_cast<int>(plan->decode_ctx.size());
    if ((chunk > 0 && (!k_new_prefill || !v_new_prefill)) || (ndec > 0 && (!k_new_decode || !v_new_decode)))
        return POD_ERR_INVALID_ARGUMENT;
    if (chunk + ndec == 0) return POD_OK;
    const int hkv = plan->shape.num_kv_heads;
    const int rows = (chunk + ndec) * hkv;
    const int32_t* dec_pos =
        reinterpret_cast<const int32_t*>(static_cast<const uint8_t*>(workspace) + plan->ws.off_dec_pos);
    append_kv_kernel<<<(rows + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(k_new_prefill), static_cast<const uint4*>(v_new_prefill),
        static_cast<const uint4*>(k_new_decode), static_cast<const uint4*>(v_new_decode), static_cast<uint4*>(k_pool),
        static_cast<uint4*>(v_pool), page_indptr, page_indices, dec_pos, chunk,
        chunk > 0 ? static_cast<int>(plan->batch.prefill.position_offset) : 0, ndec, hkv, plan->batch.kv_layout,
        plan->shape.head_dim / 8);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "append_kv launch");
    return POD_OK;
}

pod_status pod_oproj_run(const void* o, const void* w, int64_t tokens, int64_t k, int64_t n, void* const* y_parts,
                         int32_t world, int64_t rows_per_rank, int32_t accumulate, void* stream) {
    if (!o || !w || !y_parts || tokens < 1 || k < 1 || n < 1 || world < 1 || world > oproj::kMaxWorld)
        return POD_ERR_INVALID_ARGUMENT;
    if (k % oproj::kBK || n % 128) {
        set_last_error("pod_oproj_run: K must be a multiple of 64 and N of 128");
        return POD_ERR_UNSUPPORTED;
    }
    if (!accumulate && world != 1) {
        set_last_error("pod_oproj_run: world > 1 needs accumulate = 1 (the reduce-scatter epilogue)");
        return POD_ERR_INVALID_ARGUMENT;
    }
    if (accumulate && (rows_per_rank < 1 || rows_per_rank * world < tokens)) {
        set_last_error("pod_oproj_run: rows_per_rank * world must cover the token rows");
        return POD_ERR_INVALID_ARGUMENT;
    }
    OprojParams p{};
    for (int r = 0; r < world; ++r) {
        if (!y_parts[r]) return POD_ERR_INVALID_ARGUMENT;
        p.y[r] = static_cast<float*>(y_parts[r]);
    }
    p.world = world;
    p.accumulate = accumulate;
    p.rows_per_rank = accumulate ? rows_per_rank : tokens;
    p.tokens = tokens;
    p.k = k;
    p.n = n;
    EncodeTiledFn enc = encode_fn();
    if (!enc) {
        set_last_error("cuTensorMapEncodeTiled unavailable");
        return POD_ERR_CUDA;
    }
    CUtensorMap ta, tb;
    const cuuint32_t estr[2] = {1, 1};
    {  // A = O [tokens][K]: box 64 K x 128 rows, SW128 (rows past `tokens` read as zero)
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(tokens)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(k) * 2};
        const cuuint32_t box[2] = {64, oproj::kBM};
        if (enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(o), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            set_last_error("cuTensorMapEncodeTiled(o_proj A) failed");
            return POD_ERR_CUDA;
        }
    }
    {  // B = W [K][N]: box 64 N x 64 K rows, SW128 (MN-major operand)
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(k)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(n) * 2};
        const cuuint32_t box[2] = {64, oproj::kBK};
        if (enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            set_last_error("cuTensorMapEncodeTiled(o_proj B) failed");
            return POD_ERR_CUDA;
        }
    }
    {  // per device: the large dynamic shared memory limit
        constexpr int kMaxDev = 64;
        static std::once_flag once[kMaxDev];
        static cudaError_t err[kMaxDev];
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess || dev < 0 || dev >= kMaxDev) return cuda_fail(e, "cudaGetDevice");
        std::call_once(once[dev], [&] {
            err[dev] = cudaFuncSetAttribute(oproj_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            oproj::Cfg<128>::kSmem);
            if (err[dev] == cudaSuccess)
                err[dev] = cudaFuncSetAttribute(oproj_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                oproj::Cfg<256>::kSmem);
        });
        if (err[dev] != cudaSuccess) return cuda_fail(err[dev], "o_proj attributes");
    }
    // 128 x 256 tiles when N allows (half the A re-reads per output), else 128 x 128
    const unsigned gy = static_cast<unsigned>((tokens + oproj::kBM - 1) / oproj::kBM);
    if (n % 256 == 0)
        oproj_kernel<256><<<dim3(static_cast<unsigned>(n / 256), gy), oproj::kThreads, oproj::Cfg<256>::kSmem,
                             static_cast<cudaStream_t>(stream)>>>(p, ta, tb);
    else
        oproj_kernel<128><<<dim3(static_cast<unsigned>(n / 128), gy), oproj::kThreads, oproj::Cfg<128>::kSmem,
                             static_cast<cudaStream_t>(stream)>>>(p, ta, tb);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "o_proj launch");
    return POD_OK;
}

const char* pod_last_error(void) { return g_last_error.c_str(); }

pod_status pod_attn_occupancy(const pod_plan* plan, int32_t* fused, int32_t* prefill, int32_t* decode) {
    if (!plan || !fused || !prefill || !decode) return POD_ERR_INVALID_ARGUMENT;
    const int G = plan->shape.num_q_heads / plan->shape.num_kv_heads;
    if (G != 4) return POD_ERR_UNSUPPORTED;
    int a = 0;
    pod_status st = set_kernel_attributes<4, 1>();
    if (st != POD_OK) return st;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, pod_fused_kernel<4, 1>, kThreads, kSmemBytes);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy");
    // one persistent kernel serves all three launch kinds
    *fused = a;
    *prefill = a;
    *decode = a;
    return POD_OK;
}

}  // extern "C"
