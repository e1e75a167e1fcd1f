// pod_sm.cuh -- the warp-specialised POD kernel (POD_POLICY_WARPSPEC): one CTA per
// SM that owns the whole SM (227 KB smem, 512 TMEM columns, 16 warps) and runs a
// prefill engine and a decode engine side by side, each binding work items from
// its own pool at runtime.  Included by pod_attn.cu (uses its helpers).
//
//   warps 0-3   softmax of prefill M-block A   (TMEM lane quadrant = warp % 4)
//   warps 4-7   softmax of prefill M-block B
//   warp  8     prefill TMA producer (K/V tiles through the page table)
//   warp  9     prefill MMA issuer: S = Q K^T and O += P V, both TS-MMAs (Q, P in TMEM)
//   warps 10-15 decode group: 6 warps stream one (request, KV head, split) item,
//               each through its own TMA ring of head-pages, LSE-merged in smem
//
// Why: a decode CTA co-resident with a prefill CTA is bounded by the shared
// memory it can keep in flight (~96 KB ring -> ~34 GB/s per SM next to a prefill
// CTA); with one CTA per SM the prefill keeps Q, S, P and O in TMEM and
// needs only 64 KB of K/V stages, and the decode group gets 144 KB of rings.  The
// prefill engine runs two 128-row M-blocks over the same K/V tiles (half the K/V
// traffic per row), ping-ponging the tensor core between the blocks' softmax.
// Two tile widths share the layout: 32-key tiles with double-buffered S
// (prefill_item_sm, decode-dominant plans) and 64-key tiles with one S buffer per
// block (prefill_item_sm64, prefill-dominant plans; RunParams::pf_tn64).  The most
// prefill-dominant plans (RunParams::pf_db) run a second kernel instance (kE = 1): 64-key
// tiles with two S buffers per block, Q in shared memory (prefill_item_db, SmLay<1>).
// Plans with RunParams::vs_pages read V from the per-launch fp16 shadow (no conversion).
//
// Role binding is still SM-aware and dynamic: every SM hosts both roles for as
// long as both pools have work (the placement the POD scheduler aims for,
// PAPER.md:379), an engine whose pool is exhausted retires, and the claims are
// atomic tickets on the same counters (gpu_sim.hpp:114-131).
#pragma once

#ifndef POD_SM_SOFTMAX_HIGH
#define POD_SM_SOFTMAX_HIGH 0
#endif
#ifndef POD_SM_MERGED_EMPTY
#define POD_SM_MERGED_EMPTY 1
#endif
#ifndef POD_SM_MMA_SLEEP
#define POD_SM_MMA_SLEEP 0
#endif
#ifndef POD_SM_SOFTMAX_SLEEP
#define POD_SM_SOFTMAX_SLEEP 0
#endif
// wait helper: spin (try_wait) or back off with __nanosleep(kNs)
template <int kNs>
__device__ __forceinline__ void sm_wait(uint32_t bar, uint32_t parity) {
    if constexpr (kNs > 0)
        ptx::mbar_wait_relaxed<kNs>(bar, parity);
    else
        ptx::mbar_wait(bar, parity);
}
// Warp-uniform copy of the engines' loop state: every lane holds the same values, but the
// compiler only keeps them (and the descriptors / stage offsets derived from them) on the
// uniform datapath -- no R2UR per MMA issue -- once they come out of a shuffle broadcast.
#ifndef POD_SM_UNIFORM_STATE
#define POD_SM_UNIFORM_STATE 1
#endif
__device__ __forceinline__ int wuni(int x) { return POD_SM_UNIFORM_STATE ? __shfl_sync(0xffffffffu, x, 0) : x; }
namespace sm3 {
#ifndef POD_SM_DUAL_MMA
#define POD_SM_DUAL_MMA 0
#endif
#ifndef POD_SM_DEC_WARPS
#define POD_SM_DEC_WARPS (6 - POD_SM_DUAL_MMA)
#endif
#ifndef POD_SM_DEC_STAGES
#define POD_SM_DEC_STAGES 3
#endif
constexpr int kDW = POD_SM_DEC_WARPS;   // decode warps
static_assert(POD_SM_DUAL_MMA || kDW == kSmDecodeWarps, "planner's decode-warp count");
constexpr int kDS = POD_SM_DEC_STAGES;  // ring stages per decode warp
// With POD_SM_DUAL_MMA, warp 9 issues block A's MMAs and warp 10 block B's (each
// block's chain in its own issuing thread); by default warp 9 issues both and the
// sixth decode warp takes warp 10's place (measured faster fused).
constexpr bool kDualMma = POD_SM_DUAL_MMA != 0;
constexpr int kProdWarp = 8, kMmaWarp = 9, kMmaWarpB = kDualMma ? 10 : 9, kDecWarp0 = kDualMma ? 11 : 10;
constexpr int kPrefillThreads = kDecWarp0 * 32;
constexpr int kThreads = (kDecWarp0 + kDW) * 32;
// Prefill K/V tiles of 32 keys (2 pages): S is double-buffered per block inside
// the block's 64 TMEM columns, so QK_X(t+1) runs while the softmax of tile t does.
constexpr int kTN = 32;
#ifndef POD_SM_PROD_SLEEP
#define POD_SM_PROD_SLEEP 128  // producer back-off (ns) while waiting for a free stage
#endif
// timing experiments only (tools/micro/build_variant.sh); all 0 in the product
#ifndef POD_SM_EXP_NOVWAIT
#define POD_SM_EXP_NOVWAIT 0
#endif
#ifndef POD_SM_EXP_ST0
#define POD_SM_EXP_ST0 0
#endif
#ifndef POD_SM_EXP_SPLITCONST
#define POD_SM_EXP_SPLITCONST 0
#endif
#ifndef POD_SM_UNIFORM_WARP
#define POD_SM_UNIFORM_WARP 1
#endif
#ifndef POD_SM_LAZY_PV
#define POD_SM_LAZY_PV 1
#endif
#ifndef POD_SM_STAGES
#define POD_SM_STAGES 4
#endif
constexpr int kNS = POD_SM_STAGES;                             // K and V ring stages
constexpr uint32_t kStage = kTN * kHeadDim * 2;                // 8 KB: [d-half][32 keys][64 d], SW128
constexpr uint32_t kOffKs = 0;
constexpr uint32_t kOffVs = kNS * kStage;
static_assert(kNS * kStage >= 8 * 4096, "the epilogue's 8 warp tiles (store_o_rows) fit the K ring");
#ifndef POD_SM64_BATCHED_PV
#define POD_SM64_BATCHED_PV 1  // 64-key engine: the 8 PV MMAs of a tile in one elected asm block
#endif
#ifndef POD_SM64_KSTAGES
#define POD_SM64_KSTAGES 2  // K ring stages of the 64-key pair engine (V: 2)
#endif
// the prefill rings: 32-key engine K + V (64 KB), or the 64-key engine's K + V stages
constexpr uint32_t kPfRingBytes = (POD_SM64_KSTAGES + 2) * 16384u > 2 * kNS * kStage ? (POD_SM64_KSTAGES + 2) * 16384u
                                                                                      : 2 * kNS * kStage;
constexpr uint32_t kOffDec = kPfRingBytes;                     // decode rings (64 KB in)
constexpr uint32_t kOffBars = kOffDec + kDW * kDS * kDecStageBytes;
// prefill mbarriers: 0 qA, 1 qB, 2-5 k_full, 6-9 k_empty, 10-13 v_full, 14-17 v_empty,
// 18-19 sA[2], 20-21 sB[2], 22-23 pA[2], 24-25 pB[2], 26-27 pvA[2], 28-29 pvB[2]
// (single MMA issuer: bars 6-9 are per-stage kv_empty, committed once both K and V of a
//  tile are consumed; bars 14-17 unused.  POD_SM_DUAL_MMA: k_empty / v_empty take two
//  arrivals, one commit per block's issuing thread)
// (pv per S buffer: a waiter is never more than one completion behind on a
// barrier, so parity waits stay unambiguous even when the softmax skips them)
constexpr int kBarKF = 2, kBarKE = kBarKF + kNS, kBarVF = kBarKE + kNS, kBarVE = kBarVF + kNS;
constexpr int kBarS = kBarVE + kNS, kBarP = kBarS + 4, kBarPV = kBarP + 4;
constexpr int kNumBars = kBarPV + 4;
constexpr uint32_t kOffDecBars = kOffBars + kNumBars * 8;
constexpr uint32_t kOffMisc = kOffDecBars + kDW * kDS * 8;     // tmem slot, claim slots
constexpr uint32_t kSmem = kOffMisc + 64;
static_assert(kSmem <= 232448, "one CTA per SM: <= 227 KB dynamic smem");
static_assert(kOffDec % 1024 == 0 && kDecStageBytes % 1024 == 0, "SW128 stages are 1024-aligned");
// TMEM columns (512): Q_A, Q_B (bf16 pairs), S_A[2], S_B[2] (fp32 / P over S), O_A, O_B
constexpr uint32_t kQA = 0, kQB = 64, kSA = 128, kSB = 192, kOA = 256, kOB = 384;

struct PfState {
    int g = 0;            // K/V tiles issued (stage = g % kNS, phase = (g / kNS) & 1)
    int n[2] = {0, 0};    // tiles per block (S buffer = n & 1; s/p/pv phases (n >> 1) & 1)
    int nq[2] = {0, 0};   // Q loads per block (q_full phases)
    int npv[2][2] = {{0, 0}, {0, 0}};  // pv commits per (block, S buffer) (POD_SM_LAZY_PV)
};
__device__ __forceinline__ PfState uniform(const PfState& a) {
    PfState u;
    u.g = wuni(a.g);
    u.n[0] = wuni(a.n[0]);
    u.n[1] = wuni(a.n[1]);
    u.nq[0] = wuni(a.nq[0]);
    u.nq[1] = wuni(a.nq[1]);
    u.npv[0][0] = wuni(a.npv[0][0]);
    u.npv[0][1] = wuni(a.npv[0][1]);
    u.npv[1][0] = wuni(a.npv[1][0]);
    u.npv[1][1] = wuni(a.npv[1][1]);
    return u;
}

// S = Q K^T for one 32-key tile: A = Q (TMEM, 128 rows x 128 d), B = K (smem,
// K-major SW128 [d-half][32 keys][64 d]), N = 32.
template <int kFmt>
__device__ __forceinline__ void issue_qk32(uint32_t tmem_s, uint32_t tmem_q, uint32_t sK) {
    if (POD_SM_NOMMA) return;  // timing experiment only
    constexpr uint32_t idesc = ptx::idesc_f16(kFmt, kMBlock, kTN, 0);
    ptx::umma_ts_k128_elect<kTN * 128>(tmem_s, tmem_q, ptx::sw128_desc(sK, 16, 1024), idesc);
}
// O (+)= P V for one 32-key tile: A = P (TMEM; hi in columns [0,16), lo in [16,32)),
// B = V (smem, MN-major SW128 [d-half][32 keys][64 d]), N = 128.
template <int kFmt>  // kFmt: format of P and V (fp16 under POD_PRECISION_F16PV)
__device__ __forceinline__ void issue_pv32(uint32_t tmem_o, uint32_t tmem_p, uint32_t sV, bool accumulate,
                                           bool split) {
    if (POD_SM_NOMMA) return;  // timing experiment only
    constexpr uint32_t idesc = ptx::idesc_f16(kFmt, kMBlock, kHeadDim, 1);
    static_assert(kTN == 32, "umma_pv32_elect: two K-steps, lo part 16 columns after hi");
    const uint64_t b = ptx::sw128_desc(sV, 2048, 1024);  // page-major V (prefill_load_v_pages)
    if (split)
        ptx::umma_pv32_elect<true>(tmem_o, tmem_p, b, idesc, accumulate ? 1u : 0u);
    else
        ptx::umma_pv32_elect<false>(tmem_o, tmem_p, b, idesc, accumulate ? 1u : 0u);
}
// The 4 TMA boxes (2 pages x 2 d-halves, 128B swizzle) of one 32-key tile.
__device__ __forceinline__ void load_tile32(const RunParams& p, const CUtensorMap* tm, uint32_t dst, uint32_t bar,
                                            int kt, int kv_head, const PageIds& ids) {
    const int ph0 = ids.get(min(kt / 16, ids.n - 1)), ph1 = ids.get(min(kt / 16 + 1, ids.n - 1));
#pragma unroll
    for (int pg = 0; pg < 2; ++pg) {
#pragma unroll
        for (int dh = 0; dh < 2; ++dh) {
            const uint32_t d = dst + dh * (kTN * 128) + pg * 2048;
            const int phys = pg ? ph1 : ph0;
            if (p.kv_layout == POD_KV_HND)
                ptx::tma_load_4d_elect(d, tm, bar, dh * 64, 0, kv_head, phys);
            else
                ptx::tma_load_4d_elect(d, tm, bar, dh * 64, kv_head, 0, phys);
        }
    }
}
}  // namespace sm3

// Epilogue of one softmax warp (its 32 rows of a block): O (TMEM, 128 fp32 columns) x inv
// to the rows' outputs.  A lane owns a row, so direct stores scatter every instruction over
// 32 rows (16 B pieces 512 B - 16 KB apart); measured at C1 the item epilogues all run at
// once and took ~11k cycles.  Instead each 32-column chunk goes through a warp-private 4 KB
// smem tile (XOR-swizzled 16 B chunks: conflict-free both ways) and leaves as whole 128 B row
// segments, 4 rows per store instruction.  `tile` is in the K ring, idle once the item's
// last PV of this block completed (every QK of the item was issued before it).
__device__ __forceinline__ void store_o_rows(uint32_t o_addr, float inv, const ORow& orow, bool row_ok,
                                             uint32_t tile, int lane, int hd) {
    // destination of the 8 rows this lane writes: rows 4i + lane / 8
    char* dst[8];
    bool ok[8];
    const unsigned long long mine = reinterpret_cast<unsigned long long>(orow.ptr);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = 4 * i + (lane >> 3);
        dst[i] = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, mine, r));
        ok[i] = __shfl_sync(0xffffffffu, row_ok ? 1 : 0, r) != 0;
    }
    const int c4 = lane & 7;  // the 16 B column chunk this lane writes
#pragma unroll 1
    for (int ch = 0; ch < kHeadDim / 32; ++ch) {
        float o[32];
        ptx::tmem_ld32(o_addr + ch * 32, o);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint32_t a = tile + lane * 128u + ((static_cast<uint32_t>(c) ^ (lane & 7)) << 4);
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(o[4 * c] * inv),
                         "f"(o[4 * c + 1] * inv), "f"(o[4 * c + 2] * inv), "f"(o[4 * c + 3] * inv)
                         : "memory");
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int r = 4 * i + (lane >> 3);
            const uint32_t a = tile + r * 128u + ((static_cast<uint32_t>(c4) ^ (r & 7)) << 4);
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
            if (ok[i] && ch * 32 + 4 * c4 < hd) store4(ORow{dst[i], orow.fmt}, ch * 32 + 4 * c4, v);
        }
        __syncwarp();
    }
    ptx::fence_proxy_async_smem();  // the next item's TMA loads (async proxy) reuse the tile's bytes
}

// One prefill item of the warp-specialised engine: up to two 128-row M-blocks of
// one (q tile, KV head, KV split) CtaTask over the same 32-key K/V tiles.
template <int kFmt>
__device__ void prefill_item_sm(const RunParams& p, const CUtensorMap* tmk, const CUtensorMap* tmv /* 5-D page map */, int item,
                                uint32_t sbase, uint32_t tmem, sm3::PfState& ps, int warp, int lane) {
    using namespace sm3;
    const PrefillCta job = p.pctas[item];
    const int G = p.group;
    const int rpb = kMBlock / G;
    const int nblocks = (job.rows + rpb - 1) / rpb;  // 1 or 2
    const bool hasB = nblocks > 1;
    const BlockRange rA = prefill_block(p, job, 0);
    const BlockRange rB = hasB ? prefill_block(p, job, 1) : rA;
    // 32-key tiles from the (page-aligned) first key up to the last key either block sees
    const int kv_hi = min(job.kv_end, p.offset + (hasB ? rB.r0 + rB.nrows : rA.r0 + rA.nrows));
    const int kt0 = rA.kt0;
    const int nt = kv_hi > job.kv_begin ? (kv_hi - kt0 + kTN - 1) / kTN : 0;
    const PfState s0 = uniform(ps);
    if (nt > 0) {
        ps.g += nt;
        ps.n[0] += nt;
        ps.nq[0] += 1;
        if (hasB) {
            ps.n[1] += nt;
            ps.nq[1] += 1;
        }
        // pv commits (see pv_commit below): tiles max(0, nt-2) .. nt-1, one per S buffer
        for (int t = max(0, nt - 2); t < nt; ++t) {
            ps.npv[0][(s0.n[0] + t) & 1] += 1;
            if (hasB) ps.npv[1][(s0.n[1] + t) & 1] += 1;
        }
    }
    // POD_SM_LAZY_PV: PV_X(t) gets its own commit only for the last two tiles.  Earlier,
    // "PV_X(t-1) done" is implied by S_X(t+1)'s commit (issued after PV_X(t-1) by the same
    // thread, in-order pipe), which the softmax waits for anyway.
    auto pv_commit = [&](int t) { return !POD_SM_LAZY_PV || t + 2 >= nt; };
    const int pbeg = p.page_indptr[0];
    const int npages = p.page_indptr[1] - pbeg;
    const uint32_t bar0 = sbase + kOffBars;
    auto bar = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
    const uint32_t sK = sbase + kOffKs, sV = sbase + kOffVs;
    const int first = s0.n[0] == 0 ? 0 : 1;  // trace only the CTA's first item

    if (warp == kProdWarp) {
        // ------------------------------------------------ TMA producer --
        PageIds ids;
        ids.init(p.page_indices + pbeg, npages, kt0 / 16);
        for (int t = 0; t <= nt && nt > 0; ++t) {
            if (t < nt) {  // K of tile t
                const int gg = s0.g + t, st = gg % kNS;
                if (gg >= kNS) ptx::mbar_wait_relaxed<POD_SM_PROD_SLEEP>(bar(kBarKE + st), ((gg / kNS) - 1) & 1);
                if (POD_SM_NOLOAD && gg >= kNS) {  // timing experiment: stale K, no TMA
                    if (lane == 0) ptx::mbar_arrive(bar(kBarKF + st));
                } else {
                    ptx::mbar_arrive_expect_tx_elect(bar(kBarKF + st), kStage);
                    load_tile32(p, tmk, sK + st * kStage, bar(kBarKF + st), kt0 + t * kTN, job.kv_head, ids);
                }
            }
            if (t > 0) {  // V of tile t-1 (single issuer: its stage was freed with K's)
                const int gg = s0.g + t - 1, st = gg % kNS;
                if (!POD_SM_MERGED_EMPTY && gg >= kNS)
                    ptx::mbar_wait_relaxed<POD_SM_PROD_SLEEP>(bar(kBarVE + st), ((gg / kNS) - 1) & 1);
                if (POD_SM_NOLOAD && gg >= kNS) {
                    if (lane == 0) ptx::mbar_arrive(bar(kBarVF + st));
                } else {
                    if (p.vs_pages && t == 1) ptx::griddep_wait();  // the fp16 V shadow (see prefill_item)
                    ptx::mbar_arrive_expect_tx_elect(bar(kBarVF + st), kStage);
                    prefill_load_v_pages<2>(tmv, sV + st * kStage, bar(kBarVF + st), kt0 + (t - 1) * kTN, job.kv_head,
                                            ids, p.vs_pages);
                }
            }
        }
    } else if (!kDualMma && warp == kMmaWarp) {
        // the P-split flag is hoisted out of the loop (a runtime branch per PV cost ~7 %)
        // kPv: 0 = bf16 hi + lo (two PV MMAs), 1 = one P in the data format, 2 = fp16 P x
        // fp16 V (POD_PRECISION_F16PV: block A's softmax warps convert V(t) before P_A(t))
        auto mma_issuer = [&](auto pv_c) {
            constexpr int kPv = decltype(pv_c)::value;
            constexpr bool kSplit = kPv == 0;
            constexpr int kPvFmt = kPv == 2 ? 0 : kFmt;
            // -------------------------------------------------- MMA issuer --
            // Per block, QK_X(t+2) reuses the S buffer of tile t after PV_X(t) (in-order
            // pipe), so the softmax of tile t+1 overlaps PV_X(t) and QK_X(t+2); the two
            // blocks interleave on the tensor core.
            if (nt > 0) {
                sm_wait<POD_SM_MMA_SLEEP>(bar(0), s0.nq[0] & 1);
                if (hasB) sm_wait<POD_SM_MMA_SLEEP>(bar(1), s0.nq[1] & 1);
                for (int j = 0; j < 2 && j < nt; ++j) {
                    const int gg = s0.g + j, st = gg % kNS;
                    sm_wait<POD_SM_MMA_SLEEP>(bar(kBarKF + st), (gg / kNS) & 1);
                    ptx::tc_fence_after();
                    const int bA = (s0.n[0] + j) & 1, bB = (s0.n[1] + j) & 1;
                    issue_qk32<kFmt>(tmem + kSA + 32 * bA, tmem + kQA, sK + st * kStage);
                    ptx::umma_commit_elect(bar(kBarS + bA));
                    if (hasB) {
                        issue_qk32<kFmt>(tmem + kSB + 32 * bB, tmem + kQB, sK + st * kStage);
                        ptx::umma_commit_elect(bar(kBarS + 2 + bB));
                    }
                    if (!POD_SM_MERGED_EMPTY) ptx::umma_commit_elect(bar(kBarKE + st));
                }
                for (int t = 0; t < nt; ++t) {
                    const int gg = s0.g + t, st = gg % kNS;
                    const int g2 = gg + 2, st2 = g2 % kNS;
                    const bool more = t + 2 < nt;
                    const int nA = s0.n[0] + t, bA = nA & 1;
                    sm_wait<POD_SM_MMA_SLEEP>(bar(kBarP + bA), (nA >> 1) & 1);
                    trace_stamp(p, first, t, 4);
                    if (!POD_SM_EXP_NOVWAIT) sm_wait<POD_SM_MMA_SLEEP>(bar(kBarVF + st), (gg / kNS) & 1);
                    trace_stamp(p, first, t < 128 ? 384 + t : 9999, 4);
                    ptx::tc_fence_after();
                    issue_pv32<kPvFmt>(tmem + kOA, tmem + kSA + 32 * bA, sV + (POD_SM_EXP_ST0 ? 0 : st) * kStage,
                                       t > 0, kSplit);
                    trace_stamp(p, first, t < 128 ? 384 + t : 9999, 5);
                    if (pv_commit(t)) ptx::umma_commit_elect(bar(kBarPV + bA));
                    trace_stamp(p, first, t, 5);
                    if (more) {
                        sm_wait<POD_SM_MMA_SLEEP>(bar(kBarKF + st2), (g2 / kNS) & 1);
                        trace_stamp(p, first, t < 128 ? 384 + t : 9999, 6);
                        ptx::tc_fence_after();
                        issue_qk32<kFmt>(tmem + kSA + 32 * bA, tmem + kQA, sK + (POD_SM_EXP_ST0 ? 0 : st2) * kStage);
                        ptx::umma_commit_elect(bar(kBarS + bA));
                    }
                    trace_stamp(p, first, t, 6);
                    if (hasB) {
                        const int nB = s0.n[1] + t, bB = nB & 1;
                        sm_wait<POD_SM_MMA_SLEEP>(bar(kBarP + 2 + bB), (nB >> 1) & 1);
                        trace_stamp(p, first, t < 128 ? 384 + t : 9999, 7);
                        ptx::tc_fence_after();
                        issue_pv32<kPvFmt>(tmem + kOB, tmem + kSB + 32 * bB, sV + (POD_SM_EXP_ST0 ? 0 : st) * kStage,
                                           t > 0, kSplit);
                        if (pv_commit(t)) ptx::umma_commit_elect(bar(kBarPV + 2 + bB));
                        if (more) {
                            issue_qk32<kFmt>(tmem + kSB + 32 * bB, tmem + kQB, sK + (POD_SM_EXP_ST0 ? 0 : st2) * kStage);
                            ptx::umma_commit_elect(bar(kBarS + 2 + bB));
                        }
                    }
                    if (POD_SM_MERGED_EMPTY) {
                        // K and V of tile t are both consumed (QK(t) ran before PV(t)): one
                        // commit frees the stage for the producer
                        ptx::umma_commit_elect(bar(kBarKE + st));
                    } else {
                        ptx::umma_commit_elect(bar(kBarVE + st));
                        if (more) ptx::umma_commit_elect(bar(kBarKE + st2));
                    }
                }
            }
        };
        if (kFmt == 1 && p.p_f16)
            mma_issuer(std::integral_constant<int, 2>{});
        else if (POD_SM_EXP_SPLITCONST || p.p_split != 0)
            mma_issuer(std::integral_constant<int, 0>{});
        else
            mma_issuer(std::integral_constant<int, 1>{});
    } else if (kDualMma && (warp == kMmaWarp || warp == kMmaWarpB)) {
        // ------------------------------------------ MMA issuers (per block) --
        // Block X: QK_X(t+2) reuses the S buffer of tile t after PV_X(t) (in-order
        // per issuing thread), so the softmax of tile t+1 overlaps PV_X(t) and
        // QK_X(t+2).  A commit only tracks its own thread's MMAs, so the K/V empty
        // barriers count two arrivals: one per block thread (block A's thread
        // arrives twice when the item has no block B).
        const int X = warp == kMmaWarpB ? 1 : 0;
        const int rel = hasB ? 1 : 2;
        auto release = [&](uint32_t b) {
            ptx::umma_commit_elect(b);
            if (rel == 2) ptx::umma_commit_elect(b);
        };
        if (nt > 0 && (X == 0 || hasB)) {
            const uint32_t tS = tmem + (X ? kSB : kSA), tQ = tmem + (X ? kQB : kQA), tO = tmem + (X ? kOB : kOA);
            ptx::mbar_wait(bar(X), s0.nq[X] & 1);
            for (int j = 0; j < 2 && j < nt; ++j) {
                const int gg = s0.g + j, st = gg % kNS;
                ptx::mbar_wait(bar(kBarKF + st), (gg / kNS) & 1);
                ptx::tc_fence_after();
                const int bx = (s0.n[X] + j) & 1;
                issue_qk32<kFmt>(tS + 32 * bx, tQ, sK + st * kStage);
                ptx::umma_commit_elect(bar(kBarS + 2 * X + bx));
                if (!POD_SM_MERGED_EMPTY) release(bar(kBarKE + st));
            }
            for (int t = 0; t < nt; ++t) {
                const int gg = s0.g + t, st = gg % kNS;
                const int g2 = gg + 2, st2 = g2 % kNS;
                const bool more = t + 2 < nt;
                const int n = s0.n[X] + t, bx = n & 1;
                ptx::mbar_wait(bar(kBarP + 2 * X + bx), (n >> 1) & 1);
                trace_stamp(p, first, X ? (t < 128 ? 384 + t : 9999) : (t < 256 ? t : 9999), 4);
                ptx::mbar_wait(bar(kBarVF + st), (gg / kNS) & 1);
                ptx::tc_fence_after();
                issue_pv32<kFmt>(tO, tS + 32 * bx, sV + st * kStage, t > 0, p.p_split != 0);
                if (pv_commit(t)) ptx::umma_commit_elect(bar(kBarPV + 2 * X + bx));
                trace_stamp(p, first, X ? (t < 128 ? 384 + t : 9999) : (t < 256 ? t : 9999), 5);
                if (more) {
                    ptx::mbar_wait(bar(kBarKF + st2), (g2 / kNS) & 1);
                    ptx::tc_fence_after();
                    issue_qk32<kFmt>(tS + 32 * bx, tQ, sK + st2 * kStage);
                    ptx::umma_commit_elect(bar(kBarS + 2 * X + bx));
                }
                trace_stamp(p, first, X ? (t < 128 ? 384 + t : 9999) : (t < 256 ? t : 9999), 6);
                if (POD_SM_MERGED_EMPTY) {
                    release(bar(kBarKE + st));  // K(t) and V(t) both consumed by this thread
                } else {
                    release(bar(kBarVE + st));
                    if (more) release(bar(kBarKE + st2));
                }
            }
        }
    } else {
        // ------------------------------------ softmax (4 warps per block) --
        const int X = warp >> 2;  // block
        if (X == 1 && !hasB) return;
        const int q = warp & 3;   // TMEM lane quadrant
        const BlockRange br = X ? rB : rA;
        const int m = q * 32 + lane;  // row of the block
        const int my_r = br.r0 + m / G;
        const bool row_ok = (m / G) < br.nrows;
        const int vis = p.offset + my_r;
        const int qhead = job.kv_head * G + m % G;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
        const uint32_t o_addr = lane_base + (X ? kOB : kOA);
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
        if (nt == 0) {
            if (row_ok) {
                for (int c = 0; c < p.hd; c += 4) store4(orow, c, make_float4(0.f, 0.f, 0.f, 0.f));
                *lrow = -INFINITY;
            }
            return;
        }
        // ---- Q row -> TMEM (A operand of QK^T); rows past the chunk are zero
        {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(static_cast<const uint16_t*>(p.q_prefill) +
                                                                    (static_cast<size_t>(my_r) * p.hq + qhead) * p.hd);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                float qv[32];
#pragma unroll
                for (int c = 0; c < 32; c += 4) {  // (32 hf + c) pairs = d 64 hf + 2c; zero past the head dim
                    const uint4 v = row_ok && 64 * hf + 2 * c < p.hd
                                        ? __ldg(reinterpret_cast<const uint4*>(src + 32 * hf + c))
                                        : make_uint4(0u, 0u, 0u, 0u);
                    qv[c] = __uint_as_float(v.x);
                    qv[c + 1] = __uint_as_float(v.y);
                    qv[c + 2] = __uint_as_float(v.z);
                    qv[c + 3] = __uint_as_float(v.w);
                }
                ptx::tmem_st32(lane_base + (X ? kQB : kQA) + 32 * hf, qv);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(bar(X));
        }
        // POD_PRECISION_F16PV: block A converts V(t) to fp16 in smem before its P(t)
        // arrival (PV_B(t) is issued after PV_A(t)); V(t+1) is converted right after
        // P(t) is handed over, while the next S is computed, off the critical path.
        auto v_to_f16 = [&](int t) {
            const int gg = s0.g + t, st = gg % kNS;
            ptx::mbar_wait(bar(kBarVF + st), (gg / kNS) & 1);
            v_stage_to_f16<kStage, 128>(sV + st * kStage, q * 32 + lane);
        };
        if (kFmt == 1 && p.p_f16 && !p.vs_pages && X == 0) v_to_f16(0);
        float m_run = -INFINITY, l_run = 0.f;
        for (int t = 0; t < nt; ++t) {
            const int n = s0.n[X] + t, b = n & 1;
            const uint32_t s_addr = lane_base + (X ? kSB : kSA) + 32 * b;
            if (lane == 0 && q == 0) trace_stamp(p, first, X ? (t < 128 ? 384 + t : 9999) : (t < 256 ? t : 9999), 0);
            sm_wait<POD_SM_SOFTMAX_SLEEP>(bar(kBarS + 2 * X + b), (n >> 1) & 1);
            if (lane == 0 && q == 0) trace_stamp(p, first, X ? (t < 128 ? 384 + t : 9999) : (t < 256 ? t : 9999), 1);
            ptx::tc_fence_after();
            if (POD_SOFTMAX_SKIP) {  // timing experiment only: P = S bits, no softmax work
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(bar(kBarP + 2 * X + b));
                continue;
            }
            float s[kTN];
            ptx::tmem_ld32(s_addr, s);
            ptx::tmem_wait_ld();
            const int kb = kt0 + t * kTN;
            const int lo = max(job.kv_begin - kb, 0);
            const int hi = row_ok ? min(min(job.kv_end, vis + 1) - kb, kTN) : 0;
            if (!__all_sync(0xffffffffu, lo == 0 && hi == kTN)) {
#pragma unroll
                for (int c = 0; c < kTN; ++c)
                    if (c < lo || c >= hi) s[c] = -INFINITY;
            }
            const float tmax = row_max<kTN>(s);
            const float m_new = fmaxf(m_run, tmax * p.sl2);
            const bool need = m_new > m_run + 8.f;  // lazy rescale (see prefill_item)
            const float m_use = need ? m_new : m_run;
            const float factor = need ? ptx::ex2(m_run - m_new) : 1.f;
            l_run *= factor;
            m_run = m_use;
            // O is rescaled only when the reference max moved: then wait for
            // PV_X(t-1), the newest MMA writing O_X (PV_X(t) needs our arrival).
            if (t > 0 && __any_sync(0xffffffffu, need)) {
                if (!POD_SM_LAZY_PV)
                    ptx::mbar_wait(bar(kBarPV + 2 * X + ((n - 1) & 1)), ((n - 1) >> 1) & 1);
                else if (t + 1 < nt)  // S_X(t+1) complete => PV_X(t-1) complete
                    ptx::mbar_wait(bar(kBarS + 2 * X + ((n + 1) & 1)), ((n + 1) >> 1) & 1);
                else
                    ptx::mbar_wait(bar(kBarPV + 2 * X + ((n - 1) & 1)), s0.npv[X][(n - 1) & 1] & 1);
                ptx::tc_fence_after();
#pragma unroll 1
                for (int ch = 0; ch < kHeadDim / 32; ++ch) {
                    float o[32];
                    ptx::tmem_ld32(o_addr + ch * 32, o);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 32; ++c) o[c] *= factor;
                    ptx::tmem_st32(o_addr + ch * 32, o);
                }
            }
            const float neg_m = m_use == -INFINITY ? 0.f : -m_use;
            float lsum;
            if (kFmt == 1 && p.p_f16)
                lsum = softmax_p_row<kFmt, 3, kTN>(s, p.sl2, neg_m, s_addr);
            else if (kFmt == 1 && p.p_split)
                lsum = softmax_p_row<kFmt, 1, kTN>(s, p.sl2, neg_m, s_addr);
            else if (p.p_split)
                lsum = softmax_p_row<kFmt, 2, kTN>(s, p.sl2, neg_m, s_addr);
            else
                lsum = softmax_p_row<kFmt, 0, kTN>(s, p.sl2, neg_m, s_addr);
            l_run += lsum;
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0 && q == 0) trace_stamp(p, first, X ? (t < 128 ? 384 + t : 9999) : (t < 256 ? t : 9999), 2);
            if (lane == 0 && q == 3) trace_stamp(p, first, X ? (t < 128 ? 384 + t : 9999) : (t < 256 ? t : 9999), 3);
            if (lane == 0) ptx::mbar_arrive(bar(kBarP + 2 * X + b));
            if (kFmt == 1 && p.p_f16 && !p.vs_pages && X == 0 && t + 1 < nt) v_to_f16(t + 1);  // off the P(t) -> PV(t) path
        }
        // ------------------------------------------------- epilogue --
        {  // the last PV's commit covers every earlier MMA of this thread
            const int nl = s0.n[X] + nt - 1;
            ptx::mbar_wait(bar(kBarPV + 2 * X + (nl & 1)), POD_SM_LAZY_PV ? s0.npv[X][nl & 1] & 1 : (nl >> 1) & 1);
            // the other S buffer's PV barrier completed its phase for tile nt-2 (implied by the
            // wait above, in-order pipe); observing it keeps every phase waited before the
            // next item commits to the barrier again (compute-sanitizer synccheck)
            if (POD_SM_LAZY_PV && nt >= 2)
                ptx::mbar_wait(bar(kBarPV + 2 * X + ((nl - 1) & 1)), s0.npv[X][(nl - 1) & 1] & 1);
        }
        ptx::tc_fence_after();
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        store_o_rows(o_addr, inv, orow, row_ok, sbase + kOffKs + static_cast<uint32_t>(warp) * 4096u, lane, p.hd);
        if (row_ok) *lrow = l_run > 0.f ? (m_run + ptx::lg2(l_run)) * kLn2 : -INFINITY;
        ptx::tc_fence_before();
    }
}


// ---------------------------------------------------------------------------
// The pair engine over 64-key K/V tiles with ONE S buffer per block (plans with
// pf_tn64: prefill-dominant batches, pod_plan.cpp).
// TMEM keeps the same columns (Q_A | Q_B | S_A | S_B | O_A | O_B, S now 64 keys
// wide): per 64 keys a block issues 8 QK (N = 64) + 8 PV MMAs instead of 2 x 12,
// and half the barrier hops.  With S single-buffered, QK_X(t+1) follows PV_X(t)
// in the in-order pipe, and S_X(t) complete implies PV_X(t-1) complete, so the
// lazy O rescale needs no extra wait.  K and V rings: 2 stages of 16 KB each with
// separate empty barriers (K freed after both QKs, V after both PVs).
#ifndef POD_SM64_SPIN_MMA
#define POD_SM64_SPIN_MMA 0  // MMA issuer polls P_X with test_wait (no suspend) instead of try_wait
#endif
#ifndef POD_SM64_SPIN_SOFTMAX
#define POD_SM64_SPIN_SOFTMAX 0  // softmax warps poll S_X with test_wait
#endif
namespace sm64 {
__device__ __forceinline__ void wait_mma(uint32_t bar, uint32_t parity) {
    if (POD_SM64_SPIN_MMA)
        ptx::mbar_wait_spin(bar, parity);
    else
        ptx::mbar_wait(bar, parity);
}
__device__ __forceinline__ void wait_softmax(uint32_t bar, uint32_t parity) {
    if (POD_SM64_SPIN_SOFTMAX)
        ptx::mbar_wait_spin(bar, parity);
    else
        ptx::mbar_wait(bar, parity);
}
constexpr int kTN = 64;
constexpr int kNS = 2;                      // V stages
constexpr int kNSK = POD_SM64_KSTAGES;      // K stages
constexpr uint32_t kStage = kTN * kHeadDim * 2;  // 16 KB: [d-half][64 keys][64 d], SW128
static_assert((kNS + kNSK) * kStage <= sm3::kPfRingBytes, "the prefill ring region holds both rings");
static_assert(kNSK <= sm3::kNS, "K stage barriers");
static_assert(kNSK * kStage >= 8 * 4096, "the epilogue's 8 warp tiles (store_o_rows) fit the K ring");
__device__ __forceinline__ void load_tile64(const RunParams& p, const CUtensorMap* tm, uint32_t dst, uint32_t bar,
                                            int kt, int kv_head, const PageIds& ids) {
    int ph[4];
#pragma unroll
    for (int pg = 0; pg < 4; ++pg) ph[pg] = ids.get(min(kt / 16 + pg, ids.n - 1));
#pragma unroll
    for (int pg = 0; pg < 4; ++pg) {
#pragma unroll
        for (int dh = 0; dh < 2; ++dh) {
            const uint32_t d = dst + dh * (kTN * 128) + pg * 2048;
            if (p.kv_layout == POD_KV_HND)
                ptx::tma_load_4d_elect(d, tm, bar, dh * 64, 0, kv_head, ph[pg]);
            else
                ptx::tma_load_4d_elect(d, tm, bar, dh * 64, kv_head, 0, ph[pg]);
        }
    }
}
template <int kFmt>
__device__ __forceinline__ void issue_qk64(uint32_t tmem_s, uint32_t tmem_q, uint32_t sK) {
    constexpr uint32_t idesc = ptx::idesc_f16(kFmt, kMBlock, kTN, 0);
    ptx::umma_ts_k128_elect<kTN * 128>(tmem_s, tmem_q, ptx::sw128_desc(sK, 16, 1024), idesc);
}
}  // namespace sm64

template <int kFmt>
__device__ void prefill_item_sm64(const RunParams& p, const CUtensorMap* tmk, const CUtensorMap* tmv /* 5-D page map */, int item,
                                  uint32_t sbase, uint32_t tmem, sm3::PfState& ps, int warp, int lane) {
    using namespace sm3;
    using sm64::kTN;
    using sm64::kNS;
    using sm64::kStage;
    using sm64::kNSK;
    const PrefillCta job = p.pctas[item];
    const int G = p.group;
    const int rpb = kMBlock / G;
    const int nblocks = (job.rows + rpb - 1) / rpb;  // 1 or 2
    const bool hasB = nblocks > 1;
    const BlockRange rA = prefill_block(p, job, 0);
    const BlockRange rB = hasB ? prefill_block(p, job, 1) : rA;
    const int kv_hi = min(job.kv_end, p.offset + (hasB ? rB.r0 + rB.nrows : rA.r0 + rA.nrows));
    const int kt0 = rA.kt0;
    const int nt = kv_hi > job.kv_begin ? (kv_hi - kt0 + kTN - 1) / kTN : 0;
    const PfState s0 = uniform(ps);
    if (nt > 0) {  // g: tiles through the rings; n: S / P completions; npv[X][0]: PV commits
        ps.g += nt;
        ps.n[0] += nt;
        ps.nq[0] += 1;
        ps.npv[0][0] += 1;
        if (hasB) {
            ps.n[1] += nt;
            ps.nq[1] += 1;
            ps.npv[1][0] += 1;
        }
    }
    const int pbeg = p.page_indptr[0];
    const int npages = p.page_indptr[1] - pbeg;
    const uint32_t bar0 = sbase + kOffBars;
    auto bar = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
    const uint32_t sK = sbase + kOffKs, sV = sbase + kOffKs + kNSK * kStage;
    // debug trace (POD_TRACE_STAMPS builds): CTA 0's first item; row t = block A + MMA A,
    // row 384 + t = block B + MMA B + producer (tools/profile_run.py --trace64)
    const int first = s0.n[0] == 0 ? 0 : 1;
    auto rowB = [&](int t) { return t < 384 ? 384 + t : 9999; };

    if (warp == kProdWarp) {
        // ------------------------------------------------ TMA producer --
        PageIds ids;
        ids.init(p.page_indices + pbeg, npages, kt0 / 16);
        for (int t = 0; t < nt; ++t) {
            const int gg = s0.g + t, st = gg % kNS, sk = gg % kNSK;
            if (gg >= kNSK) ptx::mbar_wait_relaxed<POD_SM_PROD_SLEEP>(bar(kBarKE + sk), ((gg / kNSK) - 1) & 1);
            ptx::mbar_arrive_expect_tx_elect(bar(kBarKF + sk), kStage);
            sm64::load_tile64(p, tmk, sK + sk * kStage, bar(kBarKF + sk), kt0 + t * kTN, job.kv_head, ids);
            if (lane == 0) trace_stamp(p, first, rowB(t), 6);
            if (gg >= kNS) ptx::mbar_wait_relaxed<POD_SM_PROD_SLEEP>(bar(kBarVE + st), ((gg / kNS) - 1) & 1);
            if (p.vs_pages && t == 0) ptx::griddep_wait();  // the fp16 V shadow (see prefill_item)
            ptx::mbar_arrive_expect_tx_elect(bar(kBarVF + st), kStage);
            prefill_load_v_pages<4>(tmv, sV + st * kStage, bar(kBarVF + st), kt0 + t * kTN, job.kv_head, ids, p.vs_pages);
            if (lane == 0) trace_stamp(p, first, rowB(t), 7);
        }
    } else if (warp == kMmaWarp) {
        // -------------------------------------------------- MMA issuer --
        auto mma_issuer = [&](auto pv_c) {  // kPv as in prefill_item_sm
            constexpr int kPv = decltype(pv_c)::value;
            constexpr bool kSplit = kPv == 0;
            constexpr int kPvFmt = kPv == 2 ? 0 : kFmt;
            if (nt == 0) return;
            ptx::mbar_wait(bar(0), s0.nq[0] & 1);
            if (hasB) ptx::mbar_wait(bar(1), s0.nq[1] & 1);
            {
                const int gg = s0.g, sk = gg % kNSK;
                ptx::mbar_wait(bar(kBarKF + sk), (gg / kNSK) & 1);
                ptx::tc_fence_after();
                sm64::issue_qk64<kFmt>(tmem + kSA, tmem + kQA, sK + sk * kStage);
                ptx::umma_commit_elect(bar(kBarS + 0));
                if (hasB) {
                    sm64::issue_qk64<kFmt>(tmem + kSB, tmem + kQB, sK + sk * kStage);
                    ptx::umma_commit_elect(bar(kBarS + 1));
                }
                ptx::umma_commit_elect(bar(kBarKE + sk));
            }
            for (int t = 0; t < nt; ++t) {
                const int gg = s0.g + t, st = gg % kNS;
                const int g1 = gg + 1, sk1 = g1 % kNSK;
                const bool more = t + 1 < nt, last = t + 1 == nt;
#pragma unroll
                for (int X = 0; X < 2; ++X) {
                    if (X == 1 && !hasB) break;
                    const int n = s0.n[X] + t;
                    sm64::wait_mma(bar(kBarP + X), n & 1);
                    if (lane == 0) trace_stamp(p, first, X ? rowB(t) : t, 4);
                    if (X == 0) ptx::mbar_wait(bar(kBarVF + st), (gg / kNS) & 1);
                    ptx::tc_fence_after();
                    if (POD_SM64_BATCHED_PV) {
                        constexpr uint32_t idesc_pv = ptx::idesc_f16(kPvFmt, kMBlock, kHeadDim, 1);
                        ptx::umma_pv64_elect<kSplit>(tmem + (X ? kOB : kOA), tmem + (X ? kSB : kSA),
                                                     ptx::sw128_desc(sV + st * kStage, 2048, 1024), idesc_pv,
                                                     t > 0 ? 1u : 0u);
                    } else {
                        prefill_issue_pv<kPvFmt>(tmem + (X ? kOB : kOA), tmem + (X ? kSB : kSA), sV + st * kStage,
                                                 t > 0, kSplit);
                    }
                    if (last) ptx::umma_commit_elect(bar(kBarPV + X));
                    if (more) {
                        if (X == 0) {
                            ptx::mbar_wait(bar(kBarKF + sk1), (g1 / kNSK) & 1);
                            ptx::tc_fence_after();
                        }
                        sm64::issue_qk64<kFmt>(tmem + (X ? kSB : kSA), tmem + (X ? kQB : kQA), sK + sk1 * kStage);
                        ptx::umma_commit_elect(bar(kBarS + X));
                    }
                    if (lane == 0) trace_stamp(p, first, X ? rowB(t) : t, 5);
                }
                ptx::umma_commit_elect(bar(kBarVE + st));          // V(t): both PVs issued above
                if (more) ptx::umma_commit_elect(bar(kBarKE + sk1));  // K(t+1): both QKs
            }
        };
        if (kFmt == 1 && p.p_f16)
            mma_issuer(std::integral_constant<int, 2>{});
        else if (p.p_split != 0)
            mma_issuer(std::integral_constant<int, 0>{});
        else
            mma_issuer(std::integral_constant<int, 1>{});
    } else if (warp < kProdWarp) {
        // ------------------------------------ softmax (4 warps per block) --
        const int X = warp >> 2;  // block
        if (X == 1 && !hasB) return;
        const int q = warp & 3;   // TMEM lane quadrant
        const BlockRange br = X ? rB : rA;
        const int m = q * 32 + lane;
        const int my_r = br.r0 + m / G;
        const bool row_ok = (m / G) < br.nrows;
        const int vis = p.offset + my_r;
        const int qhead = job.kv_head * G + m % G;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
        const uint32_t o_addr = lane_base + (X ? kOB : kOA);
        const uint32_t s_addr = lane_base + (X ? kSB : kSA);
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
        if (nt == 0) {
            if (row_ok) {
                for (int c = 0; c < p.hd; c += 4) store4(orow, c, make_float4(0.f, 0.f, 0.f, 0.f));
                *lrow = -INFINITY;
            }
            return;
        }
        {  // Q row -> TMEM (A operand of QK^T); rows past the chunk are zero
            const uint32_t* src = reinterpret_cast<const uint32_t*>(static_cast<const uint16_t*>(p.q_prefill) +
                                                                    (static_cast<size_t>(my_r) * p.hq + qhead) * p.hd);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                float qv[32];
#pragma unroll
                for (int c = 0; c < 32; c += 4) {  // (32 hf + c) pairs = d 64 hf + 2c; zero past the head dim
                    const uint4 v = row_ok && 64 * hf + 2 * c < p.hd
                                        ? __ldg(reinterpret_cast<const uint4*>(src + 32 * hf + c))
                                        : make_uint4(0u, 0u, 0u, 0u);
                    qv[c] = __uint_as_float(v.x);
                    qv[c + 1] = __uint_as_float(v.y);
                    qv[c + 2] = __uint_as_float(v.z);
                    qv[c + 3] = __uint_as_float(v.w);
                }
                ptx::tmem_st32(lane_base + (X ? kQB : kQA) + 32 * hf, qv);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(bar(X));
        }
        // POD_PRECISION_F16PV: as in prefill_item_sm (V(t+1) converted after P(t) is handed over)
        auto v_to_f16 = [&](int t) {
            const int gg = s0.g + t, st = gg % kNS;
            ptx::mbar_wait(bar(kBarVF + st), (gg / kNS) & 1);
            v_stage_to_f16<kStage, 128>(sV + st * kStage, q * 32 + lane);
        };
        if (kFmt == 1 && p.p_f16 && !p.vs_pages && X == 0) v_to_f16(0);
        float m_run = -INFINITY, l_run = 0.f;
        for (int t = 0; t < nt; ++t) {
            const int n = s0.n[X] + t;
            if (lane == 0 && q == 0) trace_stamp(p, first, X ? rowB(t) : t, 0);
            sm64::wait_softmax(bar(kBarS + X), n & 1);  // also: PV_X(t-1) complete
            if (lane == 0 && q == 0) trace_stamp(p, first, X ? rowB(t) : t, 1);
            ptx::tc_fence_after();
            float s[kTN];
            ptx::tmem_ld32(s_addr, *reinterpret_cast<float(*)[32]>(&s[0]));
            ptx::tmem_ld32(s_addr + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
            ptx::tmem_wait_ld();
            if (lane == 0 && q == 0 && X == 0) trace_stamp(p, first, t, 6);
            const int kb = kt0 + t * kTN;
            const int lo = max(job.kv_begin - kb, 0);
            const int hi = row_ok ? min(min(job.kv_end, vis + 1) - kb, kTN) : 0;
            if (!__all_sync(0xffffffffu, lo == 0 && hi == kTN)) {
#pragma unroll
                for (int c = 0; c < kTN; ++c)
                    if (c < lo || c >= hi) s[c] = -INFINITY;
            }
            const float tmax = row_max<kTN>(s);
            const float m_new = fmaxf(m_run, tmax * p.sl2);
            const bool need = m_new > m_run + 8.f;  // lazy rescale (see prefill_item)
            const float m_use = need ? m_new : m_run;
            const float factor = need ? ptx::ex2(m_run - m_new) : 1.f;
            l_run *= factor;
            m_run = m_use;
            if (t > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
                for (int ch = 0; ch < kHeadDim / 32; ++ch) {
                    float o[32];
                    ptx::tmem_ld32(o_addr + ch * 32, o);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 32; ++c) o[c] *= factor;
                    ptx::tmem_st32(o_addr + ch * 32, o);
                }
            }
            const float neg_m = m_use == -INFINITY ? 0.f : -m_use;
            float lsum;
            if (kFmt == 1 && p.p_f16)
                lsum = softmax_p_row<kFmt, 3, kTN>(s, p.sl2, neg_m, s_addr);
            else if (kFmt == 1 && p.p_split)
                lsum = softmax_p_row<kFmt, 1, kTN>(s, p.sl2, neg_m, s_addr);
            else if (p.p_split)
                lsum = softmax_p_row<kFmt, 2, kTN>(s, p.sl2, neg_m, s_addr);
            else
                lsum = softmax_p_row<kFmt, 0, kTN>(s, p.sl2, neg_m, s_addr);
            l_run += lsum;
            if (lane == 0 && q == 0 && X == 0) trace_stamp(p, first, t, 7);
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0 && q == 0) trace_stamp(p, first, X ? rowB(t) : t, 2);
            if (lane == 0 && q == 3) trace_stamp(p, first, X ? rowB(t) : t, 3);
            if (lane == 0) ptx::mbar_arrive(bar(kBarP + X));
            if (kFmt == 1 && p.p_f16 && !p.vs_pages && X == 0 && t + 1 < nt) v_to_f16(t + 1);  // off the P(t) -> PV(t) path
        }
        if (lane == 0 && warp == 0) trace_stamp(p, first, 766, 0);
        ptx::mbar_wait(bar(kBarPV + X), s0.npv[X][0] & 1);  // the last PV (commit covers all)
        if (lane == 0 && warp == 0) trace_stamp(p, first, 766, 1);
        ptx::tc_fence_after();
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        store_o_rows(o_addr, inv, orow, row_ok, sbase + kOffKs + static_cast<uint32_t>(warp) * 4096u, lane, p.hd);
        if (lane == 0 && warp == 0) trace_stamp(p, first, 766, 2);
        if (row_ok) *lrow = l_run > 0.f ? (m_run + ptx::lg2(l_run)) * kLn2 : -INFINITY;
        ptx::tc_fence_before();
    }
}

// ---------------------------------------------------------------------------
// The pair engine over 64-key tiles with DOUBLE-buffered S per block (prefill-dominant
// plans, pf_tn64; the kE = 1 kernel instance).  The single-S 64-key engine cannot start
// QK_X(t+1) before the softmax of tile t has handed P over (P lives over S), so each
// block's chain is softmax -> P hop -> PV + QK -> S hop per tile.  With two
// S buffers per block QK_X(t+2) runs while the softmax of tile t+1 does, as in the
// two-CTA kernel's prefill CTA (the fastest prefill engine of the repo) -- but TMEM then
// has no room for Q (S_A[2] | S_B[2] | O_A | O_B = 512 columns), so Q sits in shared
// memory and QK^T is an SS-MMA, and the decode group keeps 2 ring stages per warp:
//   smem  K ring [0, 32K) | V ring [32K, 64K) | Q_A | Q_B (SW128, 32 KB each) | decode
// V comes from the fp16 shadow (pod_plan::vs_pages) for F16PV plans, so no per-tile
// conversion sits on the softmax warps either.
namespace db {
constexpr int kTN = 64, kNS = 2;
constexpr uint32_t kStage = kTN * kHeadDim * 2;       // 16 KB: K [d-half][64 keys][64 d]; V page-major
constexpr uint32_t kQBytes = kMBlock * kHeadDim * 2;  // 32 KB per block
constexpr uint32_t kOffK = 0, kOffV = kNS * kStage, kOffQ = 2 * kNS * kStage;
constexpr uint32_t kPfBytes = kOffQ + 2 * kQBytes;    // 128 KB
constexpr uint32_t kSA = 0, kSB = 128, kOA = 256, kOB = 384;  // S_X[b] at kSX + 64 b
static_assert(kNS <= sm3::kNS, "stage barriers");
static_assert(kNS * kStage >= 8 * 4096, "the epilogue's 8 warp tiles (store_o_rows) fit the K ring");
template <int kFmt>
__device__ __forceinline__ void issue_qk(uint32_t tmem_s, uint32_t sQ, uint32_t sK) {
    constexpr uint32_t idesc = ptx::idesc_f16(kFmt, kMBlock, kTN, 0);
    ptx::umma_ss_k128_elect<kMBlock * 128, kTN * 128>(tmem_s, ptx::sw128_desc(sQ, 16, 1024),
                                                      ptx::sw128_desc(sK, 16, 1024), idesc);
}
}  // namespace db

template <int kFmt, uint32_t kOffBars>
__device__ void prefill_item_db(const RunParams& p, const CUtensorMap* tmk, const CUtensorMap* tmv /* 5-D page map */,
                                int item, uint32_t sbase, uint32_t tmem, sm3::PfState& ps, int warp, int lane) {
    using namespace sm3;
    using db::kTN;
    using db::kNS;
    using db::kStage;
    const PrefillCta job = p.pctas[item];
    const int G = p.group;
    const int rpb = kMBlock / G;
    const int nblocks = (job.rows + rpb - 1) / rpb;  // 1 or 2
    const bool hasB = nblocks > 1;
    const BlockRange rA = prefill_block(p, job, 0);
    const BlockRange rB = hasB ? prefill_block(p, job, 1) : rA;
    const int kv_hi = min(job.kv_end, p.offset + (hasB ? rB.r0 + rB.nrows : rA.r0 + rA.nrows));
    const int kt0 = rA.kt0;
    const int nt = kv_hi > job.kv_begin ? (kv_hi - kt0 + kTN - 1) / kTN : 0;
    const PfState s0 = uniform(ps);
    if (nt > 0) {  // as prefill_item_sm: tiles, S / P completions, Q loads, lazy PV commits
        ps.g += nt;
        ps.n[0] += nt;
        ps.nq[0] += 1;
        if (hasB) {
            ps.n[1] += nt;
            ps.nq[1] += 1;
        }
        for (int t = max(0, nt - 2); t < nt; ++t) {
            ps.npv[0][(s0.n[0] + t) & 1] += 1;
            if (hasB) ps.npv[1][(s0.n[1] + t) & 1] += 1;
        }
    }
    // PV_X(t) commits only for the last two tiles (one per S buffer); earlier, "PV_X(t-1)
    // done" is implied by S_X(t+1)'s commit (prefill_item_sm)
    auto pv_commit = [&](int t) { return t + 2 >= nt; };
    const int pbeg = p.page_indptr[0];
    const int npages = p.page_indptr[1] - pbeg;
    const uint32_t bar0 = sbase + kOffBars;
    auto bar = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
    const uint32_t sK = sbase + db::kOffK, sV = sbase + db::kOffV, sQ = sbase + db::kOffQ;

    if (warp == kProdWarp) {
        // ------------------------------------------------ TMA producer --
        // K(t), then V(t-1): K stages free after both QK(t) (issued two tiles ahead), V stages
        // after both PV(t)
        PageIds ids;
        ids.init(p.page_indices + pbeg, npages, kt0 / 16);
        for (int t = 0; t <= nt && nt > 0; ++t) {
            if (t < nt) {
                const int gg = s0.g + t, st = gg % kNS;
                if (gg >= kNS) ptx::mbar_wait_relaxed<POD_SM_PROD_SLEEP>(bar(kBarKE + st), ((gg / kNS) - 1) & 1);
                ptx::mbar_arrive_expect_tx_elect(bar(kBarKF + st), kStage);
                sm64::load_tile64(p, tmk, sK + st * kStage, bar(kBarKF + st), kt0 + t * kTN, job.kv_head, ids);
            }
            if (t > 0) {
                const int gg = s0.g + t - 1, st = gg % kNS;
                if (gg >= kNS) ptx::mbar_wait_relaxed<POD_SM_PROD_SLEEP>(bar(kBarVE + st), ((gg / kNS) - 1) & 1);
                if (p.vs_pages && t == 1) ptx::griddep_wait();  // the fp16 V shadow (see prefill_item)
                ptx::mbar_arrive_expect_tx_elect(bar(kBarVF + st), kStage);
                prefill_load_v_pages<4>(tmv, sV + st * kStage, bar(kBarVF + st), kt0 + (t - 1) * kTN, job.kv_head,
                                        ids, p.vs_pages);
            }
        }
    } else if (warp == kMmaWarp) {
        // -------------------------------------------------- MMA issuer --
        auto mma_issuer = [&](auto pv_c) {  // kPv as in prefill_item_sm
            constexpr int kPv = decltype(pv_c)::value;
            constexpr bool kSplit = kPv == 0;
            constexpr int kPvFmt = kPv == 2 ? 0 : kFmt;
            constexpr uint32_t idesc_pv = ptx::idesc_f16(kPvFmt, kMBlock, kHeadDim, 1);
            if (nt == 0) return;
            ptx::mbar_wait(bar(0), s0.nq[0] & 1);
            if (hasB) ptx::mbar_wait(bar(1), s0.nq[1] & 1);
            for (int j = 0; j < 2 && j < nt; ++j) {
                const int gg = s0.g + j, st = gg % kNS;
                ptx::mbar_wait(bar(kBarKF + st), (gg / kNS) & 1);
                ptx::tc_fence_after();
                const int bA = (s0.n[0] + j) & 1, bB = (s0.n[1] + j) & 1;
                db::issue_qk<kFmt>(tmem + db::kSA + 64 * bA, sQ, sK + st * kStage);
                ptx::umma_commit_elect(bar(kBarS + bA));
                if (hasB) {
                    db::issue_qk<kFmt>(tmem + db::kSB + 64 * bB, sQ + db::kQBytes, sK + st * kStage);
                    ptx::umma_commit_elect(bar(kBarS + 2 + bB));
                }
                ptx::umma_commit_elect(bar(kBarKE + st));  // K(j): both QKs issued
            }
            for (int t = 0; t < nt; ++t) {
                const int gg = s0.g + t, st = gg % kNS;
                const int g2 = gg + 2, st2 = g2 % kNS;
                const bool more = t + 2 < nt;
#pragma unroll
                for (int X = 0; X < 2; ++X) {
                    if (X == 1 && !hasB) break;
                    const int n = s0.n[X] + t, b = n & 1;
                    const uint32_t tS = tmem + (X ? db::kSB : db::kSA) + 64 * b;
                    ptx::mbar_wait(bar(kBarP + 2 * X + b), (n >> 1) & 1);
                    if (X == 0) ptx::mbar_wait(bar(kBarVF + st), (gg / kNS) & 1);
                    ptx::tc_fence_after();
                    ptx::umma_pv64_elect<kSplit>(tmem + (X ? db::kOB : db::kOA), tS,
                                                 ptx::sw128_desc(sV + st * kStage, 2048, 1024), idesc_pv,
                                                 t > 0 ? 1u : 0u);
                    if (pv_commit(t)) ptx::umma_commit_elect(bar(kBarPV + 2 * X + b));
                    if (more) {  // QK_X(t+2) reuses S_X[b] after PV_X(t) read its P (in-order pipe)
                        if (X == 0) {
                            ptx::mbar_wait(bar(kBarKF + st2), (g2 / kNS) & 1);
                            ptx::tc_fence_after();
                        }
                        db::issue_qk<kFmt>(tS, sQ + X * db::kQBytes, sK + st2 * kStage);
                        ptx::umma_commit_elect(bar(kBarS + 2 * X + b));
                    }
                }
                ptx::umma_commit_elect(bar(kBarVE + st));             // V(t): both PVs issued
                if (more) ptx::umma_commit_elect(bar(kBarKE + st2));  // K(t+2): both QKs issued
            }
        };
        if (kFmt == 1 && p.p_f16)
            mma_issuer(std::integral_constant<int, 2>{});
        else if (p.p_split != 0)
            mma_issuer(std::integral_constant<int, 0>{});
        else
            mma_issuer(std::integral_constant<int, 1>{});
    } else if (warp < kProdWarp) {
        // ------------------------------------ softmax (4 warps per block) --
        const int X = warp >> 2;
        if (X == 1 && !hasB) return;
        const int q = warp & 3;
        const BlockRange br = X ? rB : rA;
        const int m = q * 32 + lane;
        const int my_r = br.r0 + m / G;
        const bool row_ok = (m / G) < br.nrows;
        const int vis = p.offset + my_r;
        const int qhead = job.kv_head * G + m % G;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
        const uint32_t o_addr = lane_base + (X ? db::kOB : db::kOA);
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
        if (nt == 0) {
            if (row_ok) {
                for (int c = 0; c < p.hd; c += 4) store4(orow, c, make_float4(0.f, 0.f, 0.f, 0.f));
                *lrow = -INFINITY;
            }
            return;
        }
        {  // Q row -> shared memory, SW128 K-major (A operand of the SS QK^T); zero past the chunk / head dim
            const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(p.q_prefill) +
                                                              (static_cast<size_t>(my_r) * p.hq + qhead) * p.hd);
            const uint32_t dst = sQ + X * db::kQBytes + static_cast<uint32_t>(m) * 128u;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint4 v = row_ok && 8 * j < p.hd ? __ldg(src + j) : make_uint4(0u, 0u, 0u, 0u);
                const uint32_t a = dst + (j >> 3) * (kMBlock * 128u) + ((static_cast<uint32_t>(j & 7) ^ (m & 7)) << 4);
                asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                             : "memory");
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(bar(X));
        }
        // POD_PRECISION_F16PV without the shadow (it is on for these plans with bf16 data): block
        // A converts V(t) before its P(t) arrival, as in prefill_item_sm
        auto v_to_f16 = [&](int t) {
            const int gg = s0.g + t, st = gg % kNS;
            ptx::mbar_wait(bar(kBarVF + st), (gg / kNS) & 1);
            v_stage_to_f16<kStage, 128>(sV + st * kStage, q * 32 + lane);
        };
        const bool convert = kFmt == 1 && p.p_f16 && !p.vs_pages && X == 0;
        float m_run = -INFINITY, l_run = 0.f;
        for (int t = 0; t < nt; ++t) {
            const int n = s0.n[X] + t, b = n & 1;
            const uint32_t s_addr = lane_base + (X ? db::kSB : db::kSA) + 64 * b;
            ptx::mbar_wait(bar(kBarS + 2 * X + b), (n >> 1) & 1);
            ptx::tc_fence_after();
            float s[kTN];
            ptx::tmem_ld32(s_addr, *reinterpret_cast<float(*)[32]>(&s[0]));
            ptx::tmem_ld32(s_addr + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
            ptx::tmem_wait_ld();
            const int kb = kt0 + t * kTN;
            const int lo = max(job.kv_begin - kb, 0);
            const int hi = row_ok ? min(min(job.kv_end, vis + 1) - kb, kTN) : 0;
            if (!__all_sync(0xffffffffu, lo == 0 && hi == kTN)) {
#pragma unroll
                for (int c = 0; c < kTN; ++c)
                    if (c < lo || c >= hi) s[c] = -INFINITY;
            }
            const float tmax = row_max<kTN>(s);
            const float m_new = fmaxf(m_run, tmax * p.sl2);
            const bool need = m_new > m_run + 8.f;  // lazy rescale (see prefill_item)
            const float m_use = need ? m_new : m_run;
            const float factor = need ? ptx::ex2(m_run - m_new) : 1.f;
            l_run *= factor;
            m_run = m_use;
            if (t > 0 && __any_sync(0xffffffffu, need)) {  // wait for PV_X(t-1), the newest MMA writing O_X
                if (t + 1 < nt)  // S_X(t+1) complete => PV_X(t-1) complete
                    ptx::mbar_wait(bar(kBarS + 2 * X + ((n + 1) & 1)), ((n + 1) >> 1) & 1);
                else
                    ptx::mbar_wait(bar(kBarPV + 2 * X + ((n - 1) & 1)), s0.npv[X][(n - 1) & 1] & 1);
                ptx::tc_fence_after();
#pragma unroll 1
                for (int ch = 0; ch < kHeadDim / 32; ++ch) {
                    float o[32];
                    ptx::tmem_ld32(o_addr + ch * 32, o);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 32; ++c) o[c] *= factor;
                    ptx::tmem_st32(o_addr + ch * 32, o);
                }
            }
            const float neg_m = m_use == -INFINITY ? 0.f : -m_use;
            float lsum;
            // one pair in 8 of the exponentials on the FMA pipe (ex2_poly2): with two S buffers
            // per block the two blocks' softmax phases overlap and share the MUFU (fused C2 B=8
            // 333 -> 321 us; the single-S and two-CTA engines measured no gain or a loss)
            constexpr int kPoly = 1;
            if (kFmt == 1 && p.p_f16)
                lsum = softmax_p_row<kFmt, 3, kTN, kPoly>(s, p.sl2, neg_m, s_addr);
            else if (kFmt == 1 && p.p_split)
                lsum = softmax_p_row<kFmt, 1, kTN, kPoly>(s, p.sl2, neg_m, s_addr);
            else if (p.p_split)
                lsum = softmax_p_row<kFmt, 2, kTN, kPoly>(s, p.sl2, neg_m, s_addr);
            else
                lsum = softmax_p_row<kFmt, 0, kTN, kPoly>(s, p.sl2, neg_m, s_addr);
            l_run += lsum;
            if (convert) v_to_f16(t);  // V(t) before P(t) goes to the MMA issuer
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(bar(kBarP + 2 * X + b));
        }
        // ------------------------------------------------- epilogue --
        {
            const int nl = s0.n[X] + nt - 1;
            ptx::mbar_wait(bar(kBarPV + 2 * X + (nl & 1)), s0.npv[X][nl & 1] & 1);
            if (nt >= 2) ptx::mbar_wait(bar(kBarPV + 2 * X + ((nl - 1) & 1)), s0.npv[X][(nl - 1) & 1] & 1);
        }
        ptx::tc_fence_after();
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        store_o_rows(o_addr, inv, orow, row_ok, sbase + db::kOffK + static_cast<uint32_t>(warp) * 4096u, lane, p.hd);
        if (row_ok) *lrow = l_run > 0.f ? (m_run + ptx::lg2(l_run)) * kLn2 : -INFINITY;
        ptx::tc_fence_before();
    }
}

// Shared-memory layout of the two kernel instances: kE = 0 (32- / 64-key single-S engines,
// six decode warps x 3 ring stages) and kE = 1 (the double-S 64-key engine: Q in smem,
// six decode warps x 2 ring stages).
template <int kE>
struct SmLay {
    static constexpr int kDW = sm3::kDW, kDS = sm3::kDS;
    static constexpr uint32_t kOffDec = sm3::kOffDec, kOffBars = sm3::kOffBars, kOffDecBars = sm3::kOffDecBars,
                              kOffMisc = sm3::kOffMisc, kSmem = sm3::kSmem;
};
#ifndef POD_DB_DEC_WARPS
#define POD_DB_DEC_WARPS 4  // the double-S instance's decode group: warps x ring stages (6 x 2: C2 B=8 322 vs 316 us)
#endif
#ifndef POD_DB_DEC_STAGES
#define POD_DB_DEC_STAGES 3
#endif
template <>
struct SmLay<1> {
    static constexpr int kDW = POD_DB_DEC_WARPS, kDS = POD_DB_DEC_STAGES;
    static constexpr uint32_t kOffDec = db::kPfBytes;
    static constexpr uint32_t kOffBars = kOffDec + kDW * kDS * kDecStageBytes;
    static constexpr uint32_t kOffDecBars = kOffBars + sm3::kNumBars * 8;
    static constexpr uint32_t kOffMisc = kOffDecBars + kDW * kDS * 8;
    static constexpr uint32_t kSmem = kOffMisc + 64;
    static_assert(kSmem <= 232448, "one CTA per SM: <= 227 KB dynamic smem");
    static_assert(kOffDec % 1024 == 0, "SW128 stages are 1024-aligned");
};

__device__ __forceinline__ void sm_log_claim(const RunParams& p, int op, int id, int32_t* slot_out) {
    *slot_out = -1;
    if (!p.role_log || id < 0) return;
    const uint32_t sm = ptx::smid();
    const uint32_t slot = atomicAdd(&p.ctr->arrival, 1u);
    int32_t* rec = p.role_log + 8 * slot;
    rec[0] = static_cast<int32_t>(sm);
    rec[1] = static_cast<int32_t>(atomicAdd(&p.ctr->sm_ctr[sm], 1u));
    rec[2] = op;
    rec[3] = id;
    rec[4] = static_cast<int32_t>(slot);
    rec[5] = static_cast<int32_t>(ptx::globaltimer() & 0x7fffffff);
    rec[7] = static_cast<int32_t>(blockIdx.x);
    *slot_out = static_cast<int32_t>(slot);
}

// One CTA per SM; both engines bind items from their pools until drained.
template <int G, int kFmt, int kE>
__global__ void __launch_bounds__(sm3::kThreads, 1)
    pod_sm_kernel(const __grid_constant__ RunParams p, const __grid_constant__ CUtensorMap tmk,
                  const __grid_constant__ CUtensorMap tmv, const __grid_constant__ CUtensorMap tdk,
                  const __grid_constant__ CUtensorMap tdv) {
    using namespace sm3;
    using L = SmLay<kE>;
    constexpr int kDS = L::kDS, kDW = L::kDW;  // (kDW < sm3::kDW leaves the last warps idle)
    constexpr uint32_t kOffDec = L::kOffDec, kOffBars = L::kOffBars, kOffDecBars = L::kOffDecBars,
                       kOffMisc = L::kOffMisc;
    extern __shared__ __align__(1024) uint8_t smem[];
    // Logical warp roles (0-7 softmax, 8 producer, 9 MMA, 10.. decode).  With
    // POD_SM_SOFTMAX_HIGH the decode group takes the lowest hardware warp ids and the
    // softmax warps the highest (the SMSP arbiter favours higher warp ids); TMEM lane
    // quadrants follow the hardware id, which keeps warp % 4 for every softmax warp.
    // warp index broadcast from lane 0: the compiler then knows it (and every role's loop
    // state) is warp-uniform and keeps MMA / TMA operands on the uniform datapath
    const int hw_warp = POD_SM_UNIFORM_WARP ? __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0)
                                            : static_cast<int>(threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    static_assert(!POD_SM_SOFTMAX_HIGH || (kDecWarp0 == 10 && sm3::kThreads == 512), "role remap layout");
    const int warp = !POD_SM_SOFTMAX_HIGH ? hw_warp
                     : hw_warp >= 8       ? hw_warp - 8    // softmax: hardware warps 8-15 (quadrant = hw % 4)
                     : hw_warp >= 6       ? hw_warp + 2    // producer, MMA: hardware warps 6, 7
                                          : hw_warp + 10;  // decode group: hardware warps 0-5
    const int tid = warp * 32 + lane;
    // debug builds: CTA entry / exit times after the per-tile trace (tools/profile_run.py --cta-times)
    int32_t* cta_t = POD_TRACE_STAMPS && p.trace && p.role_log ? p.role_log + p.trace + 768 * 8 + 2 * blockIdx.x
                                                               : nullptr;
    if (cta_t && tid == 0) cta_t[0] = static_cast<int32_t>(ptx::globaltimer() & 0x7fffffff);
    if (tid == 0) trace_stamp(p, 0, 767, 0);  // debug trace: CTA entry (clock64, row 767)
    const uint32_t sbase = ptx::smem_u32(smem);
    volatile int32_t* misc = reinterpret_cast<volatile int32_t*>(smem + kOffMisc);  // [0] tmem, [2..3] pf, [4..5] dec
    if (tid == 0) {
        if (sbase & 1023u) __trap();
        // q_full (0, 1) and p_full (22-25): one arrival per softmax warp of the block
        for (int i = 0; i < kNumBars; ++i)
            ptx::mbar_init(sbase + kOffBars + 8 * i, (i <= 1 || (i >= kBarP && i < kBarP + 4)) ? kPrefillWarps
                                                     : (kDualMma && i >= kBarKE && i < kBarVE + kNS && !(i >= kBarVF && i < kBarVE)) ? 2 : 1);
        for (int i = 0; i < kDW * kDS; ++i) ptx::mbar_init(sbase + kOffDecBars + 8 * i, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) {
        if (p.num_pctas > 0) ptx::tmem_alloc(ptx::smem_u32(const_cast<int32_t*>(misc)), 512);
        ptx::tmem_relinquish();
    }
    if (warp == kProdWarp && lane == 0) {
        ptx::prefetch_tmap(&tmk);
        ptx::prefetch_tmap(&tmv);
        ptx::prefetch_tmap(&tdk);
        ptx::prefetch_tmap(&tdv);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();

    if (warp < kDecWarp0) {
        // ============================================ prefill engine ===
        // The CTA owns all 512 columns, so the allocation starts at lane 0, column 0:
        // a compile-time TMEM base keeps every MMA operand in uniform registers.
        if (p.num_pctas > 0 && tid == 0 && misc[0] != 0) __trap();
        constexpr uint32_t tmem = 0u;
        PfState ps;
        int prev_slot = -1;
        while (p.num_pctas > 0) {
            ptx::named_bar_sync(1, kPrefillThreads);  // the previous item is complete in every warp
            if (warp == kProdWarp && lane == 0) {
                if (prev_slot >= 0) p.role_log[8 * prev_slot + 6] = static_cast<int32_t>(ptx::globaltimer() & 0x7fffffff);
                int id = static_cast<int>(atomicAdd(&p.ctr->cta_assign[0], 1u));
                if (id >= p.num_pctas) id = -1;
                int32_t slot;
                sm_log_claim(p, 0, id, &slot);
                misc[2] = id;
                misc[3] = slot;
            }
            ptx::named_bar_sync(1, kPrefillThreads);
            const int id = wuni(misc[2]);
            prev_slot = misc[3];
            if (id < 0) break;
            if constexpr (kE == 1) {
                prefill_item_db<kFmt, kOffBars>(p, &tmk, p.vs_pages ? &tmv : &tdv, id, sbase, tmem, ps, warp, lane);
            } else if (p.pf_tn64) {
                const int fi = ps.n[0] == 0 ? 0 : 1;  // debug trace: the CTA's first item
                if (tid == 0) trace_stamp(p, fi, 767, 1);
                prefill_item_sm64<kFmt>(p, &tmk, p.vs_pages ? &tmv : &tdv, id, sbase, tmem, ps, warp, lane);
                if (lane == 0 && (warp == 0 || warp == kProdWarp || warp == kMmaWarp))
                    trace_stamp(p, fi, 767, warp == 0 ? 2 : warp == kProdWarp ? 3 : 4);  // role done
            }
            else
                prefill_item_sm<kFmt>(p, &tmk, p.vs_pages ? &tmv : &tdv, id, sbase, tmem, ps, warp, lane);
        }
        ptx::tc_fence_before();
        ptx::named_bar_sync(1, kPrefillThreads);
        ptx::tc_fence_after();
        if (warp == 0 && p.num_pctas > 0) ptx::tmem_dealloc(tmem, 512);
    } else {
        // ============================================= decode engine ===
        const int dw = warp - kDecWarp0;
        int dpos = 0;
        while (p.num_dctas > 0 && dw < kDW) {
            if (dw == 0 && lane == 0) {
                int id = static_cast<int>(atomicAdd(&p.ctr->cta_assign[1], 1u));
                if (id >= p.num_dctas) id = -1;
                int32_t slot;
                sm_log_claim(p, 1, id, &slot);
                misc[4] = id;
                misc[5] = slot;
            }
            ptx::named_bar_sync(3, kDW * 32);
            const int id = wuni(misc[4]), slot = misc[5];
            ptx::named_bar_sync(3, kDW * 32);
            if (id < 0) break;
            decode_item<G, kFmt, kDW, kDS>(p, &tdk, &tdv, id, dw, sbase + kOffDec, sbase + kOffDecBars,
                                           reinterpret_cast<float*>(smem + kOffDec), 2, dpos);
            if (slot >= 0 && dw == 0 && lane == 0)
                p.role_log[8 * slot + 6] = static_cast<int32_t>(ptx::globaltimer() & 0x7fffffff);
        }
    }
    ptx::griddep_launch_dependents();  // the split merge may start launching (it waits for completion)
    __syncthreads();
    if (cta_t && tid == 0) cta_t[1] = static_cast<int32_t>(ptx::globaltimer() & 0x7fffffff);
    if (tid == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(&p.ctr->done, 1u);
        if (prev == gridDim.x - 1) {
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
