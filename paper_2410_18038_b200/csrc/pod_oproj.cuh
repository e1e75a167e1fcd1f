// pod_oproj.cuh -- the o_proj consumer of the attention output (SURVEY.md §8(f) N4,
// second half): Y = O W with O [tokens][K] (this rank's heads, K = Hq/T x d, bf16) and
// W [K][N] (the rows of W_o that belong to those heads, bf16), fp32 accumulate.
//
// Under KV-head-group TP the attention output never needs an all-gather: o_proj is
// row-parallel (Y = sum_r O_r W_r), so each rank multiplies its own slice and the
// partial products are REDUCED.  This kernel does the reduction in its epilogue:
// every output tile is added (red.global.add.v4.f32) straight into the row owner's Y
// through a peer pointer (CUDA IPC mapping over NVLink / NVSwitch), i.e. a GEMM with a
// fused reduce-scatter over token rows: rank t owns rows [t*R, (t+1)*R) of Y and
// receives every rank's contribution to them tile by tile while the GEMMs run.  With
// one rank (or accumulate = 0) it is a plain GEMM storing fp32.
//
// Tiles: 128 x kBN output per CTA, K in steps of 64 through a TMA ring (A = O K-major
// SW128, B = W MN-major SW128 as kBN / 64 column chunks of 8 KB), tcgen05.mma kind::f16
// M128 N kBN K16 issued by one warp, the fp32 accumulator in kBN TMEM columns, 4 epilogue
// warps.  kBN = 256 (N % 256 == 0): one CTA per SM, 4 x 48 KB stages, half the A
// re-reads per output of kBN = 128 (two CTAs per SM, 3 x 32 KB stages, one CTA's epilogue
// overlapping the other's main loop).  The epilogue stages each warp's 32 rows x 32
// columns through a swizzled 4 KB smem tile (the ring is idle once the accumulator is
// complete), so every store / reduction instruction covers 4 whole 128 B row segments
// instead of 32 scattered 16 B pieces.  Included by pod_attn.cu.
#pragma once

namespace oproj {
constexpr int kBM = 128, kBK = 64, kMaxWorld = 8, kThreads = 192;  // warps 0-3 epilogue, 4 TMA, 5 MMA
constexpr uint32_t kABytes = kBM * kBK * 2;                          // 16 KB: [128 rows][64 K], SW128
template <int kBN>
struct Cfg {
    static constexpr int kStages = kBN == 256 ? 4 : 3;
    static constexpr int kCtasPerSm = kBN == 256 ? 1 : 2;
    static constexpr uint32_t kBBytes = kBK * kBN * 2;  // [kBN / 64 chunks][64 K rows][64 N]
    static constexpr uint32_t kStageBytes = kABytes + kBBytes;
    static constexpr uint32_t kOffBars = kStages * kStageBytes;
    static constexpr uint32_t kSmem = kOffBars + 256;
    static_assert(kStages * kStageBytes >= 4 * 4096, "the epilogue's warp tiles fit the ring");
};
}  // namespace oproj

struct OprojParams {
    float* y[oproj::kMaxWorld];  // Y of every rank (peer-mapped), fp32 [rows_per_rank][n]
    int32_t world;
    int32_t accumulate;  // 1: red.add into the row owner's Y; 0: store (world == 1)
    int64_t rows_per_rank;
    int64_t tokens;
    int64_t k;
    int64_t n;
};

__device__ __forceinline__ void red_add_v4(float* addr, float4 v) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

template <int kBN>
__global__ void __launch_bounds__(oproj::kThreads, oproj::Cfg<kBN>::kCtasPerSm)
    oproj_kernel(const __grid_constant__ OprojParams p, const __grid_constant__ CUtensorMap tma,
                 const __grid_constant__ CUtensorMap tmb) {
    using namespace oproj;
    using C = Cfg<kBN>;
    constexpr int kStages = C::kStages;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t bars = sbase + C::kOffBars;
    auto full = [&](int s) { return bars + 8u * s; };
    auto empty = [&](int s) { return bars + 8u * (kStages + s); };
    const uint32_t acc_full = bars + 8u * (2 * kStages);
    volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem + C::kOffBars + 8 * (2 * kStages + 1));
    const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
    const int nk = static_cast<int>(p.k / kBK);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(full(s), 1);
            ptx::mbar_init(empty(s), 1);
        }
        ptx::mbar_init(acc_full, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) {
        ptx::tmem_alloc(ptx::smem_u32(const_cast<uint32_t*>(tmem_slot)), kBN);
        ptx::tmem_relinquish();
    }
    if (warp == 4 && lane == 0) {
        ptx::prefetch_tmap(&tma);
        ptx::prefetch_tmap(&tmb);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 4) {
        // ------------------------------------------------ TMA producer --
        for (int kt = 0; kt < nk; ++kt) {
            const int s = kt % kStages;
            if (kt >= kStages) ptx::mbar_wait(empty(s), ((kt / kStages) - 1) & 1);
            const uint32_t sa = sbase + s * C::kStageBytes, sb = sa + kABytes;
            ptx::mbar_arrive_expect_tx_elect(full(s), C::kStageBytes);
            ptx::tma_load_2d_elect(sa, &tma, full(s), kt * kBK, m0);
#pragma unroll
            for (int j = 0; j < kBN / 64; ++j) ptx::tma_load_2d_elect(sb + j * 8192, &tmb, full(s), n0 + 64 * j, kt * kBK);
        }
    } else if (warp == 5) {
        // -------------------------------------------------- MMA issuer --
        constexpr uint32_t idesc = ptx::idesc_f16(1, kBM, kBN, 1);  // bf16, B MN-major
        for (int kt = 0; kt < nk; ++kt) {
            const int s = kt % kStages;
            ptx::mbar_wait(full(s), (kt / kStages) & 1);
            ptx::tc_fence_after();
            const uint32_t sa = sbase + s * C::kStageBytes, sb = sa + kABytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
                // A: K-major, 16 K = 32 B inside the 128 B swizzle row; B: MN-major, 16 K rows
                // = 2 KB, the 64-wide n-chunks 8 KB apart (LBO)
                ptx::umma_f16_ss_elect(tmem, ptx::sw128_desc(sa + kk * 32, 16, 1024),
                                       ptx::sw128_desc(sb + kk * 2048, 8192, 1024), idesc, (kt | kk) > 0 ? 1u : 0u);
            }
            ptx::umma_commit_elect(empty(s));
        }
        ptx::umma_commit_elect(acc_full);
    } else {
        // --------------------------------------------------- epilogue --
        // (the ring is idle once acc_full fires: every MMA, hence every stage read, is done)
        ptx::mbar_wait(acc_full, 0);
        ptx::tc_fence_after();
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
        const uint32_t tile = sbase + static_cast<uint32_t>(warp) * 4096u;
        // destinations of the 8 rows this lane writes per chunk: rows 4i + lane / 8 of the warp
        const int c4 = lane & 7;
        float* dst[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t row = m0 + warp * 32 + 4 * i + (lane >> 3);
            dst[i] = nullptr;
            if (row < p.tokens) {
                const int owner = p.accumulate ? static_cast<int>(row / p.rows_per_rank) : 0;
                const int64_t lr = p.accumulate ? row % p.rows_per_rank : row;
                dst[i] = p.y[owner] + lr * p.n + n0 + 4 * c4;
            }
        }
#pragma unroll 1
        for (int ch = 0; ch < kBN / 32; ++ch) {
            float v[32];
            ptx::tmem_ld32(lane_base + ch * 32, v);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint32_t a = tile + lane * 128u + ((static_cast<uint32_t>(c) ^ (lane & 7)) << 4);
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v[4 * c]), "f"(v[4 * c + 1]),
                             "f"(v[4 * c + 2]), "f"(v[4 * c + 3])
                             : "memory");
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = 4 * i + (lane >> 3);
                const uint32_t a = tile + r * 128u + ((static_cast<uint32_t>(c4) ^ (r & 7)) << 4);
                float4 q;
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
                             : "r"(a));
                if (dst[i]) {
                    if (p.accumulate)
                        red_add_v4(dst[i] + ch * 32, q);
                    else
                        *reinterpret_cast<float4*>(dst[i] + ch * 32) = q;
                }
            }
            __syncwarp();
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, kBN);
    }
}
