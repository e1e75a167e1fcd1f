// Microbenchmark: synchronisation latencies of the prefill pipeline's building blocks
// (one CTA per SM, 148 CTAs; clock64 cycles per iteration, max over CTAs).
//   0  tcgen05.commit -> mbarrier wait, same thread (no MMA in flight)
//   1  mbarrier.arrive -> wait, same thread
//   2  ping-pong: warp 1 commits bar A, warp 2 waits A and arrives B, warp 1 waits B
//   3  one QK tile (8 TS MMAs, N32) + commit + wait: MMA latency of a tile
//   4  one QK + one PV (hi+lo) tile + commit + wait
//   5  issue cost only: clock around the 8 QK MMAs (no wait)
//   6  issue cost only: clock around one commit (no wait)
//   7  12 MMAs (QK + PV) issued back to back x n, one commit at the end: throughput
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2410_18038_b200/csrc/sm100_ptx.cuh"
using namespace pod;

template <int kTest>
__global__ void __launch_bounds__(128, 1) sync_lat(int n, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bars[2];
    const int warp = threadIdx.x / 32;
    const uint32_t sb = ptx::smem_u32(smem);
    const uint32_t ba = ptx::smem_u32(&bars[0]), bb = ptx::smem_u32(&bars[1]);
    if (threadIdx.x == 0) {
        ptx::mbar_init(ba, 1);
        ptx::mbar_init(bb, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) {
        ptx::tmem_alloc(ptx::smem_u32(&tmem_slot), 512);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    constexpr uint32_t idesc_qk = ptx::idesc_f16(1, 128, 32, 0);
    constexpr uint32_t idesc_pv = ptx::idesc_f16(1, 128, 128, 1);
    const uint64_t bk = ptx::sw128_desc(sb, 16, 1024);
    const uint64_t bv = ptx::sw128_desc(sb + 65536, 32 * 128, 1024);
    long long acc = 0;
    if (threadIdx.x == 0) ptx::mbar_arrive(bb);  // bb: phase 0 complete (tests 9, 10)
    __syncthreads();
    if (warp == 1) {
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
            if constexpr (kTest == 0) {
                ptx::umma_commit_elect(ba);
                ptx::mbar_wait(ba, ph);
                ph ^= 1;
            } else if constexpr (kTest == 1) {
                if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(ba);
                ptx::mbar_wait(ba, ph);
                ph ^= 1;
            } else if constexpr (kTest == 2) {
                ptx::umma_commit_elect(ba);
                ptx::mbar_wait(bb, ph);
                ph ^= 1;
            } else if constexpr (kTest == 3 || kTest == 4) {
                ptx::umma_ts_k128_elect<32 * 128>(tmem + 128, tmem, bk, idesc_qk);
                if constexpr (kTest == 4) ptx::umma_pv32_elect<true>(tmem + 256, tmem + 128, bv, idesc_pv, 1u);
                ptx::umma_commit_elect(ba);
                ptx::mbar_wait(ba, ph);
                ph ^= 1;
            } else if constexpr (kTest == 5) {
                const long long a = clock64();
                ptx::umma_ts_k128_elect<32 * 128>(tmem + 128, tmem, bk, idesc_qk);
                acc += clock64() - a;
            } else if constexpr (kTest == 6) {
                const long long a = clock64();
                ptx::umma_commit_elect(ba);
                acc += clock64() - a;
            } else if constexpr (kTest == 7) {
                ptx::umma_ts_k128_elect<32 * 128>(tmem + 128, tmem, bk, idesc_qk);
                ptx::umma_pv32_elect<true>(tmem + 256, tmem + 128, bv, idesc_pv, 1u);
            } else if constexpr (kTest == 8) {  // + one commit per tile, never waited
                ptx::umma_ts_k128_elect<32 * 128>(tmem + 128, tmem, bk, idesc_qk);
                ptx::umma_pv32_elect<true>(tmem + 256, tmem + 128, bv, idesc_pv, 1u);
                ptx::umma_commit_elect(bb);
            } else if constexpr (kTest == 9) {  // + wait on a completed barrier + fence per tile
                ptx::mbar_wait(bb, 0);  // phase 0 of bb completed before the loop
                ptx::tc_fence_after();
                ptx::umma_ts_k128_elect<32 * 128>(tmem + 128, tmem, bk, idesc_qk);
                ptx::umma_pv32_elect<true>(tmem + 256, tmem + 128, bv, idesc_pv, 1u);
            } else if constexpr (kTest == 10) {  // the kernel's per-tile sync pattern, no real waiting
                ptx::mbar_wait(bb, 0);
                ptx::tc_fence_after();
                ptx::umma_pv32_elect<true>(tmem + 256, tmem + 128, bv, idesc_pv, 1u);
                ptx::mbar_wait(bb, 0);
                ptx::tc_fence_after();
                ptx::umma_ts_k128_elect<32 * 128>(tmem + 128, tmem, bk, idesc_qk);
                ptx::umma_commit_elect(ba);
                ptx::mbar_wait(bb, 0);
                ptx::tc_fence_after();
                ptx::umma_pv32_elect<true>(tmem + 384, tmem + 192, bv, idesc_pv, 1u);
                ptx::umma_ts_k128_elect<32 * 128>(tmem + 192, tmem + 64, bk, idesc_qk);
                ptx::umma_commit_elect(ba);
                ptx::umma_commit_elect(ba);
            } else if constexpr (kTest == 11) {  // same MMAs as 10, no sync at all
                ptx::umma_pv32_elect<true>(tmem + 256, tmem + 128, bv, idesc_pv, 1u);
                ptx::umma_ts_k128_elect<32 * 128>(tmem + 128, tmem, bk, idesc_qk);
                ptx::umma_pv32_elect<true>(tmem + 384, tmem + 192, bv, idesc_pv, 1u);
                ptx::umma_ts_k128_elect<32 * 128>(tmem + 192, tmem + 64, bk, idesc_qk);
            }
        }
        if constexpr (kTest >= 5 && kTest != 8 && kTest != 10) {
            ptx::umma_commit_elect(ba);
            ptx::mbar_wait(ba, 0);
        }
        const long long t1 = clock64();  // tests 8, 10: issue-side time (queue tail < 1 us of 1000 tiles)
        if constexpr (kTest == 8 || kTest == 10) __nanosleep(100000);  // let the un-waited commits land
        if (threadIdx.x == 32) out[blockIdx.x] = (kTest == 5 || kTest == 6) ? acc : t1 - t0;
    } else if (warp == 2 && kTest == 2) {
        uint32_t ph = 0;
        for (int i = 0; i < n; ++i) {
            ptx::mbar_wait(ba, ph);
            ph ^= 1;
            if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(bb);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

// Replica of the pair engine's single-issuer loop (pod_sm.cuh prefill_item_sm) with the
// softmax replaced by one responder warp per block (wait S, arrive P), no TMA:
// cycles per tile-pair.  order as the kernel: PV_A, QK_A(t+2), PV_B, QK_B(t+2).
template <int kNoMma, int kResp, int kProd>
__global__ void __launch_bounds__(512, 1) pipe_replica(int n, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bars[16];  // s[X][b] 2X+b, p[X][b] 4+2X+b, kfull 8+st, kvempty 12+st
    const int warp = threadIdx.x / 32;
    const uint32_t sb = ptx::smem_u32(smem);
    auto bar = [&](int i) { return ptx::smem_u32(&bars[i]); };
    if (threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) ptx::mbar_init(bar(i), (i >= 4 && i < 8) ? kResp : 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) {
        ptx::tmem_alloc(ptx::smem_u32(&tmem_slot), 512);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    constexpr uint32_t idesc_qk = ptx::idesc_f16(1, 128, 32, 0);
    constexpr uint32_t idesc_pv = ptx::idesc_f16(1, 128, 128, 1);
    const uint64_t bk = ptx::sw128_desc(sb, 16, 1024);
    const uint64_t bv = ptx::sw128_desc(sb + 65536, 32 * 128, 1024);
    const uint32_t kQ[2] = {0, 64}, kS[2] = {128, 192}, kO[2] = {256, 384};
    if (warp == 1) {
        const long long t0 = clock64();
        for (int j = 0; j < 2; ++j)
            for (int X = 0; X < 2; ++X) {
                if (kProd && X == 0) ptx::mbar_wait(bar(8 + j), 0);
                if (!kNoMma) ptx::umma_ts_k128_elect<32 * 128>(tmem + kS[X] + 32 * j, tmem + kQ[X], bk, idesc_qk);
                ptx::umma_commit_elect(bar(2 * X + j));
            }
        for (int t = 0; t < n; ++t) {
            const int b = t & 1;
            const bool more = t + 2 < n;
            for (int X = 0; X < 2; ++X) {
                ptx::mbar_wait(bar(4 + 2 * X + b), (t >> 1) & 1);
                ptx::tc_fence_after();
                if (!kNoMma) ptx::umma_pv32_elect<true>(tmem + kO[X], tmem + kS[X] + 32 * b, bv, idesc_pv, 1u);
                if (more) {
                    if (kProd && X == 0) {
                        const int g2 = t + 2;
                        ptx::mbar_wait(bar(8 + (g2 & 3)), (g2 >> 2) & 1);
                        ptx::tc_fence_after();
                    }
                    if (!kNoMma) ptx::umma_ts_k128_elect<32 * 128>(tmem + kS[X] + 32 * b, tmem + kQ[X], bk, idesc_qk);
                    ptx::umma_commit_elect(bar(2 * X + b));
                }
            }
            if (kProd) ptx::umma_commit_elect(bar(12 + (t & 3)));  // stage of tile t free
        }
        ptx::umma_commit_elect(bar(2));  // spare: wait for the tail via a last commit on s_B[0]...
        const long long t1 = clock64();
        if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
    } else if (kProd && warp == 12) {  // producer: stage ring of 4, arrive instead of TMA
        for (int g = 0; g < n; ++g) {
            if (g >= 4) ptx::mbar_wait_relaxed<>(bar(12 + (g & 3)), ((g >> 2) - 1) & 1);
            if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(bar(8 + (g & 3)));
        }
    } else if (warp >= 2 && warp < 2 + 2 * kResp) {
        const int X = (warp - 2) / kResp;
        for (int t = 0; t < n; ++t) {
            const int b = t & 1;
            ptx::mbar_wait(bar(2 * X + b), (t >> 1) & 1);
            ptx::tc_fence_after();
            __syncwarp();
            if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(bar(4 + 2 * X + b));
        }
    }
    __nanosleep(20000);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 1024 * 8);
    long long h[1024];
    const char* names[12] = {"commit -> wait (same thread)", "arrive -> wait (same thread)",
                            "ping-pong commit/wait/arrive/wait", "QK tile (8 MMA N32) + commit + wait",
                            "QK + PV(hi+lo) tile + commit + wait", "issue of 8 QK MMAs (clock around)",
                            "issue of one commit (clock around)", "QK+PV tiles back to back (throughput)",
                            "QK+PV + commit per tile (no wait)", "wait(done)+fence + QK+PV per tile",
                            "kernel pattern, 2 blocks (waits satisfied)", "same MMAs, 2 blocks, no sync"};
    for (int test = 0; test < 12; ++test) {
        auto k = test == 0 ? sync_lat<0> : test == 1 ? sync_lat<1> : test == 2 ? sync_lat<2> : test == 3 ? sync_lat<3>
               : test == 4 ? sync_lat<4> : test == 5 ? sync_lat<5> : test == 6 ? sync_lat<6> : test == 7 ? sync_lat<7>
               : test == 8 ? sync_lat<8> : test == 9 ? sync_lat<9> : test == 10 ? sync_lat<10> : sync_lat<11>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        const int n = 1000;
        for (int rep = 0; rep < 2; ++rep) k<<<148, 128, 200 * 1024>>>(n, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("err %s\n", cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%-45s %.1f cycles/iter\n", names[test], double(mx) / n);
    }
    {
      for (int v = 0; v < 6; ++v) {
        auto k = v == 0 ? pipe_replica<0, 1, 0> : v == 1 ? pipe_replica<1, 1, 0> : v == 2 ? pipe_replica<0, 4, 0>
               : v == 3 ? pipe_replica<0, 4, 1> : v == 4 ? pipe_replica<1, 4, 1> : pipe_replica<0, 1, 1>;
        const char* vn[6] = {"replica: MMAs, 1 responder/block", "replica: no MMAs, 1 responder/block",
                             "replica: MMAs, 4 responders/block", "replica: MMAs, 4 resp, producer ring",
                             "replica: no MMAs, 4 resp, producer ring", "replica: MMAs, 1 resp, producer ring"};
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        const int n = 1000;
        for (int rep = 0; rep < 2; ++rep) k<<<148, 512, 200 * 1024>>>(n, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("err %s\n", cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%-45s %.1f cycles/tile-pair\n", vn[v], double(mx) / n);
      }
    }
    return 0;
}
