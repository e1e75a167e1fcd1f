// Microbenchmark: the pair engine's per-tile MMA sequence issued back to back by
// one thread (no waits): PV_A (hi/lo x 2 K-steps, N=128), QK_A (8 x N=32),
// PV_B, QK_B -- and variants -- cycles per tile.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2410_18038_b200/csrc/sm100_ptx.cuh"
using namespace pod;

template <int kVariant, bool kContend>
__global__ void __launch_bounds__(384, 1) pair_mma(int n, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32;
    const uint32_t sb = ptx::smem_u32(smem);
    if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); ptx::fence_mbar_init(); }
    if (warp == 0) { ptx::tmem_alloc(ptx::smem_u32(&tmem_slot), 512); ptx::tmem_relinquish(); }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (kContend && warp >= 4) {  // 8 'softmax' warps: tcgen05.ld 32 cols + st 16 cols per iteration
        const int q = warp & 3;
        const uint32_t base = (static_cast<uint32_t>(q * 32) << 16);
        float acc = 0.f;
        for (int i = 0; i < n * 2; ++i) {
            float v[32];
            ptx::tmem_ld32(base + 128 + 32 * (i & 3), v);
            ptx::tmem_wait_ld();
            uint32_t h[16];
            for (int c = 0; c < 16; ++c) h[c] = __float_as_uint(v[2 * c] + acc);
            ptx::tmem_st16(base + 128 + 64 * (warp >= 8) + 32 * (i & 1), h);
            ptx::tmem_wait_st();
            acc += v[0];
        }
        if (acc == 12345.f) out[0] = 1;
    }
    if (warp == 1) {
        constexpr uint32_t id_qk = ptx::idesc_f16(1, 128, 32, 0);
        constexpr uint32_t id_qk64 = ptx::idesc_f16(1, 128, 64, 0);
        constexpr uint32_t id_pv = ptx::idesc_f16(1, 128, 128, 1);
        const uint64_t bk = ptx::sw128_desc(sb, 16, 1024), bv = ptx::sw128_desc(sb + 65536, 4096, 1024);
        long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
#pragma unroll
            for (int X = 0; X < 2; ++X) {
                const uint32_t o = 256 + 128 * X, sx = 128 + 64 * X + 32 * (i & 1), q = 64 * X;
                if (kVariant == 0) {  // 32-key tile, batched asm
                    ptx::umma_pv32_elect<true>(o, sx, bv, id_pv, 1u);
                    ptx::umma_ts_k128_elect<4096>(sx, q, bk, id_qk);
                } else if (kVariant == 1) {  // 32-key tile, PV only
                    ptx::umma_pv32_elect<true>(o, sx, bv, id_pv, 1u);
                } else if (kVariant == 2) {  // 32-key tile, QK only
                    ptx::umma_ts_k128_elect<4096>(sx, q, bk, id_qk);
                } else {  // 64-key tile equivalent: QK N=64 x 8, PV 8 MMAs
                    ptx::umma_pv32_elect<true>(o, sx, bv, id_pv, 1u);
                    ptx::umma_pv32_elect<true>(o, sx, bv, id_pv, 1u);
                    ptx::umma_ts_k128_elect<4096>(sx, q, bk, id_qk64);
                }
            }
        }
        ptx::umma_commit_elect(ptx::smem_u32(&bar));
        ptx::mbar_wait(ptx::smem_u32(&bar), 0);
        long long t1 = clock64();
        if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tmem_slot, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    long long h[148];
    const char* names[4] = {"32-key tile: PV(hi/lo,2 ksteps)+QK(N32) x2 blocks", "PV only", "QK only",
                            "64-key equivalent: 2xPV32 + QK N64, x2 blocks"};
    const double nominal[4] = {2 * (256 + 128), 2 * 256, 2 * 128, 2 * (512 + 256)};
    for (int v = 0; v < 4; ++v) {
      for (int contend = 0; contend < 2; ++contend) {
        auto k = contend ? (v == 0 ? pair_mma<0, true> : v == 1 ? pair_mma<1, true> : v == 2 ? pair_mma<2, true> : pair_mma<3, true>)
                         : (v == 0 ? pair_mma<0, false> : v == 1 ? pair_mma<1, false> : v == 2 ? pair_mma<2, false> : pair_mma<3, false>);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
        k<<<148, 384, 128 * 1024>>>(1024, d);
        k<<<148, 384, 128 * 1024>>>(1024, d);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%-55s %s: %.0f cycles per tile (nominal %.0f)\n", names[v], contend ? "+TMEM ld/st" : "alone      ",
               double(mx) / 1024, nominal[v]);
      }
    }
    return 0;
}
