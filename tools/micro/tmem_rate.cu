// Microbenchmark: tcgen05.ld / tcgen05.st throughput (4 warps, one per TMEM lane
// quadrant), alone and while warp 4 issues TS-MMAs (M128 N128 K16, A from TMEM).
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2410_18038_b200/csrc/sm100_ptx.cuh"
using namespace pod;

template <int kMode>  // 0: ld only, 1: st only, 2: mma only, 3: ld + mma, 4: ld+st + mma
__global__ void __launch_bounds__(192, 1) tmem_rate(int n, long long* out, float* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); ptx::fence_mbar_init(); }
    if (warp == 0) { ptx::tmem_alloc(ptx::smem_u32(&tmem_slot), 512); ptx::tmem_relinquish(); }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    long long t0 = clock64();
    float acc = 0.f;
    if (warp < 4 && kMode != 2) {
        const uint32_t base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
        for (int i = 0; i < n; ++i) {
            float v[32];
            if (kMode == 0 || kMode == 3 || kMode == 4) {
                ptx::tmem_ld32(base + (i & 3) * 32, v);
                ptx::tmem_wait_ld();
                acc += v[0] + v[31];
            }
            if (kMode == 1 || kMode == 4) {
                for (int c = 0; c < 32; ++c) v[c] = acc + c;
                ptx::tmem_st32(base + 128 + (i & 3) * 32, v);
                ptx::tmem_wait_st();
            }
        }
    }
    if (warp == 4 && kMode >= 2) {
        constexpr uint32_t idesc = ptx::idesc_f16(1, 128, 128, 1);
        const uint64_t b = ptx::sw128_desc(ptx::smem_u32(smem), 16, 1024);
        for (int i = 0; i < n / 4; ++i)
            ptx::umma_f16_ts_elect(tmem + 256, tmem + 128 + (i & 7) * 8, b + ((i & 7) * 2), idesc, 1u);
        ptx::umma_commit_elect(ptx::smem_u32(&bar));
        ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    }
    long long t1 = clock64();
    sink[blockIdx.x * 192 + threadIdx.x] = acc;
    if (lane == 0) out[blockIdx.x * 8 + warp] = t1 - t0;
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
    long long* d; float* sink;
    cudaMalloc(&d, 148 * 8 * 8); cudaMalloc(&sink, 148 * 192 * 4);
    long long h[148 * 8];
    const int n = 4096;
    const char* names[5] = {"ld x32 (4 KB/warp-instr) only", "st x32 only", "TS-MMA only (n/4 MMAs)",
                            "ld + TS-MMA", "ld + st + TS-MMA"};
    for (int mode = 0; mode < 5; ++mode) {
        auto k = mode == 0 ? tmem_rate<0> : mode == 1 ? tmem_rate<1> : mode == 2 ? tmem_rate<2> : mode == 3 ? tmem_rate<3> : tmem_rate<4>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        k<<<148, 192, 64 * 1024>>>(n, d, sink);
        k<<<148, 192, 64 * 1024>>>(n, d, sink);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        long long ldw = 0, mw = 0;
        for (int b = 0; b < 148; ++b) { for (int w = 0; w < 4; ++w) ldw = h[b * 8 + w] > ldw ? h[b * 8 + w] : ldw; mw = h[b * 8 + 4] > mw ? h[b * 8 + 4] : mw; }
        printf("%-32s: softmax-warps %.1f cyc/iter (%.0f B/cyc/SM per op kind), mma warp %.1f cyc/MMA\n", names[mode],
               double(ldw) / n, 4.0 * 4096 / (double(ldw) / n), double(mw) / (n / 4));
    }
    return 0;
}
