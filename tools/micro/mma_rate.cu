// Microbenchmark: tcgen05.mma issue throughput for the prefill shapes.
// One CTA per SM; thread 0 issues `n` MMAs of one shape back to back (operands are
// whatever is in smem/TMEM), commits, waits, and records clock64 deltas.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2410_18038_b200/csrc/sm100_ptx.cuh"
using namespace pod;

template <int kShape>
__global__ void __launch_bounds__(128, 1) mma_rate(int n, long long* out) {
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
    const uint32_t tmem = tmem_slot;
    long long t0 = 0, t1 = 0;
    if (warp == 1) {
        // shapes: 0 SS M128 N64 K16; 1 TS M128 N128 K16 (A tmem); 2 SS M128 N128 K16; 3 TS M128 N64 K16
        constexpr uint32_t N = kShape == 6 ? 32 : kShape == 7 ? 16 : (kShape == 1 || kShape == 2 || kShape >= 4) ? 128 : 64;
        constexpr uint32_t idesc = ptx::idesc_f16(1, 128, N, (kShape == 1 || kShape == 4 || kShape == 5) ? 1 : 0);
        const uint64_t a = ptx::sw128_desc(sb, 16, 1024);
        const uint64_t b = ptx::sw128_desc(sb + 65536, 16, 1024);
        __syncwarp();
        t0 = clock64();
        for (int i = 0; i < n; ++i) {
            if constexpr (kShape == 0 || kShape == 2)
                ptx::umma_f16_ss_elect(tmem, a + ((i & 7) * 2), b + ((i & 7) * 2), idesc, 1u);
            else if constexpr (kShape == 4) {  // operands through vector registers (R2UR per MMA)
                const uint32_t tm = *reinterpret_cast<volatile uint32_t*>(&tmem_slot);
                ptx::umma_f16_ts_elect(tm + 256, tm + (i & 7) * 8, b + ((i & 7) * 2), idesc, 1u);
            } else if constexpr (kShape == 6 || kShape == 7) {  // TS N32 / N16 (vector-reg tmem)
                const uint32_t tm = *reinterpret_cast<volatile uint32_t*>(&tmem_slot);
                ptx::umma_f16_ts_elect(tm + 256, tm + (i & 7) * 8, b + ((i & 7) * 2), idesc, 1u);
            } else if constexpr (kShape == 5) {  // lane-0 issue (divergent branch, no elect)
                const uint32_t tm = *reinterpret_cast<volatile uint32_t*>(&tmem_slot);
                if ((threadIdx.x & 31) == 0) ptx::umma_f16_ts(tm + 256, tm + (i & 7) * 8, b + ((i & 7) * 2), idesc, 1u);
            } else
                ptx::umma_f16_ts_elect(tmem + 256, tmem + (i & 7) * 8, b + ((i & 7) * 2), idesc, 1u);
        }
        ptx::umma_commit_elect(ptx::smem_u32(&bar));
        ptx::mbar_wait(ptx::smem_u32(&bar), 0);
        t1 = clock64();
        if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 1024 * 8);
    long long h[1024];
    const char* names[8] = {"SS M128 N64 K16", "TS M128 N128 K16 (A=TMEM, B MN-major)", "SS M128 N128 K16",
                            "TS M128 N64 K16 (A=TMEM)", "TS N128, tmem via vector reg + elect", "TS N128, lane-0 branch", "TS N32 (vector tmem, elect)", "TS N16 (vector tmem, elect)"};
    for (int shape = 0; shape < 8; ++shape) {
        for (int grid : {1, 148}) {
            for (int n : {64, 1024}) {
                auto k = shape == 0 ? mma_rate<0> : shape == 1 ? mma_rate<1> : shape == 2 ? mma_rate<2> : shape == 3 ? mma_rate<3> : shape == 4 ? mma_rate<4> : shape == 5 ? mma_rate<5> : shape == 6 ? mma_rate<6> : mma_rate<7>;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                k<<<grid, 128, 200 * 1024>>>(n, d);
                k<<<grid, 128, 200 * 1024>>>(n, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
                long long mx = 0;
                for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("%-40s grid %3d n %5d: %.1f cycles/mma\n", names[shape], grid, n, double(mx) / n);
            }
        }
    }
    return 0;
}
