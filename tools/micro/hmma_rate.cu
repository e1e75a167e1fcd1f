// Microbenchmark: legacy mma.sync.m16n8k16 (bf16, fp32 acc) throughput per warp / per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int kChains>
__global__ void hmma_rate(int n, long long* out, float* sink) {
    float d[kChains][4] = {};
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long t1 = clock64();
    float s = 0;
    for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
    long long* d; float* sink;
    cudaMalloc(&d, 4096 * 8); cudaMalloc(&sink, 4096 * 1024 * 4);
    long long h[4096];
    const int n = 4096;
    for (int warps : {1, 4, 8, 16}) {
        for (int chains : {1, 2, 8}) {
            auto k = chains == 1 ? hmma_rate<1> : chains == 2 ? hmma_rate<2> : hmma_rate<8>;
            k<<<148, warps * 32>>>(n, d, sink);
            k<<<148, warps * 32>>>(n, d, sink);
            cudaDeviceSynchronize();
            cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            const double per = double(mx) / (n * chains);  // cycles per HMMA per warp
            printf("warps/CTA %2d chains %d: %.1f cycles per HMMA per warp; SM rate %.2f HMMA/cycle\n", warps, chains,
                   per, warps / per);
        }
    }
    return 0;
}
