// Microbenchmark: MUFU.EX2 vs FFMA2 vs the FA4-style polynomial exp2, per warp and per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d)
                 : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
                   "l"(*reinterpret_cast<uint64_t*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}

template <int kOp, int kChains>
__global__ void rate(int n, long long* out, float* sink) {
    float v[kChains];
    float2 w[kChains];
    for (int c = 0; c < kChains; ++c) {
        v[c] = -0.001f * (threadIdx.x + c);
        w[c] = make_float2(v[c], v[c] * 0.5f);
    }
    const float2 m = make_float2(0.999f, 0.998f), a = make_float2(1e-7f, 2e-7f);
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (kOp == 0) v[c] = ex2(v[c]) - 1.0f;          // MUFU + FADD
            else if (kOp == 1) w[c] = ffma2(w[c], m, a);     // FFMA2
            else if (kOp == 2) { v[c] = ex2(v[c]); }          // MUFU only (dependent)
            else if (kOp == 3) {                              // F2FP f32x2 -> f16x2 (+ back via PRMT-free add)
                uint32_t h;
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(v[c]), "f"(w[c].x));
                v[c] = __uint_as_float(h);
            } else if (kOp == 4) {                            // F2FP f32x2 -> bf16x2
                uint32_t h;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(v[c]), "f"(w[c].x));
                v[c] = __uint_as_float(h);
            } else if (kOp == 5) {                            // FMNMX3
                asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(v[c]) : "f"(w[c].x), "f"(w[c].y));
            } else if (kOp == 6) {                            // ex2.approx.f16x2
                uint32_t h = __float_as_uint(v[c]);
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h));
                v[c] = __uint_as_float(h);
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int c = 0; c < kChains; ++c) s += v[c] + w[c].x + w[c].y;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int kOp, int kChains>
void run(const char* name, long long* d, float* sink) {
    long long h[148];
    const int n = 2048;
    for (int warps : {1, 4, 8, 16}) {
        rate<kOp, kChains><<<148, warps * 32>>>(n, d, sink);
        rate<kOp, kChains><<<148, warps * 32>>>(n, d, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        const double per = double(mx) / (n * kChains);  // cycles per instruction per warp
        printf("%-12s warps/CTA %2d chains %2d: %6.2f cycles per warp-instr; SM rate %.3f warp-instr/cycle = %.1f lanes/clk\n",
               name, warps, kChains, per, warps / per, 32.0 * warps / per);
    }
}

int main() {
    long long* d; float* sink;
    cudaMalloc(&d, 4096 * 8); cudaMalloc(&sink, 4096 * 1024 * 4);
    run<2, 16>("mufu.ex2", d, sink);
    run<0, 16>("ex2+fadd", d, sink);
    run<1, 16>("ffma2", d, sink);
    run<3, 16>("cvt.f16x2", d, sink);
    run<4, 16>("cvt.bf16x2", d, sink);
    run<5, 16>("max3", d, sink);
    run<6, 16>("ex2.f16x2", d, sink);
    return 0;
}
