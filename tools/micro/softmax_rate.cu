// Microbenchmark: the prefill softmax row step for a 64-key tile (tree max, exp2 via
// MUFU, fp32 row sum, fp16 P packing) from registers, per warp and per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
          "l"(*reinterpret_cast<uint64_t*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
    return *reinterpret_cast<float2*>(&d);
}
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

template <int kVariant>
__global__ void softmax_rate(int n, long long* out, uint32_t* sink) {
    float s[64];
    for (int c = 0; c < 64; ++c) s[c] = 0.01f * ((threadIdx.x * 7 + c * 13) % 97);
    const float sl2 = 0.1275f;
    float m_run = -1e30f, l_run = 0.f;
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
        const float tmax = row_max<64>(s);
        const float m_new = fmaxf(m_run, tmax * sl2);
        const bool need = m_new > m_run + 8.f;
        const float m_use = need ? m_new : m_run;
        l_run *= need ? ex2(m_run - m_new) : 1.f;
        m_run = m_use;
        const float2 sl2v = make_float2(sl2, sl2), nm2 = make_float2(-m_use, -m_use);
        float2 ls[4] = {};
        uint32_t hi[32];
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
            const float2 x = ffma2(make_float2(s[c], s[c + 1]), sl2v, nm2);
            const float p0 = ex2(x.x), p1 = ex2(x.y);
            ls[(c / 2) % (kVariant == 1 ? 4 : 2)] = fadd2(ls[(c / 2) % (kVariant == 1 ? 4 : 2)], make_float2(p0, p1));
            __half2 h = __floats2half2_rn(p0, p1);
            hi[c / 2] = *reinterpret_cast<uint32_t*>(&h);
        }
        l_run += ls[0].x + ls[0].y + ls[1].x + ls[1].y + ls[2].x + ls[2].y + ls[3].x + ls[3].y;
#pragma unroll
        for (int c = 0; c < 32; ++c) acc ^= hi[c];
        s[it & 63] += 1e-7f * acc;  // keep the loop from being hoisted
    }
    long long t1 = clock64();
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(l_run);
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
    long long* d; uint32_t* sink;
    cudaMalloc(&d, 4096 * 8); cudaMalloc(&sink, 4096 * 1024 * 4);
    long long h[148];
    const int n = 512;
    for (int v : {0, 1}) for (int warps : {4, 8, 16}) {
        auto k = v == 0 ? softmax_rate<0> : softmax_rate<1>;
        k<<<148, warps * 32>>>(n, d, sink);
        k<<<148, warps * 32>>>(n, d, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("variant %d warps/CTA %2d (%d per SMSP): %.0f cycles per 64-key row step per warp\n", v, warps,
               warps / 4, double(mx) / n);
    }
    return 0;
}
