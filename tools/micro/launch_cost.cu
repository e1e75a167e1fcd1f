// Microbenchmark: device time of an (almost) empty kernel vs its launch shape --
// dynamic smem (0 / 100 KB / 213 KB), 512 threads, 148 CTAs -- after an L2-flushing memset.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) empty_kernel(int* out) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) sm[0] = blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && sm[0] < 0) out[0] = 1;
}

int main() {
    int* out;
    char* buf;
    cudaMalloc(&out, 4);
    cudaMalloc(&buf, 512 << 20);
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int smem : {16, 100 * 1024, 213 * 1024}) {
        for (int flush : {0, 1}) {
            float best = 1e9, sum = 0;
            for (int it = 0; it < 20; ++it) {
                if (flush) cudaMemsetAsync(buf, it, 512 << 20);
                cudaEventRecord(a);
                empty_kernel<<<148, 512, smem>>>(out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaError_t e = cudaEventElapsedTime(&ms, a, b);
                if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                if (it >= 3) { best = ms < best ? ms : best; sum += ms; }
            }
            printf("smem %6d B, flush %d: empty kernel %.2f us (min %.2f)\n", smem, flush, sum / 17 * 1000, best * 1000);
        }
    }
    return 0;
}
