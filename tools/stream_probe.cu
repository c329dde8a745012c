// stream_probe.cu -- developer probe: achievable HBM bandwidth on this B200 for the
// stencil's stream mix (3 reads + 1 in-place write per point, fp32), elementwise
// and float4-vectorised, no stencil arithmetic.  The stencil kernel's roofline
// fraction is judged against the measured copy peak; this probe says how much
// of that a 3:1 read/write mix can reach.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/stream_probe.cu -o /tmp/stream_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mix3r1w(const float4* __restrict__ a, const float4* __restrict__ b, float4* c, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 x = a[i], y = b[i], z = c[i];
        z.x = fmaf(x.x, y.x, z.x);
        z.y = fmaf(x.y, y.y, z.y);
        z.z = fmaf(x.z, y.z, z.z);
        z.w = fmaf(x.w, y.w, z.w);
        c[i] = z;
    }
}
__global__ void copy(const float4* __restrict__ a, float4* __restrict__ c, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) c[i] = a[i];
}

int main() {
    const size_t N = 512ull * 512 * 512;  // points (C3)
    float *a, *b, *c, *d;
    cudaMalloc(&a, N * 4);
    cudaMalloc(&b, N * 4);
    cudaMalloc(&c, N * 4);
    cudaMalloc(&d, N * 4);
    cudaMemset(a, 0, N * 4);
    cudaMemset(b, 0, N * 4);
    cudaMemset(c, 0, N * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            for (int it = 0; it < 20; ++it) mix3r1w<<<blocks, 256>>>((float4*)a, (float4*)b, (float4*)c, N / 4);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= 20;
            printf("mix 3r+1w  blocks=%5d: %.3f ms  %.0f GB/s (16 B/pt)\n", blocks, ms, 16.0 * N / ms / 1e6);
            cudaEventRecord(e0);
            for (int it = 0; it < 20; ++it) copy<<<blocks, 256>>>((float4*)a, (float4*)d, N / 4);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= 20;
            printf("copy       blocks=%5d: %.3f ms  %.0f GB/s (8 B/pt)\n", blocks, ms, 8.0 * N / ms / 1e6);
        }
    }
    return 0;
}
