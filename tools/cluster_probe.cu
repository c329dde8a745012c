// Cluster-barrier latency probe (B200): cycles per iteration of {optional DSMEM store to a neighbour;
// cluster barrier} for 8-CTA clusters of 1024 / 256 threads.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void probe(long long* out, int iters) {
    __shared__ float buf[2048];
    cg::cluster_group cl = cg::this_cluster();
    const int r = cl.block_rank(), n = cl.num_blocks();
    float* peer = cl.map_shared_rank(buf, (r + 1) % n);
    buf[threadIdx.x] = 0.f;
    cl.sync();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE & 1) peer[threadIdx.x] = (float)i;  // one DSMEM store per thread
        if (MODE & 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        else if (MODE & 4) {  // CTA barrier + one thread's fence + relaxed cluster barrier
            __syncthreads();
            if (threadIdx.x == 0) asm volatile("fence.acq_rel.cluster;" ::: "memory");
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
        } else asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
}

template <int MODE>
void run(int threads) {
    long long* d;
    cudaMalloc(&d, 64 * sizeof(long long));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 8;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, probe<MODE>, d, 1000);
    long long h[8];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("mode %d threads %4d: %lld cycles/iter (%s)\n", MODE, threads, h[0], cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    for (int t : {1024, 256}) {
        run<0>(t);  // relaxed barrier only
        run<1>(t);  // DSMEM store + relaxed barrier
        run<2>(t);  // release/acquire barrier
        run<3>(t);  // DSMEM store + release/acquire barrier
        run<5>(t);  // DSMEM store + syncthreads + one-thread fence + relaxed barrier
    }
}
