// aw_fwi.cu -- NEXT-3: device kernels of the adjoint-state
// FWI gradient.  The propagations (forward, checkpoint recompute, adjoint in
// reversed time) reuse the stencil kernels of aw_stream.cu / aw_kernels.cu;
// this file holds the three kernels the gradient adds:
//
//   imaging   G += psi^k * D^n,  D^n = fl32(fl32(u^{n+1} - 2u^n) + u^{n-1}),  n = nt-1-k
//   residual  res = fl32(rec - d_obs), the time-reversed residual as the adjoint wavelet, J
//   finalize  grad = fl32(-(double)G / dt^2)
//
// The readings (misfit, adjoint recursion, imaging condition) are DESIGN.md §3
// Q23-Q26; the fp32 sequence is the one of oracle_fwi_gradient (FP32CANON),
// which makes the GPU gradient value-identical to the oracle's.  The paper
// motivates the whole project with inversion
// but defines no gradient itself.
#include "aw_internal.h"

namespace aw {

// Flat float4 walk over the owned planes (rows padded to 32 floats, so plane % 4 == 0).
// HBM-bound: reads psi, u^{n+1}, u^n, u^{n-1}, G and writes G: 24 B per point.
__global__ void fwi_imaging_kernel(const float4* __restrict__ psi, const float4* __restrict__ u1,
                                   const float4* __restrict__ u0, const float4* __restrict__ um1,
                                   float4* __restrict__ G, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 p = psi[i], a = u1[i], b = u0[i], c = um1[i];
        float4 g = G[i];
        // D = fl32(fl32(u1 - 2 u0) + um1): fma(-2, u0, u1) rounds u1 - 2u0 (2u0 exact) once
        g.x = __fmaf_rn(p.x, __fadd_rn(__fmaf_rn(-2.0f, b.x, a.x), c.x), g.x);
        g.y = __fmaf_rn(p.y, __fadd_rn(__fmaf_rn(-2.0f, b.y, a.y), c.y), g.y);
        g.z = __fmaf_rn(p.z, __fadd_rn(__fmaf_rn(-2.0f, b.z, a.z), c.z), g.z);
        g.w = __fmaf_rn(p.w, __fadd_rn(__fmaf_rn(-2.0f, b.w, a.w), c.w), g.w);
        G[i] = g;
    }
}

static int stream_blocks(int64_t n4) {
    int64_t b = (n4 + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;  // 8 resident 256-thread CTAs per SM, grid-stride beyond
    return b < 1 ? 1 : (int)b;
}

cudaError_t launch_fwi_imaging(const Geom& g, const float* psi, const float* u1, const float* u0, const float* um1,
                               float* G, cudaStream_t s) {
    const int64_t off = (int64_t)g.R * g.plane;  // wavefield buffers start at plane -R
    const int64_t n4 = (int64_t)g.nz * g.plane / 4;
    fwi_imaging_kernel<<<stream_blocks(n4), 256, 0, s>>>(
        reinterpret_cast<const float4*>(psi + off), reinterpret_cast<const float4*>(u1 + off),
        reinterpret_cast<const float4*>(u0 + off), reinterpret_cast<const float4*>(um1 + off),
        reinterpret_cast<float4*>(G), n4);
    return cudaGetLastError();
}

// One CTA of 1024 threads: every thread sums a fixed strided subset in fp64, then a fixed-shape
// tree in shared memory -> a deterministic J (the order differs from the oracle's sequential sum,
// so J agrees to rounding, not bit for bit; res and wadj are exact).
__global__ void __launch_bounds__(1024) fwi_residual_kernel(const float* __restrict__ rec,
                                                            const float* __restrict__ dobs, float* __restrict__ res,
                                                            float* __restrict__ wadj, int nt, int nr, double* J) {
    __shared__ double part[1024];
    const int64_t tot = (int64_t)nt * nr;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < tot; i += blockDim.x) {
        const float r = __fsub_rn(rec[i], dobs[i]);
        res[i] = r;
        const int64_t n = i / nr, c = i - n * nr;
        wadj[(int64_t)(nt - 1 - n) * nr + c] = r;  // adjoint step k injects res[nt-1-k]
        acc = __fma_rn((double)r, (double)r, acc);
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) part[threadIdx.x] = __dadd_rn(part[threadIdx.x], part[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *J = __dmul_rn(0.5, part[0]);
}

cudaError_t launch_fwi_residual(const float* rec, const float* dobs, float* res, float* wadj, int nt, int nr,
                                double* J, cudaStream_t s) {
    fwi_residual_kernel<<<1, 1024, 0, s>>>(rec, dobs, res, wadj, nt, nr, J);
    return cudaGetLastError();
}

__global__ void fwi_finalize_kernel(float* __restrict__ G, int64_t n, double dt2) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        G[i] = __double2float_rn(-__ddiv_rn((double)G[i], dt2));
}

cudaError_t launch_fwi_finalize(const Geom& g, float* G, double dt, cudaStream_t s) {
    const int64_t n = (int64_t)g.nz * g.plane;
    fwi_finalize_kernel<<<stream_blocks(n / 4), 256, 0, s>>>(G, n, dt * dt);
    return cudaGetLastError();
}

// NEXT-4 multi-shot: acc = fl32(acc + grad), the per-shot gradients summed in call order
__global__ void fwi_accumulate_kernel(float4* __restrict__ acc, const float4* __restrict__ G, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 a = acc[i];
        const float4 g = G[i];
        a.x = __fadd_rn(a.x, g.x);
        a.y = __fadd_rn(a.y, g.y);
        a.z = __fadd_rn(a.z, g.z);
        a.w = __fadd_rn(a.w, g.w);
        acc[i] = a;
    }
}

cudaError_t launch_fwi_accumulate(const Geom& g, float* acc, const float* G, cudaStream_t s) {
    const int64_t n4 = (int64_t)g.nz * g.plane / 4;
    fwi_accumulate_kernel<<<stream_blocks(n4), 256, 0, s>>>(reinterpret_cast<float4*>(acc),
                                                             reinterpret_cast<const float4*>(G), n4);
    return cudaGetLastError();
}

}  // namespace aw
