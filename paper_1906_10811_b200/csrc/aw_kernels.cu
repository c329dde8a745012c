// aw_kernels.cu -- reference-grade device kernels of libaw (sm_100a).
//
// Every floating-point operation of the update is written with an explicit
// rounding intrinsic (__fmul_rn/__fadd_rn/__fsub_rn/__fmaf_rn) so that nvcc can
// neither contract nor reorder it: the per-point sequence is the canonical one
// of SURVEY.md §8(c).6 (restated in DESIGN.md §2), which makes the GPU
// value-identical to the fp32 oracle rather than merely close.
//
//   L   = C0 * u_p                                        (PAPER.md:417 centre term)
//   for d = ndim-1 .. 0, j = 1..R:  L = fma(C[d][j], u_{p-j e_d} + u_{p+j e_d}, L)
//   t   = 2 u_p - u^{n-1}_p
//   w   = fma(b_p, L, t)                                  (b = dt^2/m, division hoisted,
//   u^{n+1}_p = fma(a_p, w, (1 - a_p) * u^{n-1}_p)         PAPER.md:788-826; a = m/(m+eta dt/2))
#include <algorithm>

#include "aw_internal.h"

namespace aw {

// ---------------------------------------------------------------------------
// Coefficient precompute, fp64 then one rounding to fp32.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void coeff1(float m, float eta, double dt, double dt2, float& b, float& a) {
    const double mm = (double)m;
    const double den = __dadd_rn(mm, __dmul_rn(__dmul_rn((double)eta, dt), 0.5));
    b = __double2float_rn(__ddiv_rn(dt2, mm));
    a = __double2float_rn(__ddiv_rn(mm, den));
}

// n is a multiple of 4 (rows are padded to 32 floats); float4 streams, 4 points per thread-iteration.
__global__ void coeffs_kernel(const float4* __restrict__ m, const float4* __restrict__ eta, float4* __restrict__ b,
                              float4* __restrict__ a, int64_t n4, double dt) {
    const double dt2 = __dmul_rn(dt, dt);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 mm = m[i];
        const float4 e = eta ? eta[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 bb, aa;
        coeff1(mm.x, e.x, dt, dt2, bb.x, aa.x);
        coeff1(mm.y, e.y, dt, dt2, bb.y, aa.y);
        coeff1(mm.z, e.z, dt, dt2, bb.z, aa.z);
        coeff1(mm.w, e.w, dt, dt2, bb.w, aa.w);
        b[i] = bb;
        if (a) a[i] = aa;
    }
}

cudaError_t launch_coeffs(const float* m, const float* eta, float* b, float* a, int64_t n, double dt,
                          cudaStream_t s) {
    const int64_t n4 = n / 4;
    int blocks = (int)((n4 + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    coeffs_kernel<<<blocks, 256, 0, s>>>((const float4*)m, (const float4*)eta, (float4*)b, (float4*)a, n4, dt);
    return cudaGetLastError();
}

// Model validation: m > 0 finite, eta >= 0 finite at every owned point.
// flat float4 walk over the padded arrays; x = element index mod pitch (pitch % 4 == 0)
__global__ void validate_kernel(const float4* __restrict__ m, const float4* __restrict__ eta, int64_t n4, int nx,
                                int64_t pitch, unsigned* flag, unsigned epoch) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)((4 * i) % pitch);
        const float4 v = m[i];
        const float4 e = eta ? eta[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float mv[4] = {v.x, v.y, v.z, v.w}, ev[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (x + c < nx) bad |= !(mv[c] > 0.0f) || !isfinite(mv[c]) || !(ev[c] >= 0.0f) || !isfinite(ev[c]);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMax(flag, epoch);
}

cudaError_t launch_validate_model(const float* m, const float* eta, const Geom& g, unsigned* flag, unsigned epoch,
                                  cudaStream_t s) {
    const int64_t n4 = (int64_t)g.nz * g.plane / 4;
    int blocks = (int)((n4 + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    validate_kernel<<<blocks, 256, 0, s>>>((const float4*)m, (const float4*)eta, n4, g.nx, g.pitch, flag, epoch);
    return cudaGetLastError();
}

// Copy m (and eta) from dense C-order device arrays into the padded model layout (pitch-padded rows,
// padding 0) and validate them in the same pass (aw_set_model with device inputs: one launch instead
// of memsets + 2D copies + the validation kernel).  x = blockIdx.x * 256 + threadIdx.x covers the
// padded row, blockIdx.y strides over the rows: coalesced, no integer division.
__global__ void __launch_bounds__(256) stage_model_kernel(const float* __restrict__ ms, const float* __restrict__ es,
                                                          float* __restrict__ md, float* __restrict__ ed,
                                                          int64_t rows, int nx, int64_t pitch, unsigned* flag,
                                                          unsigned epoch) {
    bool bad = false;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < pitch) {
#pragma unroll 4
        for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
            float mv = 0.0f, ev = 0.0f;
            if (x < nx) {
                mv = ms[row * nx + x];
                if (es) ev = es[row * nx + x];
                bad |= !(mv > 0.0f) || !isfinite(mv) || !(ev >= 0.0f) || !isfinite(ev);
            }
            md[row * pitch + x] = mv;
            if (ed) ed[row * pitch + x] = ev;
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMax(flag, epoch);
}

cudaError_t launch_stage_model(const float* m_src, const float* eta_src, float* m_dst, float* eta_dst, const Geom& g,
                               unsigned* bad, unsigned epoch, cudaStream_t s) {
    const int64_t rows = (int64_t)g.nz * g.ny;
    const int bx = (int)((g.pitch + 255) / 256);
    int by = (int)std::min<int64_t>(rows, std::max<int64_t>(1, 148 * 16 / bx));
    if (by < 1) by = 1;
    stage_model_kernel<<<dim3(bx, by), 256, 0, s>>>(m_src, eta_src, m_dst, eta_dst, rows, g.nx, g.pitch, bad, epoch);
    return cudaGetLastError();
}

// Source scales s = fl32((w64 * dt^2) / (m_c + (eta_c * dt) * 0.5))
__global__ void source_scales_kernel(const float* __restrict__ m, const float* __restrict__ eta,
                                     const int64_t* __restrict__ moff, const double* __restrict__ w64,
                                     float* __restrict__ s_out, int nent, double dt) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nent) return;
    int64_t o = moff[i];
    double mm = (double)m[o];
    double e = eta ? (double)eta[o] : 0.0;
    double den = __dadd_rn(mm, __dmul_rn(__dmul_rn(e, dt), 0.5));
    double dt2 = __dmul_rn(dt, dt);
    s_out[i] = __double2float_rn(__ddiv_rn(__dmul_rn(w64[i], dt2), den));
}

cudaError_t launch_source_scales(const float* m, const float* eta, const int64_t* moff, const double* w64,
                                 float* s_out, int nent, double dt, cudaStream_t s) {
    if (nent <= 0) return cudaSuccess;
    source_scales_kernel<<<(nent + 127) / 128, 128, 0, s>>>(m, eta, moff, w64, s_out, nent, dt);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// v1 stencil: one thread per point, global loads, canonical op order.
// Zero ghosts: x/y by bounds checks, z by the (zeroed or exchanged) halo planes.
// In a team the first/last R owned planes are also stored into the
// neighbours' halo planes (peer memory) -- the fused exchange.
// ---------------------------------------------------------------------------
template <int NDIM, int R>
__global__ void __launch_bounds__(256) stencil_v1_kernel(Geom g, Coefs c, const float* __restrict__ ucur,
                                                         const float* uprev, float* unext, const float* __restrict__ b,
                                                         const float* __restrict__ a, float* __restrict__ lo,
                                                         int64_t lo_off, float* __restrict__ hi, int64_t hi_off) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = (NDIM == 3) ? (int)(blockIdx.y * blockDim.y + threadIdx.y) : 0;
    const int z = (NDIM == 3) ? (int)blockIdx.z : (int)(blockIdx.y * blockDim.y + threadIdx.y);
    if (x >= g.nx || y >= g.ny || z >= g.nz) return;
    const int64_t o = (int64_t)z * g.plane + (int64_t)y * g.pitch + x;  // model index
    const int64_t ou = o + (int64_t)R * g.plane;                          // wavefield index
    const float* p = ucur + ou;
    const float uc = p[0];
    float L = __fmul_rn(c.C0, uc);
    // axis ndim-1 (x, contiguous)
#pragma unroll
    for (int j = 1; j <= R; ++j) {
        float lo_v = (x - j >= 0) ? p[-j] : 0.0f;
        float hi_v = (x + j < g.nx) ? p[j] : 0.0f;
        L = __fmaf_rn(c.C[NDIM - 1][j], __fadd_rn(lo_v, hi_v), L);
    }
    if (NDIM == 3) {
        // axis 1 (y)
#pragma unroll
        for (int j = 1; j <= R; ++j) {
            float lo_v = (y - j >= 0) ? p[-(int64_t)j * g.pitch] : 0.0f;
            float hi_v = (y + j < g.ny) ? p[(int64_t)j * g.pitch] : 0.0f;
            L = __fmaf_rn(c.C[1][j], __fadd_rn(lo_v, hi_v), L);
        }
    }
    // axis 0 (z): halo planes
#pragma unroll
    for (int j = 1; j <= R; ++j)
        L = __fmaf_rn(c.C[0][j], __fadd_rn(p[-(int64_t)j * g.plane], p[(int64_t)j * g.plane]), L);
    const float um = uprev[ou];  // u^{n-1}: the output buffer itself (in place) or a history level
    const float t = __fsub_rn(__fmul_rn(2.0f, uc), um);
    const float w = __fmaf_rn(b[o], L, t);
    const float aa = a ? a[o] : 1.0f;
    const float r = __fmul_rn(__fsub_rn(1.0f, aa), um);
    const float un = __fmaf_rn(aa, w, r);
    unext[ou] = un;
    if (lo && z < R) lo[lo_off + o] = un;
    if (hi && z >= g.nz - R) hi[hi_off + o - (int64_t)(g.nz - R) * g.plane] = un;
}

template <int NDIM>
static cudaError_t launch_v1_ndim(const Geom& g, const Coefs& c, const float* ucur, const float* uprev, float* unext,
                                  const float* b,
                                  const float* a, float* lo, int64_t lo_off, float* hi, int64_t hi_off,
                                  cudaStream_t s) {
    dim3 block, grid;
    if (NDIM == 3) {
        block = dim3(64, 4, 1);
        grid = dim3((g.nx + 63) / 64, (g.ny + 3) / 4, g.nz);
    } else {
        block = dim3(128, 2, 1);
        grid = dim3((g.nx + 127) / 128, (g.nz + 1) / 2, 1);
    }
    switch (g.R) {
#define AW_CASE(RR) \
    case RR: stencil_v1_kernel<NDIM, RR><<<grid, block, 0, s>>>(g, c, ucur, uprev, unext, b, a, lo, lo_off, hi, hi_off); break;
        AW_CASE(1) AW_CASE(2) AW_CASE(3) AW_CASE(4) AW_CASE(5) AW_CASE(6) AW_CASE(7) AW_CASE(8)
#undef AW_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_stencil_v1(const Geom& g, const Coefs& c, const float* ucur, const float* uprev, float* unext,
                              const float* b, const float* a, const Halo& halo, int parity_next, cudaStream_t s) {
    float* lo = halo.lo[parity_next];
    float* hi = halo.hi[parity_next];
    if (g.ndim == 3) return launch_v1_ndim<3>(g, c, ucur, uprev, unext, b, a, lo, halo.lo_off, hi, halo.hi_off, s);
    return launch_v1_ndim<2>(g, c, ucur, uprev, unext, b, a, lo, halo.lo_off, hi, halo.hi_off, s);
}

// ---------------------------------------------------------------------------
// Per-step sparse work: receivers read u^n, injection adds into
// u^{n+1} in CSR order (corner ascending, then source ascending; Q11).
// Step index n = *d_base + i (d_base advanced once per graph / run chunk).
// ---------------------------------------------------------------------------
__global__ void sparse_step_kernel(Geom g, Sparse sp, const float* __restrict__ ucur, float* __restrict__ unext,
                                   const int64_t* __restrict__ d_base, int i, float* __restrict__ lo,
                                   int64_t lo_off, float* __restrict__ hi, int64_t hi_off) {
    const int64_t n = *d_base + i;
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < sp.nrl) {
        float acc = 0.0f;
        for (int beta = 0; beta < sp.nc; ++beta) {
            int64_t off = sp.rec_off[(int64_t)t * sp.nc + beta];
            if (off < 0) continue;
            acc = __fmaf_rn(sp.rec_w[(int64_t)t * sp.nc + beta], ucur[off], acc);
        }
        sp.traces[n * sp.nr + sp.rec_id[t]] = acc;
        return;
    }
    t -= sp.nrl;
    if (t < sp.nuc) {
        const int64_t off = sp.inj_off[t];
        float v = unext[off];
        const float* q = sp.wavelet + n * sp.ns;
        for (int e = sp.inj_ptr[t]; e < sp.inj_ptr[t + 1]; ++e) v = __fmaf_rn(sp.inj_s[e], q[sp.inj_src[e]], v);
        unext[off] = v;
        // keep the neighbours' halo copies of boundary planes consistent (team mode)
        const int z = sp.inj_plane[t];
        const int64_t o = off - (int64_t)g.R * g.plane;  // model-layout index
        if (lo && z < g.R) lo[lo_off + o] = v;
        if (hi && z >= g.nz - g.R) hi[hi_off + o - (int64_t)(g.nz - g.R) * g.plane] = v;
    }
}

cudaError_t launch_sparse_step(const Geom& g, const Sparse& sp, const float* ucur, float* unext,
                               const int64_t* d_base, int i, const Halo& halo, int parity_next, cudaStream_t s) {
    int n = sp.nrl + sp.nuc;
    if (n <= 0) return cudaSuccess;
    sparse_step_kernel<<<(n + 127) / 128, 128, 0, s>>>(g, sp, ucur, unext, d_base, i, halo.lo[parity_next],
                                                       halo.lo_off, halo.hi[parity_next], halo.hi_off);
    return cudaGetLastError();
}

__global__ void advance_kernel(int64_t* d_base, int64_t by) { *d_base += by; }

// start of an aw_run: step base, cleared NaN flag and exchange-wait counters in one launch (instead of a
// pageable host-to-device copy and two memsets)
__global__ void run_init_kernel(DevCtl* ctl, int64_t base) {
    ctl->base = base;
    ctl->flag = 0u;
    ctl->wait_ns = 0ull;
    ctl->nwait = 0ull;
}

cudaError_t launch_run_init(DevCtl* ctl, int64_t base, cudaStream_t s) {
    run_init_kernel<<<1, 1, 0, s>>>(ctl, base);
    return cudaGetLastError();
}

cudaError_t launch_advance(int64_t* d_base, int64_t by, cudaStream_t s) {
    advance_kernel<<<1, 1, 0, s>>>(d_base, by);
    return cudaGetLastError();
}

// NaN/Inf check of the owned wavefield and of trace rows [t0, t1).
__global__ void check_finite_kernel(Geom g, const float* __restrict__ u, const float* __restrict__ traces,
                                    int64_t t0, int64_t t1, int nr, unsigned* flag) {
    // owned planes incl. the (always zero) pitch padding: a flat float4 walk
    const float4* u4 = reinterpret_cast<const float4*>(u + (int64_t)g.R * g.plane);
    const int64_t n4 = (int64_t)g.nz * g.plane / 4;
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = u4[i];
        bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
    }
    if (traces) {
        int64_t tot = (t1 - t0) * nr;
        for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < tot; k += (int64_t)gridDim.x * blockDim.x)
            bad |= !isfinite(traces[t0 * nr + k]);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

cudaError_t launch_check_finite(const Geom& g, const float* u, const float* traces, int64_t t0, int64_t t1,
                                int nr, unsigned* flag, cudaStream_t s) {
    check_finite_kernel<<<148 * 8, 256, 0, s>>>(g, u, traces, t0, t1, nr, flag);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Team handshake: after step n a rank publishes "level n+1 halo delivered"
// into its neighbours' flag words (system-scope release); before step n a
// rank waits until both neighbours published level n (acquire).  Because the
// flag is raised only after the whole step (stencil + injection) completed,
// it also certifies that the neighbour finished reading the halo buffer that
// the next step overwrites (no WAR hazard with two physical levels).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Levels are encoded (epoch << 32) + level + 1 with the epoch and the step base read from the
// device control block, so the kernels are parameter-free per step and can be graph-captured.
__global__ void team_wait_kernel(DevCtl* ctl, int has_lo, int has_hi, int i) {
    if (threadIdx.x != 0) return;
    const unsigned long long want = (ctl->epoch << 32) + (unsigned long long)(ctl->base + i + 1);
    // team_flags[0]: from rank-1, [1]: from rank+1
    const volatile unsigned long long* flags = ctl->team_flags;
    unsigned long long t0 = 0;
    for (int k = 0;; ++k) {
        unsigned long long f0, f1;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f0) : "l"(flags + 0) : "memory");
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f1) : "l"(flags + 1) : "memory");
        if ((!has_lo || f0 >= want) && (!has_hi || f1 >= want)) break;
        if (k == 0) t0 = global_ns();
        __nanosleep(200);
    }
    if (t0) {  // exchange-time accounting (aw_run_stats.ms_exchange)
        ctl->wait_ns += global_ns() - t0;
        ctl->nwait += 1;
    }
}

cudaError_t launch_team_wait(DevCtl* ctl, bool has_lo, bool has_hi, int i, cudaStream_t s) {
    team_wait_kernel<<<1, 32, 0, s>>>(ctl, has_lo, has_hi, i);
    return cudaGetLastError();
}

__global__ void team_signal_kernel(unsigned long long* peer_lo_flag, unsigned long long* peer_hi_flag,
                                   const DevCtl* ctl, int i) {
    if (threadIdx.x != 0) return;
    // this step produced level base + i + 1
    unsigned long long v = (ctl->epoch << 32) + (unsigned long long)(ctl->base + i + 2);
    __threadfence_system();  // halo stores of this step (stencil + injection) before the flag
    if (peer_lo_flag) atomicMax_system(peer_lo_flag, v);
    if (peer_hi_flag) atomicMax_system(peer_hi_flag, v);
}

cudaError_t launch_team_signal(unsigned long long* peer_lo_flag, unsigned long long* peer_hi_flag,
                               const DevCtl* ctl, int i, cudaStream_t s) {
    team_signal_kernel<<<1, 32, 0, s>>>(peer_lo_flag, peer_hi_flag, ctl, i);
    return cudaGetLastError();
}

// Raise flag words to at least v (monotone, so late signals of an older epoch never lower them).
__global__ void team_raise_kernel(unsigned long long* f0, unsigned long long* f1, unsigned long long v) {
    if (threadIdx.x != 0) return;
    __threadfence_system();
    if (f0) atomicMax_system(f0, v);
    if (f1) atomicMax_system(f1, v);
}

cudaError_t launch_team_raise(unsigned long long* f0, unsigned long long* f1, unsigned long long v,
                              cudaStream_t s) {
    team_raise_kernel<<<1, 32, 0, s>>>(f0, f1, v);
    return cudaGetLastError();
}

}  // namespace aw
