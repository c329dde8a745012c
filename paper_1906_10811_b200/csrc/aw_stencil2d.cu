// aw_stencil2d.cu -- the 2D hot path (SURVEY.md §8(a) rows a5+a6 for ndim = 2): star Laplacian of
// order k = 2R fused with the damped leapfrog update, on B200 (sm_100a).
//
// 2D grids have no streaming axis, so each CTA owns one 64 x 32 output tile (x contiguous, z rows):
//  * one TMA 2D box brings the u^n tile with its R-wide halo into shared memory (x ghosts: TMA's
//    out-of-bounds zero fill; z ghosts: the zeroed halo rows of the wavefield buffer), while every
//    thread already loads its u^{n-1}, b, a pairs from global memory (64-bit, coalesced);
//  * 8 warps x 4 rows; lane l owns the adjacent columns x0+2l, x0+2l+1, so all arithmetic is
//    packed FFMA2/FADD2/FMUL2 on point pairs and the store is one 64-bit STG per row;
//  * ~12-18 KB of shared memory per CTA: many CTAs per SM overlap their loads.
// HBM-bound at 16 algorithmic B per point update (+4 where eta != 0).  Sources and receivers run
// in the sparse kernel after it (aw_kernels.cu), exactly as for the reference-grade v1 kernel.
//
// Per point the canonical sequence of SURVEY §8(c).6, axis 1 (x) then axis 0 (z):
//   L = C0*u; x pairs j = 1..R; z pairs; t = 2u - u^{n-1}; w = fma(b, L, t);
//   u^{n+1} = fma(a, w, (1-a) u^{n-1})
// with explicit-rounding intrinsics: value-identical to the oracle and to stencil_v1_kernel.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <unordered_map>

#include "aw_internal.h"

namespace aw {

struct Tile2DPlan {
    int ntx = 0, ntz = 0;
    int resident = 0;  // SMs x resident CTAs on the grid's device (queried at the first launch)
    std::unordered_map<const void*, CUtensorMap> maps;  // u^n buffers seen so far (2, or a FWI ring)
};

namespace {

__device__ __forceinline__ uint32_t s2_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

struct S2Args {
    Coefs c;
    const float* uprev;  // u^{n-1} buffer base (plane -R)
    float* unext;        // u^{n+1} buffer base
    const float* b;      // model layout
    const float* a;      // null: no damping
    int64_t pitch;
    int nx, nz, R, ntx, ntz;
};

// TMA ring depth: 1 = one CTA per tile (grid = #tiles); S > 1 = persistent grid whose CTAs prefetch
// the boxes of their next S-1 tiles.  Measured on 16384^2 (profiles/r1/bench_2d.jsonl): S = 3 is
// slower here (so 8: 0.85 vs 0.75 ms) -- unlike the diffusion kernel, each tile also issues its own
// u^{n-1}, b, a loads, which the one-tile CTAs already overlap with the box -- so S = 1 for every R.
template <int R>
constexpr int s2_stages() { return 1; }
// tile height (8 warps, TY/8 rows per thread): 64 halves the z-halo overhead at high orders
#ifndef AW_S2_TALL_R
#define AW_S2_TALL_R 9  // off: 64-row tiles measured no faster here (so 12: 0.854 vs 0.86 ms on 16384^2)
#endif
template <int R>
constexpr int s2_ty() { return R >= AW_S2_TALL_R ? 64 : 32; }

template <int R>
__global__ void __launch_bounds__(256) stencil2d_kernel(const __grid_constant__ CUtensorMap tm,
                                                        const __grid_constant__ S2Args A) {
    constexpr int TX = 64, TY = s2_ty<R>(), RY = TY / 8, S = s2_stages<R>();
    constexpr int RP = (R + 3) / 4 * 4;  // TMA box rows must be multiples of 32 B
    constexpr int TXP = TX + 2 * RP, TYP = TY + 2 * R;
    constexpr int K = (R + 1) / 2;
    constexpr int STAGE_BYTES = TXP * TYP * 4;
    constexpr int STAGE_STRIDE = (STAGE_BYTES + 127) / 128 * 128;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * STAGE_STRIDE);
    const int ntiles = A.ntx * A.ntz;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto issue = [&](int t, int s) {
        const int x0 = (t % A.ntx) * TX, z0 = (t / A.ntx) * TY;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s2_smem(bar + s)),
                     "r"(STAGE_BYTES)
                     : "memory");
        // buffer row of plane z is z + R, so the box of planes [z0-R, z0+TY+R) starts at row z0
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(s2_smem(smem + s * STAGE_STRIDE)),
            "l"(&tm), "r"(x0 - RP), "r"(z0), "r"(s2_smem(bar + s))
            : "memory");
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s2_smem(bar + s)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < S; ++s)
            if (blockIdx.x + s * (int)gridDim.x < ntiles) issue(blockIdx.x + s * gridDim.x, s);
    }
    __syncthreads();  // barriers initialised before anyone waits on them
    const int ly = warp * RY;
    const float2 C0 = make_float2(A.c.C0, A.c.C0);
    const float2 two = make_float2(2.f, 2.f), one = make_float2(1.f, 1.f);
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % S;
        const int x0 = (t % A.ntx) * TX, z0 = (t / A.ntx) * TY;
        // this thread's u^{n-1}, b, a pairs: issued before waiting for the tile
        const int xa = x0 + 2 * lane;
        const bool inA = xa < A.nx, inB = xa + 1 < A.nx;
        float2 um[RY], bb[RY], aa[RY];
#pragma unroll
        for (int i = 0; i < RY; ++i) {
            const int z = z0 + ly + i;
            um[i] = bb[i] = make_float2(0.f, 0.f);
            aa[i] = make_float2(1.f, 1.f);
            if (z >= A.nz || !inA) continue;
            const int64_t o = (int64_t)z * A.pitch + xa;
            const float* pu = A.uprev + o + (int64_t)R * A.pitch;
            if (inB) {
                um[i] = *reinterpret_cast<const float2*>(pu);
                bb[i] = __ldg(reinterpret_cast<const float2*>(A.b + o));
                if (A.a) aa[i] = __ldg(reinterpret_cast<const float2*>(A.a + o));
            } else {
                um[i].x = pu[0];
                bb[i].x = __ldg(A.b + o);
                if (A.a) aa[i].x = __ldg(A.a + o);
            }
        }
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
            "@!P1 bra WAIT_%=;\n"
            "}\n" ::"r"(s2_smem(bar + s)), "r"((uint32_t)((it / S) & 1))
            : "memory");
        const float* tile = reinterpret_cast<const float*>(smem + s * STAGE_STRIDE);
        const float* Qs = tile + ly * TXP + RP + 2 * lane;  // plane z0+ly-R, column pair of this lane
        float2 col[RY + 2 * R];
#pragma unroll
        for (int r = 0; r < RY + 2 * R; ++r) col[r] = *reinterpret_cast<const float2*>(Qs + r * TXP);
#pragma unroll
        for (int i = 0; i < RY; ++i) {
            const int z = z0 + ly + i;
            const float* row = Qs + (i + R) * TXP;
            const float2 uc = col[i + R];
            float2 L = __fmul2_rn(C0, uc);
            float2 v[2 * K + 1];
#pragma unroll
            for (int k = -K; k <= K; ++k) v[K + k] = *reinterpret_cast<const float2*>(row + 2 * k);
#pragma unroll
            for (int j = 1; j <= R; ++j) {  // axis 1 (x) first: pair sums u[x-j] + u[x+j] of both columns
                const int m = j >> 1;
                const float2 lo = (j & 1) ? make_float2(v[K - m - 1].y, v[K - m].x) : v[K - m];
                const float2 hi = (j & 1) ? make_float2(v[K + m].y, v[K + m + 1].x) : v[K + m];
                L = __ffma2_rn(make_float2(A.c.C[1][j], A.c.C[1][j]), __fadd2_rn(lo, hi), L);
            }
#pragma unroll
            for (int j = 1; j <= R; ++j)  // then axis 0 (z)
                L = __ffma2_rn(make_float2(A.c.C[0][j], A.c.C[0][j]), __fadd2_rn(col[i + R - j], col[i + R + j]), L);
            const float2 t2 = __ffma2_rn(two, uc, make_float2(-um[i].x, -um[i].y));  // 2u exact: one rounding
            const float2 w = __ffma2_rn(bb[i], L, t2);
            const float2 r1 = __fmul2_rn(__fadd2_rn(one, make_float2(-aa[i].x, -aa[i].y)), um[i]);
            const float2 un = __ffma2_rn(aa[i], w, r1);
            if (z < A.nz && inA) {
                float* o = A.unext + (int64_t)(z + R) * A.pitch + xa;
                if (inB) *reinterpret_cast<float2*>(o) = un;
                else o[0] = un.x;
            }
        }
        if (S > 1) {
            __syncthreads();  // every warp finished reading stage s
            if (tid == 0 && t + S * (int)gridDim.x < ntiles) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the TMA rewrite
                issue(t + S * gridDim.x, s);
            }
        }
    }
}

template <int R>
constexpr size_t s2_smem_bytes() {
    constexpr int RP = (R + 3) / 4 * 4, TXP = 64 + 2 * RP, TYP = s2_ty<R>() + 2 * R;
    return s2_stages<R>() * (((TXP * TYP * 4 + 127) / 128) * 128) + 8 * s2_stages<R>();
}

PFN_cuTensorMapEncodeTiled_v12000 s2_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

template <int R>
cudaError_t s2_launch(Tile2DPlan* p, const Geom& g, const Coefs& c, const float* ucur, const float* uprev,
                      float* unext, const float* b, const float* a, cudaStream_t s) {
    constexpr int RP = (R + 3) / 4 * 4;
    auto it = p->maps.find(ucur);
    if (it == p->maps.end()) {
        auto enc = s2_encode_fn();
        if (!enc) return cudaErrorNotSupported;
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)g.nx, (cuuint64_t)(g.nz + 2 * g.R)};
        cuuint64_t strides[1] = {(cuuint64_t)g.pitch * 4};
        cuuint32_t box[2] = {(cuuint32_t)(64 + 2 * RP), (cuuint32_t)(s2_ty<R>() + 2 * R)};
        cuuint32_t estr[2] = {1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ucur), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
        it = p->maps.emplace(ucur, m).first;
    }
    S2Args A;
    A.c = c;
    A.uprev = uprev;
    A.unext = unext;
    A.b = b;
    A.a = a;
    A.pitch = g.pitch;
    A.nx = g.nx;
    A.nz = g.nz;
    A.R = g.R;
    A.ntx = p->ntx;
    static_assert(s2_smem_bytes<R>() <= 48 * 1024, "fits the default dynamic shared memory limit");
    A.ntz = (g.nz + s2_ty<R>() - 1) / s2_ty<R>();
    if (!p->resident) {  // resident CTAs on the current device (persistent grid when S > 1)
        int dev = 0, sms = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stencil2d_kernel<R>, 256, s2_smem_bytes<R>());
        p->resident = sms * (occ < 1 ? 1 : occ);
    }
    const int ntiles = p->ntx * A.ntz;
    const int grid = (s2_stages<R>() == 1 || ntiles < p->resident) ? ntiles : p->resident;
    stencil2d_kernel<R><<<grid, 256, s2_smem_bytes<R>(), s>>>(it->second, A);
    return cudaGetLastError();
}

}  // namespace

cudaError_t tile2d_prepare(const Geom& g, Tile2DPlan** plan) {
    *plan = nullptr;
    if (g.ndim != 2 || g.R < 1 || g.R > AW_MAXR) return cudaErrorNotSupported;
    Tile2DPlan* p = new Tile2DPlan();
    p->ntx = (g.nx + 63) / 64;
    p->ntz = (g.nz + 31) / 32;
    *plan = p;
    return cudaSuccess;
}

void tile2d_release(Tile2DPlan* p) { delete p; }

void tile2d_forget_maps(Tile2DPlan* p) {
    if (p) p->maps.clear();
}

cudaError_t launch_stencil_tile2d(Tile2DPlan* p, const Geom& g, const Coefs& c, const float* ucur, const float* uprev,
                                  float* unext, const float* b, const float* a, cudaStream_t s) {
    if (!p) return cudaErrorNotSupported;
    switch (g.R) {
        case 1: return s2_launch<1>(p, g, c, ucur, uprev, unext, b, a, s);
        case 2: return s2_launch<2>(p, g, c, ucur, uprev, unext, b, a, s);
        case 3: return s2_launch<3>(p, g, c, ucur, uprev, unext, b, a, s);
        case 4: return s2_launch<4>(p, g, c, ucur, uprev, unext, b, a, s);
        case 5: return s2_launch<5>(p, g, c, ucur, uprev, unext, b, a, s);
        case 6: return s2_launch<6>(p, g, c, ucur, uprev, unext, b, a, s);
        case 7: return s2_launch<7>(p, g, c, ucur, uprev, unext, b, a, s);
        case 8: return s2_launch<8>(p, g, c, ucur, uprev, unext, b, a, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace aw
