// aw_diffusion.cu -- NEXT-2: the paper's own benchmark operator on B200.
//
//   u_t = nu (u_xx + u_yy)          PAPER.md:732-736 [Evaluation > Examined problem]
//   Devito: TimeFunction(time_order=1, space_order=so), Eq(u.dt, v*(u.dx2+u.dy2)),
//   solve(eqn, u.forward)           PAPER.md:738-744  -> forward Euler
//
// The paper ran this operator through OPS-generated CUDA on a GTX 1080 and
// reports "peak utilisation" 20%/7% (advanced DSE) and 62%/28% (aggressive DSE,
// divisions hoisted) for the lowest/highest space order.
// Here: one hand-written sm_100a kernel per step, all divisions hoisted into
// the fp32 tables C[d][j] = fl32(c_j/h_d^2), C0, D = fl32(nu*dt) (computed once
// on the host), and the canonical per-point sequence (DESIGN.md §3 Q22)
//   L = C0*u; for d = 1, 0 (fastest first), j = 1..R: L = fma(C[d][j], u_-j + u_+j, L)
//   u_next = fma(D, L, u)
// with explicit-rounding intrinsics, so the result is value-identical to the
// fp32 oracle (oracle_diffusion_run).
//
// Kernel: one CTA per 64x32 output tile.  A single TMA 2D box load brings the
// tile plus its R-wide halo into shared memory (OOB zero fill = the zero
// padding of PAPER.md:455-491), then 8 warps compute 4 rows x 2 columns each
// with packed FFMA2/FADD2 on adjacent column pairs (2l, 2l+1; 64-bit shared
// loads and stores) and store coalesced rows.
// Many CTAs per SM (11-16 KB smem each) overlap their loads; HBM-bound at
// 8 algorithmic B per point update (read u, write u_next).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/aw.h"
#include "aw_internal.h"

extern "C" aw_status aw_internal_fail(aw_status st, const char* msg);

#ifndef AW_DIFF_TALL
#define AW_DIFF_TALL 1
#endif
#ifndef AW_DIFF_TALL_R
#define AW_DIFF_TALL_R 5  // tall tiles measured slower for R = 3, 4 (profiles/r1/diffusion_next2.jsonl)
#endif

namespace aw {
namespace {

__device__ __forceinline__ uint32_t smem_u32d(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct DiffArgs {
    float C[2][AW_MAXR + 1];  // [axis][j]
    float C0, D;
    float* out;               // row-pitched output
    int64_t pitch;
    int nx, ny;               // axis 1 (x, contiguous), axis 0 (rows)
    int ntx, nty;             // 64 x 32 tiles
};

// TMA ring depth: S = 1 with one CTA per tile (grid = #tiles) is the plain tiled kernel, best for
// R <= 2 where the kernel is store-bound; S = 3 with a persistent grid overlaps the load of the next
// tiles with the compute of this one, best for R >= 3 (profiles/r1/diffusion_next2.jsonl)
template <int R>
constexpr int diff_stages() { return R <= 2 ? 1 : 3; }
// tile height: taller tiles halve the y-halo overhead ((TY+2R)/TY) and the per-row column loads
// ((RY+2R)/RY) at high orders; 8 warps, RY = TY/8 rows per thread
template <int R>
constexpr int diff_ty() { return AW_DIFF_TALL && R >= AW_DIFF_TALL_R ? 64 : 32; }

template <int R>
__global__ void __launch_bounds__(256) diffusion_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ DiffArgs A) {
    constexpr int TX = 64, TY = diff_ty<R>(), RY = TY / 8, S = diff_stages<R>();
    constexpr int RP = (R + 3) / 4 * 4;  // TMA inner box row must be a multiple of 32 B
    constexpr int TXP = TX + 2 * RP, TYP = TY + 2 * R;
    constexpr int STAGE_BYTES = TXP * TYP * 4;
    constexpr int STAGE_STRIDE = (STAGE_BYTES + 127) / 128 * 128;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * STAGE_STRIDE);
    const int ntiles = A.ntx * A.nty;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // persistent CTA: tiles blockIdx.x, +gridDim.x, ... through a ring of S TMA stages, so the load
    // of the tiles S ahead overlaps the compute of this one (a one-tile CTA waits for its load)
    auto issue = [&](int t, int s) {
        const int x0 = (t % A.ntx) * TX, y0 = (t / A.ntx) * TY;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32d(bar + s)),
                     "r"(STAGE_BYTES)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(smem_u32d(smem + s * STAGE_STRIDE)),
            "l"(&tm), "r"(x0 - RP), "r"(y0 - R), "r"(smem_u32d(bar + s))
            : "memory");
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32d(bar + s)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < S; ++s)
            if (blockIdx.x + s * gridDim.x < ntiles) issue(blockIdx.x + s * gridDim.x, s);
    }
    __syncthreads();
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % S;
    const float* tile = reinterpret_cast<const float*>(smem + s * STAGE_STRIDE);
    const int x0 = (t % A.ntx) * TX, y0 = (t / A.ntx) * TY;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32d(bar + s)), "r"((uint32_t)((it / S) & 1))
        : "memory");

    // lane l owns the adjacent columns x0+2l, x0+2l+1: 64-bit shared loads and global stores
    const int ly = warp * RY;
    constexpr int K = (R + 1) / 2;
    const float* Qs = tile + ly * TXP + RP + 2 * lane;  // row ly-R .. of the halo'd tile, column pair
    float2 col[RY + 2 * R];
#pragma unroll
    for (int r = 0; r < RY + 2 * R; ++r) col[r] = *reinterpret_cast<const float2*>(Qs + r * TXP);
    const float2 C0 = make_float2(A.C0, A.C0), D = make_float2(A.D, A.D);
    const int xa = x0 + 2 * lane;
#pragma unroll
    for (int i = 0; i < RY; ++i) {
        const int y = y0 + ly + i;
        const float* row = Qs + (i + R) * TXP;
        const float2 uc = col[i + R];
        float2 L = __fmul2_rn(C0, uc);
        float2 v[2 * K + 1];  // columns (2l + 2k, 2l + 2k + 1), k = -K..K
#pragma unroll
        for (int k = -K; k <= K; ++k) v[K + k] = *reinterpret_cast<const float2*>(row + 2 * k);
#pragma unroll
        for (int j = 1; j <= R; ++j) {  // axis 1 (x, contiguous) first: u[x-j] + u[x+j] of both columns
            const int m = j >> 1;
            if (j & 1) {  // odd j: the two columns' pairs sit in different float2s -- two packed adds,
                // each keeps one useful half, then scalar fmas (no register moves to re-pair halves)
                const float2 sa = __fadd2_rn(v[K - m - 1], v[K + m]);      // .y = u[2l-j] + u[2l+j]
                const float2 sb = __fadd2_rn(v[K - m], v[K + m + 1]);      // .x = u[2l+1-j] + u[2l+1+j]
                L.x = __fmaf_rn(A.C[1][j], sa.y, L.x);
                L.y = __fmaf_rn(A.C[1][j], sb.x, L.y);
            } else {
                L = __ffma2_rn(make_float2(A.C[1][j], A.C[1][j]), __fadd2_rn(v[K - m], v[K + m]), L);
            }
        }
#pragma unroll
        for (int j = 1; j <= R; ++j)  // then axis 0 (rows)
            L = __ffma2_rn(make_float2(A.C[0][j], A.C[0][j]), __fadd2_rn(col[i + R - j], col[i + R + j]), L);
        const float2 un = __ffma2_rn(D, L, uc);
        if (y < A.ny && xa < A.nx) {
            float* o = A.out + (int64_t)y * A.pitch + xa;
            if (xa + 1 < A.nx) *reinterpret_cast<float2*>(o) = un;  // 8-B aligned: x0 % 64 == 0, pitch % 32 == 0
            else o[0] = un.x;
        }
    }
    __syncthreads();  // every warp finished reading stage s
    if (tid == 0 && t + S * (int)gridDim.x < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the TMA rewrite
        issue(t + S * gridDim.x, s);
    }
    }
}

template <int R>
size_t diff_smem() {
    constexpr int RP = (R + 3) / 4 * 4, TXP = 64 + 2 * RP, TYP = diff_ty<R>() + 2 * R;
    return diff_stages<R>() * (((TXP * TYP * 4 + 127) / 128) * 128) + 8 * diff_stages<R>();
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// exact FD weights, independently of aw_api.cu's copy (same closed form)
void weights(int k, double* c) {
    typedef __int128 i128;
    auto gcd = [](i128 a, i128 b) {
        if (a < 0) a = -a;
        if (b < 0) b = -b;
        while (b) {
            i128 t = a % b;
            a = b;
            b = t;
        }
        return a;
    };
    auto fact = [](int n) {
        i128 f = 1;
        for (int i = 2; i <= n; ++i) f *= i;
        return f;
    };
    const int m = k / 2;
    i128 sn = 0, sd = 1;
    for (int j = 1; j <= m; ++j) {
        i128 n = 2 * fact(m) * fact(m) * ((j % 2) ? 1 : -1), d = (i128)j * j * fact(m - j) * fact(m + j);
        i128 g = gcd(n, d);
        n /= g;
        d /= g;
        c[j] = (double)(int64_t)n / (double)(int64_t)d;
        i128 nn = sn * d + n * sd, dd = sd * d;
        g = gcd(nn, dd);
        sn = nn / g;
        sd = dd / g;
    }
    i128 n0 = -2 * sn, g = gcd(n0, sd);
    c[0] = (double)(int64_t)(n0 / g) / (double)(int64_t)(sd / g);
}

}  // namespace
}  // namespace aw

struct aw_diffusion {
    int R = 0, nx = 0, ny = 0;
    int64_t pitch = 0;
    double h[2] = {1, 1}, nu = 0;
    float* buf[2] = {nullptr, nullptr};
    int cur = 0;
    int64_t steps = 0;
    cudaStream_t s = nullptr, ext = nullptr;
    cudaEvent_t ev_sync = nullptr, ev0 = nullptr, ev1 = nullptr;
    CUtensorMap tm[2];
    int device = 0;
    bool poisoned = false;
    int opt_timing = 0, opt_graph = 64;
    std::vector<cudaEvent_t> tev;
    cudaGraphExec_t graph = nullptr;
    int graph_G = 0, graph_parity = -1;
    double graph_dt = 0;
    aw_run_stats stats{};
    int64_t launches = 0;
    aw::DiffArgs args{};
    int resident = 0;  // SMs x resident CTAs of the kernel instance (0 = not queried yet)
};

namespace {

aw_status dfail(aw_diffusion* d, cudaError_t e, const char* what) {
    if (d) d->poisoned = true;
    char buf[256];
    snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
    cudaGetLastError();
    return aw_internal_fail(e == cudaErrorMemoryAllocation ? AW_ENOMEM : AW_ECUDA, buf);
}

#define DCK(call)                                   \
    do {                                            \
        cudaError_t e_ = (call);                    \
        if (e_ != cudaSuccess) return dfail(d, e_, #call); \
    } while (0)

template <int R>
cudaError_t launch_diff(aw_diffusion* d, int src, cudaStream_t s) {
    aw::DiffArgs A = d->args;
    A.out = d->buf[1 - src];
    A.nty = (d->ny + aw::diff_ty<R>() - 1) / aw::diff_ty<R>();
    if (!d->resident) {  // resident CTAs of this instance on the handle's device (persistent grid)
        int sms = 0, occ = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, aw::diffusion_kernel<R>, 256, aw::diff_smem<R>());
        d->resident = sms * (occ < 1 ? 1 : occ);
    }
    const int ntiles = A.ntx * A.nty;
    const int grid = (aw::diff_stages<R>() == 1 || ntiles < d->resident) ? ntiles : d->resident;
    aw::diffusion_kernel<R><<<grid, 256, aw::diff_smem<R>(), s>>>(d->tm[src], A);
    return cudaGetLastError();
}

cudaError_t launch_step(aw_diffusion* d, int src, cudaStream_t s) {
    switch (d->R) {
        case 1: return launch_diff<1>(d, src, s);
        case 2: return launch_diff<2>(d, src, s);
        case 3: return launch_diff<3>(d, src, s);
        case 4: return launch_diff<4>(d, src, s);
        case 5: return launch_diff<5>(d, src, s);
        case 6: return launch_diff<6>(d, src, s);
        case 7: return launch_diff<7>(d, src, s);
        case 8: return launch_diff<8>(d, src, s);
    }
    return cudaErrorInvalidValue;
}

template <int R>
cudaError_t set_attr() {
    return cudaFuncSetAttribute(aw::diffusion_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)aw::diff_smem<R>());
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

extern "C" {

aw_status aw_diffusion_create(aw_diffusion** out, int ndim, const int64_t* shape, const double* extent,
                              int space_order, double nu, void* stream) {
    if (!out) return aw_internal_fail(AW_EINVAL, "out is NULL");
    *out = nullptr;
    if (ndim != 2) return aw_internal_fail(ndim == 3 ? AW_EUNSUPPORTED : AW_EINVAL, "diffusion: ndim must be 2");
    if (!shape || !extent) return aw_internal_fail(AW_EINVAL, "shape/extent NULL");
    if (space_order < 2 || space_order > 16 || (space_order & 1))
        return aw_internal_fail(AW_EINVAL, "space_order must be even in [2, 16]");
    if (!(nu > 0) || !std::isfinite(nu)) return aw_internal_fail(AW_EINVAL, "nu must be finite and > 0");
    const int R = space_order / 2;
    for (int d = 0; d < 2; ++d) {
        if (shape[d] < R + 1 || shape[d] > (1 << 30)) return aw_internal_fail(AW_EINVAL, "bad shape");
        if (!(extent[d] > 0) || !std::isfinite(extent[d])) return aw_internal_fail(AW_EINVAL, "extent must be > 0");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return aw_internal_fail(AW_ECUDA, "no CUDA device available (libaw has no CPU fallback)");
    }
    aw_diffusion* d = new aw_diffusion();
    cudaGetDevice(&d->device);
    d->R = R;
    d->ny = (int)shape[0];
    d->nx = (int)shape[1];
    d->pitch = ((int64_t)d->nx + 31) / 32 * 32;
    d->nu = nu;
    d->ext = (cudaStream_t)stream;
    for (int a = 0; a < 2; ++a) d->h[a] = extent[a] / (double)(shape[a] - 1);
    // axis tables (division hoisting); axis 0 = rows, axis 1 = x
    double c[AW_MAXR + 1];
    aw::weights(space_order, c);
    std::memset(&d->args, 0, sizeof d->args);
    double s0 = 0.0;
    for (int a = 0; a < 2; ++a) {
        const double h2 = d->h[a] * d->h[a];
        for (int j = 1; j <= R; ++j) d->args.C[a][j] = (float)(c[j] / h2);
        s0 = s0 + c[0] / h2;
    }
    d->args.C0 = (float)s0;
    d->args.pitch = d->pitch;
    d->args.nx = d->nx;
    d->args.ny = d->ny;
    d->args.ntx = (d->nx + 63) / 64;
    const size_t bytes = (size_t)d->ny * d->pitch * sizeof(float);
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&d->s, cudaStreamNonBlocking)) || (e = cudaEventCreate(&d->ev0)) ||
        (e = cudaEventCreate(&d->ev1)) || (e = cudaEventCreateWithFlags(&d->ev_sync, cudaEventDisableTiming)) ||
        (e = cudaMalloc((void**)&d->buf[0], bytes)) || (e = cudaMalloc((void**)&d->buf[1], bytes)) ||
        (e = cudaMemsetAsync(d->buf[0], 0, bytes, d->s)) || (e = cudaMemsetAsync(d->buf[1], 0, bytes, d->s))) {
        aw_status st = dfail(nullptr, e, "diffusion create");
        aw_diffusion_destroy(d);
        return st;
    }
    switch (R) {
        case 1: e = set_attr<1>(); break;
        case 2: e = set_attr<2>(); break;
        case 3: e = set_attr<3>(); break;
        case 4: e = set_attr<4>(); break;
        case 5: e = set_attr<5>(); break;
        case 6: e = set_attr<6>(); break;
        case 7: e = set_attr<7>(); break;
        case 8: e = set_attr<8>(); break;
    }
    auto enc = aw::encode_fn();
    const int RP = (R + 3) / 4 * 4;
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        cuuint64_t dims[2] = {(cuuint64_t)d->nx, (cuuint64_t)d->ny};
        cuuint64_t strides[1] = {(cuuint64_t)d->pitch * 4};
        const int TY = R >= AW_DIFF_TALL_R && AW_DIFF_TALL ? 64 : 32;  // = aw::diff_ty<R>()
        cuuint32_t box[2] = {(cuuint32_t)(64 + 2 * RP), (cuuint32_t)(TY + 2 * R)};
        cuuint32_t estr[2] = {1, 1};
        if (!enc || enc(&d->tm[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d->buf[b], dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            e = cudaErrorInvalidValue;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(d->s);
    if (e != cudaSuccess) {
        aw_status st = dfail(nullptr, e, "diffusion setup");
        aw_diffusion_destroy(d);
        return st;
    }
    *out = d;
    return AW_OK;
}

void aw_diffusion_destroy(aw_diffusion* d) {
    if (!d) return;
    if (d->s) cudaStreamSynchronize(d->s);
    if (d->graph) cudaGraphExecDestroy(d->graph);
    for (auto e : d->tev) cudaEventDestroy(e);
    for (int b = 0; b < 2; ++b)
        if (d->buf[b]) cudaFree(d->buf[b]);
    if (d->ev0) cudaEventDestroy(d->ev0);
    if (d->ev1) cudaEventDestroy(d->ev1);
    if (d->ev_sync) cudaEventDestroy(d->ev_sync);
    if (d->s) cudaStreamDestroy(d->s);
    cudaGetLastError();
    delete d;
}

static aw_status d_enter(aw_diffusion* d) {
    if (d->poisoned) return aw_internal_fail(AW_ESTATE, "handle poisoned by an earlier CUDA error");
    DCK(cudaSetDevice(d->device));
    if (d->ext) {
        DCK(cudaEventRecord(d->ev_sync, d->ext));
        DCK(cudaStreamWaitEvent(d->s, d->ev_sync, 0));
    }
    return AW_OK;
}
static aw_status d_leave(aw_diffusion* d) {
    if (d->ext) {
        DCK(cudaEventRecord(d->ev_sync, d->s));
        DCK(cudaStreamWaitEvent(d->ext, d->ev_sync, 0));
    }
    return AW_OK;
}

aw_status aw_diffusion_set(aw_diffusion* d, const float* u) {
    if (!d) return aw_internal_fail(AW_EINVAL, "null handle");
    aw_status st = d_enter(d);
    if (st) return st;
    d->cur = 0;
    d->steps = 0;
    const size_t bytes = (size_t)d->ny * d->pitch * sizeof(float);
    DCK(cudaMemsetAsync(d->buf[0], 0, bytes, d->s));
    if (u)
        DCK(cudaMemcpy2DAsync(d->buf[0], d->pitch * 4, u, (size_t)d->nx * 4, (size_t)d->nx * 4, d->ny,
                              is_device_ptr(u) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, d->s));
    DCK(cudaStreamSynchronize(d->s));
    return d_leave(d);
}

aw_status aw_diffusion_run(aw_diffusion* d, int nt, double dt) {
    if (!d) return aw_internal_fail(AW_EINVAL, "null handle");
    if (nt < 0 || !(dt > 0) || !std::isfinite(dt)) return aw_internal_fail(AW_EINVAL, "nt >= 0 and dt > 0 required");
    aw_status st = d_enter(d);
    if (st) return st;
    d->args.D = (float)(d->nu * dt);  // fl32(nu*dt): one rounding of the fp64 product
    int64_t launches = 0;
    DCK(cudaEventRecord(d->ev0, d->s));
    int done = 0;
    const int G = d->opt_graph;
    if (!d->opt_timing && G > 0 && nt >= G) {
        if (!d->graph || d->graph_G != G || d->graph_parity != d->cur || d->graph_dt != dt) {
            if (d->graph) cudaGraphExecDestroy(d->graph);
            d->graph = nullptr;
            cudaGraph_t gr;
            DCK(cudaStreamBeginCapture(d->s, cudaStreamCaptureModeThreadLocal));
            int c = d->cur;
            for (int i = 0; i < G; ++i) {
                cudaError_t e = launch_step(d, c, d->s);
                if (e != cudaSuccess) {
                    cudaStreamEndCapture(d->s, &gr);
                    return dfail(d, e, "diffusion capture");
                }
                c = 1 - c;
            }
            DCK(cudaStreamEndCapture(d->s, &gr));
            DCK(cudaGraphInstantiate(&d->graph, gr, 0));
            cudaGraphDestroy(gr);
            d->graph_G = G;
            d->graph_parity = d->cur;
            d->graph_dt = dt;
        }
        while (nt - done >= G && (G % 2 == 0 || d->cur == d->graph_parity)) {
            DCK(cudaGraphLaunch(d->graph, d->s));
            done += G;
            launches += G;
            if (G & 1) d->cur = 1 - d->cur;
        }
    }
    if (d->opt_timing)
        while ((int)d->tev.size() < 2 * nt) {
            cudaEvent_t e;
            DCK(cudaEventCreate(&e));
            d->tev.push_back(e);
        }
    const int first = done;
    for (; done < nt; ++done) {
        const int i = done - first;
        if (d->opt_timing) DCK(cudaEventRecord(d->tev[2 * i], d->s));
        DCK(launch_step(d, d->cur, d->s));
        if (d->opt_timing) DCK(cudaEventRecord(d->tev[2 * i + 1], d->s));
        d->cur = 1 - d->cur;
        ++launches;
    }
    DCK(cudaEventRecord(d->ev1, d->s));
    if ((st = d_leave(d))) return st;
    DCK(cudaStreamSynchronize(d->s));
    float ms = 0.f;
    DCK(cudaEventElapsedTime(&ms, d->ev0, d->ev1));
    d->stats.ms_total = ms;
    d->stats.launches = launches;
    d->launches += launches;
    d->stats.launches_total = d->launches;
    d->stats.points = (int64_t)d->nx * d->ny;
    d->stats.gpts = ms > 0 ? (double)d->stats.points * nt / (ms * 1e6) : 0.0;
    d->stats.kernel = AW_KERNEL_STREAM;
    d->stats.eta_tiles = 0;
    if (d->opt_timing) {
        double sum = 0;
        for (int i = 0; i < nt - first; ++i) {
            float e = 0.f;
            DCK(cudaEventElapsedTime(&e, d->tev[2 * i], d->tev[2 * i + 1]));
            sum += e;
        }
        d->stats.ms_stencil = sum;
        d->stats.n_stencil = nt - first;
    } else {
        d->stats.ms_stencil = -1;
        d->stats.n_stencil = 0;
    }
    d->steps += nt;
    return AW_OK;
}

aw_status aw_diffusion_read(aw_diffusion* d, float* out) {
    if (!d || !out) return aw_internal_fail(AW_EINVAL, "null argument");
    aw_status st = d_enter(d);
    if (st) return st;
    DCK(cudaMemcpy2DAsync(out, (size_t)d->nx * 4, d->buf[d->cur], d->pitch * 4, (size_t)d->nx * 4, d->ny,
                          is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, d->s));
    DCK(cudaStreamSynchronize(d->s));
    return d_leave(d);
}

aw_status aw_diffusion_stats(const aw_diffusion* d, aw_run_stats* out) {
    if (!d || !out) return aw_internal_fail(AW_EINVAL, "null argument");
    *out = d->stats;
    out->launches_total = d->launches;
    return AW_OK;
}

aw_status aw_diffusion_set_option(aw_diffusion* d, int option, int64_t value) {
    if (!d) return aw_internal_fail(AW_EINVAL, "null handle");
    if (option == AW_OPT_TIMING) {
        d->opt_timing = value != 0;
        return AW_OK;
    }
    if (option == AW_OPT_GRAPH_STEPS) {
        if (value < 0 || value > 4096) return aw_internal_fail(AW_EINVAL, "graph steps out of range");
        d->opt_graph = (int)value;
        return AW_OK;
    }
    return aw_internal_fail(AW_EINVAL, "unsupported option for diffusion");
}

}  // extern "C"
