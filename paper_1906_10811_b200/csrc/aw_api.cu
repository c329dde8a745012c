// aw_api.cu -- host runtime of libaw: the C-ABI of include/aw.h.
//
// Validation, device layout, sparse setup (fp64 index/weight computation,
// SURVEY.md §8(c).4), FD-weight and axis-coefficient tables (§8(c).1-2), the
// on-device time loop (CUDA graphs of G steps or timed direct launches), the
// multi-slab team (fused peer-memory halo stores + flag handshake), and stats.
// No CPU compute fallback exists: every step of the path runs in the kernels
// of aw_kernels.cu / aw_stream.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/aw.h"
#include <cstddef>

#include "aw_internal.h"

using aw::Coefs;
using aw::Geom;
using aw::Halo;

namespace {

thread_local std::string g_err;

aw_status fail(aw_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

// ---------------------------------------------------------------------------
// Exact FD weights: c_j = 2(-1)^{j+1}(m!)^2 / (j^2 (m-j)! (m+j)!),
// c_0 = -2 sum c_j, as reduced rationals in 128-bit integers, then one
// correctly rounded fp64 division each.
// ---------------------------------------------------------------------------
typedef __int128 i128;
i128 igcd(i128 a, i128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        i128 t = a % b;
        a = b;
        b = t;
    }
    return a;
}
struct Rat {
    i128 n, d;
};
Rat rat_norm(i128 n, i128 d) {
    if (d < 0) n = -n, d = -d;
    i128 g = igcd(n, d);
    if (g == 0) g = 1;
    return {n / g, d / g};
}
void fd_weights(int k, double* c) {
    const int m = k / 2;
    auto fact = [](int n) {
        i128 f = 1;
        for (int i = 2; i <= n; ++i) f *= i;
        return f;
    };
    Rat sum{0, 1};
    for (int j = 1; j <= m; ++j) {
        i128 num = 2 * fact(m) * fact(m) * ((j % 2) ? 1 : -1);
        i128 den = (i128)j * j * fact(m - j) * fact(m + j);
        Rat cj = rat_norm(num, den);
        c[j] = (double)(int64_t)cj.n / (double)(int64_t)cj.d;
        sum = rat_norm(sum.n * cj.d + cj.n * sum.d, sum.d * cj.d);
    }
    Rat c0 = rat_norm(-2 * sum.n, sum.d);
    c[0] = (double)(int64_t)c0.n / (double)(int64_t)c0.d;
}

int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

enum PtrKind { PK_HOST, PK_DEVICE };
PtrKind ptr_kind(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return PK_HOST;
    }
    return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) ? PK_DEVICE : PK_HOST;
}

struct Team;

}  // namespace

struct aw_grid {
    // geometry
    int ndim = 0;
    int64_t shape[3] = {1, 1, 1};
    double extent[3] = {0, 0, 0}, origin[3] = {0, 0, 0}, h[3] = {1, 1, 1};
    int so = 0, R = 0;
    int rank = 0, world = 1, device = 0;
    int64_t z0 = 0;
    Geom geom{};
    Coefs coefs{};
    // streams
    cudaStream_t s = nullptr;
    cudaStream_t ext = nullptr;
    cudaEvent_t ev_sync = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
    // pinned host staging of the small uploads (sparse tables): the copies are truly asynchronous; the
    // event guards the buffer's reuse (the previous upload must have left it)
    char* h_stage = nullptr;
    size_t h_stage_cap = 0;
    cudaEvent_t ev_stage = nullptr;
    bool stage_pending = false;
    unsigned model_epoch = 0;  // aw_set_model calls (device-side validation writes the failing epoch)
    bool poisoned = false;
    // device memory.  The dense arrays (2 wavefield levels, m, eta, b, a) live in one block: the
    // library's own allocation (dense_lib) or the caller's workspace (aw_bind_workspace).
    float* ubuf[2] = {nullptr, nullptr};
    size_t ubytes = 0;  // per wavefield buffer
    float *m = nullptr, *eta = nullptr, *b = nullptr, *a = nullptr;
    size_t mbytes = 0;
    char* dense = nullptr;      // block in use (nullptr: AW_DIST_WORKSPACE and nothing bound yet)
    char* dense_lib = nullptr;  // the library's block (freed when a workspace is bound)
    size_t dense_bytes = 0;
    char* ws = nullptr;         // bound caller workspace
    size_t ws_bytes = 0;
    size_t ws_slot_off[2] = {0, 0}, ws_slot_cap[2] = {0, 0};  // sparse arena slots: [0] sources, [1] receivers
    size_t src_need = 0, rec_need = 0;                         // bytes of the current sparse arenas
    std::map<void*, size_t> lib_allocs;                        // the library's own device allocations
    aw::DevCtl* ctl = nullptr;  // device control block (step base, epoch, flags, team words)
    int64_t* d_base = nullptr;  // &ctl->base
    unsigned* d_flag = nullptr; // &ctl->flag
    unsigned long long* d_team_flags = nullptr;  // ctl->team_flags: [0] from rank-1, [1] from rank+1
    // state
    bool have_model = false, have_damp = false, coeffs_valid = false, dt_set = false;
    double dt = 0.0;
    int cur = 0;  // physical buffer holding u^n
    int64_t steps = 0;
    // sources
    int ns = 0, src_nt = 0;
    std::vector<int64_t> src_corner_lin;  // [ns][nc]
    std::vector<double> src_w64;          // [ns][nc]
    std::vector<int> ent_src, ent_beta;   // owned entries in CSR order
    std::vector<int64_t> h_inj_lin;       // owned unique injection corners (CSR order)
    std::vector<int> h_inj_ptr;           // their CSR ranges
    float* d_wavelet = nullptr;
    int64_t* d_inj_off = nullptr;
    int* d_inj_plane = nullptr;
    int* d_inj_ptr = nullptr;
    int* d_inj_src = nullptr;
    int64_t* d_inj_moff = nullptr;
    double* d_inj_w64 = nullptr;
    float* d_inj_s = nullptr;
    int nuc = 0, nent = 0;
    // receivers
    int nr = 0, rec_nt = 0;
    std::vector<int64_t> rec_corner_lin;
    std::vector<float> rec_w32;
    int nrl = 0;
    int* d_rec_id = nullptr;
    int64_t* d_rec_off = nullptr;
    float* d_rec_w = nullptr;
    float* d_traces = nullptr;
    // options
    int opt_kernel = AW_KERNEL_AUTO;
    int opt_timing = 0;
    int opt_graph = 16;
    int opt_check = 1;
    // stream kernel plan
    aw::StreamPlan* plan = nullptr;
    aw::Tile2DPlan* t2 = nullptr;          // 2D tiled kernel (AUTO in 2D, single slab)
    int eta_tiles_pct = 100;
    int kernel_used = AW_KERNEL_V1;
    // graphs: key = (G << 1) | parity
    // captured graphs per (G, parity): a few entries, each with the signature of every launch parameter
    // it captured (buffers, tensor maps, sparse tables, ...), so a setup call that changes nothing the
    // graph uses (e.g. the same sources re-added, a new model in the same arrays) keeps the graph
    struct GraphEntry {
        std::string sig;
        cudaGraphExec_t exec;
    };
    std::map<int64_t, std::vector<GraphEntry>> graphs;
    // timing events pool
    std::vector<cudaEvent_t> tev;
    // team
    Halo halo{};
    unsigned long long* peer_flag_lo = nullptr;  // &flags_{rank-1}[1]
    unsigned long long* peer_flag_hi = nullptr;  // &flags_{rank+1}[0]
    std::vector<void*> ipc_opened;
    std::vector<std::pair<cudaIpcMemHandle_t, void*>> ipc_opened_h;
    bool team_connected = false;
    bool halo_dirty = false;  // LOCAL set_wavefield in a team: exchange before the next run
    int64_t nz_lo = 0;
    unsigned long long epoch = 1;
    // stats
    aw_run_stats stats{};
    int64_t launch_count = 0;  // kernels launched since creation
    // device arenas of the sparse data (grown, never shrunk: no allocation in steady state)
    char* src_arena = nullptr;
    size_t src_cap = 0;
    char* rec_arena = nullptr;
    size_t rec_cap = 0;
    // NEXT-3 FWI gradient: adjoint injection tables (receivers as sources), per-call buffers,
    // the forward history ring + checkpoint pool (kept between calls)
    std::vector<double> rec_w64;           // receivers' fp64 multilinear weights [nr][nc]
    bool adj_valid = false;                // adjoint tables built for the current receivers
    int adj_nuc = 0, adj_nent = 0;
    std::vector<int64_t> h_adj_lin;
    std::vector<int> h_adj_ptr;
    char* adj_arena = nullptr;
    size_t adj_cap = 0;
    int64_t* d_adj_off = nullptr;
    int* d_adj_plane = nullptr;
    int* d_adj_ptr = nullptr;
    int* d_adj_src = nullptr;
    int64_t* d_adj_moff = nullptr;
    double* d_adj_w64 = nullptr;
    float* d_adj_s = nullptr;
    char* fwi_arena = nullptr;             // d_obs, residual, adjoint wavelet, J, G
    size_t fwi_cap = 0;
    float* fwi_pool = nullptr;             // nbuf wavefield-sized buffers
    int64_t fwi_pool_nbuf = 0;
    int opt_ckpt = 0;                      // AW_OPT_CHECKPOINT_STEPS (0 = auto)
    int opt_accum = 0;                     // AW_OPT_FWI_ACCUMULATE
    bool acc_valid = false;                // d_Gacc holds the sum of the gradients since the option was set
    float* d_Gacc = nullptr;
    // NEXT-1 temporal blocking (two steps per launch): third wavefield buffer, readiness
    int opt_temporal = 0;                  // AW_OPT_TEMPORAL (off: measured slower on B200, DESIGN.md NEXT-1)
    int opt_resident = AW_RESIDENT_AUTO;   // AW_OPT_RESIDENT (small-grid multi-step kernel)
    bool resident_used = false;            // the last run used the resident kernel
    bool resident2d_used = false;          // the last run used the 2D one-CTA resident kernel
    std::vector<int64_t> h_rec_off;        // owned receivers' corner offsets (resident kernel's item lists)
    bool rec_items_dirty = true;           // h_rec_off changed since the lists were built
    float* ubuf_spare = nullptr;
    bool tb_ready = false;
    int n_timed = 0;                       // timed stencil launches of the last run (AW_OPT_TIMING)
    unsigned long long* ts0 = nullptr;     // AW_OPT_TIMING = 2: per-launch first-CTA start (device ns)
    unsigned long long* ts1 = nullptr;     //                    per-launch last-CTA end
    int ts_cap = 0;
    bool ts_on = false;                    // the last run recorded device timestamps
    bool wave_invalid = false;             // after aw_fwi_gradient until aw_reset / aw_set_wavefield
};

namespace {

#define CK(call)                                                                                          \
    do {                                                                                                  \
        cudaError_t e_ = (call);                                                                          \
        if (e_ != cudaSuccess) {                                                                          \
            g->poisoned = true;                                                                           \
            return fail(AW_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
        }                                                                                                 \
    } while (0)

#define CHECK_STATE(g)                                                                 \
    do {                                                                               \
        if (!(g)) return fail(AW_EINVAL, "null grid handle");                          \
        if ((g)->poisoned) return fail(AW_ESTATE, "handle poisoned by an earlier CUDA error"); \
    } while (0)

void free_graphs(aw_grid* g) {
    for (auto& kv : g->graphs)
        for (auto& e : kv.second) cudaGraphExecDestroy(e.exec);
    g->graphs.clear();
}

// The library's own device allocations are tracked (aw_run_stats.lib_device_bytes).
cudaError_t lmalloc(aw_grid* g, void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) g->lib_allocs[*p] = bytes;
    return e;
}
bool in_ws(const aw_grid* g, const void* p) {
    return g->ws && p >= (const void*)g->ws && p < (const void*)(g->ws + g->ws_bytes);
}
template <class T>
void dfree(aw_grid* g, T*& p) {  // frees library memory only (never a pointer into the workspace)
    if (p && !in_ws(g, p)) {
        cudaFree((void*)p);
        g->lib_allocs.erase((void*)p);
    }
    p = nullptr;
}
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Synchronise the library stream with the caller's stream (entry) ...
aw_status enter(aw_grid* g) {
    cudaError_t e = cudaSetDevice(g->device);
    if (e != cudaSuccess) {
        g->poisoned = true;
        return fail(AW_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    }
    if (g->ext) {
        CK(cudaEventRecord(g->ev_sync, g->ext));
        CK(cudaStreamWaitEvent(g->s, g->ev_sync, 0));
    }
    return AW_OK;
}
// ... and back (exit): the caller's stream waits for the library's work.
aw_status leave(aw_grid* g) {
    if (g->ext) {
        CK(cudaEventRecord(g->ev_sync, g->s));
        CK(cudaStreamWaitEvent(g->ext, g->ev_sync, 0));
    }
    return AW_OK;
}

// Copy a dense [rows][nx] fp32 array (host or device) into a pitched device array.
aw_status copy_in(aw_grid* g, float* dst, int64_t dst_pitch, const float* src, int64_t nx, int64_t rows) {
    if (rows <= 0) return AW_OK;
    cudaMemcpyKind kind = ptr_kind(src) == PK_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpy2DAsync(dst, dst_pitch * sizeof(float), src, nx * sizeof(float), nx * sizeof(float), rows, kind,
                         g->s));
    return AW_OK;
}
aw_status copy_out(aw_grid* g, float* dst, const float* src, int64_t src_pitch, int64_t nx, int64_t rows) {
    if (rows <= 0) return AW_OK;
    cudaMemcpyKind kind = ptr_kind(dst) == PK_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(cudaMemcpy2DAsync(dst, nx * sizeof(float), src, src_pitch * sizeof(float), nx * sizeof(float), rows, kind,
                         g->s));
    return AW_OK;
}

int64_t rows_per_plane(const aw_grid* g) { return g->ndim == 3 ? g->shape[1] : 1; }
int64_t nx_of(const aw_grid* g) { return g->shape[g->ndim - 1]; }

// Sparse setup for one point: corners (global linear index,
// -1 = skipped) and fp64 weights.  Returns false if the point is outside.
bool locate(const aw_grid* g, const double* x, int64_t* corner, double* w, int64_t* base0) {
    int64_t i[3];
    double f[3];
    for (int d = 0; d < g->ndim; ++d) {
        double p = (x[d] - g->origin[d]) / g->h[d];
        if (!(p >= 0.0 && p <= (double)(g->shape[d] - 1))) return false;
        double fl = std::floor(p);
        i[d] = (int64_t)fl;
        f[d] = p - fl;
    }
    *base0 = i[0];
    const int nc = 1 << g->ndim;
    for (int beta = 0; beta < nc; ++beta) {
        int64_t lin = 0;
        double wt = 1.0;
        bool skip = false;
        for (int d = 0; d < g->ndim; ++d) {
            const int up = (beta >> d) & 1;
            const int64_t idx = i[d] + up;
            if (idx >= g->shape[d]) skip = true;
            const double wd = up ? f[d] : (1.0 - f[d]);
            wt = (d == 0) ? wd : wt * wd;
            lin = lin * g->shape[d] + idx;
        }
        corner[beta] = skip ? -1 : lin;
        w[beta] = skip ? 0.0 : wt;
    }
    return true;
}

int64_t lin_div(const aw_grid* g) { return g->ndim == 3 ? g->shape[1] * g->shape[2] : g->shape[1]; }

// global linear index -> (plane relative to z0, offset in a wavefield buffer, model index)
void lin_to_local(const aw_grid* g, int64_t lin, int64_t* zl, int64_t* uoff, int64_t* moff) {
    const int64_t per_plane = lin_div(g);
    int64_t z = lin / per_plane;
    int64_t rem = lin % per_plane;
    int64_t y = 0, x = rem;
    if (g->ndim == 3) {
        y = rem / g->shape[2];
        x = rem % g->shape[2];
    }
    *zl = z - g->z0;
    *moff = (*zl) * g->geom.plane + y * g->geom.pitch + x;
    *uoff = *moff + (int64_t)g->R * g->geom.plane;
}


// Injection CSR over this rank's owned corners of n points: entries sorted by
// corner (global linear index) ascending, then point index, then corner bit pattern.  Used for the
// sources and, in the FWI adjoint (NEXT-3), for the receivers injecting the residual.
struct E {
    int64_t lin;
    int s, beta;
};
struct InjTables {
    std::vector<E> ents;
    std::vector<int64_t> off, moff, lin;   // per unique corner: buffer offset; per entry: model offset
    std::vector<int> plane, ptr, src, ent_src, ent_beta;
    std::vector<double> w;
};
void build_injection(const aw_grid* g, int n, const std::vector<int64_t>& corner, const std::vector<double>& w,
                     InjTables* t) {
    const int nc = 1 << g->ndim;
    for (int s = 0; s < n; ++s)
        for (int beta = 0; beta < nc; ++beta) {
            int64_t lin = corner[(size_t)s * nc + beta];
            if (lin < 0) continue;
            int64_t z = lin / lin_div(g);
            if (z < g->z0 || z >= g->z0 + g->geom.nz) continue;
            t->ents.push_back({lin, s, beta});
        }
    std::stable_sort(t->ents.begin(), t->ents.end(), [](const E& a, const E& b) {
        return a.lin != b.lin ? a.lin < b.lin : (a.s != b.s ? a.s < b.s : a.beta < b.beta);
    });
    const std::vector<E>& ents = t->ents;
    for (size_t e = 0; e < ents.size(); ++e) {
        int64_t zl, uoff, moff;
        lin_to_local(g, ents[e].lin, &zl, &uoff, &moff);
        if (e == 0 || ents[e].lin != ents[e - 1].lin) {
            t->off.push_back(uoff);
            t->plane.push_back((int)zl);
            t->ptr.push_back((int)e);
            t->lin.push_back(ents[e].lin);
        }
        t->moff.push_back(moff);
        t->src.push_back(ents[e].s);
        t->w.push_back(w[(size_t)ents[e].s * nc + ents[e].beta]);
        t->ent_src.push_back(ents[e].s);
        t->ent_beta.push_back(ents[e].beta);
    }
    t->ptr.push_back((int)ents.size());
}

// The dense block: u^a, u^b (wavefield layout, planes [-R, nz+R)), then four model-layout arrays
// (m, eta, b, a).  aw_set_model swaps the roles of m<->b and eta<->a (staging), so after the first
// placement the pointers, not the offsets, say which array is which.
constexpr size_t kDenseAlign = 4096;
// AW_RESIDENT_AUTO picks the resident multi-step kernel up to this many points (~128 MB at 16 B per
// point: the working set fits in the 126 MB L2, and a step takes microseconds, so launch gaps matter)
constexpr int64_t kResidentAutoPoints = 8LL << 20;
void place_dense(aw_grid* g, char* base) {
    const size_t U = align_up(g->ubytes, kDenseAlign), M = align_up(g->mbytes, kDenseAlign);
    g->dense = base;
    g->ubuf[0] = (float*)base;
    g->ubuf[1] = (float*)(base + U);
    g->m = (float*)(base + 2 * U);
    g->eta = (float*)(base + 2 * U + M);
    g->b = (float*)(base + 2 * U + 2 * M);
    g->a = (float*)(base + 2 * U + 3 * M);
}
#define NEED_DENSE(g)                                                                                   \
    do {                                                                                                \
        if (!(g)->dense) return fail(AW_ESTATE, "no device memory bound yet (AW_DIST_WORKSPACE): call "   \
                                                "aw_bind_workspace first");                             \
    } while (0)

unsigned long long enc(const aw_grid* g, int64_t level) {
    return (g->epoch << 32) + (unsigned long long)(level + 1);
}
bool team_mode(const aw_grid* g) { return g->world > 1; }

void free_sources(aw_grid* g) {  // the device arrays are views into g->src_arena
    g->d_wavelet = nullptr;
    g->d_inj_off = nullptr;
    g->d_inj_plane = nullptr;
    g->d_inj_ptr = nullptr;
    g->d_inj_src = nullptr;
    g->d_inj_moff = nullptr;
    g->d_inj_w64 = nullptr;
    g->d_inj_s = nullptr;
    g->ns = g->src_nt = g->nuc = g->nent = 0;
    g->src_need = 0;
    g->src_corner_lin.clear();
    g->src_w64.clear();
    g->ent_src.clear();
    g->ent_beta.clear();
    g->h_inj_lin.clear();
    g->h_inj_ptr.clear();
}
void free_receivers(aw_grid* g) {  // views into g->rec_arena
    g->d_rec_id = nullptr;
    g->d_rec_off = nullptr;
    g->d_rec_w = nullptr;
    g->d_traces = nullptr;
    g->nr = g->rec_nt = g->nrl = 0;
    g->rec_need = 0;
    g->rec_corner_lin.clear();
    g->rec_w32.clear();
    g->rec_w64.clear();
    g->h_rec_off.clear();
    g->rec_items_dirty = true;
    g->adj_valid = false;
}

// Packs several host arrays into one device arena (16-B aligned slices) with a single copy.
struct Packer {
    std::vector<char> host;
    size_t off = 0;
    template <class T>
    size_t add(const std::vector<T>& v) {  // returns the slice offset
        size_t o = off;
        off = (off + v.size() * sizeof(T) + 15) / 16 * 16;
        host.resize(off);
        if (!v.empty()) std::memcpy(host.data() + o, v.data(), v.size() * sizeof(T));
        return o;
    }
    size_t reserve(size_t bytes) {  // uninitialised slice (filled on the device)
        size_t o = off;
        off = (off + bytes + 15) / 16 * 16;
        return o;
    }
};

// Asynchronous upload of host bytes through the handle's pinned staging buffer (stream-ordered on g->s).
aw_status upload(aw_grid* g, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return AW_OK;
    if (g->stage_pending) {  // the previous upload must have left the buffer
        CK(cudaEventSynchronize(g->ev_stage));
        g->stage_pending = false;
    }
    if (g->h_stage_cap < bytes) {
        if (g->h_stage) CK(cudaFreeHost(g->h_stage));
        g->h_stage = nullptr;
        g->h_stage_cap = 0;
        const size_t want = std::max<size_t>(bytes + bytes / 2, 4096);
        CK(cudaHostAlloc((void**)&g->h_stage, want, cudaHostAllocDefault));
        g->h_stage_cap = want;
    }
    std::memcpy(g->h_stage, src, bytes);
    CK(cudaMemcpyAsync(dst, g->h_stage, bytes, cudaMemcpyHostToDevice, g->s));
    CK(cudaEventRecord(g->ev_stage, g->s));
    g->stage_pending = true;
    return AW_OK;
}

// Queue a copy of the device control block into the pinned staging buffer and synchronise the stream:
// afterwards g->h_stage holds the DevCtl as of the end of the queued work (one round trip).
aw_status readback_ctl(aw_grid* g) {
    if (g->stage_pending) {
        CK(cudaEventSynchronize(g->ev_stage));
        g->stage_pending = false;
    }
    if (g->h_stage_cap < sizeof(aw::DevCtl)) {
        if (g->h_stage) CK(cudaFreeHost(g->h_stage));
        g->h_stage = nullptr;
        g->h_stage_cap = 0;
        CK(cudaHostAlloc((void**)&g->h_stage, 4096, cudaHostAllocDefault));
        g->h_stage_cap = 4096;
    }
    CK(cudaMemcpyAsync(g->h_stage, g->ctl, sizeof(aw::DevCtl), cudaMemcpyDeviceToHost, g->s));
    CK(cudaStreamSynchronize(g->s));
    return AW_OK;
}

// slot: 0 = the sources' arena, 1 = the receivers' (placed in the bound workspace when they fit),
// -1 = an arena that always lives in library memory (FWI)
aw_status ensure_arena(aw_grid* g, char** arena, size_t* cap, size_t bytes, int slot = -1) {
    if (slot >= 0 && g->ws && g->ws_slot_cap[slot] >= bytes) {
        char* w = g->ws + g->ws_slot_off[slot];
        if (*arena != w) {
            if (*arena && !in_ws(g, *arena)) {
                CK(cudaStreamSynchronize(g->s));
                dfree(g, *arena);
            }
            *arena = w;
            *cap = g->ws_slot_cap[slot];
        }
        return AW_OK;
    }
    if (*cap >= bytes && *arena) return AW_OK;
    if (*arena) {
        CK(cudaStreamSynchronize(g->s));
        dfree(g, *arena);
        *arena = nullptr;
        *cap = 0;
    }
    size_t want = bytes + bytes / 2 + 256;
    cudaError_t e = lmalloc(g, (void**)arena, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? AW_ENOMEM : AW_ECUDA, "sparse arena: %s", cudaGetErrorString(e));
    }
    *cap = want;
    return AW_OK;
}

aw::Sparse sparse_view(const aw_grid* g) {
    aw::Sparse sp;
    std::memset(&sp, 0, sizeof sp);  // padding too: the bytes are part of graph signatures
    sp.nrl = g->nrl;
    sp.nr = g->nr;
    sp.rec_id = g->d_rec_id;
    sp.rec_off = g->d_rec_off;
    sp.rec_w = g->d_rec_w;
    sp.traces = g->d_traces;
    sp.nuc = g->nuc;
    sp.ns = g->ns;
    sp.inj_off = g->d_inj_off;
    sp.inj_plane = g->d_inj_plane;
    sp.inj_ptr = g->d_inj_ptr;
    sp.inj_src = g->d_inj_src;
    sp.inj_s = g->d_inj_s;
    sp.nent = g->nent;
    sp.wavelet = g->d_wavelet;
    sp.nc = 1 << g->ndim;
    return sp;
}

// dt-dependent tables: b, a, source scales, the streaming plan.
aw_status prepare(aw_grid* g, double dt) {
    if (g->coeffs_valid && g->dt_set && g->dt == dt) return AW_OK;
    int64_t n = (int64_t)g->geom.nz * g->geom.plane;
    CK(aw::launch_coeffs(g->m, g->have_damp ? g->eta : nullptr, g->b, g->have_damp ? g->a : nullptr, n, dt, g->s));
    CK(aw::launch_source_scales(g->m, g->have_damp ? g->eta : nullptr, g->d_inj_moff, g->d_inj_w64, g->d_inj_s,
                                g->nent, dt, g->s));
    g->launch_count += 1 + (g->nent > 0 ? 1 : 0);
    const bool want_stream = g->opt_kernel != AW_KERNEL_V1 && g->ndim == 3;
    if (g->plan && !want_stream) {
        aw::stream_release(g->plan);
        g->plan = nullptr;
    }
    g->kernel_used = AW_KERNEL_V1;
    g->tb_ready = false;
    g->eta_tiles_pct = g->have_damp ? 100 : 0;
    if (want_stream) {
        const float* ub[2] = {g->ubuf[0], g->ubuf[1]};
        const float* a = g->have_damp ? g->a : nullptr;
        // the plan (tensor maps, grid, flag buffer) is built once per handle; later runs only
        // refresh the maps and the eta flags (no allocation, no host synchronisation)
        cudaError_t e = g->plan ? aw::stream_refresh(g->plan, g->geom, ub, g->b, a, g->s)
                                : aw::stream_prepare(g->geom, ub, g->b, a, &g->plan, g->s);
        if (e == cudaSuccess)
            e = aw::stream_set_injection(g->plan, g->geom, g->z0, g->h_inj_lin.data(), g->h_inj_ptr.data(), g->nuc,
                                         g->s);
        if (e == cudaSuccess) {
            g->kernel_used = AW_KERNEL_STREAM;
            g->launch_count += a ? 2 : 0;
            g->tb_ready = false;
            if (g->opt_temporal && !team_mode(g)) {
                if (!g->ubuf_spare) {
                    CK(lmalloc(g, (void**)&g->ubuf_spare, g->ubytes));
                    CK(cudaMemsetAsync(g->ubuf_spare, 0, g->ubytes, g->s));  // zero halo planes for good
                }
                CK(aw::stream_tb_prepare(g->plan, g->geom, 0));
                g->tb_ready = true;
            }
        } else if (e == cudaErrorNotSupported) {
            cudaGetLastError();
            if (g->opt_kernel == AW_KERNEL_STREAM)
                return fail(AW_EUNSUPPORTED, "no streaming-kernel specialisation for this configuration");
        } else {
            CK(e);
        }
    } else if (g->opt_kernel == AW_KERNEL_STREAM) {
        return fail(AW_EUNSUPPORTED, "the streaming kernel is 3D only");
    } else if (g->ndim == 2 && g->opt_kernel == AW_KERNEL_AUTO && !team_mode(g)) {
        if (!g->t2) CK(aw::tile2d_prepare(g->geom, &g->t2));
        g->kernel_used = AW_KERNEL_TILE2D;
    }
    g->dt = dt;
    g->dt_set = true;
    g->coeffs_valid = true;
    return AW_OK;
}

// Enqueue one time step (local index i relative to *d_base) reading buffer
// `cur` (u^n) and writing buffer 1-cur (u^{n+1} over u^{n-1}).
aw_status enqueue_step(aw_grid* g, int i, int cur, cudaEvent_t e0, cudaEvent_t e1, int64_t* launches) {
    const int nxt = 1 - cur;
    if (team_mode(g)) {
        // the wanted level comes from the device (step base + i, epoch): graph-capturable
        CK(aw::launch_team_wait(g->ctl, g->halo.lo[0] != nullptr, g->halo.hi[0] != nullptr, i, g->s));
        ++*launches;
    }
    if (e0) CK(cudaEventRecord(e0, g->s));
    // receivers + injection inside the stencil kernel (AW_NO_FUSE=1: separate sparse kernel, for A/B runs)
    static const bool no_fuse = aw::dev_knob("AW_NO_FUSE") != nullptr;
    const bool fused = g->kernel_used == AW_KERNEL_STREAM && !no_fuse;
    if (g->kernel_used == AW_KERNEL_STREAM) {
        aw::Sparse sp = sparse_view(g);
        if (!fused) sp.nrl = sp.nuc = 0;
        CK(aw::launch_stencil_stream(g->plan, g->geom, g->coefs, cur, g->ubuf[cur], g->ubuf[nxt], g->b,
                                     g->have_damp ? g->a : nullptr, g->halo, nxt, sp, g->d_base, i, g->s));
    } else if (g->kernel_used == AW_KERNEL_TILE2D) {
        CK(aw::launch_stencil_tile2d(g->t2, g->geom, g->coefs, g->ubuf[cur], g->ubuf[nxt], g->ubuf[nxt], g->b,
                                     g->have_damp ? g->a : nullptr, g->s));
    } else {
        CK(aw::launch_stencil_v1(g->geom, g->coefs, g->ubuf[cur], g->ubuf[nxt], g->ubuf[nxt], g->b,
                                 g->have_damp ? g->a : nullptr,
                                 g->halo, nxt, g->s));
    }
    ++*launches;
    if (e1) CK(cudaEventRecord(e1, g->s));
    if (!fused && g->nrl + g->nuc > 0) {
        CK(aw::launch_sparse_step(g->geom, sparse_view(g), g->ubuf[cur], g->ubuf[nxt], g->d_base, i, g->halo, nxt,
                                  g->s));
        ++*launches;
    }
    // (the 3D streaming kernel raises the neighbours' flags itself, as soon as its boundary items are done)
    if (team_mode(g) && (g->peer_flag_lo || g->peer_flag_hi) && g->kernel_used != AW_KERNEL_STREAM) {
        CK(aw::launch_team_signal(g->peer_flag_lo, g->peer_flag_hi, g->ctl, i, g->s));
        ++*launches;
    }
    return AW_OK;
}

// Every value a captured step launch takes from the handle (see enqueue_step).
std::string graph_signature(const aw_grid* g) {
    std::string sig;
    auto put = [&](const void* p, size_t n) { sig.append((const char*)p, n); };
    put(&g->kernel_used, sizeof g->kernel_used);
    put(g->ubuf, sizeof g->ubuf);
    put(&g->b, sizeof g->b);
    const float* a = g->have_damp ? g->a : nullptr;
    put(&a, sizeof a);
    put(&g->coefs, sizeof g->coefs);
    put(&g->geom, sizeof g->geom);
    const aw::Sparse sp = sparse_view(g);
    put(&sp, sizeof sp);
    put(&g->halo, sizeof g->halo);
    put(&g->peer_flag_lo, sizeof g->peer_flag_lo);
    put(&g->peer_flag_hi, sizeof g->peer_flag_hi);
    put(&g->ctl, sizeof g->ctl);
    put(&g->t2, sizeof g->t2);
    put(&g->plan, sizeof g->plan);
    aw::stream_plan_signature(g->plan, &sig);
    return sig;
}

aw_status get_graph(aw_grid* g, int G, int cur, cudaGraphExec_t* out) {
    const int64_t key = ((int64_t)G << 1) | cur;
    const std::string sig = graph_signature(g);
    std::vector<aw_grid::GraphEntry>& ents = g->graphs[key];
    for (size_t k = 0; k < ents.size(); ++k)
        if (ents[k].sig == sig) {
            *out = ents[k].exec;
            if (k) std::swap(ents[k], ents[0]);  // most recent first
            return AW_OK;
        }
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(g->s, cudaStreamCaptureModeThreadLocal));
    int64_t dummy = 0;
    int c = cur;
    aw_status st = AW_OK;
    for (int i = 0; i < G && st == AW_OK; ++i) {
        st = enqueue_step(g, i, c, nullptr, nullptr, &dummy);
        c = 1 - c;
    }
    if (st == AW_OK) {
        cudaError_t e = aw::launch_advance(g->d_base, G, g->s);
        if (e != cudaSuccess) st = fail(AW_ECUDA, "advance: %s", cudaGetErrorString(e));
    }
    cudaError_t e = cudaStreamEndCapture(g->s, &graph);
    if (st != AW_OK) {
        g->poisoned = true;
        return st;
    }
    CK(e);
    cudaGraphExec_t exec;
    CK(cudaGraphInstantiate(&exec, graph, 0));
    cudaGraphDestroy(graph);
    // two entries cover aw_set_model's alternating staging arrays; older ones are dropped
    constexpr size_t kKeep = 3;
    if (ents.size() >= kKeep) {
        CK(cudaStreamSynchronize(g->s));  // the dropped graph may still be in flight
        cudaGraphExecDestroy(ents.back().exec);
        ents.pop_back();
    }
    ents.insert(ents.begin(), aw_grid::GraphEntry{sig, exec});
    *out = exec;
    return AW_OK;
}

aw_status check_run_args(aw_grid* g, int nt, double dt) {
    if (nt < 0) return fail(AW_EINVAL, "nt must be >= 0 (got %d)", nt);
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(AW_EINVAL, "dt must be finite and > 0");
    if (!g->have_model) return fail(AW_ESTATE, "aw_set_model has not been called");
    if (g->dt_set && g->steps > 0 && dt != g->dt)
        return fail(AW_EINVAL, "dt is fixed at %.17g until aw_reset (got %.17g)", g->dt, dt);
    if (g->ns > 0 && g->steps + nt > g->src_nt)
        return fail(AW_EINVAL, "wavelet covers %d steps, run needs %lld", g->src_nt, (long long)(g->steps + nt));
    if (g->nr > 0 && g->steps + nt > g->rec_nt)
        return fail(AW_EINVAL, "trace buffer covers %d steps, run needs %lld", g->rec_nt,
                    (long long)(g->steps + nt));
    return AW_OK;
}

// Copy my boundary planes of the current level into the neighbours' halos
// (after a LOCAL set_wavefield) and publish the level.
aw_status team_prologue(aw_grid* g) {
    const int64_t R = g->R, plane = g->geom.plane;
    const int c = g->cur;
    if (g->halo.lo[c]) {
        CK(cudaMemcpyAsync(g->halo.lo[c] + g->halo.lo_off, g->ubuf[c] + R * plane, R * plane * sizeof(float),
                           cudaMemcpyDefault, g->s));
    }
    if (g->halo.hi[c]) {
        CK(cudaMemcpyAsync(g->halo.hi[c] + g->halo.hi_off, g->ubuf[c] + (int64_t)g->geom.nz * plane,
                           R * plane * sizeof(float), cudaMemcpyDefault, g->s));
    }
    CK(aw::launch_team_raise(g->peer_flag_lo, g->peer_flag_hi, enc(g, g->steps), g->s));
    return AW_OK;
}

aw_status run_begin(aw_grid* g, int nt, double dt) {
    NEED_DENSE(g);
    aw_status st = check_run_args(g, nt, dt);
    if (st) return st;
    if (team_mode(g) && !g->team_connected) return fail(AW_ESTATE, "team handle is not connected");
    if ((st = enter(g))) return st;
    if ((st = prepare(g, dt))) return st;
    if (g->halo_dirty) {
        if ((st = team_prologue(g))) return st;
        g->halo_dirty = false;
    }
    // small grids: the resident multi-step kernel (one launch for the run, per-item step counters)
    const int64_t npts = (int64_t)g->geom.nz * g->geom.ny * g->geom.nx;
    g->resident_used = g->kernel_used == AW_KERNEL_STREAM && !team_mode(g) && !(g->tb_ready && nt >= 2) &&
                       g->opt_timing != 1 &&
                       (g->opt_resident == AW_RESIDENT_ON ||
                        (g->opt_resident == AW_RESIDENT_AUTO && npts <= kResidentAutoPoints)) &&
                       aw::stream_resident_ready(g->plan);
    // small 2D grids: one CTA holds the grid in shared memory for the whole run
    g->resident2d_used = g->kernel_used == AW_KERNEL_TILE2D && !team_mode(g) && g->opt_resident != AW_RESIDENT_OFF &&
                         aw::resident2d_fits(g->geom, sparse_view(g), g->have_damp);
    if (g->resident_used) {
        if (g->rec_items_dirty) {
            CK(aw::stream_set_receivers(g->plan, g->geom, g->h_rec_off.data(), g->nrl, 1 << g->ndim, g->s));
            g->rec_items_dirty = false;
        }
        CK(aw::stream_resident_begin(g->plan, g->s));
    }
    // AW_OPT_TIMING = 2: the streaming kernel stamps its first-CTA start / last-CTA end per launch
    // (production path, CUDA graphs kept); the arrays are sized for the run and reset here
    g->ts_on = g->opt_timing == 2 && g->kernel_used == AW_KERNEL_STREAM && !(g->tb_ready && nt >= 2);
    if (g->ts_on) {
        if (g->ts_cap < nt) {
            const int cap = std::max(nt, 1024);
            dfree(g, g->ts0);
            dfree(g, g->ts1);
            CK(lmalloc(g, (void**)&g->ts0, (size_t)cap * sizeof(unsigned long long)));
            CK(lmalloc(g, (void**)&g->ts1, (size_t)cap * sizeof(unsigned long long)));
            g->ts_cap = cap;
        }
        CK(cudaMemsetAsync(g->ts0, 0xff, (size_t)g->ts_cap * sizeof(unsigned long long), g->s));
        CK(cudaMemsetAsync(g->ts1, 0, (size_t)g->ts_cap * sizeof(unsigned long long), g->s));
        aw::stream_set_timestamps(g->plan, g->ts0, g->ts1, g->ts_cap);
    } else if (g->plan) {
        aw::stream_set_timestamps(g->plan, nullptr, nullptr, 0);
    }
    CK(cudaEventRecord(g->ev_t0, g->s));
    CK(aw::launch_run_init(g->ctl, g->steps, g->s));  // step base, NaN flag, exchange-wait counters
    g->launch_count += 1;
    return AW_OK;
}

// Enqueue the nt steps.  Direct launches (with per-stencil events when
// timing) or graphs of G steps.
aw_status run_enqueue(aw_grid* g, int nt, int64_t* launches) {
    const bool timing = g->opt_timing == 1;  // per-launch events (direct launches); 2 = device timestamps
    const int G = g->opt_graph;
    if (timing && (int64_t)g->tev.size() < 2 * (int64_t)nt) {
        while ((int64_t)g->tev.size() < 2 * (int64_t)nt) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            g->tev.push_back(e);
        }
    }
    g->n_timed = timing ? nt : 0;
    static const bool no_fuse = aw::dev_knob("AW_NO_FUSE") != nullptr;
    if (g->tb_ready && !team_mode(g) && !no_fuse && nt >= 2) {
        // NEXT-1: two steps per launch over three rotating buffers (direct launches, one per pass)
        const float* a = g->have_damp ? g->a : nullptr;
        const aw::Sparse sp = sparse_view(g);
        int done = 0, timed = 0;
        while (nt - done >= 2) {
            float* X = g->ubuf[g->cur];
            float* Y = g->ubuf[1 - g->cur];
            float* V = g->ubuf_spare;
            if (timing) CK(cudaEventRecord(g->tev[2 * timed], g->s));
            CK(aw::launch_stencil_tb(g->plan, g->geom, g->coefs, X, Y, V, g->b, a, sp, g->d_base, done, g->s));
            if (timing) CK(cudaEventRecord(g->tev[2 * timed + 1], g->s));
            ++timed;
            ++*launches;
            g->ubuf[g->cur] = Y;      // u^{n+2}
            g->ubuf[1 - g->cur] = V;  // u^{n+1}
            g->ubuf_spare = X;
            done += 2;
        }
        if (done < nt) {  // odd remainder: one ordinary step on the permuted buffers
            if (timing) CK(cudaEventRecord(g->tev[2 * timed], g->s));
            CK(aw::launch_stencil_stream_bufs(g->plan, g->geom, g->coefs, g->ubuf[g->cur], g->ubuf[1 - g->cur],
                                              g->ubuf[1 - g->cur], g->b, a, sp, 0, g->d_base, done, g->s));
            if (timing) CK(cudaEventRecord(g->tev[2 * timed + 1], g->s));
            ++timed;
            ++*launches;
            g->cur = 1 - g->cur;
        }
        g->n_timed = timing ? timed : 0;
        // the per-parity maps and any captured graphs refer to the old buffer order
        const float* ub[2] = {g->ubuf[0], g->ubuf[1]};
        CK(aw::stream_remap(g->plan, g->geom, ub, g->b, a));
        free_graphs(g);
        return AW_OK;
    }
    if (g->resident2d_used) {
        if (timing) CK(cudaEventRecord(g->tev[0], g->s));
        CK(aw::launch_stencil_resident2d(g->geom, g->coefs, g->ubuf[g->cur], g->ubuf[1 - g->cur], g->b,
                                         g->have_damp ? g->a : nullptr, sparse_view(g), g->d_base, 0, nt, g->s));
        if (timing) CK(cudaEventRecord(g->tev[1], g->s));
        g->n_timed = timing && nt > 0 ? 1 : 0;
        *launches += nt > 0 ? 1 : 0;
        if (nt & 1) g->cur = 1 - g->cur;
        return AW_OK;
    }
    if (g->resident_used) {
        // small grids: every step of the run in one launch of the resident kernel
        CK(aw::launch_stencil_resident(g->plan, g->geom, g->coefs, g->cur, g->ubuf, g->b,
                                       g->have_damp ? g->a : nullptr, sparse_view(g), g->d_base, 0, nt, g->s));
        ++*launches;
        if (nt & 1) g->cur = 1 - g->cur;
        return AW_OK;
    }
    int done = 0;
    if (!timing && G > 0) {  // team steps too: their waits and signals read the level from the device
        while (nt - done >= G) {
            cudaGraphExec_t exec;
            aw_status st = get_graph(g, G, g->cur, &exec);
            if (st) return st;
            CK(cudaGraphLaunch(exec, g->s));
            const int per_step = 1 + (g->kernel_used != AW_KERNEL_STREAM && g->nrl + g->nuc > 0 ? 1 : 0) +
                                 (team_mode(g) ? 1 + ((g->peer_flag_lo || g->peer_flag_hi) &&
                                                              g->kernel_used != AW_KERNEL_STREAM ? 1 : 0) : 0);
            *launches += (int64_t)G * per_step + 1;
            done += G;
            if (G & 1) g->cur = 1 - g->cur;
        }
        // the graphs advanced *d_base to steps + done
    }
    const int first = done;
    for (int i = 0; done < nt; ++i, ++done) {
        cudaEvent_t e0 = timing ? g->tev[2 * i] : nullptr, e1 = timing ? g->tev[2 * i + 1] : nullptr;
        aw_status st = enqueue_step(g, done - first, g->cur, e0, e1, launches);
        if (st) return st;
        g->cur = 1 - g->cur;
    }
    return AW_OK;
}

aw_status run_end(aw_grid* g, int nt, int64_t launches) {
    const int64_t t0 = g->steps;
    if (g->opt_check) {
        CK(aw::launch_check_finite(g->geom, g->ubuf[g->cur], g->nr > 0 ? g->d_traces : nullptr, t0, t0 + nt,
                                   g->nr, g->d_flag, g->s));
        ++launches;
    }
    CK(cudaEventRecord(g->ev_t1, g->s));
    // the control block comes back with the run's own synchronisation (pinned staging, no second
    // round trip)
    aw_status st = readback_ctl(g);
    if (st) return st;
    if ((st = leave(g))) return st;
    aw::DevCtl ctl;
    std::memcpy(&ctl, g->h_stage, sizeof ctl);
    const unsigned flag = ctl.flag;
    g->stats.ms_exchange = (double)ctl.wait_ns * 1e-6;
    g->stats.exchange_waits = (int64_t)ctl.nwait;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, g->ev_t0, g->ev_t1));
    g->stats.ms_total = ms;
    g->stats.launches = launches;
    g->launch_count += launches;
    g->stats.launches_total = g->launch_count;
    g->stats.points = (int64_t)g->geom.nz * g->geom.ny * g->geom.nx;
    g->stats.gpts = ms > 0 ? (double)g->stats.points * nt / (ms * 1e6) : 0.0;
    g->stats.kernel = g->kernel_used;
    g->stats.resident = g->resident_used || g->resident2d_used ? 1 : 0;
    if (g->plan) g->eta_tiles_pct = aw::stream_eta_tiles_pct(g->plan);
    g->stats.eta_tiles = g->eta_tiles_pct;
    if (g->ts_on) {
        std::vector<unsigned long long> t0(g->ts_cap), t1(g->ts_cap);
        CK(cudaMemcpy(t0.data(), g->ts0, t0.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(t1.data(), g->ts1, t1.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        double sum_ns = 0.0;
        int64_t n = 0;
        for (int k = 0; k < g->ts_cap; ++k)
            if (t1[k] != 0 && t0[k] != ~0ull && t1[k] >= t0[k]) {
                sum_ns += (double)(t1[k] - t0[k]);
                ++n;
            }
        g->stats.ms_stencil = sum_ns * 1e-6;
        g->stats.n_stencil = g->resident_used ? (n > 0 ? nt : 0) : n;  // time steps the timed launches cover
        g->stats.timed_launches = n;
    } else if (g->opt_timing == 1) {
        double sum = 0.0;
        for (int i = 0; i < g->n_timed; ++i) {
            float e = 0.f;
            CK(cudaEventElapsedTime(&e, g->tev[2 * i], g->tev[2 * i + 1]));
            sum += e;
        }
        g->stats.ms_stencil = sum;
        g->stats.n_stencil = nt;  // time steps covered by the timed launches (two per temporal-blocking pass)
        g->stats.timed_launches = g->n_timed;
    } else {
        g->stats.ms_stencil = -1.0;
        g->stats.n_stencil = 0;
    }
    g->steps += nt;
    if (flag) return fail(AW_ENONFINITE, "NaN/Inf in the wavefield or traces after steps [%lld, %lld)",
                          (long long)t0, (long long)g->steps);
    return AW_OK;
}


// ---------------------------------------------------------------------------
// NEXT-3: adjoint-state FWI gradient (host orchestration; kernels in aw_fwi.cu)
// ---------------------------------------------------------------------------

// Adjoint injection tables: the receivers inject the residual like sources (DESIGN.md §3 Q24), so
// their corners get the source treatment -- CSR by corner then receiver, scales
// s = fl32(w64 dt^2 / (m_c + eta_c dt/2)) (computed on the device per call).
aw_status fwi_build_adjoint(aw_grid* g) {
    if (g->adj_valid) return AW_OK;
    InjTables t;
    build_injection(g, g->nr, g->rec_corner_lin, g->rec_w64, &t);
    g->h_adj_lin = t.lin;
    g->h_adj_ptr = t.ptr;
    g->adj_nuc = (int)t.off.size();
    g->adj_nent = (int)t.ents.size();
    Packer pk;
    const size_t o_off = pk.add(t.off), o_plane = pk.add(t.plane), o_ptr = pk.add(t.ptr), o_src = pk.add(t.src),
                 o_moff = pk.add(t.moff), o_w = pk.add(t.w);
    const size_t small = pk.off;
    const size_t o_s = pk.reserve((size_t)g->adj_nent * sizeof(float));
    aw_status st = ensure_arena(g, &g->adj_arena, &g->adj_cap, pk.off);
    if (st) return st;
    char* A = g->adj_arena;
    g->d_adj_off = (int64_t*)(A + o_off);
    g->d_adj_plane = (int*)(A + o_plane);
    g->d_adj_ptr = (int*)(A + o_ptr);
    g->d_adj_src = (int*)(A + o_src);
    g->d_adj_moff = (int64_t*)(A + o_moff);
    g->d_adj_w64 = (double*)(A + o_w);
    g->d_adj_s = (float*)(A + o_s);
    CK(cudaMemcpyAsync(A, pk.host.data(), small, cudaMemcpyHostToDevice, g->s));
    CK(cudaStreamSynchronize(g->s));  // pk.host dies here
    g->adj_valid = true;
    return AW_OK;
}

// Checkpoint schedule: segments of K steps; the history ring holds the K+2 levels of one segment,
// every later segment start keeps its two levels (u^{jK-1}, u^{jK}).  Buffers: K + 2 + 2(nseg - 1).
int64_t fwi_buffers(int nt, int K) { return (int64_t)K + 2 + 2 * ((int64_t)(nt + K - 1) / K - 1); }

int fwi_choose_K(const aw_grid* g, int nt, int64_t max_bufs) {
    if (g->opt_ckpt > 0) return std::min(g->opt_ckpt, nt);
    for (int K = nt; K >= 1; --K)  // largest segment that fits: fewest recomputed steps (nt - K)
        if (fwi_buffers(nt, K) <= max_bufs) return K;
    return 0;
}

// One time step on explicit buffers (history ring or adjoint pair); single slab.
aw_status fwi_step(aw_grid* g, const float* ucur, const float* uprev, float* unext, const aw::Sparse& sp, int inj_set,
                   int step_i, int64_t* launches) {
    const float* a = g->have_damp ? g->a : nullptr;
    if (g->kernel_used == AW_KERNEL_STREAM) {
        CK(aw::launch_stencil_stream_bufs(g->plan, g->geom, g->coefs, ucur, uprev, unext, g->b, a, sp, inj_set,
                                          g->d_base, step_i, g->s));
        ++*launches;
    } else {
        Halo none{};
        if (g->kernel_used == AW_KERNEL_TILE2D)
            CK(aw::launch_stencil_tile2d(g->t2, g->geom, g->coefs, ucur, uprev, unext, g->b, a, g->s));
        else
            CK(aw::launch_stencil_v1(g->geom, g->coefs, ucur, uprev, unext, g->b, a, none, 0, g->s));
        ++*launches;
        if (sp.nrl + sp.nuc > 0) {
            CK(aw::launch_sparse_step(g->geom, sp, ucur, unext, g->d_base, step_i, none, 0, g->s));
            ++*launches;
        }
    }
    return AW_OK;
}
}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* aw_last_error(void) { return g_err.c_str(); }

// internal (aw_internal.h): lets the other translation units set the thread-local error text
aw_status aw_internal_fail(aw_status st, const char* msg) { return fail(st, "%s", msg); }
int aw_abi_version(void) { return AW_ABI_VERSION; }

double aw_critical_dt(int ndim, const double* spacing, int space_order, double vmax) {
    if (ndim < 1 || ndim > 3 || !spacing || space_order < 2 || space_order > 16 || (space_order & 1) || !(vmax > 0))
        return 0.0;
    double c[AW_MAXR + 1];
    fd_weights(space_order, c);
    double S = std::fabs(c[0]);
    for (int j = 1; j <= space_order / 2; ++j) S += 2.0 * std::fabs(c[j]);
    double sum = 0.0;
    for (int d = 0; d < ndim; ++d) sum += S / (spacing[d] * spacing[d]);
    return 2.0 / (vmax * std::sqrt(sum));
}

aw_status aw_grid_create(aw_grid** out, int ndim, const int64_t* shape, const double* extent, const double* origin,
                         int space_order, const aw_dist* dist) {
    if (!out) return fail(AW_EINVAL, "out is NULL");
    *out = nullptr;
    if (ndim == 1) return fail(AW_EUNSUPPORTED, "1D grids are not supported");
    if (ndim < 2 || ndim > 3) return fail(AW_EINVAL, "ndim must be 2 or 3 (got %d)", ndim);
    if (!shape || !extent) return fail(AW_EINVAL, "shape/extent is NULL");
    if (space_order < 2 || space_order > 16 || (space_order & 1))
        return fail(AW_EINVAL, "space_order must be even in [2, 16] (got %d)", space_order);
    const int R = space_order / 2;
    for (int d = 0; d < ndim; ++d) {
        if (shape[d] < R + 1) return fail(AW_EINVAL, "shape[%d]=%lld < k/2+1", d, (long long)shape[d]);
        if (shape[d] > (1ll << 31) - 1) return fail(AW_EINVAL, "shape[%d] too large", d);
        if (!(extent[d] > 0.0) || !std::isfinite(extent[d])) return fail(AW_EINVAL, "extent[%d] must be > 0", d);
        if (origin && !std::isfinite(origin[d])) return fail(AW_EINVAL, "origin[%d] not finite", d);
    }
    int rank = 0, world = 1, device = -1;
    unsigned dflags = 0;
    cudaStream_t ext = nullptr;
    if (dist) {
        rank = dist->rank;
        world = dist->world;
        device = dist->device;
        ext = (cudaStream_t)dist->stream;
        dflags = dist->flags;
        if (dflags & ~(unsigned)AW_DIST_WORKSPACE) return fail(AW_EINVAL, "unknown aw_dist flags 0x%x", dflags);
        if (world < 1 || rank < 0 || rank >= world) return fail(AW_EINVAL, "bad rank/world %d/%d", rank, world);
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(AW_ECUDA, "no CUDA device available (libaw has no CPU fallback)");
    }
    if (device < 0) {
        if (cudaGetDevice(&device) != cudaSuccess) return fail(AW_ECUDA, "cudaGetDevice failed");
    }
    if (device >= ndev) return fail(AW_EINVAL, "device %d >= device count %d", device, ndev);
    // slab of axis 0: nearly equal split
    int64_t z0 = 0, nz = 0;
    {
        aw_status pst = aw_slab_partition(shape[0], world, rank, R, &z0, &nz);
        if (pst) return pst;
    }

    aw_grid* g = new aw_grid();
    g->ndim = ndim;
    g->so = space_order;
    g->R = R;
    g->rank = rank;
    g->world = world;
    g->device = device;
    g->z0 = z0;
    g->ext = ext;
    for (int d = 0; d < ndim; ++d) {
        g->shape[d] = shape[d];
        g->extent[d] = extent[d];
        g->origin[d] = origin ? origin[d] : 0.0;
        g->h[d] = extent[d] / (double)(shape[d] - 1);
    }
    Geom& G = g->geom;
    G.ndim = ndim;
    G.R = R;
    G.nz = (int)nz;
    G.ny = (int)rows_per_plane(g);
    G.nx = (int)nx_of(g);
    G.pitch = round_up(G.nx, AW_PITCH_ALIGN);
    G.plane = (int64_t)G.ny * G.pitch;
    // axis coefficients
    double c[AW_MAXR + 1];
    fd_weights(space_order, c);
    double s0 = 0.0;
    std::memset(&g->coefs, 0, sizeof g->coefs);
    for (int d = 0; d < ndim; ++d) {
        double h2 = g->h[d] * g->h[d];
        for (int j = 1; j <= R; ++j) g->coefs.C[d][j] = (float)(c[j] / h2);
        g->coefs.C[d][0] = (float)(c[0] / h2);
        s0 = s0 + c[0] / h2;
    }
    g->coefs.C0 = (float)s0;
    // fault-injection test hook ("perturbing one weight"): proves the parity
    // tests can fail.  Never set in production; tests/test_gpu_faults.py uses it in a subprocess.
    if (getenv("AW_DEBUG_PERTURB")) g->coefs.C[0][1] = nextafterf(g->coefs.C[0][1], 0.0f);

    aw_status st = AW_OK;
    auto bad = [&](cudaError_t e, const char* what) {
        if (e == cudaSuccess) return false;
        st = fail(e == cudaErrorMemoryAllocation ? AW_ENOMEM : AW_ECUDA, "%s: %s", what, cudaGetErrorString(e));
        cudaGetLastError();
        return true;
    };
    do {
        if (bad(cudaSetDevice(device), "cudaSetDevice")) break;
        if (bad(cudaStreamCreateWithFlags(&g->s, cudaStreamNonBlocking), "stream")) break;
        if (bad(cudaEventCreateWithFlags(&g->ev_sync, cudaEventDisableTiming), "event")) break;
        if (bad(cudaEventCreate(&g->ev_t0), "event") || bad(cudaEventCreate(&g->ev_t1), "event")) break;
        if (bad(cudaEventCreateWithFlags(&g->ev_stage, cudaEventDisableTiming), "event")) break;
        g->ubytes = (size_t)(nz + 2 * R) * G.plane * sizeof(float);
        g->mbytes = (size_t)nz * G.plane * sizeof(float);
        g->dense_bytes = 2 * align_up(g->ubytes, kDenseAlign) + 4 * align_up(g->mbytes, kDenseAlign);
        if (bad(lmalloc(g, (void**)&g->ctl, sizeof(aw::DevCtl)), "cudaMalloc control block")) break;
        g->d_base = &g->ctl->base;
        g->d_flag = &g->ctl->flag;
        g->d_team_flags = g->ctl->team_flags;
        if (bad(cudaMemsetAsync(g->ctl, 0, sizeof(aw::DevCtl), g->s), "memset")) break;
        if (!(dflags & AW_DIST_WORKSPACE)) {
            if (bad(lmalloc(g, (void**)&g->dense_lib, g->dense_bytes), "cudaMalloc of the grid arrays")) break;
            place_dense(g, g->dense_lib);
            if (bad(cudaMemsetAsync(g->dense, 0, g->dense_bytes, g->s), "memset")) break;
        }
        if (bad(cudaMemcpyAsync(&g->ctl->epoch, &g->epoch, sizeof g->epoch, cudaMemcpyHostToDevice, g->s), "epoch"))
            break;
        if (bad(cudaStreamSynchronize(g->s), "sync")) break;
    } while (0);
    if (st != AW_OK) {
        aw_grid_destroy(g);
        return st;
    }
    *out = g;
    return AW_OK;
}

void aw_grid_destroy(aw_grid* g) {
    if (!g) return;
    cudaSetDevice(g->device);
    if (g->s) cudaStreamSynchronize(g->s);
    free_graphs(g);
    if (g->plan) aw::stream_release(g->plan);
    aw::tile2d_release(g->t2);
    for (void* p : g->ipc_opened) cudaIpcCloseMemHandle(p);
    free_sources(g);
    free_receivers(g);
    dfree(g, g->src_arena);
    dfree(g, g->rec_arena);
    dfree(g, g->adj_arena);
    dfree(g, g->fwi_arena);
    dfree(g, g->fwi_pool);
    dfree(g, g->d_Gacc);
    // the third temporal-blocking buffer is the library's even when the rotation moved it into ubuf[]
    for (float* p : {g->ubuf[0], g->ubuf[1], g->ubuf_spare})
        if (p && g->lib_allocs.count((void*)p)) {
            cudaFree(p);
            g->lib_allocs.erase((void*)p);
        }
    dfree(g, g->dense_lib);
    dfree(g, g->ctl);
    dfree(g, g->ts0);
    dfree(g, g->ts1);
    for (cudaEvent_t e : g->tev) cudaEventDestroy(e);
    if (g->ev_sync) cudaEventDestroy(g->ev_sync);
    if (g->ev_t0) cudaEventDestroy(g->ev_t0);
    if (g->ev_t1) cudaEventDestroy(g->ev_t1);
    if (g->ev_stage) cudaEventDestroy(g->ev_stage);
    if (g->h_stage) cudaFreeHost(g->h_stage);
    if (g->s) cudaStreamDestroy(g->s);
    cudaGetLastError();
    delete g;
}

size_t aw_workspace_bytes(const aw_grid* g) {
    if (!g) return 0;
    return g->dense_bytes + align_up(g->src_need, 256) + align_up(g->rec_need, 256);
}

aw_status aw_bind_workspace(aw_grid* g, void* dev_ptr, size_t bytes) {
    CHECK_STATE(g);
    if (!dev_ptr) return fail(AW_EINVAL, "workspace pointer is NULL");
    if ((uintptr_t)dev_ptr % 256) return fail(AW_EINVAL, "workspace must be 256-B aligned");
    if (bytes < g->dense_bytes)
        return fail(AW_EINVAL, "workspace of %zu B < the %zu B of the grid arrays", bytes, g->dense_bytes);
    if (team_mode(g) && g->team_connected) return fail(AW_ESTATE, "bind the workspace before the team connects");
    if (g->ws) return fail(AW_ESTATE, "a workspace is already bound to this handle");
    {
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, dev_ptr) != cudaSuccess) {
            cudaGetLastError();
            return fail(AW_EINVAL, "workspace is not CUDA memory");
        }
        if (at.type != cudaMemoryTypeDevice || at.device != g->device)
            return fail(AW_EINVAL, "workspace must be device memory on device %d", g->device);
    }
    char* nb = (char*)dev_ptr;
    aw_status st = enter(g);
    if (st) return st;
    // 1. the dense block: copy the current contents (zeros when nothing was allocated yet)
    char* old = g->dense;
    if (old) CK(cudaMemcpyAsync(nb, old, g->dense_bytes, cudaMemcpyDeviceToDevice, g->s));
    else CK(cudaMemsetAsync(nb, 0, g->dense_bytes, g->s));
    // 2. the sparse arenas: source slot, then the receiver slot takes the rest of the workspace
    const size_t tail0 = g->dense_bytes, tail = bytes - g->dense_bytes;
    const size_t src_slot = std::min(tail, align_up(g->src_need, 256));
    size_t slot_off[2] = {tail0, tail0 + src_slot};
    size_t slot_cap[2] = {src_slot, tail - src_slot};
    struct Move {
        char** arena;
        size_t* cap;
        size_t need;
    } mv[2] = {{&g->src_arena, &g->src_cap, g->src_need}, {&g->rec_arena, &g->rec_cap, g->rec_need}};
    char* moved_from[2] = {nullptr, nullptr};
    for (int k = 0; k < 2; ++k) {
        if (*mv[k].arena && mv[k].need > 0 && mv[k].need <= slot_cap[k]) {
            CK(cudaMemcpyAsync(nb + slot_off[k], *mv[k].arena, mv[k].need, cudaMemcpyDeviceToDevice, g->s));
            moved_from[k] = *mv[k].arena;
        }
    }
    CK(cudaStreamSynchronize(g->s));
    // 3. repoint (everything below is host bookkeeping, nothing can fail)
    auto rebase = [](auto*& p, char* from, size_t n, char* to) {
        using T = std::remove_reference_t<decltype(*p)>;
        if (p && (char*)p >= from && (char*)p < from + n) p = (T*)(to + ((char*)p - from));
    };
    if (old) {
        for (float** p : {&g->ubuf[0], &g->ubuf[1], &g->ubuf_spare, &g->m, &g->eta, &g->b, &g->a})
            rebase(*p, old, g->dense_bytes, nb);
        g->dense = nb;
    } else {
        place_dense(g, nb);
    }
    for (int k = 0; k < 2; ++k) {
        char* from = moved_from[k];
        if (!from) continue;
        char* to = nb + slot_off[k];
        if (k == 0) {
            rebase(g->d_wavelet, from, mv[k].need, to);
            rebase(g->d_inj_off, from, mv[k].need, to);
            rebase(g->d_inj_plane, from, mv[k].need, to);
            rebase(g->d_inj_ptr, from, mv[k].need, to);
            rebase(g->d_inj_src, from, mv[k].need, to);
            rebase(g->d_inj_moff, from, mv[k].need, to);
            rebase(g->d_inj_w64, from, mv[k].need, to);
            rebase(g->d_inj_s, from, mv[k].need, to);
        } else {
            rebase(g->d_rec_id, from, mv[k].need, to);
            rebase(g->d_rec_off, from, mv[k].need, to);
            rebase(g->d_rec_w, from, mv[k].need, to);
            rebase(g->d_traces, from, mv[k].need, to);
        }
    }
    // free what now lives in the workspace: the library's dense block and the moved arenas
    for (int k = 0; k < 2; ++k)
        if (moved_from[k]) {
            dfree(g, moved_from[k]);
            *mv[k].arena = nb + slot_off[k];
            *mv[k].cap = slot_cap[k];
        }
    dfree(g, g->dense_lib);
    g->ws = nb;
    g->ws_bytes = bytes;
    for (int k = 0; k < 2; ++k) {
        g->ws_slot_off[k] = slot_off[k];
        g->ws_slot_cap[k] = slot_cap[k];
    }
    // every launch parameter, tensor map and captured graph that named the old addresses is rebuilt
    g->coeffs_valid = false;
    free_graphs(g);
    return leave(g);
}

aw_status aw_local_extent(const aw_grid* g, int64_t* z0, int64_t* nz) {
    if (!g) return fail(AW_EINVAL, "null grid handle");
    if (z0) *z0 = g->z0;
    if (nz) *nz = g->geom.nz;
    return AW_OK;
}

int64_t aw_steps_done(const aw_grid* g) { return g ? g->steps : -1; }

aw_status aw_set_model(aw_grid* g, const float* m, const float* damp, int layout) {
    CHECK_STATE(g);
    NEED_DENSE(g);
    if (!m) return fail(AW_EINVAL, "m is NULL");
    if (layout != AW_GLOBAL && layout != AW_LOCAL) return fail(AW_EINVAL, "bad layout %d", layout);
    aw_status st = enter(g);
    if (st) return st;
    const int64_t nx = g->geom.nx, rows = (int64_t)g->geom.nz * g->geom.ny;
    const int64_t src_off = layout == AW_GLOBAL ? g->z0 * g->geom.ny * nx : 0;
    // Stage the new model in b (m) and a (eta): those hold dt-dependent coefficients that the next
    // run recomputes anyway.  Validate the staged copy; only a valid model is swapped in, so an
    // invalid one leaves the previous model in force (strong guarantee, include/aw.h).
    float* new_m = g->b;
    float* new_eta = g->a;
    g->coeffs_valid = false;  // b and a are overwritten from here on
    const unsigned epoch = ++g->model_epoch;
    if (ptr_kind(m) == PK_DEVICE && (!damp || ptr_kind(damp) == PK_DEVICE)) {
        // device inputs: one kernel copies both arrays into the padded staging layout (padding 0) and
        // validates them, recording `epoch` in the control block if any value is invalid
        CK(aw::launch_stage_model(m + src_off, damp ? damp + src_off : nullptr, new_m, damp ? new_eta : nullptr,
                                  g->geom, &g->ctl->model_bad, epoch, g->s));
        g->launch_count += 1;
    } else {
        // padding columns (x >= nx): 0, never read as domain points
        CK(cudaMemsetAsync(new_m, 0, g->mbytes, g->s));
        if ((st = copy_in(g, new_m, g->geom.pitch, m + src_off, nx, rows))) return st;
        if (damp) {
            CK(cudaMemsetAsync(new_eta, 0, g->mbytes, g->s));
            if ((st = copy_in(g, new_eta, g->geom.pitch, damp + src_off, nx, rows))) return st;
        }
        CK(aw::launch_validate_model(new_m, damp ? new_eta : nullptr, g->geom, &g->ctl->model_bad, epoch, g->s));
        g->launch_count += 1;
    }
    if ((st = readback_ctl(g))) return st;  // the validation decides the call's status (strong guarantee)
    unsigned bad = 0;
    std::memcpy(&bad, g->h_stage + offsetof(aw::DevCtl, model_bad), sizeof bad);
    if ((st = leave(g))) return st;
    const unsigned flag = bad == epoch;
    if (flag) return fail(AW_EINVAL, "model invalid: m must be finite and > 0, damp finite and >= 0 "
                                     "(the previous model stays in force)");
    std::swap(g->m, g->b);
    if (damp) std::swap(g->eta, g->a);
    g->have_model = true;
    g->have_damp = damp != nullptr;
    return AW_OK;
}

aw_status aw_add_sources(aw_grid* g, int ns, const double* coords, int nt_max, const float* wavelet) {
    CHECK_STATE(g);
    if (ns < 0) return fail(AW_EINVAL, "ns < 0");
    if (ns > 0 && (!coords || !wavelet || nt_max <= 0)) return fail(AW_EINVAL, "coords/wavelet/nt_max invalid");
    const int nc = 1 << g->ndim;
    std::vector<int64_t> corner((size_t)ns * nc);
    std::vector<double> w((size_t)ns * nc);
    for (int s = 0; s < ns; ++s) {
        int64_t b0;
        if (!locate(g, coords + (size_t)s * g->ndim, &corner[(size_t)s * nc], &w[(size_t)s * nc], &b0))
            return fail(AW_EINVAL, "source %d lies outside the grid", s);
    }
    aw_status st = enter(g);
    if (st) return st;
    free_sources(g);
    g->coeffs_valid = false;
    if (ns == 0) return leave(g);
    g->ns = ns;
    g->src_nt = nt_max;
    g->src_corner_lin = corner;
    g->src_w64 = w;
    // owned entries in CSR order: corner ascending, then source ascending (Q11)
    InjTables t;
    build_injection(g, ns, corner, w, &t);
    g->h_inj_lin = t.lin;
    g->h_inj_ptr = t.ptr;
    g->ent_src = t.ent_src;
    g->ent_beta = t.ent_beta;
    g->nuc = (int)t.off.size();
    g->nent = (int)t.ents.size();
    Packer pk;
    const size_t o_off = pk.add(t.off), o_plane = pk.add(t.plane), o_ptr = pk.add(t.ptr), o_src = pk.add(t.src),
                 o_moff = pk.add(t.moff), o_w = pk.add(t.w);
    const size_t small = pk.off;
    const size_t o_s = pk.reserve((size_t)g->nent * sizeof(float));
    const size_t o_wav = pk.reserve((size_t)nt_max * ns * sizeof(float));
    if ((st = ensure_arena(g, &g->src_arena, &g->src_cap, pk.off, 0))) return st;
    g->src_need = pk.off;
    char* A = g->src_arena;
    g->d_inj_off = (int64_t*)(A + o_off);
    g->d_inj_plane = (int*)(A + o_plane);
    g->d_inj_ptr = (int*)(A + o_ptr);
    g->d_inj_src = (int*)(A + o_src);
    g->d_inj_moff = (int64_t*)(A + o_moff);
    g->d_inj_w64 = (double*)(A + o_w);
    g->d_inj_s = (float*)(A + o_s);
    g->d_wavelet = (float*)(A + o_wav);
    if ((st = upload(g, A, pk.host.data(), small))) return st;
    const size_t wbytes = (size_t)nt_max * ns * sizeof(float);
    if (ptr_kind(wavelet) == PK_DEVICE) {
        CK(cudaMemcpyAsync(g->d_wavelet, wavelet, wbytes, cudaMemcpyDeviceToDevice, g->s));  // stream-ordered
    } else {
        // host memory: copied before return (a pinned buffer could otherwise change under the DMA)
        CK(cudaMemcpyAsync(g->d_wavelet, wavelet, wbytes, cudaMemcpyHostToDevice, g->s));
        CK(cudaStreamSynchronize(g->s));
        g->stage_pending = false;
    }
    return leave(g);
}

aw_status aw_add_receivers(aw_grid* g, int nr, const double* coords, int nt_max) {
    CHECK_STATE(g);
    if (nr < 0) return fail(AW_EINVAL, "nr < 0");
    if (nr > 0 && (!coords || nt_max <= 0)) return fail(AW_EINVAL, "coords/nt_max invalid");
    const int nc = 1 << g->ndim;
    std::vector<int64_t> corner((size_t)nr * nc), base0(nr);
    std::vector<double> w((size_t)nr * nc);
    for (int r = 0; r < nr; ++r)
        if (!locate(g, coords + (size_t)r * g->ndim, &corner[(size_t)r * nc], &w[(size_t)r * nc], &base0[r]))
            return fail(AW_EINVAL, "receiver %d lies outside the grid", r);
    aw_status st = enter(g);
    if (st) return st;
    free_receivers(g);
    if (nr == 0) return leave(g);
    g->nr = nr;
    g->rec_nt = nt_max;
    g->rec_corner_lin = corner;
    g->rec_w32.resize(w.size());
    for (size_t i = 0; i < w.size(); ++i) g->rec_w32[i] = (float)w[i];
    g->rec_w64 = w;
    // owner = rank owning the base corner's plane; its +1 corner may be a halo plane
    std::vector<int> ids;
    std::vector<int64_t> offs;
    std::vector<float> ws;
    for (int r = 0; r < nr; ++r) {
        if (base0[r] < g->z0 || base0[r] >= g->z0 + g->geom.nz) continue;
        ids.push_back(r);
        for (int beta = 0; beta < nc; ++beta) {
            int64_t lin = corner[(size_t)r * nc + beta];
            if (lin < 0) {
                offs.push_back(-1);
                ws.push_back(0.f);
                continue;
            }
            int64_t zl, uoff, moff;
            lin_to_local(g, lin, &zl, &uoff, &moff);
            offs.push_back(uoff);
            ws.push_back(g->rec_w32[(size_t)r * nc + beta]);
        }
    }
    g->nrl = (int)ids.size();
    g->h_rec_off = offs;
    g->rec_items_dirty = true;
    Packer pk;
    const size_t o_id = pk.add(ids), o_off = pk.add(offs), o_w = pk.add(ws);
    const size_t small = pk.off;
    const size_t o_tr = pk.reserve((size_t)nt_max * nr * sizeof(float));
    if ((st = ensure_arena(g, &g->rec_arena, &g->rec_cap, pk.off, 1))) return st;
    g->rec_need = pk.off;
    char* A = g->rec_arena;
    g->d_rec_id = (int*)(A + o_id);
    g->d_rec_off = (int64_t*)(A + o_off);
    g->d_rec_w = (float*)(A + o_w);
    g->d_traces = (float*)(A + o_tr);
    if ((st = upload(g, A, pk.host.data(), small))) return st;  // host tables via the pinned staging buffer
    CK(cudaMemsetAsync(g->d_traces, 0, (size_t)nt_max * nr * sizeof(float), g->s));
    return leave(g);
}

aw_status aw_set_wavefield(aw_grid* g, const float* u_cur, const float* u_prev, int layout) {
    CHECK_STATE(g);
    NEED_DENSE(g);
    if (layout != AW_GLOBAL && layout != AW_LOCAL) return fail(AW_EINVAL, "bad layout %d", layout);
    aw_status st = enter(g);
    if (st) return st;
    const int64_t nx = g->geom.nx, ny = g->geom.ny, plane = g->geom.plane, R = g->R, nz = g->geom.nz;
    const int64_t per_plane = ny * nx;  // dense elements per plane
    for (int which = 0; which < 2; ++which) {
        float* buf = g->ubuf[which == 0 ? g->cur : 1 - g->cur];
        const float* src = which == 0 ? u_cur : u_prev;
        {
            // LOCAL in a team: the neighbours fill my halo planes next to them (their prologue copy at
            // the next run may land before or after this call), so leave those planes alone and zero
            // the rest (owned planes, the always-zero halo at a global end).  GLOBAL: every rank fills
            // its own halos from the global array below (or zeros).
            const bool local_team = team_mode(g) && layout == AW_LOCAL;
            const int64_t zb = local_team && g->halo.lo[0] ? 0 : -R;
            const int64_t ze = local_team && g->halo.hi[0] ? nz : nz + R;
            CK(cudaMemsetAsync(buf + (zb + R) * plane, 0, (size_t)(ze - zb) * plane * sizeof(float), g->s));
        }
        if (!src) continue;
        int64_t zlo = 0, zhi = nz;  // local planes to fill
        if (layout == AW_GLOBAL && which == 0 && team_mode(g)) {
            zlo = std::max<int64_t>(-R, -g->z0);
            zhi = std::min<int64_t>(nz + R, g->shape[0] - g->z0);
        }
        const float* s0 = layout == AW_GLOBAL ? src + (g->z0 + zlo) * per_plane : src + zlo * per_plane;
        if ((st = copy_in(g, buf + (zlo + R) * plane, g->geom.pitch, s0, nx, (zhi - zlo) * ny))) return st;
    }
    if (team_mode(g)) {
        // New epoch: stale signals can no longer satisfy a wait.  With a GLOBAL array my halos are
        // already filled, so tell the neighbours they may proceed (their step stores into my
        // buffers only after this).  LOCAL: the exchange happens at the next aw_run (prologue).
        g->epoch += 1;
        CK(cudaMemcpyAsync(&g->ctl->epoch, &g->epoch, sizeof g->epoch, cudaMemcpyHostToDevice, g->s));
        if (layout == AW_GLOBAL) {
            CK(aw::launch_team_raise(g->peer_flag_lo, g->peer_flag_hi, enc(g, g->steps), g->s));
            g->launch_count += 1;
        }
    }
    CK(cudaStreamSynchronize(g->s));
    g->halo_dirty = team_mode(g) && layout == AW_LOCAL;
    g->wave_invalid = false;
    return leave(g);
}

aw_status aw_run(aw_grid* g, int nt, double dt) {
    CHECK_STATE(g);
    if (g->wave_invalid) return fail(AW_ESTATE, "call aw_reset (or aw_set_wavefield) after aw_fwi_gradient");
    aw_status st = run_begin(g, nt, dt);
    if (st) return st;
    int64_t launches = 0;
    if ((st = run_enqueue(g, nt, &launches))) return st;
    return run_end(g, nt, launches);
}

aw_status aw_fwi_gradient(aw_grid* g, int nt, double dt, const float* d_obs, float* grad, int layout,
                          float* residual, double* objective) {
    CHECK_STATE(g);
    NEED_DENSE(g);
    if (team_mode(g)) return fail(AW_EUNSUPPORTED, "aw_fwi_gradient runs on a single slab (world = 1)");
    if (nt < 1) return fail(AW_EINVAL, "nt must be >= 1 (got %d)", nt);
    if (!d_obs || !grad) return fail(AW_EINVAL, "d_obs/grad is NULL");
    if (layout != AW_GLOBAL && layout != AW_LOCAL) return fail(AW_EINVAL, "bad layout %d", layout);
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(AW_EINVAL, "dt must be finite and > 0");
    if (!g->have_model) return fail(AW_ESTATE, "aw_set_model has not been called");
    if (g->nr == 0) return fail(AW_EINVAL, "the misfit needs receivers (aw_add_receivers)");
    if (g->ns > 0 && nt > g->src_nt) return fail(AW_EINVAL, "wavelet covers %d steps, need %d", g->src_nt, nt);
    if (nt > g->rec_nt) return fail(AW_EINVAL, "trace buffer covers %d steps, need %d", g->rec_nt, nt);
    aw_status st = enter(g);
    if (st) return st;
    // start from the reset state (zero wavefields, step 0) with this dt; until aw_reset /
    // aw_set_wavefield the wavefield levels are not a forward state (also if this call fails)
    g->steps = 0;
    g->cur = 0;
    g->wave_invalid = true;
    if (!(g->dt_set && g->dt == dt)) g->coeffs_valid = false;  // any dt: the call starts from the reset state
    if ((st = prepare(g, dt))) return st;
    if ((st = fwi_build_adjoint(g))) return st;
    CK(aw::launch_source_scales(g->m, g->have_damp ? g->eta : nullptr, g->d_adj_moff, g->d_adj_w64, g->d_adj_s,
                                g->adj_nent, dt, g->s));
    int64_t launches = g->adj_nent > 0 ? 1 : 0;
    if (g->kernel_used == AW_KERNEL_STREAM) {
        cudaError_t e = aw::stream_set_injection(g->plan, g->geom, g->z0, g->h_adj_lin.data(), g->h_adj_ptr.data(),
                                                 g->adj_nuc, g->s, 1);
        CK(e);
    }

    // ---- memory: per-call arrays and the history/checkpoint pool (kept between calls) ----
    const int nr = g->nr;
    const size_t tr = (size_t)nt * nr * sizeof(float);
    const size_t fwi_bytes = 3 * ((tr + 255) / 256 * 256) + 256 + g->mbytes;
    if ((st = ensure_arena(g, &g->fwi_arena, &g->fwi_cap, fwi_bytes))) return st;
    float* d_dobs = (float*)g->fwi_arena;
    float* d_res = (float*)(g->fwi_arena + (tr + 255) / 256 * 256);
    float* d_wadj = (float*)(g->fwi_arena + 2 * ((tr + 255) / 256 * 256));
    double* d_J = (double*)(g->fwi_arena + 3 * ((tr + 255) / 256 * 256));
    float* d_G = (float*)(g->fwi_arena + 3 * ((tr + 255) / 256 * 256) + 256);
    {
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        const int64_t have = g->fwi_pool_nbuf;
        const int64_t max_bufs = have + (int64_t)((double)fr * 0.6 / (double)g->ubytes);
        const int K = fwi_choose_K(g, nt, max_bufs);
        if (K < 1) return fail(AW_ENOMEM, "not enough device memory for the FWI history (%lld buffers of %zu B)",
                               (long long)fwi_buffers(nt, 1), g->ubytes);
        const int64_t need = fwi_buffers(nt, K);
        if (need > have) {
            if (g->fwi_pool) {
                CK(cudaStreamSynchronize(g->s));
                dfree(g, g->fwi_pool);
                g->fwi_pool_nbuf = 0;
            }
            cudaError_t e = lmalloc(g, (void**)&g->fwi_pool, (size_t)need * g->ubytes);
            if (e != cudaSuccess) {
                cudaGetLastError();
                return fail(AW_ENOMEM, "FWI history pool of %lld buffers: %s", (long long)need, cudaGetErrorString(e));
            }
            g->fwi_pool_nbuf = need;
            CK(cudaMemsetAsync(g->fwi_pool, 0, (size_t)need * g->ubytes, g->s));  // zero halo planes for good
        }
        g->stats.fwi_checkpoint = K;
    }
    const int K = g->stats.fwi_checkpoint;
    const int nseg = (nt + K - 1) / K;
    // segments: the first one takes the remainder, all later ones K steps, so the last segment -- the
    // one still in the ring after the forward pass -- is full and only nt - K steps are replayed
    auto seg_lo = [&](int j) { return j == 0 ? 0 : (j >= nseg ? nt : nt - (nseg - j) * K); };
    const int S = K + 2;
    const int64_t ufl = (int64_t)(g->ubytes / sizeof(float));
    const int64_t own_off = (int64_t)g->R * g->geom.plane;                // first owned plane
    const size_t own_bytes = (size_t)g->geom.nz * g->geom.plane * sizeof(float);
    float* pool = g->fwi_pool;
    auto slot = [&](int64_t level) { return pool + (((level + 1) % S + S) % S) * ufl; };  // level -1 .. nt
    auto ckpt = [&](int j, int which) { return pool + ((int64_t)S + 2 * (j - 1) + which) * ufl; };  // j >= 1
    auto zero_level = [&](int64_t level) -> aw_status {
        CK(cudaMemsetAsync(slot(level) + own_off, 0, own_bytes, g->s));
        return AW_OK;
    };
    auto copy_level = [&](float* dst, const float* src) -> aw_status {
        CK(cudaMemcpyAsync(dst + own_off, src + own_off, own_bytes, cudaMemcpyDeviceToDevice, g->s));
        return AW_OK;
    };

    CK(cudaEventRecord(g->ev_t0, g->s));
    const int64_t zero = 0;
    CK(cudaMemcpyAsync(g->d_base, &zero, sizeof zero, cudaMemcpyHostToDevice, g->s));
    CK(cudaMemcpyAsync(d_dobs, d_obs, tr, ptr_kind(d_obs) == PK_DEVICE ? cudaMemcpyDeviceToDevice
                                                                      : cudaMemcpyHostToDevice, g->s));
    if (g->d_traces) CK(cudaMemsetAsync(g->d_traces, 0, (size_t)g->rec_nt * nr * sizeof(float), g->s));
    int64_t steps_done = 0;
    aw::Sparse fwd = sparse_view(g);  // sources + receivers (first pass)
    aw::Sparse fwd_norec = fwd;       // recompute: sources only (traces already recorded)
    fwd_norec.nrl = 0;
    aw::Sparse adj{};                 // adjoint: the receivers inject the time-reversed residual
    adj.nuc = g->adj_nuc;
    adj.ns = nr;
    adj.inj_off = g->d_adj_off;
    adj.inj_plane = g->d_adj_plane;
    adj.inj_ptr = g->d_adj_ptr;
    adj.inj_src = g->d_adj_src;
    adj.inj_s = g->d_adj_s;
    adj.wavelet = d_wadj;
    adj.nc = 1 << g->ndim;

    // ---- 1. forward pass into the history ring; checkpoints at segment starts ----
    if ((st = zero_level(-1)) || (st = zero_level(0))) return st;
    for (int n = 0; n < nt; ++n) {
        if ((st = fwi_step(g, slot(n), slot(n - 1), slot(n + 1), fwd, 0, n, &launches))) return st;
        ++steps_done;
        const int l = n + 1;
        if (l < nt && (nt - l) % K == 0) {  // l = seg_lo(j), j >= 1: keep (u^{l-1}, u^l)
            const int j = nseg - (nt - l) / K;
            if ((st = copy_level(ckpt(j, 0), slot(l - 1))) || (st = copy_level(ckpt(j, 1), slot(l)))) return st;
        }
    }
    // ---- 2. residual, misfit, adjoint wavelet ----
    CK(aw::launch_fwi_residual(g->d_traces, d_dobs, d_res, d_wadj, nt, nr, d_J, g->s));
    ++launches;
    // ---- 3. adjoint run in reversed time, segment by segment, imaging before each step ----
    float* psi[2] = {g->ubuf[0], g->ubuf[1]};
    CK(cudaMemsetAsync(psi[0], 0, g->ubytes, g->s));
    CK(cudaMemsetAsync(psi[1], 0, g->ubytes, g->s));
    CK(cudaMemsetAsync(d_G, 0, g->mbytes, g->s));
    int pc = 0;  // psi^k in psi[pc], psi^{k-1} in psi[1-pc]
    for (int j = nseg - 1; j >= 0; --j) {
        const int lo = seg_lo(j), hi = seg_lo(j + 1);
        if (j < nseg - 1) {  // recompute levels lo+1 .. hi from the checkpoint
            if (j == 0) {
                if ((st = zero_level(-1)) || (st = zero_level(0))) return st;
            } else if ((st = copy_level(slot(lo - 1), ckpt(j, 0))) || (st = copy_level(slot(lo), ckpt(j, 1)))) {
                return st;
            }
            for (int n = lo; n < hi; ++n) {
                if ((st = fwi_step(g, slot(n), slot(n - 1), slot(n + 1), fwd_norec, 0, n, &launches))) return st;
                ++steps_done;
            }
        }
        for (int n = hi - 1; n >= lo; --n) {
            const int k = nt - 1 - n;
            CK(aw::launch_fwi_imaging(g->geom, psi[pc], slot(n + 1), slot(n), slot(n - 1), d_G, g->s));
            ++launches;
            if (k == nt - 1) break;  // psi^nt pairs with no forward level
            if ((st = fwi_step(g, psi[pc], psi[1 - pc], psi[1 - pc], adj, 1, k, &launches))) return st;
            ++steps_done;
            pc = 1 - pc;
        }
    }
    // ---- 4. gradient = -G / dt^2, outputs ----
    CK(aw::launch_fwi_finalize(g->geom, d_G, dt, g->s));
    ++launches;
    const float* g_out = d_G;
    if (g->opt_accum) {  // NEXT-4: sum of the gradients of the calls since AW_OPT_FWI_ACCUMULATE was set
        if (!g->d_Gacc) CK(lmalloc(g, (void**)&g->d_Gacc, g->mbytes));
        if (g->acc_valid) {
            CK(aw::launch_fwi_accumulate(g->geom, g->d_Gacc, d_G, g->s));
            ++launches;
        } else {
            CK(cudaMemcpyAsync(g->d_Gacc, d_G, g->mbytes, cudaMemcpyDeviceToDevice, g->s));
        }
        g->acc_valid = true;
        g_out = g->d_Gacc;
    }
    CK(cudaEventRecord(g->ev_t1, g->s));
    {
        const int64_t nx = g->geom.nx, ny = g->geom.ny;
        float* dst = layout == AW_GLOBAL ? grad + g->z0 * ny * nx : grad;
        if ((st = copy_out(g, dst, g_out, g->geom.pitch, nx, (int64_t)g->geom.nz * ny))) return st;
    }
    if (residual)
        CK(cudaMemcpyAsync(residual, d_res, tr, ptr_kind(residual) == PK_DEVICE ? cudaMemcpyDeviceToDevice
                                                                                : cudaMemcpyDeviceToHost, g->s));
    double J = 0.0;
    CK(cudaMemcpyAsync(&J, d_J, sizeof J, cudaMemcpyDeviceToHost, g->s));
    if ((st = leave(g))) return st;
    CK(cudaStreamSynchronize(g->s));
    if (objective) *objective = J;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, g->ev_t0, g->ev_t1));
    g->stats.ms_total = ms;
    g->stats.ms_stencil = -1.0;
    g->stats.n_stencil = 0;
    g->stats.launches = launches;
    g->launch_count += launches;
    g->stats.launches_total = g->launch_count;
    g->stats.points = (int64_t)g->geom.nz * g->geom.ny * g->geom.nx;
    g->stats.gpts = ms > 0 ? (double)g->stats.points * nt / (ms * 1e6) : 0.0;
    g->stats.kernel = g->kernel_used;
    g->stats.resident = 0;
    g->stats.fwi_steps = steps_done;
    // the traces of the forward run stay readable; the wavefield levels hold the adjoint field
    g->steps = nt;
    g->wave_invalid = true;
    if (!std::isfinite(J)) return fail(AW_ENONFINITE, "misfit is not finite (J = %g)", J);
    return AW_OK;
}

aw_status aw_reset(aw_grid* g) {
    CHECK_STATE(g);
    NEED_DENSE(g);
    aw_status st = enter(g);
    if (st) return st;
    CK(cudaMemsetAsync(g->ubuf[0], 0, g->ubytes, g->s));
    CK(cudaMemsetAsync(g->ubuf[1], 0, g->ubytes, g->s));
    if (g->d_traces) CK(cudaMemsetAsync(g->d_traces, 0, (size_t)g->rec_nt * g->nr * sizeof(float), g->s));
    g->steps = 0;
    g->cur = 0;
    g->dt_set = false;
    g->coeffs_valid = false;
    g->wave_invalid = false;
    if (team_mode(g)) {
        // after my memsets: neighbours may start storing level-1 halos into my buffers
        g->epoch += 1;
        CK(cudaMemcpyAsync(&g->ctl->epoch, &g->epoch, sizeof g->epoch, cudaMemcpyHostToDevice, g->s));
        CK(aw::launch_team_raise(g->peer_flag_lo, g->peer_flag_hi, enc(g, 0), g->s));
        g->launch_count += 1;
        CK(cudaStreamSynchronize(g->s));  // collective: the neighbours may rely on the raised epoch
    }
    return leave(g);
}

aw_status aw_read_wavefield(aw_grid* g, int which, float* out, int layout) {
    CHECK_STATE(g);
    NEED_DENSE(g);
    if (!out) return fail(AW_EINVAL, "out is NULL");
    if (which != 0 && which != 1) return fail(AW_EINVAL, "which must be 0 or 1");
    if (layout != AW_GLOBAL && layout != AW_LOCAL) return fail(AW_EINVAL, "bad layout %d", layout);
    if (g->wave_invalid) return fail(AW_ESTATE, "no forward wavefield after aw_fwi_gradient (aw_reset first)");
    aw_status st = enter(g);
    if (st) return st;
    const float* buf = g->ubuf[which == 0 ? g->cur : 1 - g->cur];
    const int64_t nx = g->geom.nx, ny = g->geom.ny;
    float* dst = layout == AW_GLOBAL ? out + g->z0 * ny * nx : out;
    if ((st = copy_out(g, dst, buf + (int64_t)g->R * g->geom.plane, g->geom.pitch, nx, (int64_t)g->geom.nz * ny)))
        return st;
    CK(cudaStreamSynchronize(g->s));
    return leave(g);
}

aw_status aw_read_receivers(aw_grid* g, float* out) {
    CHECK_STATE(g);
    if (g->nr == 0 || g->steps == 0) return AW_OK;
    if (!out) return fail(AW_EINVAL, "out is NULL");
    aw_status st = enter(g);
    if (st) return st;
    size_t bytes = (size_t)g->steps * g->nr * sizeof(float);
    if (ptr_kind(out) == PK_DEVICE) {
        CK(cudaMemcpyAsync(out, g->d_traces, bytes, cudaMemcpyDeviceToDevice, g->s));  // stream-ordered
    } else {
        CK(cudaMemcpyAsync(out, g->d_traces, bytes, cudaMemcpyDeviceToHost, g->s));
        CK(cudaStreamSynchronize(g->s));
    }
    return leave(g);
}

aw_status aw_debug_sparse(const aw_grid* gc, int which, int64_t* corner_lin, float* w) {
    aw_grid* g = const_cast<aw_grid*>(gc);
    CHECK_STATE(g);
    const int nc = 1 << g->ndim;
    if (which == 1) {
        if (corner_lin) std::copy(g->rec_corner_lin.begin(), g->rec_corner_lin.end(), corner_lin);
        if (w) std::copy(g->rec_w32.begin(), g->rec_w32.end(), w);
        return AW_OK;
    }
    if (which != 0) return fail(AW_EINVAL, "which must be 0 or 1");
    if (corner_lin) std::copy(g->src_corner_lin.begin(), g->src_corner_lin.end(), corner_lin);
    if (w) {
        std::fill(w, w + (size_t)g->ns * nc, 0.0f);
        if (g->nent > 0) {
            std::vector<float> s(g->nent);
            CK(cudaSetDevice(g->device));
            CK(cudaMemcpy(s.data(), g->d_inj_s, g->nent * sizeof(float), cudaMemcpyDeviceToHost));
            for (int e = 0; e < g->nent; ++e) w[(size_t)g->ent_src[e] * nc + g->ent_beta[e]] = s[e];
        }
    }
    return AW_OK;
}

aw_status aw_last_run_stats(const aw_grid* g, aw_run_stats* out) {
    if (!g || !out) return fail(AW_EINVAL, "null argument");
    *out = g->stats;
    out->launches_total = g->launch_count;
    int64_t lib = 0;
    for (const auto& kv : g->lib_allocs) lib += (int64_t)kv.second;
    out->lib_device_bytes = lib + (int64_t)aw::stream_plan_bytes(g->plan);
    out->workspace_bytes = (int64_t)g->ws_bytes;
    return AW_OK;
}

aw_status aw_set_option(aw_grid* g, int option, int64_t value) {
    CHECK_STATE(g);
    switch (option) {
        case AW_OPT_KERNEL:
            if (value < AW_KERNEL_AUTO || value > AW_KERNEL_STREAM)  // TILE2D is selected by AUTO (2D)
                return fail(AW_EINVAL, "bad kernel %lld", (long long)value);
            g->opt_kernel = (int)value;
            g->coeffs_valid = false;
            if (g->plan) {
                cudaStreamSynchronize(g->s);
                aw::stream_release(g->plan);
                g->plan = nullptr;
            }
            free_graphs(g);
            return AW_OK;
        case AW_OPT_TIMING:
            if (value < 0 || value > 2) return fail(AW_EINVAL, "timing option must be 0, 1 or 2");
            g->opt_timing = (int)value;  // graphs captured with/without the timestamp arrays differ in signature
            return AW_OK;
        case AW_OPT_GRAPH_STEPS:
            if (value < 0 || value > 4096) return fail(AW_EINVAL, "graph steps out of range");
            g->opt_graph = (int)value;
            free_graphs(g);
            return AW_OK;
        case AW_OPT_CHECK_FINITE:
            g->opt_check = value != 0;
            return AW_OK;
        case AW_OPT_TEMPORAL:
            if (value < 0 || value > 1) return fail(AW_EINVAL, "temporal blocking option must be 0 or 1");
            g->opt_temporal = (int)value;
            g->coeffs_valid = false;  // re-prepare (allocates the third buffer when enabled)
            free_graphs(g);
            return AW_OK;
        case AW_OPT_FWI_ACCUMULATE:
            if (value < 0 || value > 1) return fail(AW_EINVAL, "accumulate option must be 0 or 1");
            g->opt_accum = (int)value;
            g->acc_valid = false;  // setting the option (either value) clears the sum
            return AW_OK;
        case AW_OPT_RESIDENT:
            if (value < AW_RESIDENT_OFF || value > AW_RESIDENT_AUTO) return fail(AW_EINVAL, "bad resident option");
            g->opt_resident = (int)value;
            return AW_OK;
        case AW_OPT_CHECKPOINT_STEPS:
            if (value < 0 || value > (1 << 30)) return fail(AW_EINVAL, "checkpoint steps out of range");
            g->opt_ckpt = (int)value;
            return AW_OK;
        default:
            return fail(AW_EINVAL, "unknown option %d", option);
    }
}

// ---------------------------------------------------------------------------
// Teams
// ---------------------------------------------------------------------------
// A peer address = (IPC handle of the allocation that contains it, offset into it): the wavefield
// levels share one allocation (the dense block or the caller's workspace) and the flag words sit
// inside the control block, so none of them is an allocation base.
struct aw_ipc_ptr {
    cudaIpcMemHandle_t h;
    int64_t off;
};
struct aw_team_record {
    aw_ipc_ptr u[2];
    aw_ipc_ptr flags;
    int64_t nz, R, plane, ny, nx;
    int32_t rank, world;
};

namespace {
typedef int (*PFN_memGetAddressRange)(unsigned long long*, size_t*, unsigned long long);  // cuMemGetAddressRange_v2
aw_status ipc_export(aw_grid* g, const void* p, aw_ipc_ptr* out) {
    static PFN_memGetAddressRange fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return fail(AW_ECUDA, "cuMemGetAddressRange is unavailable");
        fn = (PFN_memGetAddressRange)f;
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (fn(&base, &size, (unsigned long long)(uintptr_t)p) != 0) return fail(AW_ECUDA, "cuMemGetAddressRange failed");
    CK(cudaIpcGetMemHandle(&out->h, (void*)(uintptr_t)base));
    out->off = (int64_t)((uintptr_t)p - (uintptr_t)base);
    return AW_OK;
}
// Open a peer address; every distinct handle is opened once per handle (re-opening an open
// handle in the same process is an error) and kept until aw_grid_destroy.
aw_status ipc_open(aw_grid* g, const aw_ipc_ptr& ip, void** out) {
    for (const auto& o : g->ipc_opened_h)
        if (std::memcmp(&o.first, &ip.h, sizeof ip.h) == 0) {
            *out = (char*)o.second + ip.off;
            return AW_OK;
        }
    void* base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, ip.h, cudaIpcMemLazyEnablePeerAccess));
    g->ipc_opened.push_back(base);
    g->ipc_opened_h.push_back({ip.h, base});
    *out = (char*)base + ip.off;
    return AW_OK;
}
}  // namespace

size_t aw_team_export_size(void) { return sizeof(aw_team_record); }

aw_status aw_slab_partition(int64_t n0, int world, int rank, int R, int64_t* z0, int64_t* nz) {
    if (n0 < 1 || world < 1 || rank < 0 || rank >= world || R < 1 || !z0 || !nz)
        return fail(AW_EINVAL, "bad slab partition arguments");
    const int64_t base = n0 / world, rem = n0 % world;
    const int64_t n = base + (rank < rem ? 1 : 0);
    if (world > 1 && n < R) return fail(AW_EINVAL, "slab of %lld planes is thinner than k/2=%d", (long long)n, R);
    *z0 = rank * base + std::min<int64_t>(rank, rem);
    *nz = n;
    return AW_OK;
}

aw_status aw_team_export(aw_grid* g, void* out) {
    CHECK_STATE(g);
    NEED_DENSE(g);
    if (!out) return fail(AW_EINVAL, "out is NULL");
    aw_team_record rec;
    std::memset(&rec, 0, sizeof rec);
    CK(cudaSetDevice(g->device));
    aw_status st;
    if ((st = ipc_export(g, g->ubuf[0], &rec.u[0])) || (st = ipc_export(g, g->ubuf[1], &rec.u[1])) ||
        (st = ipc_export(g, g->d_team_flags, &rec.flags)))
        return st;
    rec.nz = g->geom.nz;
    rec.R = g->R;
    rec.plane = g->geom.plane;
    rec.ny = g->geom.ny;
    rec.nx = g->geom.nx;
    rec.rank = g->rank;
    rec.world = g->world;
    std::memcpy(out, &rec, sizeof rec);
    return AW_OK;
}

static aw_status link_neighbours(aw_grid* g, float* lo0, float* lo1, unsigned long long* lo_flags, int64_t nz_lo,
                                 float* hi0, float* hi1, unsigned long long* hi_flags) {
    g->halo.lo[0] = lo0;
    g->halo.lo[1] = lo1;
    g->halo.hi[0] = hi0;
    g->halo.hi[1] = hi1;
    g->nz_lo = nz_lo;
    g->halo.lo_off = lo0 ? (nz_lo + g->R) * g->geom.plane : 0;
    g->halo.hi_off = 0;
    g->peer_flag_lo = lo_flags ? lo_flags + 1 : nullptr;  // I am rank+1 of my lower neighbour
    g->peer_flag_hi = hi_flags ? hi_flags + 0 : nullptr;  // I am rank-1 of my upper neighbour
    g->halo.flag_lo = g->peer_flag_lo;
    g->halo.flag_hi = g->peer_flag_hi;
    g->halo.ctl = g->ctl;
    g->team_connected = true;
    free_graphs(g);
    return AW_OK;
}

aw_status aw_team_connect(aw_grid* g, const void* all_records) {
    CHECK_STATE(g);
    if (!all_records) return fail(AW_EINVAL, "records NULL");
    if (!team_mode(g)) {
        g->team_connected = true;
        return AW_OK;
    }
    const aw_team_record* recs = (const aw_team_record*)all_records;
    for (int r = 0; r < g->world; ++r)
        if (recs[r].rank != r || recs[r].world != g->world || recs[r].plane != g->geom.plane || recs[r].R != g->R)
            return fail(AW_EINVAL, "inconsistent team record of rank %d", r);
    CK(cudaSetDevice(g->device));
    void* p[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
    void* f[2] = {nullptr, nullptr};
    const int nb[2] = {g->rank - 1, g->rank + 1};
    for (int k = 0; k < 2; ++k) {
        int r = nb[k];
        if (r < 0 || r >= g->world) continue;
        aw_status st;
        if ((st = ipc_open(g, recs[r].u[0], &p[k][0])) || (st = ipc_open(g, recs[r].u[1], &p[k][1])) ||
            (st = ipc_open(g, recs[r].flags, &f[k])))
            return st;
    }
    int64_t nz_lo = g->rank > 0 ? recs[g->rank - 1].nz : 0;
    link_neighbours(g, (float*)p[0][0], (float*)p[0][1], (unsigned long long*)f[0], nz_lo, (float*)p[1][0],
                    (float*)p[1][1], (unsigned long long*)f[1]);
    CK(aw::launch_team_raise(g->peer_flag_lo, g->peer_flag_hi, enc(g, g->steps), g->s));
    CK(cudaStreamSynchronize(g->s));
    return AW_OK;
}

aw_status aw_team_connect_local(aw_grid** grids, int world) {
    if (!grids || world < 1) return fail(AW_EINVAL, "bad team");
    for (int r = 0; r < world; ++r) {
        if (!grids[r] || grids[r]->rank != r || grids[r]->world != world)
            return fail(AW_EINVAL, "grid %d is not rank %d of a %d-slab team", r, r, world);
        if (grids[r]->poisoned) return fail(AW_ESTATE, "grid %d poisoned", r);
    }
    for (int r = 0; r < world; ++r) {
        aw_grid* g = grids[r];
        aw_grid* lo = r > 0 ? grids[r - 1] : nullptr;
        aw_grid* hi = r + 1 < world ? grids[r + 1] : nullptr;
        if (lo && lo->device != g->device) {
            cudaSetDevice(g->device);
            cudaDeviceEnablePeerAccess(lo->device, 0);
            cudaGetLastError();
        }
        if (hi && hi->device != g->device) {
            cudaSetDevice(g->device);
            cudaDeviceEnablePeerAccess(hi->device, 0);
            cudaGetLastError();
        }
        link_neighbours(g, lo ? lo->ubuf[0] : nullptr, lo ? lo->ubuf[1] : nullptr, lo ? lo->d_team_flags : nullptr,
                        lo ? lo->geom.nz : 0, hi ? hi->ubuf[0] : nullptr, hi ? hi->ubuf[1] : nullptr,
                        hi ? hi->d_team_flags : nullptr);
    }
    for (int r = 0; r < world; ++r) {
        aw_grid* g = grids[r];
        CK(cudaSetDevice(g->device));
        CK(aw::launch_team_raise(g->peer_flag_lo, g->peer_flag_hi, enc(g, g->steps), g->s));
        CK(cudaStreamSynchronize(g->s));
    }
    return AW_OK;
}

aw_status aw_team_run(aw_grid** grids, int world, int nt, double dt) {
    if (!grids || world < 1) return fail(AW_EINVAL, "bad team");
    for (int r = 0; r < world; ++r) {
        CHECK_STATE(grids[r]);
        if (grids[r]->steps != grids[0]->steps) return fail(AW_ESTATE, "ranks are at different steps");
    }
    for (int r = 0; r < world; ++r) {
        aw_status st = run_begin(grids[r], nt, dt);
        if (st) return st;
    }
    std::vector<int64_t> launches(world, 0);
    // interleave the ranks step by step on their own streams
    for (int i = 0; i < nt; ++i) {
        for (int r = 0; r < world; ++r) {
            aw_grid* g = grids[r];
            if (g->opt_timing == 1 && (int64_t)g->tev.size() < 2 * (int64_t)nt) {
                while ((int64_t)g->tev.size() < 2 * (int64_t)nt) {
                    cudaEvent_t e;
                    CK(cudaEventCreate(&e));
                    g->tev.push_back(e);
                }
            }
            const bool ev = g->opt_timing == 1;
            cudaEvent_t e0 = ev ? g->tev[2 * i] : nullptr, e1 = ev ? g->tev[2 * i + 1] : nullptr;
            CK(cudaSetDevice(g->device));
            aw_status st = enqueue_step(g, i, g->cur, e0, e1, &launches[r]);
            if (st) return st;
            g->cur = 1 - g->cur;
        }
    }
    aw_status result = AW_OK;
    for (int r = 0; r < world; ++r) {
        aw_grid* g = grids[r];
        CK(cudaSetDevice(g->device));
        aw_status st = run_end(g, nt, launches[r]);
        if (st && result == AW_OK) result = st;
    }
    return result;
}

}  // extern "C"

