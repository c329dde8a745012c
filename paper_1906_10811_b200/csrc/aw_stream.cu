// aw_stream.cu -- host side of the 2.5D z-streaming stencil kernel (R-independent):
// plan construction, eta flags, injection lists, dispatch to the per-R translation units
// (aw_stream_r{1..8}.cu; the kernel itself is in aw_stream.cuh).
#include <algorithm>
#include <cstdlib>
#include <utility>
#include <vector>

#include "aw_stream.cuh"

namespace aw {

// ---------------------------------------------------------------------------
// eta flags: flags[tile][z] = 1 iff some a != 1 in the tile-plane
// ---------------------------------------------------------------------------
__global__ void eta_flags_kernel(Geom g, const float* __restrict__ a, int TX, int TY, int ntx, int nty,
                                 uint8_t* flags) {
    const int tile = blockIdx.x;
    const int z = blockIdx.y;
    const int x0 = (tile % ntx) * TX, y0 = (tile / ntx) * TY;
    bool any = false;
    for (int idx = threadIdx.x; idx < TX * TY; idx += blockDim.x) {
        int x = x0 + idx % TX, y = y0 + idx / TX;
        if (x < g.nx && y < g.ny) any |= a[(int64_t)z * g.plane + (int64_t)y * g.pitch + x] != 1.0f;
    }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) flags[(int64_t)tile * g.nz + z] = any ? 1 : 0;
}

__global__ void count_flags_kernel(const uint8_t* flags, int64_t n, unsigned long long* cnt) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += flags[i];
    atomicAdd(cnt, c);
}


static const StreamOps* stream_ops(int R) {
    switch (R) {
        case 1: return stream_ops_r1();
        case 2: return stream_ops_r2();
        case 3: return stream_ops_r3();
        case 4: return stream_ops_r4();
        case 5: return stream_ops_r5();
        case 6: return stream_ops_r6();
        case 7: return stream_ops_r7();
        case 8: return stream_ops_r8();
        default: return nullptr;
    }
}

cudaError_t stream_prepare(const Geom& g, const float* const* ubuf, const float* b, const float* a,
                           StreamPlan** plan, cudaStream_t s) {
    *plan = nullptr;
    if (g.ndim != 3) return cudaErrorNotSupported;
    StreamPlan* p = new StreamPlan();
    p->R = g.R;
    cudaError_t e = cudaSuccess;
    const StreamOps* ops = stream_ops(g.R);
    if (!ops) {
        delete p;
        return cudaErrorNotSupported;
    }
    e = ops->setup(p, g);
    if (e != cudaSuccess) {
        delete p;
        return e;
    }
    p->ntx = (g.nx + p->TX - 1) / p->TX;
    p->nty = (g.ny + p->TY - 1) / p->TY;
    // z chunks: enough items that the cyclic hand-out balances to ~1-2% (>= 8 items per CTA
    // when possible), chunks no thinner than 4R planes (warm-up overhead 2R/zc)
    const int ntiles = p->ntx * p->nty;
    int nzc = 1;
    // (the high-order kernel, zq > 1: >= 6 items per CTA -- every item start pays 2R warm-up planes)
    const int64_t per_cta = p->zq > 1 ? 6 : 8;
    while ((int64_t)ntiles * nzc < per_cta * p->grid && g.nz / (nzc * 2) >= 4 * g.R) nzc *= 2;
    if (const char* zc_env = dev_knob("AW_STREAM_ZC")) {  // development knob: planes per z chunk
        const int zc = atoi(zc_env);
        if (zc > 0) nzc = (g.nz + zc - 1) / zc;
    }
    p->zc = (g.nz + nzc - 1) / nzc;
    if (p->zq > 1 && !dev_knob("AW_STREAM_ZC"))  // the high-order kernel's full chunks: multiples of 2R+1
        p->zc = std::min(g.nz, (p->zc + p->zq - 1) / p->zq * p->zq);
    p->nzc = (g.nz + p->zc - 1) / p->zc;
    const int64_t nflags = (int64_t)ntiles * g.nz;
    if ((e = cudaMalloc(&p->flags, nflags + sizeof(unsigned long long) + 16)) != cudaSuccess) {
        delete p;
        return e;
    }
    p->d_count = reinterpret_cast<unsigned long long*>(p->flags + (nflags + 15) / 16 * 16 - 0);
    if ((e = stream_refresh(p, g, ubuf, b, a, s)) != cudaSuccess) {
        stream_release(p);
        return e;
    }
    *plan = p;
    return cudaSuccess;
}

// (Re)encode the tensor maps and recompute the per-(plane, tile) eta flags; no host sync.
cudaError_t stream_refresh(StreamPlan* p, const Geom& g, const float* const* ubuf, const float* b, const float* a,
                           cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    const StreamOps* ops = stream_ops(p->R);
    if (!ops) return cudaErrorNotSupported;
    p->map_cache.clear();  // model arrays may have moved
    e = ops->make_maps(p, g, ubuf, b, a);
    if (e != cudaSuccess) return e;
    const int ntiles = p->ntx * p->nty;
    const int64_t nflags = (int64_t)ntiles * g.nz;
    cudaMemsetAsync(p->d_count, 0, sizeof(unsigned long long), s);
    if (a) {
        dim3 grid(ntiles, g.nz);
        eta_flags_kernel<<<grid, 256, 0, s>>>(g, a, p->TX, p->TY, p->ntx, p->nty, p->flags);
        count_flags_kernel<<<148, 256, 0, s>>>(p->flags, nflags, p->d_count);
    } else {
        cudaMemsetAsync(p->flags, 0, nflags, s);
    }
    p->nflags = nflags;
    return cudaGetLastError();
}

// Percentage of (plane, tile) pairs that stream `a` (call after the stream synchronised).
int stream_eta_tiles_pct(const StreamPlan* p) {
    unsigned long long h = 0;
    if (!p || cudaMemcpy(&h, p->d_count, sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return p->nflags ? (int)(100.0 * (double)h / (double)p->nflags + 0.5) : 0;
}

void stream_plan_signature(const StreamPlan* p, std::string* sig) {
    if (!p) return;
    auto put = [&](const void* q, size_t n) { sig->append((const char*)q, n); };
    put(p->maps, sizeof p->maps);
    put(&p->flags, sizeof p->flags);
    put(p->tpsc, sizeof p->tpsc);
    put(p->tpe, sizeof p->tpe);
    put(&p->grid, sizeof p->grid);
    put(&p->ntx, sizeof p->ntx);
    put(&p->nty, sizeof p->nty);
    put(&p->nzc, sizeof p->nzc);
    put(&p->zc, sizeof p->zc);
    put(&p->ts0, sizeof p->ts0);
    put(&p->ts1, sizeof p->ts1);
    put(&p->ts_cap, sizeof p->ts_cap);
    put(p->item_inj, sizeof p->item_inj);
}

void stream_set_timestamps(StreamPlan* p, unsigned long long* ts0, unsigned long long* ts1, int cap) {
    if (!p) return;
    p->ts0 = ts0;
    p->ts1 = ts1;
    p->ts_cap = ts0 ? cap : 0;
}

size_t stream_plan_bytes(const StreamPlan* p) {
    if (!p) return 0;
    size_t n = p->flags ? (size_t)p->nflags + sizeof(unsigned long long) + 16 : 0;
    for (int k = 0; k < 2; ++k) {
        if (p->tpsc[k]) n += (size_t)p->nflags * sizeof(int2);
        n += p->tpe_cap[k] * sizeof(int4);
        if (p->item_inj[k]) n += (size_t)p->ntx * p->nty * p->nzc;
    }
    if (p->res_done) n += (size_t)p->ntx * p->nty * p->nzc * sizeof(unsigned long long);
    n += p->ritem_cap * sizeof(int);
    if (p->tb_done) n += (size_t)p->tb_nzc * p->ntx * p->nty * sizeof(unsigned long long);
    return n;
}

void stream_release(StreamPlan* p) {
    if (!p) return;
    if (p->flags) cudaFree(p->flags);
    for (int k = 0; k < 2; ++k) {
        if (p->tpsc[k]) cudaFree(p->tpsc[k]);
        if (p->tpe[k]) cudaFree(p->tpe[k]);
        if (p->item_inj[k]) cudaFree(p->item_inj[k]);
    }
    if (p->res_done) cudaFree(p->res_done);
    if (p->ritem) cudaFree(p->ritem);
    if (p->tb_done) cudaFree(p->tb_done);
    delete p;
}

// Injection lists per tile-plane for the fused kernel.  corner_lin: the owned unique injection
// corners (global row-major index, ascending), ptr: their CSR ranges into the entry arrays.
cudaError_t stream_set_injection(StreamPlan* p, const Geom& g, int64_t z0, const int64_t* corner_lin, const int* ptr,
                                 int nuc, cudaStream_t s, int set) {
    const int ntiles = p->ntx * p->nty;
    const int64_t ntp = (int64_t)ntiles * g.nz;
    cudaError_t e;
    int2*& tpsc = p->tpsc[set];
    int4*& tpe = p->tpe[set];
    size_t& tpe_cap = p->tpe_cap[set];
    if (!tpsc && (e = cudaMalloc(&tpsc, ntp * sizeof(int2))) != cudaSuccess) return e;
    std::vector<std::pair<int64_t, int4>> ents;  // key = tile*nz + z
    const int64_t per_plane = (int64_t)g.ny * g.nx;
    for (int c = 0; c < nuc; ++c) {
        const int64_t lin = corner_lin[c];
        const int z = (int)(lin / per_plane - z0);
        const int y = (int)((lin % per_plane) / g.nx), x = (int)(lin % g.nx);
        const int tile = (y / p->TY) * p->ntx + x / p->TX;
        const int pos = (y % p->TY) * 64 + (x % p->TX);
        ents.push_back({(int64_t)tile * g.nz + z, make_int4(pos, ptr[c], ptr[c + 1], 0)});
    }
    std::stable_sort(ents.begin(), ents.end(),
                     [](const std::pair<int64_t, int4>& a, const std::pair<int64_t, int4>& b) { return a.first < b.first; });
    std::vector<int2> tpsc_h;  // only the touched keys are uploaded; the rest is zero (count 0)
    if ((e = cudaMemsetAsync(tpsc, 0, ntp * sizeof(int2), s)) != cudaSuccess) return e;
    // per work item (tile, z chunk): does it hold injection corners of this set (the high-order
    // kernel runs those items on its generic path)
    const int64_t nitems = (int64_t)ntiles * p->nzc;
    uint8_t*& item_inj = p->item_inj[set];
    if (!item_inj && (e = cudaMalloc(&item_inj, nitems)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(item_inj, 0, nitems, s)) != cudaSuccess) return e;
    if (ents.empty()) return cudaSuccess;
    std::vector<int64_t> inj_items;
    for (const auto& en : ents) {
        const int64_t tile = en.first / g.nz, z = en.first % g.nz;
        const int64_t item = (z / p->zc) * ntiles + tile;
        if (inj_items.empty() || inj_items.back() != item) inj_items.push_back(item);
    }
    std::sort(inj_items.begin(), inj_items.end());
    inj_items.erase(std::unique(inj_items.begin(), inj_items.end()), inj_items.end());
    static const uint8_t one_byte = 1;  // (pageable source: the copy is staged before the call returns)
    for (int64_t it : inj_items)
        if ((e = cudaMemcpyAsync(item_inj + it, &one_byte, 1, cudaMemcpyHostToDevice, s))) return e;
    if (tpe_cap < ents.size()) {
        if (tpe) cudaFree(tpe);
        tpe = nullptr;
        tpe_cap = 0;
        if ((e = cudaMalloc(&tpe, ents.size() * sizeof(int4))) != cudaSuccess) return e;
        tpe_cap = ents.size();
    }
    std::vector<int4> tpe_h(ents.size());
    for (size_t i = 0; i < ents.size(); ++i) tpe_h[i] = ents[i].second;
    if ((e = cudaMemcpyAsync(tpe, tpe_h.data(), tpe_h.size() * sizeof(int4), cudaMemcpyHostToDevice, s)))
        return e;
    // the touched keys' {first, count} in one sparse scatter (host list of (key, value) pairs)
    std::vector<int2> vals;
    std::vector<int64_t> keys;
    for (size_t i = 0; i < ents.size();) {
        size_t j = i;
        while (j < ents.size() && ents[j].first == ents[i].first) ++j;
        keys.push_back(ents[i].first);
        vals.push_back(make_int2((int)i, (int)(j - i)));
        i = j;
    }
    for (size_t k = 0; k < keys.size(); ++k)
        if ((e = cudaMemcpyAsync(tpsc + keys[k], &vals[k], sizeof(int2), cudaMemcpyHostToDevice, s))) return e;
    return cudaStreamSynchronize(s);  // the host staging vectors die here
}

bool stream_resident_ready(const StreamPlan* p) {
    const StreamOps* ops = p ? stream_ops(p->R) : nullptr;
    return ops && ops->launch_res && p->res_ok;
}

cudaError_t stream_set_receivers(StreamPlan* p, const Geom& g, const int64_t* rec_off, int nrl, int nc,
                                 cudaStream_t s) {
    const int ntiles = p->ntx * p->nty;
    const int64_t nitems = (int64_t)ntiles * p->nzc;
    std::vector<int> cnt(nitems + 1, 0), item_of(nrl);
    for (int r = 0; r < nrl; ++r) {
        const int64_t off = rec_off[(int64_t)r * nc];  // the base corner (never skipped)
        const int z = (int)(off / g.plane) - g.R;
        const int64_t rem = off % g.plane;
        const int y = (int)(rem / g.pitch), x = (int)(rem % g.pitch);
        const int it = (z / p->zc) * ntiles + (y / p->TY) * p->ntx + x / p->TX;
        item_of[r] = it;
        ++cnt[it + 1];
    }
    std::vector<int> h(nitems + 1 + nrl);
    for (int64_t i = 0; i < nitems; ++i) cnt[i + 1] += cnt[i];
    for (int64_t i = 0; i <= nitems; ++i) h[i] = cnt[i];
    for (int r = 0; r < nrl; ++r) h[nitems + 1 + cnt[item_of[r]]++] = r;  // ascending r within an item
    cudaError_t e;
    if (p->ritem_cap < h.size()) {
        if (p->ritem) cudaFree(p->ritem);
        p->ritem = nullptr;
        p->ritem_cap = 0;
        if ((e = cudaMalloc(&p->ritem, h.size() * sizeof(int)))) return e;
        p->ritem_cap = h.size();
    }
    if (!p->res_done && (e = cudaMalloc(&p->res_done, nitems * sizeof(unsigned long long)))) return e;
    if ((e = cudaMemcpyAsync(p->ritem, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, s))) return e;
    return cudaStreamSynchronize(s);  // the host staging vector dies here
}

cudaError_t stream_resident_begin(StreamPlan* p, cudaStream_t s) {
    if (!p || !p->res_done) return cudaErrorNotSupported;
    return cudaMemsetAsync(p->res_done, 0, (size_t)p->ntx * p->nty * p->nzc * sizeof(unsigned long long), s);
}

cudaError_t launch_stencil_resident(StreamPlan* p, const Geom& g, const Coefs& c, int cur0, float* const* buf,
                                    const float* b, const float* a, const Sparse& sp, const int64_t* d_base,
                                    int step0, int nsteps, cudaStream_t s) {
    const StreamOps* ops = p ? stream_ops(p->R) : nullptr;
    if (!ops || !ops->launch_res) return cudaErrorNotSupported;
    return ops->launch_res(p, g, c, cur0, buf, b, a, sp, d_base, step0, nsteps, s);
}

cudaError_t launch_stencil_stream(StreamPlan* p, const Geom& g, const Coefs& c, int parity_cur, const float* ucur,
                                  float* unext, const float* b, const float* a, const Halo& halo, int parity_next,
                                  const Sparse& sp, const int64_t* d_base, int step_i, cudaStream_t s) {
    // u^n is read through the tensor map of buffer parity_cur (stencil) and ucur (receivers)
    if (!p) return cudaErrorNotSupported;
    const StreamOps* ops = stream_ops(p->R);
    if (!ops) return cudaErrorNotSupported;
    return ops->launch(p, g, c, parity_cur, ucur, unext, b, a, halo, parity_next, sp, d_base, step_i, s);
}

cudaError_t launch_stencil_stream_bufs(StreamPlan* p, const Geom& g, const Coefs& c, const float* ucur,
                                       const float* uprev, float* unext, const float* b, const float* a,
                                       const Sparse& sp, int inj_set, const int64_t* d_base, int step_i,
                                       cudaStream_t s) {
    if (!p || inj_set < 0 || inj_set > 1) return cudaErrorNotSupported;
    const StreamOps* ops = stream_ops(p->R);
    if (!ops) return cudaErrorNotSupported;
    return ops->launch_bufs(p, g, c, ucur, uprev, unext, b, a, sp, inj_set, d_base, step_i, s);
}

// NEXT-1: temporal-blocking plan (completion-epoch array of the A items).  Z = planes per chunk,
// >= 2R so a B chunk needs only the A chunks c-1 and c; 0 = default (16, or 2R if larger).
cudaError_t stream_tb_prepare(StreamPlan* p, const Geom& g, int Z) {
    if (!p) return cudaErrorNotSupported;
    if (Z <= 0) Z = 32;  // best of 8/16/24/32/48/64 on C3 (profiles/r1/tb_sweep.jsonl)
    if (const char* z_env = dev_knob("AW_TB_Z")) {  // development knob
        const int z = atoi(z_env);
        if (z > 0) Z = z;
    }
    if (Z < 2 * g.R) Z = 2 * g.R;
    int lead = 2;  // A phases handed out ahead of the first B phase (>= 1: B(c) must follow A(c))
    if (const char* l_env = dev_knob("AW_TB_LEAD")) lead = atoi(l_env) > 1 ? atoi(l_env) : 1;
    p->tb_lead = lead;
    const int nzc = (g.nz + Z - 1) / Z;
    const int64_t n = (int64_t)nzc * p->ntx * p->nty;
    if (p->tb_done && p->tb_Z == Z && p->tb_nzc == nzc) return cudaSuccess;
    if (p->tb_done) cudaFree(p->tb_done);
    p->tb_done = nullptr;
    cudaError_t e = cudaMalloc(&p->tb_done, n * sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
    // epochs only grow, so the array is zeroed once (synchronously: no stream is involved yet)
    if ((e = cudaMemset(p->tb_done, 0, n * sizeof(unsigned long long))) != cudaSuccess) return e;
    p->tb_Z = Z;
    p->tb_nzc = nzc;
    p->tb_epoch = 0;
    return cudaSuccess;
}

cudaError_t launch_stencil_tb(StreamPlan* p, const Geom& g, const Coefs& c, const float* x, float* y, float* v,
                              const float* b, const float* a, const Sparse& sp, const int64_t* d_base, int step_i,
                              cudaStream_t s) {
    const StreamOps* ops = p ? stream_ops(p->R) : nullptr;
    if (!ops) return cudaErrorNotSupported;
    return ops->launch_tb(p, g, c, x, y, v, b, a, sp, d_base, step_i, s);
}

// Re-encode the per-parity tensor maps after the wavefield buffers were permuted (no kernels).
cudaError_t stream_remap(StreamPlan* p, const Geom& g, const float* const* ubuf, const float* b, const float* a) {
    const StreamOps* ops = p ? stream_ops(p->R) : nullptr;
    if (!ops) return cudaErrorNotSupported;
    return ops->make_maps(p, g, ubuf, b, a);
}

}  // namespace aw
