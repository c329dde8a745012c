// aw_resident2d.cu -- small 2D grids (BASELINE.json configs[0], the 101^2 case):
// every time step of an aw_run in ONE launch of one thread-block CLUSTER whose shared memory holds
// the whole grid.
//
// The rows of the grid are split into CS nearly equal strips, one per CTA of a cluster of CS <= 8
// CTAs (one per SM).  Each CTA keeps its strip in shared memory for the whole run: both wavefield
// levels with R ghost rows above and below (and zero ghost columns), b and -- where eta != 0 -- a,
// plus its receivers' corners and weights, the injection CSR and a 32-row chunk of the wavelet, so
// no step waits on a global-memory load (traces are buffered per 32-step chunk).  For each step n of
// the run
//   * the receivers read u^n (before the step),
//   * every thread updates its column pairs (packed fp32; per half the canonical sequence of SURVEY
//     §8(c).6, axis 1 (x) then axis 0 (z)) in place over u^{n-1},
//   * the thread that owns a source corner adds the CSR-ordered injection to the value it just
//     computed (corner ascending, source ascending: Q11) before storing it,
//   * a strip's first and last R rows are also stored straight into the neighbouring CTAs' ghost
//     rows with st.async (distributed shared memory: the halo exchange fused into the update, as in
//     the 3D team kernel), each store counting its bytes on the receiving CTA's mbarrier, and
//   * step n+1 starts after a CTA barrier and the two neighbours' halo bytes of step n arrived (per-side,
//     per-step-parity mbarriers; no cluster-wide barrier or GPU-scope fence per step),
// and finally each CTA writes both levels of its strip back to the wavefield buffers (restart /
// aw_read_wavefield see exactly what the per-step kernels would have left).  No HBM traffic per
// step (traces aside): a step costs one pass over ~1 column pair per thread plus the cluster
// barrier, against ~2 launches (stencil + sparse kernel, ~3-6 us) per step of the per-step path.
//
// Every operation is an explicit-rounding intrinsic, as in stencil_v1_kernel: value-identical to
// the fp32 oracle (tests/test_gpu_resident2d.py).
#include <cooperative_groups.h>

#include <algorithm>

#include "aw_internal.h"

namespace cg = cooperative_groups;

namespace aw {

namespace {

#ifndef AW_R2_THREADS
#define AW_R2_THREADS 512  // 1024 and 256 measured 6 % and 3 % slower on C1 (tools/gpu_r2_c1ab.sh)
#endif
constexpr int kR2Threads = AW_R2_THREADS;
constexpr int kR2WavRows = 32;  // wavelet rows staged per refill (one extra barrier per 32 steps)
constexpr int kR2MaxCluster = 8;

// Shared-memory layout of one CTA (4-byte words, in this order; the same in every CTA of the cluster,
// so a neighbour's word is this CTA's offset mapped to its rank): both wavefield levels, b [, a], the
// receivers' corner indices / weights / ids, the injection corners (point index, CSR pointers,
// sources, scales) and a chunk of wavelet rows.  A level stores strip row zl in [-R, nzl + R) at
// (zl + R) * Ps + C0 + x: R ghost rows above and below (zero at the grid's ends, the neighbours'
// boundary rows inside), rows padded to an even pitch Ps >= nx + R whose tail (>= R zeros) is both
// the right ghosts of a row and the left ghosts of the next, and an even column offset C0 >= R, so
// every even x starts an 8-byte aligned column pair.  b and a use zl * Ps + x.
struct R2Plan {
    int CS, nzl_max;
    int Ps, C0, slen;
    int o_b, o_a, o_rsi, o_rw, o_rid, o_ip, o_iptr, o_isrc, o_is, o_wav, o_tr, o_mb;
    int words;
};

struct R2Args {
    Coefs c;
    float* u0;          // wavefield buffer holding u^n at entry (base = row -R)
    float* u1;          // u^{n-1} at entry
    const float* b;     // model layout (nz rows x pitch)
    const float* a;     // null: no damping
    int64_t pitch;      // global row pitch (floats)
    int nx, nz;
    int PR;             // column pairs per row, ceil(nx / 2)
    R2Plan P;
    Sparse sp;
    const int64_t* d_base;
    int step0, nsteps;
};

__host__ __device__ __forceinline__ int strip_lo(int nz, int CS, int c) { return (int)((int64_t)nz * c / CS); }

R2Plan r2_plan(const Geom& g, const Sparse& sp, bool damp, int CS) {
    R2Plan P{};
    const int R = g.R;
    P.CS = CS;
    P.nzl_max = (g.nz + CS - 1) / CS;
    P.C0 = (R + 1) / 2 * 2;
    P.Ps = (g.nx + R + 1) / 2 * 2;
    // + slack: the outermost float2 x-neighbour loads of odd R reach one column past the ghosts
    P.slen = ((P.nzl_max + 2 * R) * P.Ps + P.C0 + 4 + 3) / 4 * 4;
    int o = 2 * P.slen;
    P.o_b = o;
    o += P.nzl_max * P.Ps;
    P.o_a = o;
    if (damp) o += P.nzl_max * P.Ps;
    const int nrc = sp.nrl * sp.nc;
    P.o_rsi = o;
    o += nrc;
    P.o_rw = o;
    o += nrc;
    P.o_rid = o;
    o += sp.nrl;
    P.o_ip = o;
    o += sp.nuc;
    P.o_iptr = o;
    o += sp.nuc > 0 ? sp.nuc + 1 : 0;
    const int nent = sp.nuc > 0 ? sp.nent : 0;
    P.o_isrc = o;
    o += nent;
    P.o_is = o;
    o += nent;
    P.o_wav = o;  // per chunk row, the wavelet value of every injection entry (gathered: q[n][src_e])
    o += kR2WavRows * nent;
    P.o_tr = o;
    o += kR2WavRows * sp.nrl;
    P.o_mb = (o + 1) / 2 * 2;  // 4 mbarriers (8-byte aligned): ghost rows from below / above, by step parity
    o = P.o_mb + 8;
    P.words = o;
    return P;
}

__device__ __forceinline__ float2 ld2s(const float* p) { return *reinterpret_cast<const float2*>(p); }
// cluster barrier with release/acquire at cluster scope: orders the shared-memory (local and
// distributed) stores of a step before the neighbours' reads of the next one.  (cg's cluster.sync()
// adds a GPU-scope MEMBAR that also waits for the trace stores to global memory.)
__device__ __forceinline__ uint32_t smem_u32a(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// asynchronous store into a neighbour CTA's shared memory that counts its bytes on that CTA's mbarrier
__device__ __forceinline__ void st_async2(uint32_t addr, float2 v, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "f"(v.x), "f"(v.y), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void st_async1(uint32_t addr, float v, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(addr), "f"(v),
                 "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32a(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32a(bar)), "r"(bytes) : "memory");
}
// wait for the phase with the given parity; acquire at cluster scope (the bytes came from another CTA)
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32a(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// AS (default): the halo rows go to the neighbours with st.async, each CTA waits only for its two
// neighbours' bytes (per-side, per-step-parity mbarriers) -- no cluster-wide barrier and no GPU-scope
// fence per step; !AS: plain DSMEM stores + one cluster barrier per step (kept for A/B runs)
template <int R, bool DAMP, bool AS>
__global__ void __launch_bounds__(kR2Threads, 1) resident2d_kernel(const R2Args A) {
    extern __shared__ __align__(16) float smem[];
    cg::cluster_group cl = cg::this_cluster();
    int* smi = reinterpret_cast<int*>(smem);
    const int tid = threadIdx.x;
    const R2Plan& P = A.P;
    const int Ps = P.Ps, C0 = P.C0, CS = P.CS;
    const int cr = (int)cl.block_rank();
    const int zlo = strip_lo(A.nz, CS, cr), nzl = strip_lo(A.nz, CS, cr + 1) - zlo;
    const int nzl_dn = cr > 0 ? zlo - strip_lo(A.nz, CS, cr - 1) : 0;  // rows of the CTA below (rank cr-1)
    float* S0 = smem;
    float* S1 = smem + P.slen;
    const int* rsi = smi + P.o_rsi;  // receivers: shared-memory index of each corner (-1: skipped)
    const float* rw = smem + P.o_rw;
    const int* rid = smi + P.o_rid;  // trace column; -1: not this CTA's receiver
    const int* ip = smi + P.o_ip;    // injection corners: point index z*nx + x (ascending)
    const int* iptr = smi + P.o_iptr;
    const int* isrc = smi + P.o_isrc;
    const float* is = smem + P.o_is;
    float* wav = smem + P.o_wav;     // [row of the chunk][entry]: q[n][src_e] for the chunk's steps
    float* trb = smem + P.o_tr;      // trace rows of the current chunk (written to global once per chunk)
    const Sparse& sp = A.sp;

    // ---- load: zero everything staged per point (ghosts, pads), copy both levels (strip + ghost rows:
    // the buffers' rows z + R, z in [zlo - R, zlo + nzl + R), hold zeros beyond the grid), b, a, and
    // the sparse tables ----
    for (int i = tid; i < P.o_rsi; i += kR2Threads) smem[i] = 0.0f;
    __syncthreads();
    for (int i = tid; i < (nzl + 2 * R) * A.nx; i += kR2Threads) {
        const int r = i / A.nx, x = i - r * A.nx;  // r = zl + R
        const int64_t go = (int64_t)(zlo + r) * A.pitch + x;
        S0[r * Ps + C0 + x] = A.u0[go];
        S1[r * Ps + C0 + x] = A.u1[go];
    }
    for (int i = tid; i < nzl * A.nx; i += kR2Threads) {
        const int zl = i / A.nx, x = i - zl * A.nx;
        smem[P.o_b + zl * Ps + x] = A.b[(int64_t)(zlo + zl) * A.pitch + x];
        if (DAMP) smem[P.o_a + zl * Ps + x] = A.a[(int64_t)(zlo + zl) * A.pitch + x];
    }
    // receivers whose base corner row lies in the strip; corners: wavefield-buffer offset
    // ((z+R)*pitch + x) -> local index (its +1 row may be the first ghost row below the strip)
    for (int t = tid; t < sp.nrl; t += kR2Threads) {
        const int zb = (int)(sp.rec_off[(int64_t)t * sp.nc] / A.pitch) - R;
        const bool mine = zb >= zlo && zb < zlo + nzl;
        smi[P.o_rid + t] = mine ? sp.rec_id[t] : -1;
        for (int beta = 0; beta < sp.nc; ++beta) {
            const int64_t off = sp.rec_off[(int64_t)t * sp.nc + beta];
            const int zz = (int)(off / A.pitch);
            smi[P.o_rsi + t * sp.nc + beta] =
                off < 0 || !mine ? -1 : (zz - zlo) * Ps + C0 + (int)(off - (int64_t)zz * A.pitch);
            smem[P.o_rw + t * sp.nc + beta] = sp.rec_w[(int64_t)t * sp.nc + beta];
        }
    }
    uint32_t inj_mask = 0;  // bit k: the column pair of unit tid + 1024 k holds an injection corner
    // this thread's first corners, each packed as (csr begin << 12) | (entries << 6) | (k << 1) | h;
    // a thread with more than kInjRegs corners finds the rest by binary search
    constexpr int kInjRegs = 4;
    int inj_reg[kInjRegs];
#pragma unroll
    for (int i = 0; i < kInjRegs; ++i) inj_reg[i] = -1;
    bool inj_more = false;
    if (sp.nuc > 0) {
        int nreg = 0;
        for (int c = 0; c < sp.nuc; ++c) {
            const int64_t off = sp.inj_off[c];
            const int zz = (int)(off / A.pitch);
            const int z = zz - R, x = (int)(off - (int64_t)zz * A.pitch);
            const int u = (z - zlo) * A.PR + (x >> 1);
            if (z >= zlo && z < zlo + nzl && (u & (kR2Threads - 1)) == tid) {
                const int k = u / kR2Threads;
                inj_mask |= 1u << k;
                const int e0 = sp.inj_ptr[c], ne = sp.inj_ptr[c + 1] - e0;
                const int rec = (e0 << 12) | (ne << 6) | (k << 1) | (x & 1);
                bool placed = false;
#pragma unroll
                for (int i = 0; i < kInjRegs; ++i)
                    if (!placed && i == nreg && ne < 64 && e0 < (1 << 19)) {
                        inj_reg[i] = rec;
                        placed = true;
                    }
                if (placed) ++nreg; else inj_more = true;
            }
            if (c % kR2Threads == tid) smi[P.o_ip + c] = z * A.nx + x;
        }
        for (int i = tid; i <= sp.nuc; i += kR2Threads) smi[P.o_iptr + i] = sp.inj_ptr[i];
        const int nent = sp.inj_ptr[sp.nuc];
        for (int i = tid; i < nent; i += kR2Threads) {
            smi[P.o_isrc + i] = sp.inj_src[i];
            smem[P.o_is + i] = sp.inj_s[i];
        }
    }
    const int64_t n0 = *A.d_base + A.step0;
    // work unit u = tid + 1024 k: the column pair (2 xp, 2 xp + 1) of strip row zl, u = zl * PR + xp
    const int nunits = nzl * A.PR;
    const int q = kR2Threads / A.PR, r = kR2Threads - q * A.PR;  // u += 1024 -> (zl, xp) += (q, r) with carry
    const int zl_start = tid / A.PR, xp_start = tid - zl_start * A.PR;
    const int kcount = nunits / kR2Threads + (tid < nunits % kR2Threads ? 1 : 0);
    const int o_start = (zl_start + R) * Ps + C0 + 2 * xp_start;  // level index of the pair's first column
    const int ob_start = zl_start * Ps + 2 * xp_start;             // b / a index
    const int o_step = q * Ps + 2 * r, o_wrap = Ps - 2 * A.PR;     // index advance per 1024 units (+ row wrap)
    const bool odd_nx = A.nx & 1;
    const bool has_dn = cr > 0, has_up = cr < CS - 1;
    // a strip row zl < R is the ghost row nzl_dn + zl of the CTA below; zl >= nzl - R the ghost row
    // zl - nzl of the CTA above (the same local offset shifted by whole rows)
    const int shift_dn = nzl_dn * Ps, shift_up = -nzl * Ps;
    const float* Bs = smem + P.o_b;
    const float* As = smem + P.o_a;
    const float2 c0 = f2(A.c.C0, A.c.C0), two = f2(2.0f, 2.0f), one = f2(1.0f, 1.0f);
    // mb[0 + parity]: ghost rows from the CTA below (its last R rows), mb[2 + parity]: from the CTA above
    uint64_t* mb = reinterpret_cast<uint64_t*>(smem + P.o_mb);
    const uint32_t side_bytes = (uint32_t)R * A.nx * 4u;
    if (AS && tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init1(&mb[i]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // every CTA has loaded its strip (and initialised its barriers) before any neighbour stores into it
    cluster_barrier();

    // trace rows [n_first, n_first + rows) of this CTA's receivers from the chunk buffer to global memory
    auto flush_traces = [&](int64_t n_first, int rows) {
        for (int i = tid; i < rows * sp.nrl; i += kR2Threads) {
            const int rr = i / sp.nrl, t = i - rr * sp.nrl;
            if (rid[t] >= 0) sp.traces[(n_first + rr) * sp.nr + rid[t]] = trb[rr * sp.nrl + t];
        }
    };
    // one time step: U = u^n, W = u^{n-1} in / u^{n+1} out (in place); s = local step index
    auto step = [&](const float* __restrict__ U, float* __restrict__ W, int s) {
        const int64_t n = n0 + s;
        if (AS && tid == 0) {  // this step's halo bytes from each neighbour (the one arrival of the phase)
            if (has_dn) mbar_expect(&mb[0 + (s & 1)], side_bytes);
            if (has_up) mbar_expect(&mb[2 + (s & 1)], side_bytes);
        }
        if (s % kR2WavRows == 0 && (sp.nuc > 0 || sp.nrl > 0)) {
            // chunk start: the previous chunk's trace rows go to global memory (the GPU-scope fence of the
            // cluster barrier then waits for these stores once per chunk, not every step), and the next
            // chunk of wavelet rows comes in (the previous one is no longer read)
            if (s > 0) flush_traces(n - kR2WavRows, kR2WavRows);
            const int rows = min(kR2WavRows, A.nsteps - s);
            if (sp.nuc > 0)  // gathered: entry e of chunk row rr = q[n + rr][src_e]
                for (int i = tid; i < rows * sp.nent; i += kR2Threads) {
                    const int rr = i / sp.nent, e = i - rr * sp.nent;
                    wav[i] = sp.wavelet[(n + rr) * sp.ns + isrc[e]];
                }
            __syncthreads();
        }
        // receivers: fma chain over the corners of u^n (before the step), from the last thread down (the
        // threads past the strip's last work unit have no unit to update)
        for (int t = kR2Threads - 1 - tid; t < sp.nrl; t += kR2Threads) {
            if (rid[t] < 0) continue;
            float acc = 0.0f;
            for (int beta = 0; beta < sp.nc; ++beta) {
                const int si = rsi[t * sp.nc + beta];
                if (si < 0) continue;
                acc = __fmaf_rn(rw[t * sp.nc + beta], U[si], acc);
            }
            trb[(s % kR2WavRows) * sp.nrl + t] = acc;
        }
        float* W_dn = has_dn ? cl.map_shared_rank(W, cr - 1) : W;  // the neighbours' copies of this level
        float* W_up = has_up ? cl.map_shared_rank(W, cr + 1) : W;
        // st.async targets: the neighbours' ghost rows of W and their barriers for this step (the CTA below
        // receives from above: its mb[2 + parity]; the CTA above: its mb[0 + parity])
        // (map W's own base -- a valid local address -- then shift in 32-bit arithmetic: W + shift_up lies
        // below this CTA's window, only W + shift_up + o of a boundary row is inside the neighbour's)
        const uint32_t wa_dn = has_dn ? mapa_u32(smem_u32a(W), cr - 1) + 4u * (uint32_t)shift_dn : 0u;
        const uint32_t wa_up = has_up ? mapa_u32(smem_u32a(W), cr + 1) + 4u * (uint32_t)shift_up : 0u;
        const uint32_t mb_dn = has_dn ? mapa_u32(smem_u32a(&mb[2 + (s & 1)]), cr - 1) : 0u;
        const uint32_t mb_up = has_up ? mapa_u32(smem_u32a(&mb[0 + (s & 1)]), cr + 1) : 0u;
        int xp = xp_start, zl = zl_start, o = o_start, ob = ob_start;
#pragma unroll 2
        for (int k = 0; k < kcount; ++k) {
            // the column pair (x, x+1), x = 2 xp, as packed fp32 (per half == the scalar canonical sequence)
            const float2 uc = ld2s(U + o);
            float2 L = __fmul2_rn(c0, uc);
            {   // axis 1 (x): v[K + m] = columns (x + 2m, x + 2m + 1)
                constexpr int K = (R + 1) / 2;
                float2 v[2 * K + 1];
#pragma unroll
                for (int m = -K; m <= K; ++m) v[K + m] = ld2s(U + o + 2 * m);
#pragma unroll
                for (int j = 1; j <= R; ++j) {
                    const int m = j >> 1;
                    const float cj = A.c.C[1][j];
                    if (j & 1) {  // odd j: the pair sums sit in two float2s (one useful half each)
                        const float2 sa = __fadd2_rn(v[K - m - 1], v[K + m]);  // .y = u[x-j] + u[x+j]
                        const float2 sb = __fadd2_rn(v[K - m], v[K + m + 1]);  // .x = u[x+1-j] + u[x+1+j]
                        L.x = __fmaf_rn(cj, sa.y, L.x);
                        L.y = __fmaf_rn(cj, sb.x, L.y);
                    } else {
                        L = __ffma2_rn(f2(cj, cj), __fadd2_rn(v[K - m], v[K + m]), L);
                    }
                }
            }
#pragma unroll
            for (int j = 1; j <= R; ++j) {  // axis 0 (z)
                const float cj = A.c.C[0][j];
                L = __ffma2_rn(f2(cj, cj), __fadd2_rn(ld2s(U + o - j * Ps), ld2s(U + o + j * Ps)), L);
            }
            const float2 um = ld2s(W + o);
            // t = 2u - u^{n-1} (2u exact: one rounding), w = fma(b, L, t)
            const float2 t = __ffma2_rn(two, uc, f2(-um.x, -um.y));
            const float2 w = __ffma2_rn(ld2s(Bs + ob), L, t);
            float2 un;
            if constexpr (DAMP) {
                const float2 aa = ld2s(As + ob);
                un = __ffma2_rn(aa, w, __fmul2_rn(__fadd2_rn(one, f2(-aa.x, -aa.y)), um));
            } else {
                un = __ffma2_rn(one, w, __fmul2_rn(f2(0.0f, 0.0f), um));  // a = 1: the canonical sequence
            }
            const int x = 2 * xp;
            if ((inj_mask >> k) & 1u) {
                // injection corners of this pair: the sequential fma chain over each corner's sources in CSR
                // order (corner ascending, then source) -- corners from the registers, and (a thread with more
                // corners than registers) the rest by binary search of the staged corner list
                const float* qn = wav + (s % kR2WavRows) * sp.nent;
#pragma unroll
                for (int i = 0; i < kInjRegs; ++i) {
                    const int rec = inj_reg[i];
                    if (rec < 0 || ((rec >> 1) & 31) != k) continue;
                    const int e0 = rec >> 12, e1 = e0 + ((rec >> 6) & 63);
                    float v = (rec & 1) ? un.y : un.x;
                    for (int e = e0; e < e1; ++e) v = __fmaf_rn(is[e], qn[e], v);
                    if (rec & 1) un.y = v; else un.x = v;
                }
#pragma unroll
                for (int h = 0; h < 2 && inj_more; ++h) {
                    const int pt = (zlo + zl) * A.nx + x + h;
                    int lo = 0, hi = sp.nuc - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (ip[mid] < pt) lo = mid + 1; else hi = mid;
                    }
                    if (ip[lo] != pt || x + h >= A.nx) continue;
                    const int e0 = iptr[lo], e1 = iptr[lo + 1];
                    bool in_regs = false;  // applied above already
#pragma unroll
                    for (int i = 0; i < kInjRegs; ++i)
                        in_regs |= inj_reg[i] >= 0 && (inj_reg[i] >> 12) == e0 && ((inj_reg[i] >> 1) & 31) == k;
                    if (in_regs) continue;
                    float v = h ? un.y : un.x;
                    for (int e = e0; e < e1; ++e) v = __fmaf_rn(is[e], qn[e], v);
                    if (h) un.y = v; else un.x = v;
                }
            }
            // store: here, and (boundary rows) into the neighbours' ghost rows; a row can be both a lower
            // and an upper boundary row of a thin strip, so the two targets are tested separately
            const bool pair = !(odd_nx && xp == A.PR - 1);  // else the second column is the row's ghost
            auto put = [&](float* base) {
                if (pair) *reinterpret_cast<float2*>(base + o) = un;
                else base[o] = un.x;
            };
            put(W);
            if constexpr (AS) {
                auto put_async = [&](uint32_t wa, uint32_t mbr) {
                    if (pair) st_async2(wa + 4u * (uint32_t)o, un, mbr);
                    else st_async1(wa + 4u * (uint32_t)o, un.x, mbr);
                };
                if (has_dn && zl < R) put_async(wa_dn, mb_dn);
                if (has_up && zl >= nzl - R) put_async(wa_up, mb_up);
            } else {
                if (has_dn && zl < R) put(W_dn + shift_dn);
                if (has_up && zl >= nzl - R) put(W_up + shift_up);
            }
            o += o_step;
            ob += o_step;
            xp += r;
            zl += q;
            if (xp >= A.PR) {
                xp -= A.PR;
                ++zl;
                o += o_wrap;
                ob += o_wrap;
            }
        }
        if constexpr (AS) {
            __syncthreads();  // this CTA's rows of u^{n+1} complete, its reads of u^n done
            if (has_dn) mbar_wait_cl(&mb[0 + (s & 1)], (uint32_t)(s >> 1) & 1u);  // ghost rows of u^{n+1}
            if (has_up) mbar_wait_cl(&mb[2 + (s & 1)], (uint32_t)(s >> 1) & 1u);
        } else {
            cluster_barrier();  // u^{n+1} complete in every strip and ghost row; u^n no longer read
        }
    };
    for (int s = 0; s < A.nsteps; s += 2) {  // parity unrolled: the level pointers are fixed per call
        step(S0, S1, s);
        if (s + 1 < A.nsteps) step(S1, S0, s + 1);
    }

    if constexpr (AS) cluster_barrier();  // no CTA leaves while a neighbour may still address its memory
    if (A.nsteps > 0 && sp.nrl > 0) {  // the last (partial) chunk of trace rows
        const int s_last = (A.nsteps - 1) / kR2WavRows * kR2WavRows;
        flush_traces(n0 + s_last, A.nsteps - s_last);
    }
    // ---- write both levels of the strip back (ghost rows belong to the neighbours) ----
    for (int i = tid; i < nzl * A.nx; i += kR2Threads) {
        const int zl = i / A.nx, x = i - zl * A.nx;
        const int64_t go = (int64_t)(zlo + zl + R) * A.pitch + x;
        A.u0[go] = S0[(zl + R) * Ps + C0 + x];
        A.u1[go] = S1[(zl + R) * Ps + C0 + x];
    }
}

int max_smem_optin() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
}

// The plan: the largest cluster (8, 4, 2, 1 CTAs) whose strips are at least max(R, 2) rows (a boundary
// row then has one neighbour per side) and hold <= 32 column pairs per thread (inj_mask bits), and
// whose per-CTA shared memory fits; false when none does.
bool r2_choose(const Geom& g, const Sparse& sp, bool damp, R2Plan* out) {
    if (g.ndim != 2 || g.R < 1 || g.R > AW_MAXR || g.ny != 1 || g.nx < 1 || g.nz < 1) return false;
    const int64_t smax = max_smem_optin();
    for (int CS = kR2MaxCluster; CS >= 1; CS /= 2) {
        if (CS > 1 && g.nz / CS < std::max(g.R, 2)) continue;
        const int nzl_max = (g.nz + CS - 1) / CS;
        if ((int64_t)nzl_max * ((g.nx + 1) / 2) > 32 * kR2Threads) continue;
        const R2Plan P = r2_plan(g, sp, damp, CS);
        if ((int64_t)P.words * 4 > smax) continue;
        *out = P;
        return true;
    }
    return false;
}

template <int R, bool DAMP>
cudaError_t r2_launch_k(const R2Args& A, size_t smem, cudaStream_t s) {
    // AW_R2_SYNC=cluster (development builds): the cluster-barrier variant, for A/B runs
    static const bool sync_cluster = dev_knob("AW_R2_SYNC") != nullptr;
    auto k = sync_cluster ? resident2d_kernel<R, DAMP, false> : resident2d_kernel<R, DAMP, true>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(A.P.CS, 1, 1);
    cfg.blockDim = dim3(kR2Threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = A.P.CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, A);
}

template <int R>
cudaError_t r2_launch(const Geom& g, const Coefs& c, float* u0, float* u1, const float* b, const float* a,
                      const Sparse& sp, const int64_t* d_base, int step0, int nsteps, cudaStream_t s) {
    R2Args A;
    if (!r2_choose(g, sp, a != nullptr, &A.P)) return cudaErrorNotSupported;
    A.c = c;
    A.u0 = u0;
    A.u1 = u1;
    A.b = b;
    A.a = a;
    A.pitch = g.pitch;
    A.nx = g.nx;
    A.nz = g.nz;
    A.PR = (g.nx + 1) / 2;
    A.sp = sp;
    A.d_base = d_base;
    A.step0 = step0;
    A.nsteps = nsteps;
    const size_t smem = (size_t)A.P.words * 4;
    return a ? r2_launch_k<R, true>(A, smem, s) : r2_launch_k<R, false>(A, smem, s);
}

}  // namespace

bool resident2d_fits(const Geom& g, const Sparse& sp, bool damp) {
    R2Plan P;
    return r2_choose(g, sp, damp, &P);
}

cudaError_t launch_stencil_resident2d(const Geom& g, const Coefs& c, float* u_cur, float* u_prev, const float* b,
                                      const float* a, const Sparse& sp, const int64_t* d_base, int step0, int nsteps,
                                      cudaStream_t s) {
    if (nsteps <= 0) return cudaSuccess;
    switch (g.R) {
#define AW_CASE(RR) \
    case RR: return r2_launch<RR>(g, c, u_cur, u_prev, b, a, sp, d_base, step0, nsteps, s);
        AW_CASE(1) AW_CASE(2) AW_CASE(3) AW_CASE(4) AW_CASE(5) AW_CASE(6) AW_CASE(7) AW_CASE(8)
#undef AW_CASE
        default: return cudaErrorNotSupported;
    }
}

}  // namespace aw
