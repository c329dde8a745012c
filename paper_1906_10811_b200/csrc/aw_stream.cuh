// aw_stream.cuh -- 2.5D z-streaming stencil kernel for 3D grids (sm_100a).
// (Included by aw_stream_r{1..8}.cu, one translation unit per half-width R so the
// instantiations compile in parallel; aw_stream.cu holds the R-independent host side.)
//
// The hot loop of the path (SURVEY.md §8(a) rows a5+a6): star Laplacian of
// order k = 2R fused with the damped leapfrog update.  It is HBM-bound at
// 16 algorithmic B per point update, so the design goal is to
// stream u^n, u^{n-1}, b (and a where eta != 0) exactly once from HBM and
// write u^{n+1} once, with few enough instructions per point that the SMs
// keep up with HBM.  B200-first choices (not the paper's OPS-generated code):
//
//  * persistent grid of (#SMs x resident CTAs) CTAs; work items are
//    (xy tile, z chunk) pairs handed out cyclically, so at any time the
//    resident CTAs work on neighbouring tiles at the same z and the halo rows
//    one CTA loads are L2 hits for its neighbours;
//  * one producer warp issues TMA (cp.async.bulk.tensor.3d) loads of the u^n
//    plane tile with its halo into a ring of SU = R+1+D shared-memory stages
//    (full/empty mbarriers), plus TMA L2 prefetches PD planes ahead for every
//    stream the consumers read (u^n tiles, and the u^{n-1}, b, a tiles of
//    the output planes).  TMA's out-of-bounds zero fill is the zero-ghost
//    boundary in x and y; z ghosts are zeroed halo planes;
//  * consumer warps: lane l owns the x columns x0+l and x0+l+32 of RY rows,
//    so every operation is done on point pairs with the Blackwell packed-fp32
//    instructions (FFMA2/FADD2/FMUL2, per-lane IEEE RN == the scalar ops);
//  * z neighbours come from a register queue of 2R+1 centre values; the
//    plane loop is unrolled by 2R+1 so the queue rotates by renaming, not by
//    moves; x and y neighbours come from the resident stage of the output
//    plane (the y column is loaded once per thread and shared by its rows);
//  * interior tiles run a predicate-free path; edge tiles mask their loads
//    and stores;
//  * in a team, boundary planes are also stored into the neighbours' halo
//    planes (peer memory over NVLink): the fused exchange.
//
// Per point the arithmetic is the canonical sequence of SURVEY §8(c).6:
//   L = C0*u; x pairs j=1..R; y pairs; z pairs (fma each); t = 2u - u^{n-1};
//   w = fma(b, L, t); u^{n+1} = fma(a, w, (1-a) u^{n-1})
// so the result is value-identical to the fp32 oracle and the v1 kernel.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <unordered_map>
#include <utility>
#include <vector>

#include "aw_internal.h"

namespace aw {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Wait for the phase with the given parity.  The suspend-time hint lets the warp sleep in the
// barrier until the phase completes (up to the hint, in ns) instead of re-polling: without it the
// retry loop was ~30 % of the kernel's issued instructions (SYNCS + BRA + YIELD, ncu source page).
#ifndef AW_MBAR_SUSPEND_NS
#define AW_MBAR_SUSPEND_NS 20000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity), "n"(AW_MBAR_SUSPEND_NS)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// TMA load with an L2 cache-eviction policy (createpolicy): temporal blocking keeps the data the
// second step re-reads (evict_last) and lets the single-use streams go first (evict_first)
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 int c2, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_hint(float* p, float v, uint64_t policy) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(policy) : "memory");
}

__device__ __forceinline__ void tma_prefetch_l2_3d(const CUtensorMap* map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(c0), "r"(c1),
                 "r"(c2)
                 : "memory");
}
__device__ __forceinline__ float ldg_stream(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// packed fp32 (Blackwell FFMA2/FADD2/FMUL2): per component identical to the scalar _rn ops
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

template <int R_, int TY_, int RY_, int D_, int DP_, int PD_, int MINB_, bool ADJ_ = true, int CREG_ = 0,
          int PREG_ = 40, int QJ_ = -1>
struct Cfg {
    static constexpr int R = R_, TX = 64, TY = TY_, RY = RY_, D = D_, DP = DP_, PD = PD_, MINB = MINB_;
    // z queue: registers hold the planes z-R .. z+QJ around the output plane z (QJ_ = -1: QJ = R, the full
    // 2R+1 queue); the upper neighbours z+QJ+1 .. z+R are read from the u^n ring, which holds them anyway
    // (R-QJ more 64-bit shared loads per row, R-QJ fewer float2 registers per row, shorter unroll).
    // QJ = 0 is the half register queue (HQ): the R planes below, the output plane pushed after its update.
    static constexpr int QJ = QJ_ < 0 ? R : QJ_;
    static constexpr bool HQ = QJ == 0;
    // lane -> columns: ADJ = the adjacent pair (2l, 2l+1), read and written with 64-bit shared/global
    // accesses; otherwise (l, l+32) with 32-bit accesses (the round-1 mapping, kept for A/B runs)
    static constexpr bool ADJ = ADJ_;
    // CREG > 0: warpgroup layout -- the consumer warps form whole warpgroups and the three service
    // warps (+1 idle) a fourth one; at entry the service warpgroup gives its registers back
    // (setmaxnreg.dec to PREG) and the consumers grow to CREG (setmaxnreg.inc).  The register file
    // then holds more consumer warps than a uniform allocation would (the service warps need few).
    static constexpr int CREG = CREG_, PREG = PREG_;
    static constexpr bool WG = CREG_ > 0;
    static constexpr int CA = ADJ ? 2 : 1;   // first column = CA * lane
    static constexpr int CB = ADJ ? 1 : 32;  // second column = first + CB
    static constexpr int Q = HQ ? R : R + QJ + 1;  // z queue length (and plane-loop unroll)
    // x halo rounded up to a multiple of 4 floats: the TMA box row (TX+2RP)*4 B must be a
    // multiple of 32 B on this part (272/304-B rows trap with an illegal instruction).
    static constexpr int RP = (R + 3) / 4 * 4;
    static constexpr int TXP = TX + 2 * RP;
    static constexpr int TYP = TY + 2 * R;
    static constexpr int SU = R + 1 + D;  // u^n ring: planes [p-R, p+D]
    static constexpr int SP = DP + 1;     // (u^{n-1}, b, a) ring of the output planes
    static constexpr int NWARPS_COMP = TY / RY;
    static constexpr int NCOMP = 32 * NWARPS_COMP;
    // + u^n producer, streams producer, receivers warp (+ an idle warp completing the warpgroup)
    static constexpr int NTHREADS = NCOMP + (WG ? 128 : 96);
    static_assert(!WG || (NWARPS_COMP % 4 == 0 && NCOMP * CREG + 128 * PREG <= 65536 && CREG % 8 == 0 &&
                          PREG % 8 == 0 && PREG >= 24 && CREG <= 256),
                  "warpgroup register split");
    static constexpr int STAGE_FLOATS = TXP * TYP;
    static constexpr int STAGE_BYTES = STAGE_FLOATS * 4;                 // TMA transaction bytes
    static constexpr int STAGE_STRIDE = (STAGE_BYTES + 127) / 128 * 128;  // 128-B aligned ring slots
    static constexpr int STAGE_STRIDE_F = STAGE_STRIDE / 4;
    static constexpr int PTILE_FLOATS = TX * TY;
    static constexpr int PTILE_BYTES = PTILE_FLOATS * 4;
    static constexpr int PSTAGE_FLOATS = 3 * PTILE_FLOATS;  // u^{n-1}, b, a
    static constexpr size_t U_BYTES = (size_t)SU * STAGE_STRIDE;
    static constexpr size_t P_BYTES = (size_t)SP * PSTAGE_FLOATS * 4;
    // + full/empty barriers of both rings + 3 metadata words per streams stage
    // + full/empty barriers of both rings, then (16-B aligned) 4 metadata words per streams stage
    static constexpr size_t META_OFF = (U_BYTES + P_BYTES + (2 * SU + 2 * SP) * sizeof(uint64_t) + 15) / 16 * 16;
    static constexpr size_t SMEM = META_OFF + 4 * SP * sizeof(int);
    static_assert(TY % RY == 0, "tile shape");
    static_assert(TXP <= 256 && TYP <= 256, "TMA box dims <= 256");
};

}  // namespace

struct StreamArgs {
    Geom g;
    Coefs c;
    float* unext;            // buffer base (plane -R)
    const float* a;          // may be null (no damping)
    const uint8_t* flags;    // [ntiles][nz]: 1 if any a != 1 in the tile-plane
    float* lo;               // team halo targets (null if none)
    int64_t lo_off;
    float* hi;
    int64_t hi_off;
    int ntx, nty;            // tiles along x, y
    int nzc, zc;             // z chunks and planes per chunk
    int nitems;              // ntiles * nzc
    // fused per-step sparse work (SURVEY §8(a) a7 injection, a8 receivers)
    const int2* tpsc;        // [ntiles][nz]: {first entry, count} of injection corners in the tile-plane
    const int4* tpe;         // entries: {tile-local point ly*64+lx, csr begin, csr end, 0}
    const int* inj_src;      // [nent] source index (CSR: corner ascending, then source)
    const float* inj_s;      // [nent] fp32 scale dt^2 w / (m + eta dt/2)
    const float* wavelet;    // [nt_max][ns]
    int ns;
    int nrl, nr, nc;         // owned receivers, trace row length, corners per point
    const int* rec_id;
    const int64_t* rec_off;  // element offsets into the u^n buffer (-1: skipped corner)
    const float* rec_w;
    float* traces;           // [nt_max][nr]
    const float* ucur;       // u^n buffer base (plane -R)
    const int64_t* d_base;   // the step index is n = *d_base + step_i (graph-replay friendly)
    int step_i;
    // device-clock timing on the production path (AW_OPT_TIMING = 2, CUDA graphs kept): the first
    // CTA start and the last CTA end of launch n go to ts0[n % ts_cap] (atomicMin) and
    // ts1[n % ts_cap] (atomicMax), %globaltimer ns; null when off
    unsigned long long* ts0;
    unsigned long long* ts1;
    int ts_cap;
    // per work item: 1 if it holds injection corners (the split high-order kernel, aw_hstream.cuh,
    // runs those items on its generic path)
    const uint8_t* item_inj;
    // team (boundary first): chunk slots [0, tc_lo) are the chunks holding planes z < R, slots
    // [tc_lo, tc_nb) the chunks from tc_hi up (planes z >= nz-R), then the interior chunks; the CTA
    // completing the last of the tc_nb * ntiles boundary items raises the neighbours' flags
    int tc_lo, tc_hi, tc_nb;
    DevCtl* ctl;
    unsigned long long* flag_lo;
    unsigned long long* flag_hi;
};

// chunk of chunk slot `slot` (team order: boundary chunks first; identity otherwise)
template <bool TEAM>
__device__ __forceinline__ int chunk_of(const StreamArgs& A, int slot) {
    if constexpr (!TEAM) return slot;
    if (slot < A.tc_lo) return slot;
    if (slot < A.tc_nb) return A.tc_hi + (slot - A.tc_lo);
    return A.tc_lo + (slot - A.tc_nb);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct StreamMaps {
    CUtensorMap u;    // u^n buffer, box (TXP, TYP, 1): ring loads + L2 prefetch
    CUtensorMap un;   // u^{n-1}/u^{n+1} buffer, box (TX, TY, 1)
    CUtensorMap b;    // model layout, box (TX, TY, 1)
    CUtensorMap a;    // model layout, box (TX, TY, 1) (b again when there is no damping)
};

namespace {

struct Ring {
    uint32_t slot, phase;
    __device__ __forceinline__ void advance(uint32_t n) {
        if (++slot == n) {
            slot = 0;
            phase ^= 1;
        }
    }
};

}  // namespace

// WG layout: the service warpgroup shrinks to PREG registers per thread, the consumer warpgroups
// grow to CREG (setmaxnreg; every warp of a warpgroup executes the same instruction).  Called at
// the top of each role's branch, so ptxas allocates that branch's code under the new limit.
template <class C>
__device__ __forceinline__ void service_regs() {
    if constexpr (C::WG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::PREG));
}
template <class C>
__device__ __forceinline__ void consumer_regs() {
    if constexpr (C::WG) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::CREG));
}

// One work item (xy tile, z chunk) for a consumer thread.  INTERIOR tiles need
// no bounds predicates.  The ring positions advance exactly like the producer's.
template <class C, bool INTERIOR, bool TEAM, bool HINT = false>
__device__ __forceinline__ void consume_item(const StreamArgs& A, const float* ring, const float* pring,
                                             uint64_t* fullU, uint64_t* emptyU, uint64_t* fullP, uint64_t* emptyP,
                                             const volatile int* pmeta,
                                             int tile, int zb, int ze, int x0, int y0, int lane, int ly, Ring& ru,
                                             Ring& rp, int64_t step_n, float* out_base, uint64_t st_policy = 0) {
    constexpr int R = C::R, RY = C::RY, RP = C::RP, TXP = C::TXP, TX = C::TX, SU = C::SU, SP = C::SP, Q = C::Q;
    const Geom& g = A.g;
    const int nz = g.nz;
    const int ntiles = A.ntx * A.nty;
    const int niter = ze - zb + 2 * R;
    const int64_t pitch = g.pitch, plane = g.plane;
    const float2 C0 = f2(A.c.C0, A.c.C0);
    const float2 two = f2(2.0f, 2.0f), one = f2(1.0f, 1.0f);
    constexpr int CA = C::CA, CB = C::CB;
    // both columns of this lane as one float2 (64-bit load when ADJ)
    auto ld2 = [](const float* p) -> float2 {
        if constexpr (C::ADJ) return *reinterpret_cast<const float2*>(p);
        else return f2(p[0], p[CB]);
    };
    const int xa = x0 + CA * lane, xb = xa + CB;
    const bool inA = INTERIOR || xa < g.nx, inB = INTERIOR || xb < g.nx;
    bool ok_a[RY], ok_b[RY];
#pragma unroll
    for (int i = 0; i < RY; ++i) {
        const bool r = INTERIOR || (y0 + ly + i) < g.ny;
        ok_a[i] = inA && r;
        ok_b[i] = inB && r;
    }
    // u^{n+1} of (z, y0+ly, xa): advanced by `plane` per output plane
    // (out_base: A.unext, or the TB kernel's v / w buffer)
    float* outp = out_base + (int64_t)(zb + R) * plane + (int64_t)(y0 + ly) * pitch + xa;  // (xb = xa + CB)

    float2 q[RY][Q];
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
        for (int j = 0; j < Q; ++j) q[i][j] = f2(0.0f, 0.0f);

    for (int kb = 0; kb < niter; kb += Q) {
#pragma unroll
        for (int uq = 0; uq < Q; ++uq) {
            const int k = kb + uq;
            if (k >= niter) break;
            mbar_wait(&fullU[ru.slot], ru.phase);
            const float* P = ring + ru.slot * C::STAGE_STRIDE_F + (ly + R) * TXP + RP + CA * lane;
            if constexpr (C::QJ == R) {
                // newest plane -> queue slot uq (rotation by renaming: plane p-m sits in slot (uq-m) mod Q)
#pragma unroll
                for (int i = 0; i < RY; ++i) q[i][uq] = ld2(P + i * TXP);
            }
            const uint32_t slotR = ru.slot >= (uint32_t)R ? ru.slot - R : ru.slot + SU - R;  // plane p-R
            if constexpr (!C::HQ && C::QJ < R) {
                // partial queue: plane p-R+QJ (= z+QJ of the output plane z = p-R) -> slot uq, from the
                // iteration where it is the first one the queue needs (zb-R at k = R-QJ)
                if (k >= R - C::QJ) {
                    const uint32_t sq = slotR + C::QJ < (uint32_t)SU ? slotR + C::QJ : slotR + C::QJ - SU;
                    const float* Pq = ring + sq * C::STAGE_STRIDE_F + (ly + R) * TXP + RP + CA * lane;
#pragma unroll
                    for (int i = 0; i < RY; ++i) q[i][uq] = ld2(Pq + i * TXP);
                }
            }
            if constexpr (C::HQ) {
                // warm-up: planes zb-R .. zb-1 (p-R for R <= k < 2R) are the first outputs' lower z neighbours
                if (k >= R && k < 2 * R) {
                    const float* Pc = ring + slotR * C::STAGE_STRIDE_F + (ly + R) * TXP + RP + CA * lane;
#pragma unroll
                    for (int i = 0; i < RY; ++i) q[i][uq] = ld2(Pc + i * TXP);
                }
            }
            if (k >= 2 * R) {
                const int z = zb + k - 2 * R;  // output plane
                const float* Qs = ring + slotR * C::STAGE_STRIDE_F + ly * TXP + RP + CA * lane;
                // (u^{n-1}, b, a) tiles of the output plane
                mbar_wait(&fullP[rp.slot], rp.phase);
                const float* Pp = pring + rp.slot * C::PSTAGE_FLOATS + ly * TX + CA * lane;
                // stage metadata written by the streams producer before its arrive: use_a, injection list
                const bool use_a = pmeta[4 * rp.slot] != 0;
                const int inj_first = pmeta[4 * rp.slot + 1], inj_count = pmeta[4 * rp.slot + 2];
                // y column of the output plane (rows ly .. ly+RY-1+2R) at both x columns
                float2 col[RY + 2 * R];
#pragma unroll
                for (int r = 0; r < RY + 2 * R; ++r) col[r] = ld2(Qs + r * TXP);
                float2 res[RY];
#pragma unroll
                for (int i = 0; i < RY; ++i) {
                    const float* row = Qs + (i + R) * TXP;
                    const float2 uc = C::HQ ? col[i + R] : q[i][(uq + Q - C::QJ) % Q];
                    float2 L = mul2(C0, uc);
                    if constexpr (C::ADJ) {
                        // v[K + k] = columns (2l + 2k, 2l + 2k + 1), k = -K..K: x neighbours of both points
                        constexpr int K = (R + 1) / 2;
                        float2 v[2 * K + 1];
#pragma unroll
                        for (int k = -K; k <= K; ++k) v[K + k] = *reinterpret_cast<const float2*>(row + 2 * k);
#pragma unroll
                        for (int j = 1; j <= R; ++j) {
                            const int m = j >> 1;
                            // pair sums u[x-j] + u[x+j] of column 2l (.x) and 2l+1 (.y)
                            if (j & 1) {  // odd j: the two columns' pairs sit in different float2s -- two packed adds,
                                // each keeps one useful half, then scalar fmas (no register moves to re-pair halves)
                                const float2 sa = add2(v[K - m - 1], v[K + m]);      // .y = u[2l-j] + u[2l+j]
                                const float2 sb = add2(v[K - m], v[K + m + 1]);      // .x = u[2l+1-j] + u[2l+1+j]
                                L.x = __fmaf_rn(A.c.C[2][j], sa.y, L.x);
                                L.y = __fmaf_rn(A.c.C[2][j], sb.x, L.y);
                            } else {
                                L = fma2(make_float2(A.c.C[2][j], A.c.C[2][j]), add2(v[K - m], v[K + m]), L);
                            }
                        }
                    } else {
#pragma unroll
                        for (int j = 1; j <= R; ++j)
                            L = fma2(f2(A.c.C[2][j], A.c.C[2][j]),
                                     add2(f2(row[-j], row[32 - j]), f2(row[j], row[32 + j])), L);
                    }
#pragma unroll
                    for (int j = 1; j <= R; ++j)
                        L = fma2(f2(A.c.C[1][j], A.c.C[1][j]), add2(col[i + R - j], col[i + R + j]), L);
                    if constexpr (C::HQ) {
                        // z - j: register slot (uq - j) mod R; z + j: the ring stage of plane p - R + j
#pragma unroll
                        for (int j = 1; j <= R; ++j) {
                            const uint32_t sj = slotR + j < (uint32_t)SU ? slotR + j : slotR + j - SU;
                            const float2 up = ld2(ring + sj * C::STAGE_STRIDE_F + (ly + R + i) * TXP + RP + CA * lane);
                            L = fma2(f2(A.c.C[0][j], A.c.C[0][j]), add2(q[i][(uq + R - j) % R], up), L);
                        }
                    } else if constexpr (C::QJ < R) {
                        // plane z+m sits in slot (uq - QJ + m) mod Q for m in [-R, QJ]; above QJ: the ring
#pragma unroll
                        for (int j = 1; j <= R; ++j) {
                            float2 up;
                            if (j <= C::QJ) {
                                up = q[i][(uq + Q - C::QJ + j) % Q];
                            } else {
                                const uint32_t sj = slotR + j < (uint32_t)SU ? slotR + j : slotR + j - SU;
                                up = ld2(ring + sj * C::STAGE_STRIDE_F + (ly + R + i) * TXP + RP + CA * lane);
                            }
                            L = fma2(f2(A.c.C[0][j], A.c.C[0][j]), add2(q[i][(uq + 2 * Q - C::QJ - j) % Q], up), L);
                        }
                    } else {
#pragma unroll
                        for (int j = 1; j <= R; ++j)
                            L = fma2(f2(A.c.C[0][j], A.c.C[0][j]),
                                     add2(q[i][(uq + Q - R - j) % Q], q[i][(uq + Q - R + j) % Q]), L);
                    }
                    const float* pr = Pp + i * TX;
                    const float2 um = ld2(pr);
                    const float2 bb = ld2(pr + C::PTILE_FLOATS);
                    const float2 aa = use_a ? ld2(pr + 2 * C::PTILE_FLOATS) : one;
                    // t = 2u - u^{n-1} (2u exact: one rounding), w = fma(b, L, t)
                    const float2 t = fma2(two, uc, f2(-um.x, -um.y));
                    const float2 wv = fma2(bb, L, t);
                    const float2 rr = mul2(add2(one, f2(-aa.x, -aa.y)), um);
                    res[i] = fma2(aa, wv, rr);
                }
                if constexpr (C::HQ) {  // u^n of the output plane becomes a lower neighbour (slot uq: plane z-R done)
#pragma unroll
                    for (int i = 0; i < RY; ++i) q[i][uq] = col[i + R];
                }
                mbar_arrive(&emptyP[rp.slot]);  // every consumer thread arrives: no warp sync, no branch
                rp.advance(SP);
                // fused injection: u^{n+1}[c] = fma(s, q[n][src], u^{n+1}[c]) over the
                // corner's sources in CSR order, applied by the thread that owns the corner, before storing
                for (int e = inj_first; e < inj_first + inj_count; ++e) {
                    const int4 en = A.tpe[e];
                    const int yl = en.x >> 6, xl = en.x & 63;
                    const int owner = C::ADJ ? xl >> 1 : xl & 31;
                    const bool second = C::ADJ ? (xl & 1) : (xl >= 32);
#pragma unroll
                    for (int i = 0; i < RY; ++i) {
                        if (yl != ly + i || owner != lane) continue;
                        float v = second ? res[i].y : res[i].x;
                        const float* qn = A.wavelet + step_n * A.ns;
                        for (int k = en.y; k < en.z; ++k) v = __fmaf_rn(A.inj_s[k], qn[A.inj_src[k]], v);
                        if (second) res[i].y = v; else res[i].x = v;
                    }
                }
                if constexpr (HINT) {
#pragma unroll
                    for (int i = 0; i < RY; ++i) {
                        float* o = outp + i * pitch;
                        if (ok_a[i]) st_hint(o, res[i].x, st_policy);
                        if (ok_b[i]) st_hint(o + CB, res[i].y, st_policy);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < RY; ++i) {
                        float* o = outp + i * pitch;
                        if (C::ADJ && ok_a[i] && ok_b[i]) {
                            *reinterpret_cast<float2*>(o) = res[i];  // 8-B aligned: x0 % 64 == 0, pitch % 32 == 0
                        } else {
                            if (ok_a[i]) o[0] = res[i].x;
                            if (ok_b[i]) o[CB] = res[i].y;
                        }
                    }
                }
                if constexpr (TEAM) {
                    // fused exchange: boundary planes also go straight into the neighbours' halos.  A plane
                    // of a thin slab (R <= nz < 2R) can be both a low and a high boundary plane, so the
                    // two targets are tested separately.
                    const int64_t om = (outp - out_base) - (int64_t)R * plane;  // model-layout index
                    auto peer_store = [&](float* h) {
#pragma unroll
                        for (int i = 0; i < RY; ++i) {
                            float* o = h + i * pitch;
                            if (C::ADJ && ok_a[i] && ok_b[i]) {
                                *reinterpret_cast<float2*>(o) = res[i];  // same pitch and alignment as outp
                            } else {
                                if (ok_a[i]) o[0] = res[i].x;
                                if (ok_b[i]) o[CB] = res[i].y;
                            }
                        }
                    };
                    if (A.lo && z < R) peer_store(A.lo + A.lo_off + om);
                    if (A.hi && z >= nz - R) peer_store(A.hi + A.hi_off + om - (int64_t)(nz - R) * plane);
                }
                outp += plane;
            }
            // release the stage of plane p - R (no longer needed by any later output)
            if (k >= R) {
                mbar_arrive(&emptyU[slotR]);
            }
            ru.advance(SU);
        }
    }
    // release the last R stages of this item (planes ze .. ze+R-1)
#pragma unroll 1
    for (int m = 0; m < R; ++m) {
        const uint32_t s = ru.slot >= (uint32_t)(R - m) ? ru.slot - (R - m) : ru.slot + SU - (R - m);
        mbar_arrive(&emptyU[s]);
    }
}

template <class C, bool TEAM>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
    stream_kernel(const __grid_constant__ StreamMaps M, const __grid_constant__ StreamArgs A) {
    constexpr int R = C::R, TX = C::TX, TY = C::TY, RP = C::RP, SU = C::SU, SP = C::SP, PD = C::PD, DP = C::DP;
    extern __shared__ __align__(128) unsigned char smem[];
    float* ring = reinterpret_cast<float*>(smem);
    float* pring = reinterpret_cast<float*>(smem + C::U_BYTES);
    uint64_t* fullU = reinterpret_cast<uint64_t*>(smem + C::U_BYTES + C::P_BYTES);
    uint64_t* emptyU = fullU + SU;
    uint64_t* fullP = emptyU + SU;
    uint64_t* emptyP = fullP + SP;
    int* pmeta = reinterpret_cast<int*>(smem + C::META_OFF);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < SU; ++s) {
            mbar_init(&fullU[s], 1);
            mbar_init(&emptyU[s], C::NCOMP);  // one arrival per consumer thread
        }
        for (int s = 0; s < SP; ++s) {
            mbar_init(&fullP[s], 1);
            mbar_init(&emptyP[s], C::NCOMP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const Geom& g = A.g;
    const int nz = g.nz;
    const int ntiles = A.ntx * A.nty;

    const int64_t step_n = *A.d_base + A.step_i;
    const int ts_slot = A.ts0 ? (int)(step_n % A.ts_cap) : 0;
    if (A.ts0 && tid == 0) atomicMin(A.ts0 + ts_slot, globaltimer_ns());
    if (warp == C::NWARPS_COMP + 3) {
        service_regs<C>();  // idle warp of the service warpgroup (WG layout only)
    } else if (warp == C::NWARPS_COMP + 2) {
        service_regs<C>();
        // ---------------- receivers warp: rec[n][r] = fma chain of u^n corners --------
        for (int r = blockIdx.x + gridDim.x * lane; r < A.nrl; r += gridDim.x * 32) {
            float acc = 0.0f;
            for (int beta = 0; beta < A.nc; ++beta) {
                const int64_t off = A.rec_off[(int64_t)r * A.nc + beta];
                if (off < 0) continue;
                acc = __fmaf_rn(A.rec_w[(int64_t)r * A.nc + beta], A.ucur[off], acc);
            }
            A.traces[step_n * A.nr + A.rec_id[r]] = acc;
        }
    } else if (warp >= C::NWARPS_COMP) {
        service_regs<C>();
        // ---------------- producer warps ----------------
        // warp NWARPS_COMP: u^n plane tiles (with halo) into the ring, D planes ahead, and L2
        // prefetches PD planes ahead; warp NWARPS_COMP+1: the u^{n-1}, b, a tiles of the output
        // planes into the streams ring, DP planes ahead (+ their L2 prefetches).
        const bool is_u = warp == C::NWARPS_COMP;
        if (lane == 0) {
            if (is_u) {
                asm volatile("prefetch.tensormap [%0];" ::"l"(&M.u) : "memory");
            } else {
                asm volatile("prefetch.tensormap [%0];" ::"l"(&M.un) : "memory");
                asm volatile("prefetch.tensormap [%0];" ::"l"(&M.b) : "memory");
                if (A.a) asm volatile("prefetch.tensormap [%0];" ::"l"(&M.a) : "memory");
            }
            Ring rr{0, 0};
            for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
                const int tile = item % ntiles;
                const int zb = chunk_of<TEAM>(A, item / ntiles) * A.zc;
                const int ze = min(nz, zb + A.zc);
                const int x0 = (tile % A.ntx) * TX, y0 = (tile / A.ntx) * TY;
                const int niter = ze - zb + 2 * R;
                if (is_u) {
                    for (int kk = 0; kk < PD && kk < niter; ++kk) tma_prefetch_l2_3d(&M.u, x0 - RP, y0 - R, zb + kk);
                    for (int k = 0; k < niter; ++k) {
                        if (k + PD < niter) tma_prefetch_l2_3d(&M.u, x0 - RP, y0 - R, zb + k + PD);
                        mbar_wait(&emptyU[rr.slot], rr.phase ^ 1);
                        mbar_expect_tx(&fullU[rr.slot], C::STAGE_BYTES);
                        tma_load_3d(ring + rr.slot * C::STAGE_STRIDE_F, &M.u, &fullU[rr.slot], x0 - RP, y0 - R, zb + k);
                        rr.advance(SU);
                    }
                } else {
                    auto l2_prefetch = [&](int z) {
                        if (z >= ze) return;
                        tma_prefetch_l2_3d(&M.un, x0, y0, z + R);
                        tma_prefetch_l2_3d(&M.b, x0, y0, z);
                        if (A.a && A.flags[(int64_t)tile * nz + z]) tma_prefetch_l2_3d(&M.a, x0, y0, z);
                    };
                    for (int z = zb; z < zb + PD; ++z) l2_prefetch(z);
                    for (int z = zb; z < ze; ++z) {
                        l2_prefetch(z + PD);
                        const bool use_a = A.a && A.flags[(int64_t)tile * nz + z];  // [tile][z]: L1-friendly
                        const int2 tp = A.tpsc ? A.tpsc[(int64_t)tile * nz + z] : make_int2(0, 0);
                        float* dst = pring + rr.slot * C::PSTAGE_FLOATS;
                        mbar_wait(&emptyP[rr.slot], rr.phase ^ 1);
                        // ordered for the consumers by this arrive (release) and their wait (acquire);
                        // compute-sanitizer racecheck does not model mbarrier phases
                        pmeta[4 * rr.slot] = use_a;
                        pmeta[4 * rr.slot + 1] = tp.x;
                        pmeta[4 * rr.slot + 2] = tp.y;
                        mbar_expect_tx(&fullP[rr.slot], (use_a ? 3 : 2) * C::PTILE_BYTES);
                        tma_load_3d(dst, &M.un, &fullP[rr.slot], x0, y0, z + R);
                        tma_load_3d(dst + C::PTILE_FLOATS, &M.b, &fullP[rr.slot], x0, y0, z);
                        if (use_a) tma_load_3d(dst + 2 * C::PTILE_FLOATS, &M.a, &fullP[rr.slot], x0, y0, z);
                        rr.advance(SP);
                    }
                }
            }
        }
    } else {
        consumer_regs<C>();
        // ---------------- consumer warps ----------------
        const int ly = warp * C::RY;  // first tile row of this thread
        Ring ru{0, 0}, rp{0, 0};
        for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
            const int tile = item % ntiles;
            const int zb = chunk_of<TEAM>(A, item / ntiles) * A.zc;
            const int ze = min(nz, zb + A.zc);
            const int x0 = (tile % A.ntx) * TX, y0 = (tile / A.ntx) * TY;
            if (x0 + TX <= g.nx && y0 + TY <= g.ny)
                consume_item<C, true, TEAM>(A, ring, pring, fullU, emptyU, fullP, emptyP, pmeta, tile, zb, ze, x0, y0,
                                            lane, ly, ru, rp, step_n, A.unext);
            else
                consume_item<C, false, TEAM>(A, ring, pring, fullU, emptyU, fullP, emptyP, pmeta, tile, zb, ze, x0, y0,
                                             lane, ly, ru, rp, step_n, A.unext);
            if constexpr (TEAM) {
                if (item < A.tc_nb * ntiles && A.ctl) {
                    // a boundary item is done (its planes are in the neighbours' halos): count it; the last
                    // one of the launch raises the flags -- the neighbours' next step can start while this
                    // rank still computes its interior
                    asm volatile("bar.sync 1, %0;" ::"r"(C::NCOMP) : "memory");
                    if (tid == 0) {
                        __threadfence_system();  // cumulative: every consumer's peer stores (barrier above)
                        const unsigned nb = (unsigned)(A.tc_nb * ntiles);
                        if (atomicAdd(&A.ctl->bcount, 1u) + 1u == nb) {
                            __threadfence_system();
                            const unsigned long long v =
                                (A.ctl->epoch << 32) + (unsigned long long)(A.ctl->base + A.step_i + 2);
                            if (A.flag_lo) atomicMax_system(A.flag_lo, v);
                            if (A.flag_hi) atomicMax_system(A.flag_hi, v);
                            atomicExch(&A.ctl->bcount, 0u);  // every count of this launch is in
                        }
                    }
                }
            }
        }
    }
    if (A.ts0) {  // this CTA's end: every role done
        __syncthreads();
        if (tid == 0) atomicMax(A.ts1 + ts_slot, globaltimer_ns());
    }
}


// ---------------------------------------------------------------------------
// Small grids: the resident multi-step kernel.  One launch advances nsteps time
// steps.  Every CTA keeps its work items (item = blockIdx.x + j * gridDim.x) for all steps and runs
// them step-major with the stream_kernel roles (TMA producers, consumers, fused sparse work); there is
// no grid-wide barrier: an item starts local step i once the 27 items around it (xy tiles +-1, z
// chunks +-1 -- a superset of its halo region and of its receivers' corners) have completed step
// i-1 (per-item counters, release/acquire).  That also orders the in-place write of u^{i+1} over
// u^{i-1}: the neighbours that read those points as halo at step i-1 are done with it.  Launch
// gaps disappear and a region can run ahead of a slower one -- the bound for grids that fit in L2,
// where a step takes microseconds.  Deadlock-free: every CTA is resident and an item at step i
// waits only for items at step i-1, which every CTA processes first.
// Receivers are read per item (the item holding the receiver's base corner) by the receivers warp,
// after the item's wait; the item's completion is published only after those reads (a named
// barrier with the consumers), so u^i is neither stale nor already overwritten.
// ---------------------------------------------------------------------------
struct ResMaps {
    StreamMaps m[2];  // by the parity of the buffer holding u^n
};

struct ResArgs {
    StreamArgs s;               // geometry, coefficients, eta flags, injection lists, receivers
    float* buf[2];              // the two wavefield buffers (plane -R)
    int cur0;                   // buffer holding u^n at the launch's first step
    int nsteps;                 // steps in this launch
    int step0;                  // local index (within the run) of the first step
    unsigned long long* done;   // [nitems]: local steps completed (reset per run)
    const int* ritem_ptr;       // [nitems + 1]: receivers (indices into the owned list) by item
    const int* ritem_idx;
    int skip_wait;              // development measurement only (AW_RES_NOWAIT, dev builds): no cross-item waits
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_epoch(const unsigned long long* p, unsigned long long epoch) {
    while (ld_acquire_u64(p) < epoch) __nanosleep(64);
}
__device__ __forceinline__ void publish_done(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// lanes 0..26 each wait for one neighbour item (the item itself included) to reach `need`
__device__ __forceinline__ void wait_neighbours(const StreamArgs& A, const unsigned long long* done, int tile, int c,
                                                unsigned long long need, int lane) {
    if (need > 0 && lane < 27) {
        const int tx = tile % A.ntx + lane % 3 - 1, ty = tile / A.ntx + (lane / 3) % 3 - 1, cc = c + lane / 9 - 1;
        if (tx >= 0 && tx < A.ntx && ty >= 0 && ty < A.nty && cc >= 0 && cc < A.nzc) {
            const unsigned long long* p = done + (int64_t)cc * A.ntx * A.nty + (int64_t)ty * A.ntx + tx;
            while (ld_acquire_u64(p) < need) {
            }
        }
    }
    __syncwarp();
    // generic-proxy stores of other CTAs (and of this one) -> this CTA's async-proxy (TMA) reads
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <class C>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
    resident_kernel(const __grid_constant__ ResMaps RM, const __grid_constant__ ResArgs RA) {
    constexpr int R = C::R, TX = C::TX, TY = C::TY, RP = C::RP, SU = C::SU, SP = C::SP, PD = C::PD;
    extern __shared__ __align__(128) unsigned char smem[];
    float* ring = reinterpret_cast<float*>(smem);
    float* pring = reinterpret_cast<float*>(smem + C::U_BYTES);
    uint64_t* fullU = reinterpret_cast<uint64_t*>(smem + C::U_BYTES + C::P_BYTES);
    uint64_t* emptyU = fullU + SU;
    uint64_t* fullP = emptyU + SU;
    uint64_t* emptyP = fullP + SP;
    int* pmeta = reinterpret_cast<int*>(smem + C::META_OFF);
    const StreamArgs& A = RA.s;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < SU; ++s) {
            mbar_init(&fullU[s], 1);
            mbar_init(&emptyU[s], C::NCOMP);
        }
        for (int s = 0; s < SP; ++s) {
            mbar_init(&fullP[s], 1);
            mbar_init(&emptyP[s], C::NCOMP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const Geom& g = A.g;
    const int nz = g.nz;
    const int ntiles = A.ntx * A.nty;
    const int64_t base = *A.d_base;
    const int ts_slot = A.ts0 ? (int)((base + RA.step0) % A.ts_cap) : 0;
    if (A.ts0 && tid == 0) atomicMin(A.ts0 + ts_slot, globaltimer_ns());
    if (warp == C::NWARPS_COMP + 2) {
        // ---------------- receivers warp: per item, once its neighbours finished the
        // previous step, rec[n][r] = fma chain of the u^n corners of the item's receivers; the item's
        // consumers publish its completion only after this warp reached named barrier 2 ----------
        for (int t = 0; t < RA.nsteps; ++t) {
            const int i = RA.step0 + t;
            const float* ucur = RA.buf[RA.cur0 ^ (t & 1)];
            const int64_t step_n = base + i;
            for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
                const int e0 = RA.ritem_ptr[item], e1 = RA.ritem_ptr[item + 1];
                if (e1 > e0) {
                    wait_neighbours(A, RA.done, item % ntiles, item / ntiles, (unsigned long long)i, lane);
                    for (int e = e0 + lane; e < e1; e += 32) {
                        const int r = RA.ritem_idx[e];
                        float acc = 0.0f;
                        for (int beta = 0; beta < A.nc; ++beta) {
                            const int64_t off = A.rec_off[(int64_t)r * A.nc + beta];
                            if (off < 0) continue;
                            acc = __fmaf_rn(A.rec_w[(int64_t)r * A.nc + beta], __ldcg(ucur + off), acc);
                        }
                        A.traces[step_n * A.nr + A.rec_id[r]] = acc;
                    }
                    __syncwarp();
                }
                // the reads above happen before the item's completion is published; bar.sync (not arrive):
                // this warp must not run ahead of the consumers by a barrier generation
                __threadfence_block();
                asm volatile("bar.sync 2, %0;" ::"r"(C::NCOMP + 32) : "memory");
            }
        }
    } else if (warp == C::NWARPS_COMP) {
        // ---------------- u^n producer warp: per item, wait for the neighbours (all lanes), then lane 0
        // streams the u^n plane tiles into the ring ----------------
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&RM.m[0].u) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&RM.m[1].u) : "memory");
        }
        Ring rr{0, 0};
        for (int t = 0; t < RA.nsteps; ++t) {
            const int i = RA.step0 + t;
            const int par = RA.cur0 ^ (t & 1);
            const CUtensorMap* mu = &RM.m[par].u;
            for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
                const int tile = item % ntiles, c = item / ntiles;
                const int zb = c * A.zc;
                const int ze = min(nz, zb + A.zc);
                const int x0 = (tile % A.ntx) * TX, y0 = (tile / A.ntx) * TY;
                const int niter = ze - zb + 2 * R;
                if (!RA.skip_wait) wait_neighbours(A, RA.done, tile, c, (unsigned long long)i, lane);
                if (lane == 0) {
                    for (int kk = 0; kk < PD && kk < niter; ++kk) tma_prefetch_l2_3d(mu, x0 - RP, y0 - R, zb + kk);
                    for (int k = 0; k < niter; ++k) {
                        if (k + PD < niter) tma_prefetch_l2_3d(mu, x0 - RP, y0 - R, zb + k + PD);
                        mbar_wait(&emptyU[rr.slot], rr.phase ^ 1);
                        mbar_expect_tx(&fullU[rr.slot], C::STAGE_BYTES);
                        tma_load_3d(ring + rr.slot * C::STAGE_STRIDE_F, mu, &fullU[rr.slot], x0 - RP, y0 - R, zb + k);
                        rr.advance(SU);
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp == C::NWARPS_COMP + 1) {
        // ---------------- streams producer: u^{n-1}, b, a tiles of the output planes ----------------
        if (lane == 0) {
            Ring rr{0, 0};
            for (int t = 0; t < RA.nsteps; ++t) {
                const int i = RA.step0 + t;
                const int par = RA.cur0 ^ (t & 1);
                const StreamMaps& M = RM.m[par];
                for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
                    const int tile = item % ntiles;
                    const int zb = (item / ntiles) * A.zc;
                    const int ze = min(nz, zb + A.zc);
                    const int x0 = (tile % A.ntx) * TX, y0 = (tile / A.ntx) * TY;
                    // u^{n-1} of the item: written by its own step i-2 (this CTA's consumers)
                    if (i >= 2) wait_epoch(RA.done + item, (unsigned long long)(i - 1));
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    for (int z = zb; z < ze; ++z) {
                        const bool use_a = A.a && A.flags[(int64_t)tile * nz + z];
                        const int2 tp = A.tpsc ? A.tpsc[(int64_t)tile * nz + z] : make_int2(0, 0);
                        float* dst = pring + rr.slot * C::PSTAGE_FLOATS;
                        mbar_wait(&emptyP[rr.slot], rr.phase ^ 1);
                        pmeta[4 * rr.slot] = use_a;
                        pmeta[4 * rr.slot + 1] = tp.x;
                        pmeta[4 * rr.slot + 2] = tp.y;
                        mbar_expect_tx(&fullP[rr.slot], (use_a ? 3 : 2) * C::PTILE_BYTES);
                        tma_load_3d(dst, &M.un, &fullP[rr.slot], x0, y0, z + R);
                        tma_load_3d(dst + C::PTILE_FLOATS, &M.b, &fullP[rr.slot], x0, y0, z);
                        if (use_a) tma_load_3d(dst + 2 * C::PTILE_FLOATS, &M.a, &fullP[rr.slot], x0, y0, z);
                        rr.advance(SP);
                    }
                }
            }
        }
    } else {
        // ---------------- consumer warps ----------------
        const int ly = warp * C::RY;
        Ring ru{0, 0}, rp{0, 0};
        for (int t = 0; t < RA.nsteps; ++t) {
            const int i = RA.step0 + t;
            float* out = RA.buf[RA.cur0 ^ (t & 1) ^ 1];
            const int64_t step_n = base + i;
            for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
                const int tile = item % ntiles;
                const int zb = (item / ntiles) * A.zc;
                const int ze = min(nz, zb + A.zc);
                const int x0 = (tile % A.ntx) * TX, y0 = (tile / A.ntx) * TY;
                if (x0 + TX <= g.nx && y0 + TY <= g.ny)
                    consume_item<C, true, false>(A, ring, pring, fullU, emptyU, fullP, emptyP, pmeta, tile, zb, ze, x0,
                                                 y0, lane, ly, ru, rp, step_n, out);
                else
                    consume_item<C, false, false>(A, ring, pring, fullU, emptyU, fullP, emptyP, pmeta, tile, zb, ze, x0,
                                                  y0, lane, ly, ru, rp, step_n, out);
                // publish "item completed step i": every consumer's stores and the receivers warp's reads
                // of u^n (barrier 2), then one release
                asm volatile("fence.proxy.async.global;" ::: "memory");
                asm volatile("bar.sync 2, %0;" ::"r"(C::NCOMP + 32) : "memory");
                if (tid == 0) {
                    __threadfence();
                    publish_done(RA.done + item, (unsigned long long)(i + 1));
                }
            }
        }
    }
    if (A.ts0) {  // this CTA's end: every role done
        __syncthreads();
        if (tid == 0) atomicMax(A.ts1 + ts_slot, globaltimer_ns());
    }
}

// ---------------------------------------------------------------------------
// NEXT-1: temporal blocking, two time steps per pass.
//
// A pass reads X = u^n (with halo), Y = u^{n-1}, b, a and writes V = u^{n+1} (a third
// buffer) and W = u^{n+2} (over Y).  Work items are (tile, z-chunk) pairs of two kinds,
// handed out in phase order A(0), B(0), A(1), B(1), ...:
//   A(tile, c): step n   on planes [cZ+R, (c+1)Z+R) (A(0) from plane 0, the last to nz):
//               the ordinary consumer with inputs (X, Y, b, a), output -> V, injection q[n];
//   B(tile, c): step n+1 on planes [cZ, (c+1)Z): the same consumer with inputs
//               (V with halo, X centre, b, a), output -> W (into Y), injection q[n+1].
// B(tile, c) needs V on planes [cZ-R, (c+1)Z+R) of its tile and its four star neighbours,
// i.e. the items A(., c-1) and A(., c), which come earlier in the hand-out order: the
// u-producer waits on their completion epochs (acquire) before its TMA loads, so the pass
// is deadlock-free for any grid shape (every CTA is resident and takes items in order).
// The A phase of a chunk is ~Z planes of all tiles behind its B phase, so with Z planes of
// every field fitting in L2 the second step reads V, X, b, a from L2: the HBM traffic of a
// pass is X, Y, b, a once plus the V and W writes (~10.7 B per point update instead of 16).
// Y is overwritten by B(tile, c) only after A(tile, c) -- the only reader of those planes
// of Y -- finished (B waits for it).  Per point the arithmetic is the canonical sequence,
// so two steps of this kernel equal two steps of stream_kernel bit for bit.
// ---------------------------------------------------------------------------
struct TbMaps {
    CUtensorMap xh;  // X with halo box (TXP, TYP): A items' u^n ring
    CUtensorMap vh;  // V with halo box: B items' u^n ring
    CUtensorMap y;   // Y centre box (TX, TY): A items' u^{n-1}
    CUtensorMap xc;  // X centre box: B items' u^{n-1}
    CUtensorMap b;
    CUtensorMap a;
};

struct TbArgs {
    StreamArgs s;                  // geometry, coefficients, eta flags, injection lists, receivers (ucur = X)
    float* v;                      // V base (plane -R)
    float* w;                      // Y base: B items' output u^{n+2}
    unsigned long long* done;      // [nzc][ntiles]: epoch at which A(tile, c) completed
    unsigned long long epoch;      // this pass's epoch (monotone per plan)
    int Z, nzc, lead;              // chunk planes, chunks, A phases handed out ahead of B(0)
};

// Phase order with lead L >= 1: A(0) .. A(L-1), then B(0), A(L), B(1), A(L+1), ... (2 nzc + L phases;
// the A phases past the last chunk are empty: c = nzc marks a no-op item).
__device__ __forceinline__ void tb_decode(int item, int ntiles, int nzc, int Z, int R, int nz, int lead, int& tile,
                                          int& c, bool& isB, int& zb, int& ze) {
    const int phase = item / ntiles;
    tile = item - phase * ntiles;
    if (phase < lead) {
        c = phase;
        isB = false;
    } else {
        const int r = phase - lead;
        isB = !(r & 1);
        c = isB ? r >> 1 : lead + (r >> 1);
    }
    if (c >= nzc) {
        zb = ze = 0;
        c = nzc;
        return;
    }
    if (isB) {
        zb = c * Z;
        ze = min(nz, zb + Z);
    } else {
        zb = c == 0 ? 0 : c * Z + R;
        ze = c == nzc - 1 ? nz : min(nz, (c + 1) * Z + R);
    }
}


template <class C>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
    tb_kernel(const __grid_constant__ TbMaps M, const __grid_constant__ TbArgs T) {
    constexpr int R = C::R, TX = C::TX, TY = C::TY, RP = C::RP, SU = C::SU, SP = C::SP;
    extern __shared__ __align__(128) unsigned char smem[];
    float* ring = reinterpret_cast<float*>(smem);
    float* pring = reinterpret_cast<float*>(smem + C::U_BYTES);
    uint64_t* fullU = reinterpret_cast<uint64_t*>(smem + C::U_BYTES + C::P_BYTES);
    uint64_t* emptyU = fullU + SU;
    uint64_t* fullP = emptyU + SU;
    uint64_t* emptyP = fullP + SP;
    int* pmeta = reinterpret_cast<int*>(smem + C::META_OFF);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < SU; ++s) {
            mbar_init(&fullU[s], 1);
            mbar_init(&emptyU[s], C::NCOMP);  // one arrival per consumer thread
        }
        for (int s = 0; s < SP; ++s) {
            mbar_init(&fullP[s], 1);
            mbar_init(&emptyP[s], C::NCOMP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const StreamArgs& A = T.s;
    const Geom& g = A.g;
    const int nz = g.nz;
    const int ntiles = A.ntx * A.nty;
    const int nitems = (2 * T.nzc + T.lead) * ntiles;
    const int64_t step_n = *A.d_base + A.step_i;  // the pass advances steps n and n+1

    if (warp == C::NWARPS_COMP + 3) {  // idle warp of the service warpgroup (WG layout)
        service_regs<C>();
        return;
    }
    if (warp == C::NWARPS_COMP + 2) {
        service_regs<C>();
        // ---- receivers: rec[n] from X (read-only in this pass), rec[n+1] from V once the A items
        // owning its corners completed (they never wait, so this cannot deadlock) ----
        for (int r = blockIdx.x + gridDim.x * lane; r < A.nrl; r += gridDim.x * 32) {
            float acc = 0.0f;
            for (int beta = 0; beta < A.nc; ++beta) {
                const int64_t off = A.rec_off[(int64_t)r * A.nc + beta];
                if (off < 0) continue;
                acc = __fmaf_rn(A.rec_w[(int64_t)r * A.nc + beta], A.ucur[off], acc);
            }
            A.traces[step_n * A.nr + A.rec_id[r]] = acc;
            acc = 0.0f;
            for (int beta = 0; beta < A.nc; ++beta) {
                const int64_t off = A.rec_off[(int64_t)r * A.nc + beta];
                if (off < 0) continue;
                const int z = (int)(off / g.plane) - R;
                const int rem = (int)(off - (int64_t)(z + R) * g.plane);
                const int y = rem / (int)g.pitch, x = rem - y * (int)g.pitch;
                const int tile = (y / TY) * A.ntx + x / TX;
                const int c = z < T.Z + R ? 0 : min(T.nzc - 1, (z - R) / T.Z);
                wait_epoch(T.done + (int64_t)c * ntiles + tile, T.epoch);
                acc = __fmaf_rn(A.rec_w[(int64_t)r * A.nc + beta], __ldcg(T.v + off), acc);
            }
            A.traces[(step_n + 1) * A.nr + A.rec_id[r]] = acc;
        }
        return;
    }
    if (warp >= C::NWARPS_COMP) {
        service_regs<C>();
        // ---- producers: as in stream_kernel, with the map pair chosen by the item kind ----
        const bool is_u = warp == C::NWARPS_COMP;
        if (lane == 0) {
            const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
            Ring rr{0, 0};
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                int tile, c, zb, ze;
                bool isB;
                tb_decode(item, ntiles, T.nzc, T.Z, R, nz, T.lead, tile, c, isB, zb, ze);
                if (zb >= ze) continue;
                const int tx = tile % A.ntx, ty = tile / A.ntx;
                const int x0 = tx * TX, y0 = ty * TY;
                if (is_u) {
                    if (isB) {
                        // V of this tile and its star neighbours on chunks c-1, c must be complete
                        const int nb[5] = {tile, tx > 0 ? tile - 1 : -1, tx + 1 < A.ntx ? tile + 1 : -1,
                                           ty > 0 ? tile - A.ntx : -1, ty + 1 < A.nty ? tile + A.ntx : -1};
                        for (int cc = c > 0 ? c - 1 : 0; cc <= c; ++cc)
                            for (int q = 0; q < 5; ++q)
                                if (nb[q] >= 0) wait_epoch(T.done + (int64_t)cc * ntiles + nb[q], T.epoch);
                        // generic-proxy stores of other CTAs -> this CTA's async-proxy (TMA) reads
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    const CUtensorMap* mu = isB ? &M.vh : &M.xh;
                    const int niter = ze - zb + 2 * R;
                    for (int k = 0; k < niter; ++k) {
                        mbar_wait(&emptyU[rr.slot], rr.phase ^ 1);
                        mbar_expect_tx(&fullU[rr.slot], C::STAGE_BYTES);
                        if (isB)  // V: last readers are this item and its neighbours, soon -- default policy
                            tma_load_3d(ring + rr.slot * C::STAGE_STRIDE_F, mu, &fullU[rr.slot], x0 - RP, y0 - R, zb + k);
                        else      // X: the B items re-read it as u^{n-1}
                            tma_load_3d_hint(ring + rr.slot * C::STAGE_STRIDE_F, mu, &fullU[rr.slot], x0 - RP, y0 - R,
                                             zb + k, keep);
                        rr.advance(SU);
                    }
                } else {
                    const CUtensorMap* mp = isB ? &M.xc : &M.y;
                    for (int z = zb; z < ze; ++z) {
                        const bool use_a = A.a && A.flags[(int64_t)tile * nz + z];
                        const int2 tp = A.tpsc ? A.tpsc[(int64_t)tile * nz + z] : make_int2(0, 0);
                        float* dst = pring + rr.slot * C::PSTAGE_FLOATS;
                        mbar_wait(&emptyP[rr.slot], rr.phase ^ 1);
                        // ordered for the consumers by this arrive (release) and their wait (acquire);
                        // compute-sanitizer racecheck does not model mbarrier phases
                        pmeta[4 * rr.slot] = use_a;
                        pmeta[4 * rr.slot + 1] = tp.x;
                        pmeta[4 * rr.slot + 2] = tp.y;
                        mbar_expect_tx(&fullP[rr.slot], (use_a ? 3 : 2) * C::PTILE_BYTES);
                        // A: Y is dead after this read, b and a are re-read by B; B: last use of all three
                        const uint64_t pb = isB ? drop : keep;
                        tma_load_3d_hint(dst, mp, &fullP[rr.slot], x0, y0, z + R, drop);
                        tma_load_3d_hint(dst + C::PTILE_FLOATS, &M.b, &fullP[rr.slot], x0, y0, z, pb);
                        if (use_a) tma_load_3d_hint(dst + 2 * C::PTILE_FLOATS, &M.a, &fullP[rr.slot], x0, y0, z, pb);
                        rr.advance(SP);
                    }
                }
            }
        }
        return;
    }

    // ---- consumers ----
    consumer_regs<C>();
    const int ly = warp * C::RY;
    const uint64_t st_keep = policy_evict_last(), st_drop = policy_evict_first();
    Ring ru{0, 0}, rp{0, 0};
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        int tile, c, zb, ze;
        bool isB;
        tb_decode(item, ntiles, T.nzc, T.Z, R, nz, T.lead, tile, c, isB, zb, ze);
        const int x0 = (tile % A.ntx) * TX, y0 = (tile / A.ntx) * TY;
        if (zb < ze) {
            float* out = isB ? T.w : T.v;
            const int64_t n_inj = step_n + (isB ? 1 : 0);
            const uint64_t pol = isB ? st_drop : st_keep;  // V is re-read by B; W only by the next pass
            if (x0 + TX <= g.nx && y0 + TY <= g.ny)
                consume_item<C, true, false, true>(A, ring, pring, fullU, emptyU, fullP, emptyP, pmeta, tile, zb, ze, x0, y0,
                                             lane, ly, ru, rp, n_inj, out, pol);
            else
                consume_item<C, false, false, true>(A, ring, pring, fullU, emptyU, fullP, emptyP, pmeta, tile, zb, ze, x0,
                                              y0, lane, ly, ru, rp, n_inj, out, pol);
        }
        if (!isB && c < T.nzc) {
            // publish "A(tile, c) complete": every consumer's V stores, then one release
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("bar.sync 1, %0;" ::"r"(C::NCOMP) : "memory");
            if (tid == 0) {
                __threadfence();
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(T.done + (int64_t)c * ntiles + tile),
                             "l"(T.epoch)
                             : "memory");
            }
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct StreamPlan {
    StreamMaps maps[2];  // by parity of the u^n buffer
    uint8_t* flags = nullptr;
    int ntx = 0, nty = 0;
    int grid = 0;
    int R = 0;
    size_t smem = 0;
    int nthreads = 0;
    int TX = 0, TY = 0;
    int nzc = 1, zc = 0;
    unsigned long long* d_count = nullptr;  // tile-planes with a != 1 (inside the flags allocation)
    int64_t nflags = 0;
    int2* tpsc[2] = {nullptr, nullptr};     // [ntiles][nz] injection lists (fused sparse work), per set
    int4* tpe[2] = {nullptr, nullptr};      // set 0: sources; set 1: FWI adjoint sources (receivers)
    size_t tpe_cap[2] = {0, 0};
    // NEXT-1 temporal blocking
    unsigned long long* tb_done = nullptr;  // [tb_nzc][ntiles] completion epochs of the A items
    unsigned long long tb_epoch = 0;        // last epoch handed out (monotone)
    int tb_Z = 0, tb_nzc = 0, tb_lead = 1;
    // tensor maps of explicit-buffer launches (FWI history ring, adjoint pair), keyed by
    // (base pointer, box kind); cleared when the plan is refreshed
    std::unordered_map<uint64_t, CUtensorMap> map_cache;
    // AW_OPT_TIMING = 2: per-launch device timestamps (buffers owned by the grid handle; null = off)
    unsigned long long* ts0 = nullptr;
    unsigned long long* ts1 = nullptr;
    int ts_cap = 0;
    // split high-order kernel: z chunks are a multiple of zq planes (its unroll; 1 = any);
    // item_inj[set][item] = 1 if the item (tile, chunk) holds injection corners of that set
    int zq = 1;
    uint8_t* item_inj[2] = {nullptr, nullptr};
    // small grids: the resident multi-step kernel (per-item step counters, receivers by item)
    unsigned long long* res_done = nullptr;  // [nitems]
    int* ritem = nullptr;                    // [nitems + 1] CSR pointers, then the receiver indices
    size_t ritem_cap = 0;                    // ints allocated in ritem
    int res_ok = 0;                          // the resident kernel fits the plan's grid (occupancy)
};

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

cudaError_t encode3d(CUtensorMap* m, const void* base, const Geom& g, int planes, int bx, int by) {
    auto enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    cuuint64_t dims[3] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)g.pitch * 4, (cuuint64_t)g.plane * 4};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    // no L2 promotion: a promoted halo'd box fetches whole 256-B segments of the neighbours
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <class C>
cudaError_t setup(StreamPlan* p, const Geom& g) {
    p->smem = C::SMEM;
    p->nthreads = C::NTHREADS;
    p->TX = C::TX;
    p->TY = C::TY;
    cudaError_t e = cudaFuncSetAttribute(stream_kernel<C, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(stream_kernel<C, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(tb_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int occ = 0, occ_t = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stream_kernel<C, false>, C::NTHREADS, C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, stream_kernel<C, true>, C::NTHREADS, C::SMEM);
    if (e != cudaSuccess) return e;
    occ = occ < occ_t ? occ : occ_t;
    int occ_tb = 0;  // the temporal-blocking kernel shares the grid (all its CTAs must be resident)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_tb, tb_kernel<C>, C::NTHREADS, C::SMEM);
    if (e != cudaSuccess) return e;
    occ = occ < occ_tb ? occ : occ_tb;
    // the resident kernel too, if it fits: it is used only when all of its CTAs are co-resident
    int occ_res = 0;
    if (cudaFuncSetAttribute(resident_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) ==
            cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_res, resident_kernel<C>, C::NTHREADS, C::SMEM) ==
            cudaSuccess)
        p->res_ok = occ_res >= occ;
    cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorNotSupported;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    p->grid = sms * occ;
    return cudaSuccess;
}

template <class C>
cudaError_t make_maps(StreamPlan* p, const Geom& g, const float* const* ubuf, const float* b, const float* a) {
    for (int par = 0; par < 2; ++par) {
        StreamMaps& M = p->maps[par];
        cudaError_t e;
        if ((e = encode3d(&M.u, ubuf[par], g, g.nz + 2 * g.R, C::TXP, C::TYP))) return e;
        if ((e = encode3d(&M.un, ubuf[1 - par], g, g.nz + 2 * g.R, C::TX, C::TY))) return e;
        if ((e = encode3d(&M.b, b, g, g.nz, C::TX, C::TY))) return e;
        if ((e = encode3d(&M.a, a ? a : b, g, g.nz, C::TX, C::TY))) return e;
    }
    return cudaSuccess;
}

template <class C>
cudaError_t launch(StreamPlan* p, const Geom& g, const Coefs& c, int parity_cur, const float* ucur, float* unext,
                   const float* b, const float* a, const Halo& halo, int parity_next, const Sparse& sp,
                   const int64_t* d_base, int step_i, cudaStream_t s) {
    StreamArgs A;
    std::memset(&A, 0, sizeof A);
    A.g = g;
    A.c = c;
    A.unext = unext;
    A.a = a;
    A.flags = p->flags;
    A.lo = halo.lo[parity_next];
    A.lo_off = halo.lo_off;
    A.hi = halo.hi[parity_next];
    A.hi_off = halo.hi_off;
    A.ntx = p->ntx;
    A.nty = p->nty;
    A.nzc = p->nzc;
    A.zc = p->zc;
    A.nitems = p->ntx * p->nty * p->nzc;
    A.tpsc = sp.nuc > 0 ? p->tpsc[0] : nullptr;
    A.tpe = p->tpe[0];
    A.item_inj = sp.nuc > 0 ? p->item_inj[0] : nullptr;
    A.inj_src = sp.inj_src;
    A.inj_s = sp.inj_s;
    A.wavelet = sp.wavelet;
    A.ns = sp.ns;
    A.nrl = sp.nrl;
    A.nr = sp.nr;
    A.nc = sp.nc;
    A.rec_id = sp.rec_id;
    A.rec_off = sp.rec_off;
    A.rec_w = sp.rec_w;
    A.traces = sp.traces;
    A.ucur = ucur;
    A.d_base = d_base;
    A.step_i = step_i;
    A.ts0 = p->ts0;
    A.ts1 = p->ts1;
    A.ts_cap = p->ts_cap;
    if (A.lo || A.hi) {
        // boundary chunks first: [0, tc_lo) hold planes z < R, [tc_hi, nzc) planes z >= nz - R
        const int zc = p->zc, nzc = p->nzc;
        A.tc_lo = std::min(nzc, (g.R + zc - 1) / zc);
        A.tc_hi = std::max(A.tc_lo, std::min(nzc, std::max(0, g.nz - g.R) / zc));
        A.tc_nb = A.tc_lo + (nzc - A.tc_hi);
        A.ctl = halo.ctl;
        A.flag_lo = halo.flag_lo;
        A.flag_hi = halo.flag_hi;
        if (!A.flag_lo && !A.flag_hi) A.ctl = nullptr;  // nobody to signal
    }
    if (A.lo || A.hi)
        stream_kernel<C, true><<<p->grid, C::NTHREADS, C::SMEM, s>>>(p->maps[parity_cur], A);
    else
        stream_kernel<C, false><<<p->grid, C::NTHREADS, C::SMEM, s>>>(p->maps[parity_cur], A);
    return cudaGetLastError();
}

// One step on explicit buffers (FWI history ring / adjoint, NEXT-3): maps encoded for (ucur, uprev)
// at launch (host-side cuTensorMapEncodeTiled, ~1 us each; passed by value as __grid_constant__).
template <class C>
cudaError_t launch_bufs(StreamPlan* p, const Geom& g, const Coefs& c, const float* ucur, const float* uprev,
                        float* unext, const float* b, const float* a, const Sparse& sp, int inj_set,
                        const int64_t* d_base, int step_i, cudaStream_t s) {
    StreamMaps M;
    cudaError_t e;
    // encoding a map costs microseconds of host time per call: cache them per (buffer, box kind)
    auto cached = [&](CUtensorMap* m, const void* base, int planes, int bx, int by, int kind) -> cudaError_t {
        const uint64_t key = (uint64_t)(uintptr_t)base ^ (uint64_t)kind;  // bases are 256-B aligned
        auto it = p->map_cache.find(key);
        if (it != p->map_cache.end()) {
            *m = it->second;
            return cudaSuccess;
        }
        cudaError_t r = encode3d(m, base, g, planes, bx, by);
        if (r == cudaSuccess) p->map_cache.emplace(key, *m);
        return r;
    };
    if ((e = cached(&M.u, ucur, g.nz + 2 * g.R, C::TXP, C::TYP, 1))) return e;
    if ((e = cached(&M.un, uprev, g.nz + 2 * g.R, C::TX, C::TY, 2))) return e;
    if ((e = cached(&M.b, b, g.nz, C::TX, C::TY, 3))) return e;
    if ((e = cached(&M.a, a ? a : b, g.nz, C::TX, C::TY, 4))) return e;
    StreamArgs A;
    std::memset(&A, 0, sizeof A);
    A.g = g;
    A.c = c;
    A.unext = unext;
    A.a = a;
    A.flags = p->flags;
    A.ntx = p->ntx;
    A.nty = p->nty;
    A.nzc = p->nzc;
    A.zc = p->zc;
    A.nitems = p->ntx * p->nty * p->nzc;
    A.tpsc = sp.nuc > 0 ? p->tpsc[inj_set] : nullptr;
    A.tpe = p->tpe[inj_set];
    A.item_inj = sp.nuc > 0 ? p->item_inj[inj_set] : nullptr;
    A.inj_src = sp.inj_src;
    A.inj_s = sp.inj_s;
    A.wavelet = sp.wavelet;
    A.ns = sp.ns;
    A.nrl = sp.nrl;
    A.nr = sp.nr;
    A.nc = sp.nc;
    A.rec_id = sp.rec_id;
    A.rec_off = sp.rec_off;
    A.rec_w = sp.rec_w;
    A.traces = sp.traces;
    A.ucur = ucur;
    A.d_base = d_base;
    A.step_i = step_i;
    A.ts0 = p->ts0;
    A.ts1 = p->ts1;
    A.ts_cap = p->ts_cap;
    stream_kernel<C, false><<<p->grid, C::NTHREADS, C::SMEM, s>>>(M, A);
    return cudaGetLastError();
}

// One launch of the resident kernel: nsteps steps from local step step0 (single slab).
template <class C>
cudaError_t launch_res(StreamPlan* p, const Geom& g, const Coefs& c, int cur0, float* const* buf, const float* b,
                       const float* a, const Sparse& sp, const int64_t* d_base, int step0, int nsteps,
                       cudaStream_t s) {
    if (!p->res_done || !p->ritem || !p->res_ok) return cudaErrorNotSupported;
    ResMaps M;
    M.m[0] = p->maps[0];
    M.m[1] = p->maps[1];
    ResArgs R;
    std::memset(&R, 0, sizeof R);
    StreamArgs& A = R.s;
    A.g = g;
    A.c = c;
    A.a = a;
    A.flags = p->flags;
    A.ntx = p->ntx;
    A.nty = p->nty;
    A.nzc = p->nzc;
    A.zc = p->zc;
    A.nitems = p->ntx * p->nty * p->nzc;
    A.tpsc = sp.nuc > 0 ? p->tpsc[0] : nullptr;
    A.tpe = p->tpe[0];
    A.inj_src = sp.inj_src;
    A.inj_s = sp.inj_s;
    A.wavelet = sp.wavelet;
    A.ns = sp.ns;
    A.nrl = sp.nrl;
    A.nr = sp.nr;
    A.nc = sp.nc;
    A.rec_id = sp.rec_id;
    A.rec_off = sp.rec_off;
    A.rec_w = sp.rec_w;
    A.traces = sp.traces;
    A.d_base = d_base;
    A.ts0 = p->ts0;
    A.ts1 = p->ts1;
    A.ts_cap = p->ts_cap;
    R.buf[0] = buf[0];
    R.buf[1] = buf[1];
    R.cur0 = cur0;
    R.nsteps = nsteps;
    R.step0 = step0;
    R.done = p->res_done;
    R.ritem_ptr = p->ritem;
    R.ritem_idx = p->ritem + A.nitems + 1;
    R.skip_wait = dev_knob("AW_RES_NOWAIT") != nullptr;  // always 0 in the product library
    resident_kernel<C><<<p->grid, C::NTHREADS, C::SMEM, s>>>(M, R);
    return cudaGetLastError();
}

// One two-step pass of the temporal-blocking kernel (single slab).
template <class C>
cudaError_t launch_tb(StreamPlan* p, const Geom& g, const Coefs& c, const float* x, float* y, float* v,
                      const float* b, const float* a, const Sparse& sp, const int64_t* d_base, int step_i,
                      cudaStream_t s) {
    if (!p->tb_done) return cudaErrorNotSupported;
    TbMaps M;
    cudaError_t e;
    if ((e = encode3d(&M.xh, x, g, g.nz + 2 * g.R, C::TXP, C::TYP))) return e;
    if ((e = encode3d(&M.vh, v, g, g.nz + 2 * g.R, C::TXP, C::TYP))) return e;
    if ((e = encode3d(&M.y, y, g, g.nz + 2 * g.R, C::TX, C::TY))) return e;
    if ((e = encode3d(&M.xc, x, g, g.nz + 2 * g.R, C::TX, C::TY))) return e;
    if ((e = encode3d(&M.b, b, g, g.nz, C::TX, C::TY))) return e;
    if ((e = encode3d(&M.a, a ? a : b, g, g.nz, C::TX, C::TY))) return e;
    TbArgs T;
    std::memset(&T, 0, sizeof T);
    StreamArgs& A = T.s;
    A.g = g;
    A.c = c;
    A.a = a;
    A.flags = p->flags;
    A.ntx = p->ntx;
    A.nty = p->nty;
    A.tpsc = sp.nuc > 0 ? p->tpsc[0] : nullptr;
    A.tpe = p->tpe[0];
    A.inj_src = sp.inj_src;
    A.inj_s = sp.inj_s;
    A.wavelet = sp.wavelet;
    A.ns = sp.ns;
    A.nrl = sp.nrl;
    A.nr = sp.nr;
    A.nc = sp.nc;
    A.rec_id = sp.rec_id;
    A.rec_off = sp.rec_off;
    A.rec_w = sp.rec_w;
    A.traces = sp.traces;
    A.ucur = x;
    A.d_base = d_base;
    A.step_i = step_i;
    T.v = v;
    T.w = y;
    T.done = p->tb_done;
    T.epoch = ++p->tb_epoch;
    T.Z = p->tb_Z;
    T.nzc = p->tb_nzc;
    T.lead = p->tb_lead;
    tb_kernel<C><<<p->grid, C::NTHREADS, C::SMEM, s>>>(M, T);
    return cudaGetLastError();
}

// configuration table: (R, TY, RY, D = u^n ring lookahead, DP = streams lookahead,
//                       PD = L2 prefetch distance, min CTAs/SM)
using C1 = Cfg<1, 32, 2, 4, 4, 0, 1>;  // 16 consumer warps, 2 rows each
using C2 = Cfg<2, 32, 2, 4, 4, 0, 1>;  // 16 consumer warps, 2 rows each
using C3 = Cfg<3, 32, 2, 4, 4, 0, 1>;  // 16 consumer warps, 2 rows each
using C4 = Cfg<4, 32, 2, 4, 4, 0, 1>;  // 16 consumer warps, 2 rows each
using C5 = Cfg<5, 32, 4, 3, 3, 0, 1>;
// R = 6..8 (so 12-16; C4, C5): half register queue with 4 rows per thread (8 consumer warps, 64 x 32 tiles):
// the queue's registers pay for the taller row block, which loads each y column once for 4 rows.  On 512^3
// (ms per step, profiles/r2/ab_half_queue.jsonl): so 12 0.525 -> 0.427, so 14 0.533 -> 0.481, so 16 0.558
// -> 0.541; the same change measured no gain for R <= 5
using C6 = Cfg<6, 32, 4, 3, 2, 0, 1, true, 0, 40, 0>;
using C7 = Cfg<7, 32, 4, 2, 1, 0, 1, true, 0, 40, 0>;
using C8 = Cfg<8, 32, 4, 2, 1, 0, 1, true, 0, 40, 0>;
// development variants of R=4 (AW_STREAM_VARIANT=1/2/3), for measurements
using C4v1 = Cfg<4, 32, 4, 4, 4, 0, 1, false>;  // round-1 lane mapping (l, l+32)
using C4v2 = Cfg<4, 32, 4, 5, 3, 0, 1>;
using C4v3 = Cfg<4, 16, 2, 4, 4, 0, 1>;
// measurement variants of the high orders (AW_STREAM_VARIANT=1/2/3 with R = 6 / 8)
using C6v1 = Cfg<6, 32, 4, 2, 3, 0, 1, false>;  // the round-1 R=6 configuration
using C6v2 = Cfg<6, 16, 1, 4, 4, 0, 1>;  // 16 consumer warps, one row each
using C6v3 = Cfg<6, 32, 2, 2, 2, 0, 1>;
using C8v1 = Cfg<8, 16, 2, 3, 3, 0, 1>;
using C8v2 = Cfg<8, 16, 1, 4, 4, 0, 1>;  // 16 consumer warps, one row each
using C8v3 = Cfg<8, 16, 2, 4, 4, 0, 1, false>;
// warpgroup layout (setmaxnreg): 12 consumer warps, 24-row tiles
using C6v4 = Cfg<6, 24, 2, 2, 2, 0, 1, true, 152, 40>;
using C6v5 = Cfg<6, 24, 2, 3, 2, 0, 1, true, 152, 40>;
using C8v4 = Cfg<8, 24, 2, 2, 2, 0, 1, true, 152, 40>;
using C8v5 = Cfg<8, 24, 2, 3, 2, 0, 1, true, 152, 40>;
// half register queue (HQ): 8 and 12 consumer warps
using C6v0 = Cfg<6, 16, 2, 4, 4, 0, 1>;  // the round-1/2 product configurations (register queue of 2R+1)
using C7v0 = Cfg<7, 16, 2, 4, 4, 0, 1>;
using C8v0 = Cfg<8, 16, 2, 4, 4, 0, 1>;
using C6v6 = Cfg<6, 16, 2, 4, 4, 0, 1, true, 0, 40, 0>;
using C6v7 = Cfg<6, 24, 2, 3, 3, 0, 1, true, 0, 40, 0>;
using C8v6 = Cfg<8, 16, 2, 4, 4, 0, 1, true, 0, 40, 0>;
using C8v7 = Cfg<8, 24, 2, 3, 3, 0, 1, true, 0, 40, 0>;
using C4v4 = Cfg<4, 16, 2, 3, 3, 0, 2, true, 0, 40, 0>;   // HQ, 2 CTAs per SM
using C4v5 = Cfg<4, 32, 2, 4, 4, 0, 1, true, 0, 40, 0>;   // HQ, the product tile
using C5v6 = Cfg<5, 24, 2, 3, 3, 0, 1, true, 0, 40, 0>;
using C5v7 = Cfg<5, 32, 2, 3, 3, 0, 1, true, 0, 40, 0>;
using C6v8 = Cfg<6, 24, 2, 4, 3, 0, 1, true, 0, 40, 0>;
using C7v6 = Cfg<7, 24, 2, 3, 3, 0, 1, true, 0, 40, 0>;
// R = 6 HQ: ring depths, taller per-thread row blocks (fewer y-column loads per point)
using C6v11 = Cfg<6, 24, 2, 5, 3, 0, 1, true, 0, 40, 0>;
using C6v12 = Cfg<6, 24, 2, 4, 2, 0, 1, true, 0, 40, 0>;
using C6v13 = Cfg<6, 24, 3, 4, 3, 0, 1, true, 0, 40, 0>;   // 8 consumer warps x 3 rows
using C6v14 = Cfg<6, 32, 4, 3, 2, 0, 1, true, 0, 40, 0>;   // 8 consumer warps x 4 rows
// half queue with 4 rows per thread (8 consumer warps, 64 x 32 tiles)
using C4v6 = Cfg<4, 32, 4, 4, 4, 0, 1, true, 0, 40, 0>;
using C4v7 = Cfg<4, 32, 4, 4, 4, 0, 1>;   // the round-1 product configuration (8 consumer warps x 4 rows)
using C5v8 = Cfg<5, 32, 4, 3, 3, 0, 1, true, 0, 40, 0>;
using C6v15 = Cfg<6, 32, 4, 2, 2, 0, 1, true, 0, 40, 0>;
using C6v16 = Cfg<6, 32, 4, 3, 1, 0, 1, true, 0, 40, 0>;
using C7v12 = Cfg<7, 32, 4, 2, 1, 0, 1, true, 0, 40, 0>;
using C8v12 = Cfg<8, 32, 4, 2, 1, 0, 1, true, 0, 40, 0>;
using C8v13 = Cfg<8, 32, 4, 1, 2, 0, 1, true, 0, 40, 0>;
using C8v15 = Cfg<8, 32, 4, 1, 1, 0, 1, true, 0, 40, 0>;
using C8v16 = Cfg<8, 24, 4, 3, 2, 0, 1, true, 0, 40, 0>;   // 6 consumer warps x 4 rows
using C7v13 = Cfg<7, 32, 4, 3, 1, 0, 1, true, 0, 40, 0>;
// partial queues (z-R .. z+QJ in registers)
using C8v9 = Cfg<8, 24, 2, 3, 3, 0, 1, true, 0, 40, 2>;
using C8v10 = Cfg<8, 24, 2, 3, 3, 0, 1, true, 0, 40, 3>;
using C8v11 = Cfg<8, 16, 2, 4, 4, 0, 1, true, 0, 40, 4>;
using C7v9 = Cfg<7, 24, 2, 3, 3, 0, 1, true, 0, 40, 2>;

int variant() {
    const char* v = dev_knob("AW_STREAM_VARIANT");
    return v ? atoi(v) : 0;
}

}  // namespace

// Per-R entry points (one translation unit each): the host side dispatches through these.
struct StreamOps {
    cudaError_t (*setup)(StreamPlan*, const Geom&);
    cudaError_t (*make_maps)(StreamPlan*, const Geom&, const float* const*, const float*, const float*);
    cudaError_t (*launch)(StreamPlan*, const Geom&, const Coefs&, int, const float*, float*, const float*,
                          const float*, const Halo&, int, const Sparse&, const int64_t*, int, cudaStream_t);
    cudaError_t (*launch_bufs)(StreamPlan*, const Geom&, const Coefs&, const float*, const float*, float*,
                               const float*, const float*, const Sparse&, int, const int64_t*, int, cudaStream_t);
    cudaError_t (*launch_tb)(StreamPlan*, const Geom&, const Coefs&, const float*, float*, float*, const float*,
                             const float*, const Sparse&, const int64_t*, int, cudaStream_t);
    cudaError_t (*launch_res)(StreamPlan*, const Geom&, const Coefs&, int, float* const*, const float*, const float*,
                              const Sparse&, const int64_t*, int, int, cudaStream_t);
};
const StreamOps* stream_ops_r1();
const StreamOps* stream_ops_r2();
const StreamOps* stream_ops_r3();
const StreamOps* stream_ops_r4();
const StreamOps* stream_ops_r5();
const StreamOps* stream_ops_r6();
const StreamOps* stream_ops_r7();
const StreamOps* stream_ops_r8();

namespace {
template <class C>
const StreamOps* ops_of() {
    static const StreamOps o{setup<C>, make_maps<C>, launch<C>, launch_bufs<C>, launch_tb<C>, launch_res<C>};
    return &o;
}
}  // namespace

}  // namespace aw
