// aw_hstream.cuh -- the 2.5D z-streaming kernel for the high space orders (R = k/2 >= 6).
// (Included by aw_stream_r{6..8}.cu after aw_stream.cuh; the host side is shared.)
//
// Same operation and per-point sequence as stream_kernel, so the
// result is value-identical.  What limits stream_kernel at high orders is not HBM but the SM
// (ncu source pages of so 16): two consumer warps per scheduler to hide the LDS and
// FMA-chain latencies, 160+ registers per thread (the 2R+1-deep register queue), and a plane loop
// unrolled 2R+1 times (for the queue's renaming) whose ~57 KB of SASS overflows the 32 KB L1.5
// instruction cache.  This kernel splits a point's canonical sequence between two consumer
// warpgroup pairs at the one place the order allows it -- before the z pairs, which come last:
//
//  * A warps (in-plane part): L_xy = C0 u; x pairs j = 1..R; y pairs j = 1..R, from the halo'd
//    u^n tile of the output plane; written to a shared-memory ring (SL stages, 4 B/point).  No
//    queue, so few registers and a plain (not unrolled) plane loop of ~150 instructions;
//  * B warps (z part and update): the 2R+1-deep register queue of centre values; L = L_xy, then
//    z pairs j = 1..R; t = 2u - u^{n-1}; w = fma(b, L, t); u^{n+1} = fma(a, w, (1-a) u^{n-1}); the
//    store (+ injection and the team's peer stores on the generic path).  Its plane loop is
//    unrolled Q = 24 >= 2R+1 times for the queue's renaming, but its body is ~80 instructions, so
//    the unrolled loop (~30 KB) fits the instruction cache;
//  * every ring depth (u^n: SU, streams: SP, L_xy: SL) divides Q and every work item starts at
//    stage 0, so in B's unrolled loop all stage addresses, barriers and queue slots are
//    compile-time constants (per-stage phase bits); z chunks are a multiple of Q planes, so a full
//    chunk's loop has no trip-count checks; edge tiles, ragged chunks, items holding injection
//    corners and (in a team) boundary planes take B's generic instantiation;
//  * a service warpgroup: the u^n TMA producer (+ L2 prefetch of the streams and of the next item's
//    first planes), the u^{n-1}, b, a TMA producer, the receivers warp, one idle warp; registers are
//    redistributed with setmaxnreg (service 40, A 88, B 128 per thread);
//  * 16 consumer warps per SM instead of 8.
#pragma once
#include "aw_stream.cuh"

namespace aw {

namespace {

template <int R_, int SU_, int SP_, int SL_>
struct HCfg {
    static constexpr int R = R_, TX = 64, TY = 16, RY = 2, MINB = 1;
    static constexpr int Q = 24;  // B's plane-loop unroll = queue slots (>= 2R+1)
    static constexpr int SU = SU_, SP = SP_, SL = SL_;
    static_assert(Q >= 2 * R + 1 && Q % SU == 0 && Q % SP == 0 && Q % SL == 0 && SU <= 32, "ring geometry");
    static_assert(SU >= R + 2, "the u^n ring must hold a plane from its centre read to its output use");
    static constexpr int RP = (R + 3) / 4 * 4;  // x halo rounded up to 4 floats (TMA box rows: 32-B multiple)
    static constexpr int TXP = TX + 2 * RP;
    static constexpr int TYP = TY + 2 * R;
    static constexpr int NW_A = TY / RY, NW_B = TY / RY;  // 8 + 8 consumer warps, 2 rows x 2 columns each
    static constexpr int N_A = 32 * NW_A, N_B = 32 * NW_B;
    static constexpr int W_B = NW_A, W_S = NW_A + NW_B;  // first B warp, first service warp
    static constexpr int NTHREADS = N_A + N_B + 128;
    // setmaxnreg moves registers only within the CTA's own allocation (NTHREADS x the launch count
    // LREG); a request beyond it never completes
    static constexpr int LREG = (65536 / NTHREADS) / 8 * 8;
    static constexpr int AREG = 88, BREG = 128, PREG = 40;
    static_assert(N_A * AREG + N_B * BREG + 128 * PREG <= NTHREADS * LREG && NW_A % 4 == 0 && NW_B % 4 == 0,
                  "register split must fit the CTA's allocation");
    static constexpr int STAGE_BYTES = TXP * TYP * 4;
    static constexpr int STAGE_STRIDE = (STAGE_BYTES + 127) / 128 * 128;
    static constexpr int STAGE_STRIDE_F = STAGE_STRIDE / 4;
    static constexpr int PTILE_FLOATS = TX * TY;
    static constexpr int PTILE_BYTES = PTILE_FLOATS * 4;
    static constexpr int PSTAGE_FLOATS = 3 * PTILE_FLOATS;  // u^{n-1}, b, a
    static constexpr size_t U_BYTES = (size_t)SU * STAGE_STRIDE;
    static constexpr size_t P_BYTES = (size_t)SP * PSTAGE_FLOATS * 4;
    static constexpr size_t L_BYTES = (size_t)SL * PTILE_FLOATS * 4;
    static constexpr size_t BAR_OFF = U_BYTES + P_BYTES + L_BYTES;
    static constexpr size_t META_OFF = BAR_OFF + (2 * SU + 2 * SP + 2 * SL) * sizeof(uint64_t);
    static constexpr size_t SMEM = META_OFF + 4 * SP * sizeof(int);
    static_assert(TXP <= 256 && TYP <= 256, "TMA box");
    static_assert(SMEM <= 232448, "shared memory per CTA");
};

// Hides a value from the optimizer: without it the plane offsets of all Q unrolled iterations are
// precomputed into separate 64-bit registers instead of advancing one offset
__device__ __forceinline__ int64_t opaque(int64_t v) {
    asm volatile("" : "+l"(v));
    return v;
}

struct HBars {
    uint64_t *fullU, *emptyU, *fullP, *emptyP, *fullL, *emptyL;
};

}  // namespace

// ---- A warps: L_xy of every output plane of one item into the L ring ----
template <class C>
__device__ __forceinline__ void h_inplane(const StreamArgs& A, const float* ring, float* lring, const HBars& B,
                                          int zb, int ze, int lane, int ly, uint32_t& phU, uint32_t& phL) {
    constexpr int R = C::R, RP = C::RP, TX = C::TX, TXP = C::TXP, SU = C::SU, SL = C::SL;
    constexpr int STR = C::STAGE_STRIDE_F, PT = C::PTILE_FLOATS;
    const int niter = ze - zb + 2 * R;
    const float2 C0 = f2(A.c.C0, A.c.C0);
    const float* const rb = ring + ly * TXP + RP + 2 * lane;  // this thread's column pair, halo row ly
    float* const lb = lring + ly * TX + 2 * lane;
    int s = 0, ls = 0;
#pragma unroll 1
    for (int k = 0; k < niter; ++k) {  // plane zb-R+k in stage k mod SU
        mbar_wait(&B.fullU[s], (phU >> s) & 1u);
        phU ^= 1u << s;
        if (k >= R && k < niter - R) {  // an output plane
            const float* Qs = rb + s * STR;
            float2 col[C::RY + 2 * R];
#pragma unroll
            for (int r = 0; r < C::RY + 2 * R; ++r) col[r] = *reinterpret_cast<const float2*>(Qs + r * TXP);
            float2 L[C::RY];
#pragma unroll
            for (int i = 0; i < C::RY; ++i) {
                const float* row = Qs + (i + R) * TXP;
                L[i] = mul2(C0, col[i + R]);
                constexpr int K = (R + 1) / 2;
                float2 v[2 * K + 1];  // v[K + m] = columns (2l + 2m, 2l + 2m + 1), m = -K..K
#pragma unroll
                for (int m = -K; m <= K; ++m) v[K + m] = *reinterpret_cast<const float2*>(row + 2 * m);
#pragma unroll
                for (int jj = 1; jj <= R; ++jj) {
                    const int m = jj >> 1;
                    if (jj & 1) {  // odd: the two columns' pairs sit in different float2s
                        const float2 sa = add2(v[K - m - 1], v[K + m]);  // .y = u[2l-jj] + u[2l+jj]
                        const float2 sb = add2(v[K - m], v[K + m + 1]);  // .x = u[2l+1-jj] + u[2l+1+jj]
                        L[i].x = __fmaf_rn(A.c.C[2][jj], sa.y, L[i].x);
                        L[i].y = __fmaf_rn(A.c.C[2][jj], sb.x, L[i].y);
                    } else {
                        L[i] = fma2(f2(A.c.C[2][jj], A.c.C[2][jj]), add2(v[K - m], v[K + m]), L[i]);
                    }
                }
#pragma unroll
                for (int jj = 1; jj <= R; ++jj)
                    L[i] = fma2(f2(A.c.C[1][jj], A.c.C[1][jj]), add2(col[i + R - jj], col[i + R + jj]), L[i]);
            }
            mbar_arrive(&B.emptyU[s]);  // the halo'd tile is consumed
            mbar_wait(&B.emptyL[ls], ((phL >> ls) & 1u) ^ 1u);
            phL ^= 1u << ls;
            float* Ld = lb + ls * PT;
#pragma unroll
            for (int i = 0; i < C::RY; ++i) *reinterpret_cast<float2*>(Ld + i * TX) = L[i];
            mbar_arrive(&B.fullL[ls]);  // release: the STS above are visible to B after its wait
            ls = ls + 1 == SL ? 0 : ls + 1;
        } else {
            mbar_arrive(&B.emptyU[s]);  // a halo plane: only its centre (B) is needed
        }
        s = s + 1 == SU ? 0 : s + 1;
    }
}

// ---- B warps: z pairs + update of one item.  FAST: interior tile, full chunk (a multiple of Q
// planes), no injection corners, no peer stores.  Otherwise the generic checks. ----
template <class C, bool FAST, bool TEAM>
__device__ __forceinline__ void h_zpart(const StreamArgs& A, const float* ring, const float* pring, const float* lring,
                                        const HBars& B, const volatile int* pmeta, int tile, int zb, int ze, int x0,
                                        int y0, int lane, int ly, uint32_t& phU, uint32_t& phP, uint32_t& phL,
                                        int64_t step_n) {
    constexpr int R = C::R, RY = C::RY, RP = C::RP, TX = C::TX, TXP = C::TXP, Q = C::Q;
    constexpr int SU = C::SU, SP = C::SP, SL = C::SL, STR = C::STAGE_STRIDE_F, PT = C::PTILE_FLOATS;
    const Geom& g = A.g;
    const int nz = g.nz;
    const int niter = ze - zb + 2 * R;
    const int64_t pitch = g.pitch, plane = g.plane;
    const float2 two = f2(2.0f, 2.0f), one = f2(1.0f, 1.0f);
    const int xa = x0 + 2 * lane;
    bool ok_a[RY], ok_b[RY];
#pragma unroll
    for (int i = 0; i < RY; ++i) {
        ok_a[i] = FAST || ((y0 + ly + i) < g.ny && xa < g.nx);
        ok_b[i] = FAST || (ok_a[i] && xa + 1 < g.nx);
    }
    // model-layout offset of (output plane, row y0+ly, column xa); the u^{n+1} buffer holds the same
    // point R planes further (its plane -R is the base)
    int64_t o = (int64_t)zb * plane + (int64_t)(y0 + ly) * pitch + xa;
    float* const ubuf = A.unext + (int64_t)R * plane;
    const float* const cb = ring + (ly + R) * TXP + RP + 2 * lane;  // centre of this thread's rows
    const float* const pb = pring + ly * TX + 2 * lane;
    const float* const lb = lring + ly * TX + 2 * lane;

    float2 q[RY][Q];  // centre values of the last 2R+1 planes: plane zb-R+k in slot k mod Q
    // ---- warm-up: planes zb-R .. zb+R-1 (iterations 0 .. 2R-1) ----
#pragma unroll
    for (int k = 0; k < 2 * R; ++k) {
        const int s = k % SU;
        mbar_wait(&B.fullU[s], (phU >> s) & 1u);
        phU ^= 1u << s;
#pragma unroll
        for (int i = 0; i < RY; ++i) q[i][k] = *reinterpret_cast<const float2*>(cb + s * STR + i * TXP);
        mbar_arrive(&B.emptyU[s]);
    }
    // ---- iteration k brings plane zb-R+k (stage k mod SU) and outputs plane zb+k-2R (the item's
    // output k-2R: L stage (k-2R) mod SL, streams stage (k-2R) mod SP) ----
    for (int kb = 2 * R; kb < niter; kb += Q) {
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            const int k = kb + j;
            if constexpr (!FAST) {
                if (k >= niter) break;
            }
            const int s = (2 * R + j) % SU;  // (kb - 2R is a multiple of Q, and SU | Q)
            const int qs = (2 * R + j) % Q;  // queue slot of the newest plane
            const int qc = (R + j) % Q;      // queue slot of the output plane
            const int sl = j % SL, sp = j % SP;
            mbar_wait(&B.fullU[s], (phU >> s) & 1u);
            phU ^= 1u << s;
#pragma unroll
            for (int i = 0; i < RY; ++i) q[i][qs] = *reinterpret_cast<const float2*>(cb + s * STR + i * TXP);
            mbar_arrive(&B.emptyU[s]);
            const int z = zb + k - 2 * R;
            mbar_wait(&B.fullL[sl], (phL >> sl) & 1u);
            phL ^= 1u << sl;
            float2 L[RY];
#pragma unroll
            for (int i = 0; i < RY; ++i) L[i] = *reinterpret_cast<const float2*>(lb + sl * PT + i * TX);
            mbar_arrive(&B.emptyL[sl]);
#pragma unroll
            for (int jj = 1; jj <= R; ++jj)
#pragma unroll
                for (int i = 0; i < RY; ++i)
                    L[i] = fma2(f2(A.c.C[0][jj], A.c.C[0][jj]), add2(q[i][(qc + Q - jj) % Q], q[i][(qc + jj) % Q]),
                                L[i]);
            mbar_wait(&B.fullP[sp], (phP >> sp) & 1u);
            phP ^= 1u << sp;
            const bool use_a = pmeta[4 * sp] != 0;  // written by the streams producer before its arrive
            float2 res[RY];
#pragma unroll
            for (int i = 0; i < RY; ++i) {
                // t = 2u - u^{n-1} (2u exact: one rounding), w = fma(b, L, t), u^{n+1} = fma(a, w, (1-a) u^{n-1})
                const float* pr = pb + sp * C::PSTAGE_FLOATS + i * TX;
                const float2 um = *reinterpret_cast<const float2*>(pr);
                const float2 bb = *reinterpret_cast<const float2*>(pr + PT);
                const float2 aa = use_a ? *reinterpret_cast<const float2*>(pr + 2 * PT) : one;
                const float2 uc = q[i][qc];
                const float2 t = fma2(two, uc, f2(-um.x, -um.y));
                const float2 wv = fma2(bb, L[i], t);
                const float2 rr = mul2(add2(one, f2(-aa.x, -aa.y)), um);
                res[i] = fma2(aa, wv, rr);
            }
            mbar_arrive(&B.emptyP[sp]);
            float* outp = ubuf + o;
            if constexpr (!FAST) {
                // injection: u^{n+1}[c] = fma(s, q[n][src], u^{n+1}[c]) over the corner's
                // sources in CSR order, by the thread that owns the corner, before the store
                const int2 tp = A.tpsc ? A.tpsc[(int64_t)tile * nz + z] : make_int2(0, 0);
                for (int e = tp.x; e < tp.x + tp.y; ++e) {
                    const int4 en = A.tpe[e];
                    const int yl = en.x >> 6, xl = en.x & 63;
#pragma unroll
                    for (int i = 0; i < RY; ++i) {
                        if (yl != ly + i || (xl >> 1) != lane) continue;
                        float vv = (xl & 1) ? res[i].y : res[i].x;
                        const float* qn = A.wavelet + step_n * A.ns;
                        for (int kk = en.y; kk < en.z; ++kk) vv = __fmaf_rn(A.inj_s[kk], qn[A.inj_src[kk]], vv);
                        if (xl & 1) res[i].y = vv; else res[i].x = vv;
                    }
                }
            }
            auto store_rows = [&](float* dst) {
#pragma unroll
                for (int i = 0; i < RY; ++i) {
                    float* d = dst + i * pitch;
                    if (FAST || (ok_a[i] && ok_b[i])) {
                        *reinterpret_cast<float2*>(d) = res[i];  // 8-B aligned: x0 % 64 == 0, pitch % 32 == 0
                    } else if (ok_a[i]) {
                        d[0] = res[i].x;
                    }
                }
            };
            store_rows(outp);
            if constexpr (TEAM && !FAST) {
                // fused exchange: boundary planes also go into the neighbours' halos (a plane of a thin
                // slab can be both a low and a high boundary plane)
                if (A.lo && z < R) store_rows(A.lo + A.lo_off + o);
                if (A.hi && z >= nz - R) store_rows(A.hi + A.hi_off + o - (int64_t)(nz - R) * plane);
            }
            o = opaque(o + plane);
        }
    }
}

template <class C, bool TEAM>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB)
    hstream_kernel(const __grid_constant__ StreamMaps M, const __grid_constant__ StreamArgs A) {
    constexpr int R = C::R, TX = C::TX, TY = C::TY, RP = C::RP, SU = C::SU, SP = C::SP, SL = C::SL;
    extern __shared__ __align__(128) unsigned char smem[];
    float* ring = reinterpret_cast<float*>(smem);
    float* pring = reinterpret_cast<float*>(smem + C::U_BYTES);
    float* lring = reinterpret_cast<float*>(smem + C::U_BYTES + C::P_BYTES);
    HBars B;
    B.fullU = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    B.emptyU = B.fullU + SU;
    B.fullP = B.emptyU + SU;
    B.emptyP = B.fullP + SP;
    B.fullL = B.emptyP + SP;
    B.emptyL = B.fullL + SL;
    int* pmeta = reinterpret_cast<int*>(smem + C::META_OFF);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < SU; ++s) {
            mbar_init(&B.fullU[s], 1);
            mbar_init(&B.emptyU[s], C::N_A + C::N_B);  // every A and B thread arrives once per fill
        }
        for (int s = 0; s < SP; ++s) {
            mbar_init(&B.fullP[s], 1);
            mbar_init(&B.emptyP[s], C::N_B);
        }
        for (int s = 0; s < SL; ++s) {
            mbar_init(&B.fullL[s], C::N_A);
            mbar_init(&B.emptyL[s], C::N_B);
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
    if (warp == C::W_S + 3) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::PREG));  // idle warp of the service warpgroup
    } else if (warp == C::W_S + 2) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::PREG));
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
    } else if (warp >= C::W_S) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::PREG));
        // ---------------- producers (lane 0): warp W_S -- u^n plane tiles with halo into the u ring
        // (+ L2 prefetches of the output planes' streams and of the next item's first planes); warp
        // W_S+1 -- the u^{n-1}, b, a tiles of the output planes into the streams ring ----------------
        const bool is_u = warp == C::W_S;
        if (lane == 0) {
            if (is_u) {
                asm volatile("prefetch.tensormap [%0];" ::"l"(&M.u) : "memory");
            } else {
                asm volatile("prefetch.tensormap [%0];" ::"l"(&M.un) : "memory");
                asm volatile("prefetch.tensormap [%0];" ::"l"(&M.b) : "memory");
                if (A.a) asm volatile("prefetch.tensormap [%0];" ::"l"(&M.a) : "memory");
            }
            uint32_t pph = 0;  // per-stage phase bits of this producer's fills
            for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
                const int tile = item % ntiles;
                const int zb = (item / ntiles) * A.zc;
                const int ze = min(nz, zb + A.zc);
                const int x0 = (tile % A.ntx) * TX, y0 = (tile / A.ntx) * TY;
                const uint8_t* fl = A.flags + (int64_t)tile * nz;
                if (is_u) {
                    const int niter = ze - zb + 2 * R;
                    int s = 0;
                    for (int k = 0; k < niter; ++k) {
                        if (k == 2 * R) {
                            // the next item's warm-up planes into L2 (its start needs 2R planes at once)
                            const int nitem = item + gridDim.x;
                            if (nitem < A.nitems) {
                                const int ntile = nitem % ntiles;
                                const int nzb = (nitem / ntiles) * A.zc;
                                const int nx0 = (ntile % A.ntx) * TX, ny0 = (ntile / A.ntx) * TY;
                                for (int kk = 0; kk < 2 * R; ++kk)
                                    tma_prefetch_l2_3d(&M.u, nx0 - RP, ny0 - R, nzb + kk);
                            }
                        }
                        mbar_wait(&B.emptyU[s], ((pph >> s) & 1u) ^ 1u);
                        mbar_expect_tx(&B.fullU[s], C::STAGE_BYTES);
                        tma_load_3d(ring + s * C::STAGE_STRIDE_F, &M.u, &B.fullU[s], x0 - RP, y0 - R, zb + k);
                        pph ^= 1u << s;
                        s = s + 1 == SU ? 0 : s + 1;
                        const int z = zb + k - R;  // output ~R planes from now: its streams into L2
                        if (z >= zb && z < ze) {
                            tma_prefetch_l2_3d(&M.un, x0, y0, z + R);
                            tma_prefetch_l2_3d(&M.b, x0, y0, z);
                            if (A.a && fl[z]) tma_prefetch_l2_3d(&M.a, x0, y0, z);
                        }
                    }
                } else {
                    int sp = 0;
                    for (int z = zb; z < ze; ++z) {
                        const bool use_a = A.a && fl[z];
                        float* dst = pring + sp * C::PSTAGE_FLOATS;
                        mbar_wait(&B.emptyP[sp], ((pph >> sp) & 1u) ^ 1u);
                        // ordered for the consumers by this arrive (release) and their wait (acquire)
                        pmeta[4 * sp] = use_a;
                        mbar_expect_tx(&B.fullP[sp], (use_a ? 3 : 2) * C::PTILE_BYTES);
                        tma_load_3d(dst, &M.un, &B.fullP[sp], x0, y0, z + R);
                        tma_load_3d(dst + C::PTILE_FLOATS, &M.b, &B.fullP[sp], x0, y0, z);
                        if (use_a) tma_load_3d(dst + 2 * C::PTILE_FLOATS, &M.a, &B.fullP[sp], x0, y0, z);
                        pph ^= 1u << sp;
                        sp = sp + 1 == SP ? 0 : sp + 1;
                    }
                }
            }
        }
    } else if (warp >= C::W_B) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::BREG));
        // ---------------- B warps: z part + update ----------------
        const int ly = (warp - C::W_B) * C::RY;
        uint32_t phU = 0, phP = 0, phL = 0;  // per-stage phase bits of the consumed fills
        for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
            const int tile = item % ntiles;
            const int zb = (item / ntiles) * A.zc;
            const int ze = min(nz, zb + A.zc);
            const int x0 = (tile % A.ntx) * TX, y0 = (tile / A.ntx) * TY;
            const bool fast = x0 + TX <= g.nx && y0 + TY <= g.ny && ze - zb == A.zc && A.zc % C::Q == 0 &&
                              !(A.item_inj && A.item_inj[item]) && !(TEAM && (zb < R || ze > nz - R));
            if (fast)
                h_zpart<C, true, false>(A, ring, pring, lring, B, pmeta, tile, zb, ze, x0, y0, lane, ly, phU, phP, phL,
                                        step_n);
            else
                h_zpart<C, false, TEAM>(A, ring, pring, lring, B, pmeta, tile, zb, ze, x0, y0, lane, ly, phU, phP,
                                        phL, step_n);
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::AREG));
        // ---------------- A warps: in-plane part ----------------
        const int ly = warp * C::RY;
        uint32_t phU = 0, phL = 0;
        for (int item = blockIdx.x; item < A.nitems; item += gridDim.x) {
            const int zb = (item / ntiles) * A.zc;
            const int ze = min(nz, zb + A.zc);
            h_inplane<C>(A, ring, lring, B, zb, ze, lane, ly, phU, phL);
        }
    }
    if (A.ts0) {  // this CTA's end: every role done
        __syncthreads();
        if (tid == 0) atomicMax(A.ts1 + ts_slot, globaltimer_ns());
    }
}

namespace {

// Host side: the plan's tile geometry is the one of the matching stream_kernel configuration CS
// (the temporal-blocking kernel still runs CS on the same plan, flags and injection lists).
template <class HC, class CS>
cudaError_t setup_h(StreamPlan* p, const Geom& g) {
    static_assert(HC::R == CS::R && HC::TX == CS::TX && HC::TY == CS::TY, "shared plan geometry");
    p->smem = HC::SMEM;
    p->nthreads = HC::NTHREADS;
    p->TX = HC::TX;
    p->TY = HC::TY;
    p->zq = HC::Q;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(hstream_kernel<HC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)HC::SMEM)))
        return e;
    if ((e = cudaFuncSetAttribute(hstream_kernel<HC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)HC::SMEM)))
        return e;
    if ((e = cudaFuncSetAttribute(tb_kernel<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CS::SMEM)))
        return e;
    int occ = 0, occ_t = 0, occ_tb = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hstream_kernel<HC, false>, HC::NTHREADS, HC::SMEM)))
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, hstream_kernel<HC, true>, HC::NTHREADS, HC::SMEM)))
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_tb, tb_kernel<CS>, CS::NTHREADS, CS::SMEM))) return e;
    occ = std::min(occ, std::min(occ_t, occ_tb));  // the TB kernel shares the grid (all CTAs resident)
    if (occ < 1) return cudaErrorNotSupported;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    p->grid = sms * occ;
    return cudaSuccess;
}

template <class HC>
void fill_args_h(StreamArgs& A, StreamPlan* p, const Geom& g, const Coefs& c, const float* ucur, float* unext,
                 const float* b, const float* a, const Sparse& sp, int inj_set, const int64_t* d_base, int step_i) {
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
}

template <class HC>
cudaError_t launch_h(StreamPlan* p, const Geom& g, const Coefs& c, int parity_cur, const float* ucur, float* unext,
                     const float* b, const float* a, const Halo& halo, int parity_next, const Sparse& sp,
                     const int64_t* d_base, int step_i, cudaStream_t s) {
    // (teams: the flags are raised by stream_kernel's boundary-first signalling, which this kernel lacks)
    if (halo.lo[parity_next] || halo.hi[parity_next]) return cudaErrorNotSupported;
    StreamArgs A;
    fill_args_h<HC>(A, p, g, c, ucur, unext, b, a, sp, 0, d_base, step_i);
    A.lo = halo.lo[parity_next];
    A.lo_off = halo.lo_off;
    A.hi = halo.hi[parity_next];
    A.hi_off = halo.hi_off;
    if (A.lo || A.hi)
        hstream_kernel<HC, true><<<p->grid, HC::NTHREADS, HC::SMEM, s>>>(p->maps[parity_cur], A);
    else
        hstream_kernel<HC, false><<<p->grid, HC::NTHREADS, HC::SMEM, s>>>(p->maps[parity_cur], A);
    return cudaGetLastError();
}

// One step on explicit buffers (FWI history ring / adjoint, NEXT-3); maps cached per (buffer, box kind).
template <class HC>
cudaError_t launch_bufs_h(StreamPlan* p, const Geom& g, const Coefs& c, const float* ucur, const float* uprev,
                          float* unext, const float* b, const float* a, const Sparse& sp, int inj_set,
                          const int64_t* d_base, int step_i, cudaStream_t s) {
    StreamMaps M;
    cudaError_t e;
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
    if ((e = cached(&M.u, ucur, g.nz + 2 * g.R, HC::TXP, HC::TYP, 1))) return e;
    if ((e = cached(&M.un, uprev, g.nz + 2 * g.R, HC::TX, HC::TY, 2))) return e;
    if ((e = cached(&M.b, b, g.nz, HC::TX, HC::TY, 3))) return e;
    if ((e = cached(&M.a, a ? a : b, g.nz, HC::TX, HC::TY, 4))) return e;
    StreamArgs A;
    fill_args_h<HC>(A, p, g, c, ucur, unext, b, a, sp, inj_set, d_base, step_i);
    hstream_kernel<HC, false><<<p->grid, HC::NTHREADS, HC::SMEM, s>>>(M, A);
    return cudaGetLastError();
}

template <class HC, class CS>
const StreamOps* ops_of_h() {
    static const StreamOps o{setup_h<HC, CS>, make_maps<CS>, launch_h<HC>, launch_bufs_h<HC>, launch_tb<CS>, nullptr};
    return &o;
}

// configuration table: (R, SU = u^n ring, SP = streams ring, SL = L_xy ring), all dividing Q = 24;
// the tile geometry (64 x 16) is shared with C6..C8 (aw_stream.cuh)
using H6 = HCfg<6, 12, 4, 3>;
using H7 = HCfg<7, 12, 4, 3>;
using H8 = HCfg<8, 12, 4, 3>;

}  // namespace

}  // namespace aw
