// aw_internal.h -- private declarations of libaw (host runtime <-> device kernels).
// Not part of the ABI; see include/aw.h for the public boundary.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>

#define AW_MAXR 8          // space order <= 16
#define AW_PITCH_ALIGN 32  // x pitch in floats (128 B rows: coalescing + TMA 16-B strides)

namespace aw {

// Development knobs (environment variables for A/B measurements: AW_STREAM_VARIANT, AW_STREAM_ZC,
// AW_TB_Z, AW_TB_LEAD, AW_NO_FUSE).  Read only in development builds (AW_DEV_BUILD=1 ->
// -DAW_DEV_KNOBS); the product library ignores them.
inline const char* dev_knob(const char* name) {
#ifdef AW_DEV_KNOBS
    return getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

// Axis coefficients of the star Laplacian, fp32:
// C[d][j] = fl32(c_j / h_d^2), C0 = fl32(sum_d c_0 / h_d^2).
struct Coefs {
    float C[3][AW_MAXR + 1];
    float C0;
};

// Geometry of one rank's device arrays.  Wavefield buffers hold planes
// [-R, nz+R) of axis 0 (halo planes: zero at the global ends, the neighbour's
// boundary planes inside a team); model/coefficient arrays hold [0, nz).
// 2D grids use ny = 1 (axes (z, x)).
struct Geom {
    int ndim;
    int R;
    int nz, ny, nx;      // owned planes, axis-1 points (1 in 2D), x points
    int64_t pitch;       // floats per x row
    int64_t plane;       // ny * pitch
};

// Peer targets for the fused halo stores (team mode); null when absent.
struct DevCtl;
struct Halo {
    float* lo[2];   // rank-1's buffers (base = its plane -R); my planes [0,R) go to its planes [nz_lo, nz_lo+R)
    float* hi[2];   // rank+1's buffers; my planes [nz-R, nz) go to its planes [-R, 0)
    int64_t lo_off; // element offset of rank-1's plane nz_lo relative to its base
    int64_t hi_off; // element offset of rank+1's plane -R relative to its base (= 0)
    // boundary-first signalling from inside the 3D streaming kernel: the neighbours' flag words for
    // me (peer memory) and my control block (epoch, step base, boundary-item counter)
    unsigned long long* flag_lo;
    unsigned long long* flag_hi;
    DevCtl* ctl;
};

// Device control words of one handle (one small allocation).  base = global index of the step a
// launch calls step 0 (kernels take a step offset i, so CUDA graphs replay unchanged); epoch =
// team epoch (bumped by reset / set_wavefield); team_flags are written by the neighbours (exported
// through cudaIpc) with levels encoded (epoch << 32) + level + 1.
struct DevCtl {
    int64_t base;
    unsigned long long epoch;
    unsigned long long wait_ns;  // team: device time spent waiting for halo planes (last run)
    unsigned long long nwait;    // team: waits that blocked (last run)
    unsigned flag;               // non-finite result / invalid model
    unsigned bcount;             // team streaming kernel: boundary items completed in the current launch
    unsigned model_bad;          // aw_set_model: epoch of the last call whose model failed validation
    unsigned pad_[5];
    unsigned long long team_flags[2];  // [0]: from rank-1, [1]: from rank+1
};

// Sparse (receivers + injection CSR) device view
struct Sparse {
    // receivers owned by this rank
    int nrl;                 // number of owned receivers
    int nr;                  // global receiver count (trace row length)
    const int* rec_id;       // [nrl] global receiver index
    const int64_t* rec_off;  // [nrl][nc] element offset into a wavefield buffer (-1 = skipped)
    const float* rec_w;      // [nrl][nc]
    float* traces;           // [nt_max][nr]
    // injection CSR by corner (ascending global linear index)
    int nuc;                 // unique owned corners
    int ns;                  // global source count (wavelet row length)
    const int64_t* inj_off;  // [nuc] element offset into a wavefield buffer
    const int* inj_plane;    // [nuc] local plane index (for halo propagation)
    const int* inj_ptr;      // [nuc+1]
    const int* inj_src;      // [nent]
    const float* inj_s;      // [nent] fp32 scales
    int nent;                // injection entries (inj_ptr[nuc])
    const float* wavelet;    // [nt_max][ns]
    int nc;                  // 2^ndim
};

// ---- kernels / launchers (aw_kernels.cu) ----
cudaError_t launch_coeffs(const float* m, const float* eta, float* b, float* a, int64_t n, double dt,
                          cudaStream_t s);
// invalid value (m <= 0 or non-finite, eta < 0 or non-finite) -> *bad = epoch
cudaError_t launch_validate_model(const float* m, const float* eta, const Geom& g, unsigned* bad, unsigned epoch,
                                  cudaStream_t s);
// device inputs (C-order, nx contiguous, nz*ny rows): copy into the padded model layout (padding 0) and
// validate in one pass
cudaError_t launch_stage_model(const float* m_src, const float* eta_src, float* m_dst, float* eta_dst, const Geom& g,
                               unsigned* bad, unsigned epoch, cudaStream_t s);
cudaError_t launch_source_scales(const float* m, const float* eta, const int64_t* moff, const double* w64,
                                 float* s_out, int nent, double dt, cudaStream_t s);
// uprev = u^{n-1}: unext itself for the in-place two-buffer time loop, or another buffer
// (FWI history ring, NEXT-3)
cudaError_t launch_stencil_v1(const Geom& g, const Coefs& c, const float* ucur, const float* uprev, float* unext,
                              const float* b, const float* a, const Halo& halo, int parity_next,
                              cudaStream_t s);
cudaError_t launch_sparse_step(const Geom& g, const Sparse& sp, const float* ucur, float* unext,
                               const int64_t* d_base, int i, const Halo& halo, int parity_next,
                               cudaStream_t s);
cudaError_t launch_advance(int64_t* d_base, int64_t by, cudaStream_t s);
cudaError_t launch_run_init(DevCtl* ctl, int64_t base, cudaStream_t s);
cudaError_t launch_check_finite(const Geom& g, const float* u, const float* traces, int64_t t0,
                                int64_t t1, int nr, unsigned* flag, cudaStream_t s);
cudaError_t launch_team_wait(DevCtl* ctl, bool has_lo, bool has_hi, int i, cudaStream_t s);
cudaError_t launch_team_signal(unsigned long long* peer_lo_flag, unsigned long long* peer_hi_flag,
                               const DevCtl* ctl, int i, cudaStream_t s);
cudaError_t launch_team_raise(unsigned long long* f0, unsigned long long* f1, unsigned long long v,
                              cudaStream_t s);

// 2.5D z-streaming kernel (aw_stream.cu); returns cudaErrorNotSupported when
// the configuration has no streaming specialisation.
struct StreamPlan;
cudaError_t stream_prepare(const Geom& g, const float* const* ubuf, const float* b, const float* a,
                           StreamPlan** plan, cudaStream_t s);
cudaError_t stream_refresh(StreamPlan* p, const Geom& g, const float* const* ubuf, const float* b, const float* a,
                           cudaStream_t s);
int stream_eta_tiles_pct(const StreamPlan* p);
void stream_release(StreamPlan* p);
size_t stream_plan_bytes(const StreamPlan* p);  // device bytes the plan holds (NULL -> 0)
// appends every plan value a captured launch uses (tensor maps, tables, timestamps) to *sig
void stream_plan_signature(const StreamPlan* p, std::string* sig);
// AW_OPT_TIMING = 2: point the streaming kernel at per-launch timestamp arrays (null = off)
void stream_set_timestamps(StreamPlan* p, unsigned long long* ts0, unsigned long long* ts1, int cap);
cudaError_t launch_stencil_stream(StreamPlan* p, const Geom& g, const Coefs& c, int parity_cur,
                                  const float* ucur, float* unext, const float* b, const float* a,
                                  const Halo& halo, int parity_next, const Sparse& sp, const int64_t* d_base,
                                  int step_i, cudaStream_t s);
// injection lists per tile-plane; set 0 = the sources, set 1 = the FWI adjoint sources (receivers)
cudaError_t stream_set_injection(StreamPlan* p, const Geom& g, int64_t z0, const int64_t* corner_lin, const int* ptr,
                                 int nuc, cudaStream_t s, int set = 0);
// One step on explicit buffers (u^n = ucur, u^{n-1} = uprev, u^{n+1} -> unext; single slab, no team):
// the tensor maps are encoded for these buffers at launch.  inj_set selects the injection lists.
cudaError_t launch_stencil_stream_bufs(StreamPlan* p, const Geom& g, const Coefs& c, const float* ucur,
                                       const float* uprev, float* unext, const float* b, const float* a,
                                       const Sparse& sp, int inj_set, const int64_t* d_base, int step_i,
                                       cudaStream_t s);
// NEXT-1 temporal blocking: one launch advances two steps (u^n = x, u^{n-1} = y) -> u^{n+1} in v
// (a third buffer), u^{n+2} over y.  Single slab.  stream_tb_prepare sizes the completion array.
cudaError_t stream_tb_prepare(StreamPlan* p, const Geom& g, int Z);
cudaError_t launch_stencil_tb(StreamPlan* p, const Geom& g, const Coefs& c, const float* x, float* y, float* v,
                              const float* b, const float* a, const Sparse& sp, const int64_t* d_base, int step_i,
                              cudaStream_t s);
// re-encode the per-parity maps after the caller permuted its wavefield buffers
cudaError_t stream_remap(StreamPlan* p, const Geom& g, const float* const* ubuf, const float* b, const float* a);
// Small grids: the resident multi-step kernel (single slab).  stream_resident_ready: the plan's
// configuration has it and all its CTAs fit on the device at once.  stream_set_receivers: the owned
// receivers grouped by the work item holding their base corner (rec_off: [nrl][nc] element offsets
// into a wavefield buffer, as in Sparse; synchronises s).  stream_resident_begin: reset the per-item
// step counters (once per run, before its first resident launch).
bool stream_resident_ready(const StreamPlan* p);
cudaError_t stream_set_receivers(StreamPlan* p, const Geom& g, const int64_t* rec_off, int nrl, int nc,
                                 cudaStream_t s);
cudaError_t stream_resident_begin(StreamPlan* p, cudaStream_t s);
cudaError_t launch_stencil_resident(StreamPlan* p, const Geom& g, const Coefs& c, int cur0, float* const* buf,
                                    const float* b, const float* a, const Sparse& sp, const int64_t* d_base,
                                    int step0, int nsteps, cudaStream_t s);

// 2D tiled kernel (aw_stencil2d.cu): one CTA per 64x32 tile, TMA halo box, packed fp32 on column
// pairs; explicit buffers (in place when uprev == unext).  Sparse work stays in launch_sparse_step.
struct Tile2DPlan;
cudaError_t tile2d_prepare(const Geom& g, Tile2DPlan** plan);
void tile2d_release(Tile2DPlan* p);
cudaError_t launch_stencil_tile2d(Tile2DPlan* p, const Geom& g, const Coefs& c, const float* ucur, const float* uprev,
                                  float* unext, const float* b, const float* a, cudaStream_t s);

// Small 2D grids (aw_resident2d.cu): every step of a run in one launch of one CTA holding the whole grid in
// shared memory (single slab).  resident2d_fits: the two wavefield levels and the sparse tables fit (b, a
// are staged too when they fit, else read from global).  u_cur/u_prev: the buffers holding u^n / u^{n-1} at entry; both
// levels are written back at the end (the newest in u_cur when nsteps is even, else in u_prev).
bool resident2d_fits(const Geom& g, const Sparse& sp, bool damp);
cudaError_t launch_stencil_resident2d(const Geom& g, const Coefs& c, float* u_cur, float* u_prev, const float* b,
                                      const float* a, const Sparse& sp, const int64_t* d_base, int step0, int nsteps,
                                      cudaStream_t s);

// ---- NEXT-3 FWI kernels (aw_fwi.cu) ----
// G += psi * D,  D = fl32(fl32(u1 - 2 u0) + um1), over the owned planes (wavefield layout inputs,
// model layout G)
cudaError_t launch_fwi_imaging(const Geom& g, const float* psi, const float* u1, const float* u0, const float* um1,
                               float* G, cudaStream_t s);
// res[n][r] = fl32(rec - d_obs); wadj[nt-1-n][r] = res[n][r]; *J = 0.5 sum res^2 (fp64, fixed order)
cudaError_t launch_fwi_residual(const float* rec, const float* dobs, float* res, float* wadj, int nt, int nr,
                                double* J, cudaStream_t s);
// grad = fl32(-(double)G / dt^2) in place (model layout, padding stays 0)
cudaError_t launch_fwi_finalize(const Geom& g, float* G, double dt, cudaStream_t s);
// acc = fl32(acc + G) (model layout; NEXT-4 multi-shot gradient sums)
cudaError_t launch_fwi_accumulate(const Geom& g, float* acc, const float* G, cudaStream_t s);

}  // namespace aw
