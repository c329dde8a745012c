/*
 * aw.h -- acoustic wave propagation on B200 (sm_100a): the C-ABI boundary of
 * the hot path named by BASELINE.json:5 (north star) for arXiv 1906.10811.
 *
 *   m * u_tt - Lap(u) + eta * u_t = q          on a structured 2D/3D grid
 *
 * discretised as a space-order-k star stencil ("FD shortcuts",
 * :741 "u.dx2 + u.dy2", :746 order = space order) with the explicit update
 * obtained from solve(eq, u.forward), divisions hoisted
 * into precomputed coefficients (PAPER.md:788-826 [Evaluation > CUDA results]),
 * zero-initialised halos, time levels rotated
 * t_k = (time+k) mod n, and sparse Ricker-source injection and
 * receiver interpolation inside the time loop -- the part OPS could not
 * offload.  The exact per-point fp32 operation sequence is
 * SURVEY.md §8(c) steps 1-6 (the "canonical" order), restated in DESIGN.md §2.
 *
 * Conventions
 *  - Arrays are C-contiguous with shape (n0, n1[, n2]); axis ndim-1 is
 *    contiguous ("x"), axis 0 is the slowest ("z"), the streaming axis and the
 *    slab (multi-GPU) axis.  Coordinates are given in the same axis order.
 *  - Spacing h_d = extent_d / (n_d - 1); origin defaults to 0.
 *  - Array arguments marked [H|D] may be host or device pointers (detected
 *    with cudaPointerGetAttributes; device pointers must be on the grid's
 *    device).  [H] = host only.  All inputs are BORROWED for the duration of
 *    the call and copied; outputs are caller-allocated with the sizes stated.
 *  - Every call returns aw_status; aw_last_error() gives a thread-local text.
 *    Validation errors (AW_EINVAL / AW_EUNSUPPORTED) leave the handle
 *    unchanged.  AW_ECUDA is sticky: the handle is poisoned and every later
 *    call except aw_grid_destroy returns AW_ESTATE.
 *  - Calls on one handle are not thread-safe (concurrent reads are
 *    safe, writes require external exclusivity).  Calls are stream-ordered on
 *    the handle's stream (aw_dist.stream when given: the library's work waits
 *    for the work already queued on it, and later work queued on it waits for
 *    the library's): host inputs are consumed and host outputs are complete
 *    when a call returns; device-pointer inputs and outputs are read and
 *    written in that stream order (aw_add_sources, aw_add_receivers, aw_reset
 *    and aw_read_receivers with device pointers may return before their
 *    copies ran).  aw_set_model and aw_run return after their work
 *    completed (their status depends on it).
 *  - There is no CPU fallback: without a usable CUDA device aw_grid_create
 *    returns AW_ECUDA.
 */
#ifndef AW_H
#define AW_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define AW_ABI_VERSION 2

typedef struct aw_grid aw_grid; /* opaque; created by aw_grid_create, freed by aw_grid_destroy */

typedef enum {
    AW_OK = 0,
    AW_EINVAL = -1,        /* bad argument (shape, order, coordinate outside the grid, ...) */
    AW_ENOMEM = -2,        /* device or host allocation failed */
    AW_ECUDA = -3,         /* CUDA runtime/launch error (sticky) */
    AW_ENCCL = -4,         /* reserved (peer-memory team setup failure uses AW_ECUDA) */
    AW_ESTATE = -5,        /* call not valid in the current state (poisoned handle, no model, ...) */
    AW_EUNSUPPORTED = -6,  /* valid request the library does not implement (e.g. ndim 1) */
    AW_ENONFINITE = -7     /* NaN/Inf appeared in the receivers or the final wavefield */
} aw_status;

/* layout of array arguments for multi-rank handles */
enum { AW_GLOBAL = 0 /* array covers the whole global grid */, AW_LOCAL = 1 /* this rank's slab only */ };

/* stencil kernel selection (aw_set_option AW_OPT_KERNEL) */
enum { AW_KERNEL_AUTO = 0 /* STREAM in 3D, TILE2D in 2D */, AW_KERNEL_V1 = 1 /* one thread per point,
       reference-grade */, AW_KERNEL_STREAM = 2 /* 2.5D z-streaming TMA kernel (3D) */,
       AW_KERNEL_TILE2D = 3 /* TMA-tiled 2D kernel (reported by aw_last_run_stats; AUTO selects it) */ };

/* options */
enum {
    AW_OPT_KERNEL = 1,      /* value: AW_KERNEL_* */
    AW_OPT_TIMING = 2,      /* value 1: time every stencil launch with CUDA events (direct launches, no graphs);
                               value 2: the 3D streaming kernel stamps its first-CTA start and last-CTA end
                               per launch with the device clock (%globaltimer), CUDA graphs kept -- the
                               production path; aw_run_stats.ms_stencil / n_stencil report them */
    AW_OPT_GRAPH_STEPS = 3, /* value G >= 0: steps per captured CUDA graph (0 = no graphs) */
    AW_OPT_CHECK_FINITE = 4, /* value 0/1 (default 1): aw_run checks traces + final field */
    AW_OPT_CHECKPOINT_STEPS = 5, /* value K >= 0: aw_fwi_gradient segment length (0 = auto, see there) */
    AW_OPT_TEMPORAL = 6, /* value 0/1 (default 0): temporal blocking (NEXT-1) -- aw_run advances two steps per
                           launch with the streaming kernel (3D, single slab; a third wavefield buffer is
                           allocated); results are bit-identical to one step per launch.  Off by default:
                           measured 6-45 % slower than one step per launch on B200 (NEXT-1) */
    AW_OPT_FWI_ACCUMULATE = 7, /* value 0/1 (default 0): NEXT-4 multi-shot -- with 1, aw_fwi_gradient writes the
                           fp32 sum (in call order) of the gradients of all calls since the option was last
                           set; setting it (either value) clears the sum.  J is still per call. */
    AW_OPT_RESIDENT = 8 /* value AW_RESIDENT_* (default AUTO): small grids -- aw_run advances all nt steps in
                           ONE launch of the resident streaming kernel (3D, single slab, streaming kernel,
                           not with temporal blocking or AW_OPT_TIMING=1): every CTA keeps its work items
                           for all steps and an item starts step n+1 once its 27 neighbouring items
                           finished step n (no grid barrier, no launch gaps).  Same per-point sequence,
                           bit-identical results.  AUTO uses it up to 8 Mi points (L2-resident grids).
                           2D (AUTO kernel, single slab): grids whose two wavefield levels fit one SM's
                           shared memory (~25 K points, e.g. C1 = 101^2) run all nt steps in ONE launch of
                           one CTA holding the grid in shared memory (AUTO and ON; also with
                           AW_OPT_TIMING=1).  Same per-point sequence, bit-identical results. */
};
enum { AW_RESIDENT_OFF = 0, AW_RESIDENT_ON = 1 /* whenever supported */, AW_RESIDENT_AUTO = 2 };

/* aw_dist.flags */
enum { AW_DIST_WORKSPACE = 1 /* the caller provides the device memory of the grid's arrays with
                               aw_bind_workspace: aw_grid_create allocates none of them */ };

/* multi-rank description: one process (or virtual rank) per slab of axis 0 */
typedef struct {
    int rank;       /* 0 <= rank < world */
    int world;      /* number of slabs along axis 0 (1 = single GPU) */
    int device;     /* CUDA device ordinal to use (-1 = current device) */
    void* stream;   /* cudaStream_t to launch on (NULL = library-owned stream) */
    unsigned flags; /* AW_DIST_* bits (0 = library-allocated arrays) */
} aw_dist;

/*
 * aw_grid_create -- allocate a zero-initialised grid handle (PAPER.md:455-491
 * zero padding).
 *   ndim         2 or 3 (1 -> AW_EUNSUPPORTED)
 *   shape[ndim]  global points per axis; n_d >= k/2 + 1
 *   extent[ndim] physical length per axis, > 0 (h_d = extent_d/(n_d-1))
 *   origin[ndim] physical coordinate of node 0 (NULL = zeros)
 *   space_order  k: even, 2..16
 *   dist         NULL = one slab on the current device; otherwise the slab
 *                [z0, z0+nz) of axis 0 owned by dist->rank (nearly equal split)
 * Device memory: 2 wavefield levels with k/2 halo planes on each side of
 * axis 0 plus b, a, m, eta per owned point (fp32, x pitch padded to 128 B),
 * zero-filled ("zero-filled buffer ... allocation failure
 * surfaced as resource error" -> AW_ENOMEM).  With dist->flags &
 * AW_DIST_WORKSPACE none of these arrays is allocated: the caller binds the
 * memory with aw_bind_workspace before any call that touches them (those calls
 * return AW_ESTATE until then).
 */
aw_status aw_grid_create(aw_grid** out, int ndim, const int64_t* shape, const double* extent,
                         const double* origin, int space_order, const aw_dist* dist);

/* NULL-safe; never fails.  Must not be called while another rank of a team still runs. */
void aw_grid_destroy(aw_grid* g);

/*
 * aw_workspace_bytes -- bytes of device memory the grid's arrays need in a
 * caller-owned workspace (the north star's "PyTorch only for device memory",
 * BASELINE.json:5): the two wavefield levels, m, eta, b, a
 * (the dense part, fixed by the grid) plus the sparse arenas of the sources
 * and receivers added so far (call after aw_add_sources/aw_add_receivers to
 * include them).  0 for a NULL handle.
 *
 * aw_bind_workspace -- hand the library `bytes` bytes of device memory at
 * dev_ptr (on the grid's device, 256-B aligned, e.g. a torch uint8 tensor).
 * The dense arrays move into [0, dense) (contents copied if they already held
 * data; the library's own allocation is freed), and the rest of the workspace
 * holds the source arena, then the receiver arena; an arena that outgrows its
 * slot later falls back to a library allocation (reported in
 * aw_run_stats.lib_device_bytes).  The workspace is BORROWED: it must stay
 * allocated and untouched until aw_grid_destroy or the next bind.  Must be
 * called before a team connects (peers hold the wavefield addresses).
 * Errors: AW_EINVAL (NULL/unaligned pointer, bytes < the dense part, memory on
 * another device), AW_ESTATE (team already connected).  The handle is
 * unchanged on error.
 */
size_t aw_workspace_bytes(const aw_grid* g);
aw_status aw_bind_workspace(aw_grid* g, void* dev_ptr, size_t bytes);

/* This handle's slab of axis 0: planes [*z0, *z0 + *nz) (nearly
 * equal slabs of the slowest axis; "MPI ... domain partitioning"
 * as an OPS capability).  Either output may be NULL. */
aw_status aw_local_extent(const aw_grid* g, int64_t* z0, int64_t* nz);

/*
 * aw_set_model -- slowness squared m = 1/v^2 (> 0, finite) and damping eta
 * (>= 0, finite; NULL = 0 everywhere), fp32 [H|D], shape = global grid
 * (AW_GLOBAL) or this rank's slab (AW_LOCAL).  The dt-dependent coefficients
 * b = fl32(dt^2/m), a = fl32(m/(m + eta dt/2)) (the paper's
 * division hoisting PAPER.md:788-792) are (re)computed on the device at the
 * next aw_run.  Invalid values -> AW_EINVAL (checked on the device, on a
 * staged copy: the previous model stays in force, strong guarantee).
 */
aw_status aw_set_model(aw_grid* g, const float* m, const float* damp, int layout);

/*
 * aw_add_sources -- replace the point sources.
 *   coords [ns][ndim] fp64 [H]: physical coordinates inside the closed grid box
 *   wavelet [nt_max][ns] fp32 [H|D]: row n = source amplitudes q at step n
 * Injection at step n adds s * q[n][s] to u^{n+1} at each of the 2^ndim
 * multilinear corners, s = fl32(w*dt^2/(m_c + eta_c dt/2)),
 * corners ascending then sources ascending (Q11).  ns = 0 removes all sources.
 * A coordinate outside [o, o+(n-1)h] on any axis -> AW_EINVAL.
 */
aw_status aw_add_sources(aw_grid* g, int ns, const double* coords, int nt_max, const float* wavelet);

/*
 * aw_add_receivers -- replace the receivers; traces are recorded from u^n
 * (before step n) for steps 0..nt_max-1 (Q8).  coords [nr][ndim] fp64 [H].
 * Corner indices and fp32 weights are computed on the host in fp64 exactly as
 * SURVEY §8(c).4 (bit-exact contract).  Clears previously recorded traces.
 */
aw_status aw_add_receivers(aw_grid* g, int nr, const double* coords, int nt_max);

/*
 * aw_set_wavefield -- initial conditions / restart: u_cur = u^{n}, u_prev =
 * u^{n-1} (fp32 [H|D], NULL = zeros) for the current step counter (the two
 * levels of the leapfrog; SPEC.md:352/:639 restart ==
 * continuous run).  In a team the call is collective: every rank calls it
 * with the same layout after all ranks' previous aw_run returned (a barrier);
 * with AW_LOCAL the halo planes are exchanged at the next aw_run.
 */
aw_status aw_set_wavefield(aw_grid* g, const float* u_cur, const float* u_prev, int layout);

/*
 * aw_run -- advance nt >= 0 steps from the current state with time step dt
 * (> 0, finite).  dt is fixed by the first run until aw_reset (a different
 * dt -> AW_EINVAL).  Needs a model (AW_ESTATE otherwise); the wavelet and
 * trace buffers must cover steps_done + nt (AW_EINVAL otherwise).  For a team
 * (world > 1) every rank calls aw_run collectively.  Returns after the work
 * completed on the handle's stream; AW_ENONFINITE if NaN/Inf appeared.
 */
aw_status aw_run(aw_grid* g, int nt, double dt);

/* Zero both wavefield levels and the traces, reset the step counter and dt:
 * back to the zero-filled state of creation (PAPER.md:455-491 zero padding,
 * SPEC.md:68-76; SURVEY §8(c).5 "u^0 = u^-1 = 0").  In a team the call is
 * collective and needs a barrier before it, as aw_set_wavefield. */
aw_status aw_reset(aw_grid* g);

/* Number of steps taken since create/reset. */
int64_t aw_steps_done(const aw_grid* g);

/*
 * aw_read_wavefield -- copy u^{n} (which = 0, the newest level) or u^{n-1}
 * (which = 1) into out (fp32 [H|D], dense, global or local layout; a rank
 * asked for AW_GLOBAL writes only its own planes of the global array).  The
 * output of SURVEY §8(c).7 ("read_wavefield(0) = u^{n0+nt}"); the paper's
 * time-buffer rotation t_k = (time+k) mod n is internal.
 */
aw_status aw_read_wavefield(aw_grid* g, int which, float* out, int layout);

/*
 * aw_read_receivers -- traces [steps_done][nr] fp32 [H|D], row = step.
 * In a team each rank returns its owned receivers and zeros elsewhere; the
 * sum over ranks is the global trace set (disjoint supports, exact).
 */
aw_status aw_read_receivers(aw_grid* g, float* out);

/*
 * aw_debug_sparse -- test hook: for which = 0 (sources) / 1 (receivers), the
 * global row-major corner indices [n][2^ndim] (-1 = skipped corner) and the
 * fp32 weights (receivers) or source scales (sources; valid after a run).
 * [H] outputs.
 */
aw_status aw_debug_sparse(const aw_grid* g, int which, int64_t* corner_lin, float* w);

typedef struct {
    double ms_total;      /* wall time of the last aw_run on the stream (CUDA events) */
    double ms_stencil;    /* sum of stencil-kernel durations (AW_OPT_TIMING=1, else -1) */
    int64_t n_stencil;    /* stencil launches timed */
    int64_t launches;     /* kernels launched by the last aw_run (all kinds) */
    double gpts;          /* point updates / s of the last run (global points, this rank's time) */
    int64_t points;       /* owned points per step */
    int kernel;           /* AW_KERNEL_* actually used */
    int eta_tiles;        /* percent of stream tiles that read `a` (damping present) */
    int64_t launches_total; /* kernels launched by this handle since creation (all calls) */
    int64_t fwi_steps;    /* stencil steps of the last aw_fwi_gradient (forward + recompute + adjoint) */
    int fwi_checkpoint;   /* checkpoint segment length K used by the last aw_fwi_gradient */
    int64_t timed_launches; /* stencil launches timed by the last aw_run (AW_OPT_TIMING; a temporal-
                               blocking pass covers two of the n_stencil steps) */
    double ms_exchange;   /* team: time the last aw_run's boundary work waited for the neighbours' halo
                             planes (device clock, summed over steps of the per-step mean wait of the
                             waiting CTAs; 0 for a single slab) -- SURVEY §5 tracing row, §8(e) */
    int64_t exchange_waits; /* team: waits that found the neighbour's halo not yet delivered */
    int64_t lib_device_bytes; /* device bytes the library itself holds for this handle (cudaMalloc) */
    int64_t workspace_bytes;  /* bytes of the bound caller workspace (0 = none) */
    int32_t resident;         /* 1: the last aw_run used the resident multi-step kernel (AW_OPT_RESIDENT) */
} aw_run_stats;

aw_status aw_last_run_stats(const aw_grid* g, aw_run_stats* out);

aw_status aw_set_option(aw_grid* g, int option, int64_t value);

/* Leapfrog stability limit 2/(vmax sqrt(sum_d sum_j |c_j|/h_d^2)). */
double aw_critical_dt(int ndim, const double* spacing, int space_order, double vmax);

const char* aw_last_error(void);
int aw_abi_version(void);

/* ------------------------------------------------------------------------
 * Multi-slab teams: slabs along axis 0, per-step k/2-plane
 * halo exchange fused into the stencil kernel as direct stores into the
 * neighbours' halo planes over NVLink peer memory, with a device flag
 * handshake per step (no separate copy kernel, no host round trip).
 * ------------------------------------------------------------------------ */

/* Host-only: the slab [*z0, *z0 + *nz) of axis 0 that rank `rank` of `world`
 * owns for a grid of n0 planes (nearly equal split, the first n0 % world ranks
 * get one more plane).  AW_EINVAL if a slab would be thinner than k/2 = R
 * planes (the exchange reaches only the direct neighbours). */
aw_status aw_slab_partition(int64_t n0, int world, int rank, int R, int64_t* z0, int64_t* nz);

/* Bytes of the opaque export record of one rank (cudaIpc handles + offsets). */
size_t aw_team_export_size(void);
/* Write this rank's export record into out[aw_team_export_size()]. */
aw_status aw_team_export(aw_grid* g, void* out);
/* Connect to the neighbours from all ranks' records, concatenated in rank
 * order (world * aw_team_export_size() bytes, [H]).  Collective. */
aw_status aw_team_connect(aw_grid* g, const void* all_records);
/* Virtual ranks in one process (tests on one GPU): grids[r] has rank r. */
aw_status aw_team_connect_local(aw_grid** grids, int world);
/* Drive virtual ranks step by step on their streams (one process). */
aw_status aw_team_run(aw_grid** grids, int world, int nt, double dt);

/* ------------------------------------------------------------------------
 * NEXT-3: gradient of the least-squares data misfit by the adjoint-state
 * method -- the seismic inversion the project exists for (PAPER.md:4, :17,
 * :69, :98, :248); the paper defines no gradient, the readings are DESIGN.md
 * §3 Q23-Q26:
 *   J(m) = 1/2 sum_{n<nt} sum_r (rec[n][r] - d_obs[n][r])^2
 * for the forward run of nt steps from zero wavefields with the current
 * sources and receivers.  Adjoint field psi = the same damped leapfrog run in
 * reversed time with the time-reversed residual injected at the receivers
 * (like sources: scale w dt^2/(m + eta dt/2), CSR by corner then receiver);
 *   grad_p = -(1/dt^2) sum_{k<nt} psi^k_p (u^{n+1} - 2u^n + u^{n-1})_p,  n = nt-1-k,
 * in the fp32 sequence of oracle_fwi_gradient (value-identical to it).
 * The forward wavefield is replayed from checkpoints: segments of K steps,
 * a history ring of K+2 levels plus the two levels at each later segment
 * start (K + 2 + 2(ceil(nt/K) - 1) wavefield-sized device buffers, kept by the
 * handle between calls); nt - K forward steps are recomputed.  K =
 * AW_OPT_CHECKPOINT_STEPS, or (0) the largest K whose buffers fit in 60 % of
 * the free device memory (K = nt: no recomputation).
 *   d_obs     [nt][nr] fp32 [H|D] observed traces (row = step)
 *   grad      fp32 [H|D] dJ/dm, dense grid layout (AW_GLOBAL/AW_LOCAL as aw_read_wavefield)
 *   residual  [nt][nr] fp32 [H|D] rec - d_obs, or NULL
 *   objective J (fp64 [H]), or NULL
 * Starts from the reset state with time step dt (any dt); needs a model and
 * receivers (AW_EINVAL without receivers), sources/traces covering nt steps.
 * On return steps_done = nt and aw_read_receivers returns the forward traces;
 * the wavefield levels hold adjoint data: aw_run / aw_read_wavefield return
 * AW_ESTATE until aw_reset or aw_set_wavefield.  Single slab only (a team ->
 * AW_EUNSUPPORTED).  AW_ENOMEM if even K = 1 does not fit; AW_ENONFINITE if J
 * is not finite.
 * ------------------------------------------------------------------------ */
aw_status aw_fwi_gradient(aw_grid* g, int nt, double dt, const float* d_obs, float* grad, int layout,
                          float* residual, double* objective);

/* ------------------------------------------------------------------------
 * NEXT-2: the paper's own benchmark operator (PAPER.md:732-748 [Evaluation >
 * Examined problem]): 2D diffusion  u_t = nu (u_xx + u_yy), forward Euler
 * (time_order 1, solve(eqn, u.forward)), space order 2..16, zero padding.
 * Per point (fp32, DESIGN.md §3 Q22):  L = C0 u; pairs fastest axis first;
 * u_next = fma(fl32(nu*dt), L, u).  Same conventions as the acoustic calls:
 * [H|D] arrays, C-order (n0, n1), h_d = extent_d/(n_d-1), synchronous calls.
 * ------------------------------------------------------------------------ */
typedef struct aw_diffusion aw_diffusion;

/* ndim must be 2 (3 -> AW_EUNSUPPORTED); nu > 0; stream as in aw_dist (NULL = own). */
aw_status aw_diffusion_create(aw_diffusion** out, int ndim, const int64_t* shape, const double* extent,
                              int space_order, double nu, void* stream);
/* u^0, fp32 [H|D], dense (n0, n1); NULL = zeros.  Resets the step counter. */
aw_status aw_diffusion_set(aw_diffusion* d, const float* u);
/* advance nt >= 0 steps with time step dt (> 0; no stability check). */
aw_status aw_diffusion_run(aw_diffusion* d, int nt, double dt);
/* copy the current field into out [H|D] (n0, n1). */
aw_status aw_diffusion_read(aw_diffusion* d, float* out);
aw_status aw_diffusion_stats(const aw_diffusion* d, aw_run_stats* out);
/* AW_OPT_TIMING and AW_OPT_GRAPH_STEPS as for aw_set_option. */
aw_status aw_diffusion_set_option(aw_diffusion* d, int option, int64_t value);
void aw_diffusion_destroy(aw_diffusion* d);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* AW_H */
