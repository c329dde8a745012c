/*
 * aw_oracle.c -- plain, slow, obviously-correct CPU ORACLE for the acoustic
 * wave hot path (arXiv 1906.10811 north star, BASELINE.json:5).
 *
 *   *** TEST INFRASTRUCTURE ONLY ***
 *   Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 *   --impl reference legs may load or execute this file's library.  It shares
 *   no code, header, table or constant generator with the CUDA product path
 *   (paper_1906_10811_b200/csrc).  Inputs (m, damp, wavelet, coordinates)
 *   come from workloads/ which holds none of the method's arithmetic.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, SURVEY = SURVEY.md):
 *   m*u_tt - Lap(u) + eta*u_t = q      (BASELINE.json:5 north star)
 *   - FD shortcuts of order = space order, u.dx2 + u.dy2 (+ u.dz2)
 *        PAPER.md:172 [Background > Devito], :741 [Evaluation > Examined problem]
 *   - explicit update from solve(eq, u.forward)
 *   - zero-initialised padding / halo (zero ghosts)  PAPER.md:455-491 [ops_dat creation]
 *   - divisions hoisted into multiplications          PAPER.md:788-826 [CUDA results]
 *   - time-buffer rotation t_k = (time + k) mod n     PAPER.md:443 [ops_dat creation]
 *   The paper never runs the acoustic operator, so the
 *   discrete readings below are SURVEY.md §8(c) Q1-Q19, listed in DESIGN.md.
 *
 * Three modes:
 *   ORACLE_FP32CANON (0): the parity target.  Exactly this fp32 sequence per
 *        point (every fl32 one IEEE RN rounding, fmaf correctly rounded; the
 *        file is compiled with -ffp-contract=off so FMAs appear only where
 *        written):
 *          L   = C0 * u_p
 *          for d = ndim-1 .. 0, j = 1 .. R:   L = fmaf(C[d][j], u_{p-j e_d} + u_{p+j e_d}, L)
 *          t   = 2*u_p - uprev_p
 *          w   = fmaf(b_p, L, t)
 *          oma = 1 - a_p ;  r = oma * uprev_p
 *          unew_p = fmaf(a_p, w, r)
 *        then injection  unew[c] = fmaf(s_{s,c}, q[n][s], unew[c])  (corner
 *        ascending, then source ascending), receivers read u^n before the step.
 *   ORACLE_FP64CANON (1): the same sequence in fp64 with the SAME fp32-rounded
 *        coefficient values (isolates fp32 arithmetic noise).
 *   ORACLE_FP64EXACT (2): the textbook formula in fp64 with fp64 coefficients:
 *        unew = [dt^2 L + m(2u - uprev) + (eta dt/2) uprev] / (m + eta dt/2)
 *        injection += w64 dt^2 / den_c * q ; receivers sum w64 * u in fp64.
 *
 * Parity pins for each function are in tests/test_oracle_pins.py (P1-P12 of
 * SURVEY §8(c)); none of them reuses this file's formulas.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_FP32CANON 0
#define ORACLE_FP64CANON 1
#define ORACLE_FP64EXACT 2

#define OR_OK 0
#define OR_EINVAL -1
#define OR_ENOMEM -2

#define MAXR 8 /* space order <= 16 */

typedef __int128 i128;

static i128 gcd128(i128 a, i128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b != 0) { i128 t = a % b; a = b; b = t; }
    return a;
}

static i128 fact(int n) {
    i128 f = 1;
    for (int i = 2; i <= n; ++i) f *= i;
    return f;
}

/* ---------------------------------------------------------------------------
 * Step 1: centred FD weights for the second derivative of
 * order k = space_order ("space order"):
 *     c_j = 2 (-1)^{j+1} (m!)^2 / ( j^2 (m-j)! (m+j)! ),  j = 1..m,  m = k/2
 *     c_0 = -2 sum_j c_j
 * as exact reduced rationals num[j]/den[j], j = 0..m.
 * ------------------------------------------------------------------------- */
int oracle_fd_weights(int space_order, int64_t* num, int64_t* den) {
    if (space_order < 2 || space_order > 2 * MAXR || (space_order & 1)) return OR_EINVAL;
    int m = space_order / 2;
    i128 sn = 0, sd = 1; /* running sum of c_j, j>=1 */
    for (int j = 1; j <= m; ++j) {
        i128 n = 2 * fact(m) * fact(m);
        if (!(j & 1)) n = -n; /* (-1)^{j+1}: + for odd j */
        i128 d = (i128)j * j * fact(m - j) * fact(m + j);
        i128 g = gcd128(n, d);
        n /= g; d /= g;
        num[j] = (int64_t)n; den[j] = (int64_t)d;
        /* sn/sd += n/d */
        i128 nn = sn * d + n * sd, dd = sd * d;
        g = gcd128(nn, dd);
        sn = nn / g; sd = dd / g;
    }
    /* c_0 = -2 * sum */
    i128 n0 = -2 * sn, d0 = sd;
    i128 g = gcd128(n0, d0);
    num[0] = (int64_t)(n0 / g); den[0] = (int64_t)(d0 / g);
    return OR_OK;
}

/* fp64 value of each weight: one correctly-rounded division of the reduced
 * rational (num, den both < 2^53 for k <= 16). */
int oracle_fd_weights_f64(int space_order, double* c) {
    int64_t num[MAXR + 1], den[MAXR + 1];
    int st = oracle_fd_weights(space_order, num, den);
    if (st) return st;
    for (int j = 0; j <= space_order / 2; ++j) c[j] = (double)num[j] / (double)den[j];
    return OR_OK;
}

/* Grid spacing h_d = extent_d / (n_d - 1)  (SPEC.md:59-67 convention) */
static double spacing(const int64_t* shape, const double* extent, int d) {
    return extent[d] / (double)(shape[d] - 1);
}

/* ---------------------------------------------------------------------------
 * Step 2: axis coefficients with division hoisting
 * ("r0 = 1.0F/(h_y*h_y)"):
 *     C[d][j] = fl32(c64_j / (h_d*h_d)),   C0 = fl32(sum_d c64_0/(h_d*h_d)) (fp64, axis order)
 * C is [ndim][MAXR+1]; C[d][0] is set to fl32(c64_0/h_d^2) (unused by the step).
 * Also returns the fp64 versions (C64, C064) used by mode FP64EXACT.
 * ------------------------------------------------------------------------- */
int oracle_axis_coeffs(int ndim, const int64_t* shape, const double* extent, int space_order,
                       float* C, float* C0, double* C64, double* C064) {
    double c[MAXR + 1];
    int st = oracle_fd_weights_f64(space_order, c);
    if (st) return st;
    int R = space_order / 2;
    double s0 = 0.0;
    for (int d = 0; d < ndim; ++d) {
        double h = spacing(shape, extent, d);
        double h2 = h * h;
        for (int j = 0; j <= MAXR; ++j) {
            double v = (j <= R) ? c[j] / h2 : 0.0;
            if (C) C[d * (MAXR + 1) + j] = (float)v;
            if (C64) C64[d * (MAXR + 1) + j] = v;
        }
        s0 = s0 + c[0] / h2;
    }
    if (C0) *C0 = (float)s0;
    if (C064) *C064 = s0;
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Step 3: point coefficients, per point, from fp32 m, eta
 * and fp64 dt:   b = fl32(dt^2/m),  den = m + (eta*dt)*0.5,  a = fl32(m/den)
 * ------------------------------------------------------------------------- */
static void point_coeffs(float m, float eta, double dt, float* b, float* a, double* den) {
    double dt2 = dt * dt;
    double t = (double)eta * dt;
    double dn = (double)m + t * 0.5;
    *b = (float)(dt2 / (double)m);
    *a = (float)((double)m / dn);
    if (den) *den = dn;
}

/* ---------------------------------------------------------------------------
 * Step 4: sparse setup (bit-exact contract, BASELINE.json:5)
 * For each point and axis d:  p = (x_d - o_d)/h_d (fp64), reject unless
 * 0 <= p <= n_d-1, i = floor(p), f = p - i.  Corner beta in [0, 2^ndim):
 * bit d set -> index i_d+1, weight f_d; else index i_d, weight 1-f_d.
 * Corners with index n_d are skipped (corner = -1, weight 0).
 * w64 = product of the 1-D weights in axis order.  corner = row-major linear
 * index over the global grid.  Multilinear interpolation (Q9).
 * ------------------------------------------------------------------------- */
int oracle_sparse(int ndim, const int64_t* shape, const double* extent, const double* origin,
                  int npts, const double* coords, int64_t* corner, double* w64) {
    int nc = 1 << ndim;
    for (int s = 0; s < npts; ++s) {
        int64_t i[3];
        double f[3];
        for (int d = 0; d < ndim; ++d) {
            double o = origin ? origin[d] : 0.0;
            double h = spacing(shape, extent, d);
            double p = (coords[s * ndim + d] - o) / h;
            if (!(p >= 0.0 && p <= (double)(shape[d] - 1))) return OR_EINVAL;
            double fl = floor(p);
            i[d] = (int64_t)fl;
            f[d] = p - fl;
        }
        for (int beta = 0; beta < nc; ++beta) {
            int64_t lin = 0;
            double w = 1.0;
            int skip = 0;
            for (int d = 0; d < ndim; ++d) {
                int up = (beta >> d) & 1;
                int64_t idx = i[d] + up;
                if (idx >= shape[d]) skip = 1;
                double wd = up ? f[d] : (1.0 - f[d]);
                w = (d == 0) ? wd : w * wd;
                lin = lin * shape[d] + idx;
            }
            corner[s * nc + beta] = skip ? -1 : lin;
            w64[s * nc + beta] = skip ? 0.0 : w;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* zero-ghost access (Q3: u == 0 outside the domain)        */
static inline int inside(int ndim, const int64_t* shape, const int64_t* idx) {
    for (int d = 0; d < ndim; ++d)
        if (idx[d] < 0 || idx[d] >= shape[d]) return 0;
    return 1;
}
static inline int64_t lin_index(int ndim, const int64_t* shape, const int64_t* idx) {
    int64_t l = 0;
    for (int d = 0; d < ndim; ++d) l = l * shape[d] + idx[d];
    return l;
}

typedef struct {
    int64_t key;   /* corner linear index */
    int src;       /* source index */
    int beta;
} inj_entry;

static int inj_cmp(const void* x, const void* y) {
    const inj_entry* a = (const inj_entry*)x;
    const inj_entry* b = (const inj_entry*)y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->src != b->src) return a->src < b->src ? -1 : 1;
    return a->beta - b->beta;
}

/* ---------------------------------------------------------------------------
 * oracle_run: advance nt steps.
 *   shape/extent/origin : grid (origin may be NULL = 0)
 *   m, damp             : fp32 [N] slowness^2 and eta (damp may be NULL = 0)
 *   dt                  : time step
 *   n0                  : global index of the first step (wavelet row n0)
 *   ns, src_coords      : [ns][ndim]; wavelet [nt_total rows >= n0+nt][ns] fp32
 *   nr, rec_coords      : [nr][ndim]; rec_out [nt][nr] (float for mode 0, double else)
 *   u_cur, u_prev       : in/out level n0 and n0-1 (float for mode 0, double else),
 *                         on return levels n0+nt and n0+nt-1.
 *   nthreads            : OpenMP threads (<=0: runtime default)
 * Three logical time slots rotated as t_k = (n + k) mod 3.
 * ------------------------------------------------------------------------- */
static int oracle_run_ex(int mode, int ndim, const int64_t* shape, const double* extent, const double* origin,
                         int space_order, const float* m, const float* damp, double dt, int n0, int nt,
                         int ns, const double* src_coords, const float* wavelet, const double* wavelet64,
                         int nr, const double* rec_coords, void* rec_out,
                         void* u_cur, void* u_prev, int nthreads);

int oracle_run(int mode, int ndim, const int64_t* shape, const double* extent, const double* origin,
               int space_order, const float* m, const float* damp, double dt, int n0, int nt,
               int ns, const double* src_coords, const float* wavelet,
               int nr, const double* rec_coords, void* rec_out,
               void* u_cur, void* u_prev, int nthreads) {
    return oracle_run_ex(mode, ndim, shape, extent, origin, space_order, m, damp, dt, n0, nt, ns, src_coords,
                         wavelet, NULL, nr, rec_coords, rec_out, u_cur, u_prev, nthreads);
}

/* wavelet64 (may be NULL): fp64 amplitudes used instead of `wavelet` by the fp64 modes
 * (the FWI adjoint injects an fp64 residual in mode FP64EXACT; NEXT-3 below). */
static int oracle_run_ex(int mode, int ndim, const int64_t* shape, const double* extent, const double* origin,
                         int space_order, const float* m, const float* damp, double dt, int n0, int nt,
                         int ns, const double* src_coords, const float* wavelet, const double* wavelet64,
                         int nr, const double* rec_coords, void* rec_out,
                         void* u_cur, void* u_prev, int nthreads) {
    if (ndim < 2 || ndim > 3) return OR_EINVAL;
    if (space_order < 2 || space_order > 2 * MAXR || (space_order & 1)) return OR_EINVAL;
    if (mode < 0 || mode > 2 || nt < 0) return OR_EINVAL;
    const int R = space_order / 2;
    const int nc = 1 << ndim;
    int64_t N = 1;
    for (int d = 0; d < ndim; ++d) {
        if (shape[d] < R + 1) return OR_EINVAL;
        N *= shape[d];
    }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif

    /* Step 2: axis coefficients */
    float C[3 * (MAXR + 1)], C0;
    double C64[3 * (MAXR + 1)], C064;
    oracle_axis_coeffs(ndim, shape, extent, space_order, C, &C0, C64, &C064);

    /* Step 3: point coefficients */
    float* b = (float*)malloc(sizeof(float) * N);
    float* a = (float*)malloc(sizeof(float) * N);
    if (!b || !a) { free(b); free(a); return OR_ENOMEM; }
    for (int64_t p = 0; p < N; ++p) {
        if (!(m[p] > 0.0f) || !isfinite(m[p])) { free(b); free(a); return OR_EINVAL; }
        float eta = damp ? damp[p] : 0.0f;
        if (!(eta >= 0.0f)) { free(b); free(a); return OR_EINVAL; }
        point_coeffs(m[p], eta, dt, &b[p], &a[p], NULL);
    }
    const double dt2 = dt * dt;

    /* Step 4: sparse setup */
    int64_t* scorner = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ns > 0 ? ns : 1) * nc);
    double* sw64 = (double*)malloc(sizeof(double) * (size_t)(ns > 0 ? ns : 1) * nc);
    int64_t* rcorner = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nr > 0 ? nr : 1) * nc);
    double* rw64 = (double*)malloc(sizeof(double) * (size_t)(nr > 0 ? nr : 1) * nc);
    inj_entry* inj = (inj_entry*)malloc(sizeof(inj_entry) * (size_t)(ns > 0 ? ns : 1) * nc);
    float* s32 = (float*)malloc(sizeof(float) * (size_t)(ns > 0 ? ns : 1) * nc);
    double* s64 = (double*)malloc(sizeof(double) * (size_t)(ns > 0 ? ns : 1) * nc);
    int st = OR_OK;
    if (!scorner || !sw64 || !rcorner || !rw64 || !inj || !s32 || !s64) { st = OR_ENOMEM; goto done_sparse; }
    if (ns > 0 && oracle_sparse(ndim, shape, extent, origin, ns, src_coords, scorner, sw64)) { st = OR_EINVAL; goto done_sparse; }
    if (nr > 0 && oracle_sparse(ndim, shape, extent, origin, nr, rec_coords, rcorner, rw64)) { st = OR_EINVAL; goto done_sparse; }
    int ninj = 0;
    for (int s = 0; s < ns; ++s)
        for (int beta = 0; beta < nc; ++beta) {
            int64_t c = scorner[s * nc + beta];
            if (c < 0) continue;
            float eta = damp ? damp[c] : 0.0f;
            double den;
            float bb, aa;
            point_coeffs(m[c], eta, dt, &bb, &aa, &den);
            s32[s * nc + beta] = (float)((sw64[s * nc + beta] * dt2) / den);
            s64[s * nc + beta] = sw64[s * nc + beta] * dt2 / den;
            inj[ninj].key = c; inj[ninj].src = s; inj[ninj].beta = beta;
            ++ninj;
        }
    qsort(inj, (size_t)ninj, sizeof(inj_entry), inj_cmp); /* CSR order: corner, then source (Q11) */

    /* Three logical time slots, rotated t_k = (n+k) mod 3. */
    size_t esz = (mode == ORACLE_FP32CANON) ? sizeof(float) : sizeof(double);
    void* slot[3];
    slot[0] = malloc(esz * N); slot[1] = malloc(esz * N); slot[2] = malloc(esz * N);
    if (!slot[0] || !slot[1] || !slot[2]) { st = OR_ENOMEM; free(slot[0]); free(slot[1]); free(slot[2]); goto done_sparse; }
    /* level n lives in slot (n mod 3); n counted from 1 here so level n0-1 -> slot 0 */
    memcpy(slot[1], u_cur, esz * N);   /* level n0   -> slot (1) */
    memcpy(slot[0], u_prev, esz * N);  /* level n0-1 -> slot (0) */

    for (int step = 0; step < nt; ++step) {
        int n = n0 + step;
        /* local counter k = step+1 is level n; slots: prev (k-1)%3, cur k%3, next (k+1)%3 */
        int k = step + 1;
        void* vprev = slot[(k - 1) % 3];
        void* vcur = slot[k % 3];
        void* vnext = slot[(k + 1) % 3];

        /* 6.1 receivers read u^n (Q8) */
        for (int r = 0; r < nr; ++r) {
            if (mode == ORACLE_FP32CANON) {
                const float* u = (const float*)vcur;
                float acc = 0.0f;
                for (int beta = 0; beta < nc; ++beta) {
                    int64_t c = rcorner[r * nc + beta];
                    if (c < 0) continue;
                    acc = fmaf((float)rw64[r * nc + beta], u[c], acc);
                }
                ((float*)rec_out)[(int64_t)step * nr + r] = acc;
            } else if (mode == ORACLE_FP64CANON) {
                const double* u = (const double*)vcur;
                double acc = 0.0;
                for (int beta = 0; beta < nc; ++beta) {
                    int64_t c = rcorner[r * nc + beta];
                    if (c < 0) continue;
                    acc = fma((double)(float)rw64[r * nc + beta], u[c], acc);
                }
                ((double*)rec_out)[(int64_t)step * nr + r] = acc;
            } else {
                const double* u = (const double*)vcur;
                double acc = 0.0;
                for (int beta = 0; beta < nc; ++beta) {
                    int64_t c = rcorner[r * nc + beta];
                    if (c < 0) continue;
                    acc += rw64[r * nc + beta] * u[c];
                }
                ((double*)rec_out)[(int64_t)step * nr + r] = acc;
            }
        }

        /* 6.2 stencil + damped leapfrog update at every domain point (Q4) */
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < N; ++p) {
            int64_t idx[3], q[3];
            int64_t rem = p;
            for (int d = ndim - 1; d >= 0; --d) { idx[d] = rem % shape[d]; rem /= shape[d]; }
            if (mode == ORACLE_FP32CANON) {
                const float* u = (const float*)vcur;
                const float* um1 = (const float*)vprev;
                float L = C0 * u[p];
                for (int d = ndim - 1; d >= 0; --d) {
                    for (int j = 1; j <= R; ++j) {
                        memcpy(q, idx, sizeof(q));
                        q[d] = idx[d] - j;
                        float lo = inside(ndim, shape, q) ? u[lin_index(ndim, shape, q)] : 0.0f;
                        q[d] = idx[d] + j;
                        float hi = inside(ndim, shape, q) ? u[lin_index(ndim, shape, q)] : 0.0f;
                        float pair = lo + hi;
                        L = fmaf(C[d * (MAXR + 1) + j], pair, L);
                    }
                }
                float t = 2.0f * u[p] - um1[p];
                float w = fmaf(b[p], L, t);
                float oma = 1.0f - a[p];
                float rr = oma * um1[p];
                ((float*)vnext)[p] = fmaf(a[p], w, rr);
            } else if (mode == ORACLE_FP64CANON) {
                const double* u = (const double*)vcur;
                const double* um1 = (const double*)vprev;
                double L = (double)C0 * u[p];
                for (int d = ndim - 1; d >= 0; --d) {
                    for (int j = 1; j <= R; ++j) {
                        memcpy(q, idx, sizeof(q));
                        q[d] = idx[d] - j;
                        double lo = inside(ndim, shape, q) ? u[lin_index(ndim, shape, q)] : 0.0;
                        q[d] = idx[d] + j;
                        double hi = inside(ndim, shape, q) ? u[lin_index(ndim, shape, q)] : 0.0;
                        L = fma((double)C[d * (MAXR + 1) + j], lo + hi, L);
                    }
                }
                double t = 2.0 * u[p] - um1[p];
                double w = fma((double)b[p], L, t);
                double rr = (1.0 - (double)a[p]) * um1[p];
                ((double*)vnext)[p] = fma((double)a[p], w, rr);
            } else {
                /* textbook: L = sum_d sum_{j=-R..R} c_|j|/h_d^2 u(p + j e_d) */
                const double* u = (const double*)vcur;
                const double* um1 = (const double*)vprev;
                double L = 0.0;
                for (int d = 0; d < ndim; ++d) {
                    for (int j = -R; j <= R; ++j) {
                        memcpy(q, idx, sizeof(q));
                        q[d] = idx[d] + j;
                        double v = inside(ndim, shape, q) ? u[lin_index(ndim, shape, q)] : 0.0;
                        L += C64[d * (MAXR + 1) + (j < 0 ? -j : j)] * v;
                    }
                }
                double mm = (double)m[p];
                double he = (damp ? (double)damp[p] : 0.0) * dt * 0.5;
                ((double*)vnext)[p] = (dt2 * L + mm * (2.0 * u[p] - um1[p]) + he * um1[p]) / (mm + he);
            }
        }

        /* 6.3 injection into u^{n+1}: corner ascending, then source ascending (Q6, Q11) */
        for (int e = 0; e < ninj; ++e) {
            int s = inj[e].src, beta = inj[e].beta;
            int64_t c = inj[e].key;
            float q32 = wavelet ? wavelet[(int64_t)n * ns + s] : 0.0f;
            double q64 = wavelet64 ? wavelet64[(int64_t)n * ns + s] : (double)q32;
            if (mode == ORACLE_FP32CANON) {
                float* un = (float*)vnext;
                un[c] = fmaf(s32[s * nc + beta], q32, un[c]);
            } else if (mode == ORACLE_FP64CANON) {
                double* un = (double*)vnext;
                un[c] = fma((double)s32[s * nc + beta], q64, un[c]);
            } else {
                double* un = (double*)vnext;
                un[c] += s64[s * nc + beta] * q64;
            }
        }
        /* 6.4 rotate: implicit in the slot index (k+1)%3 */
    }
    /* after nt steps the newest level n0+nt lives in slot (nt+1)%3, the previous in nt%3 */
    memcpy(u_cur, slot[(nt + 1) % 3], esz * N);
    memcpy(u_prev, slot[nt % 3], esz * N);
    free(slot[0]); free(slot[1]); free(slot[2]);
done_sparse:
    free(scorner); free(sw64); free(rcorner); free(rw64); free(inj); free(s32); free(s64);
    free(b); free(a);
    return st;
}

/* Export the point coefficients for one (m, eta, dt) for tests. */
void oracle_point_coeffs(int64_t n, const float* m, const float* damp, double dt, float* b, float* a) {
    for (int64_t p = 0; p < n; ++p) point_coeffs(m[p], damp ? damp[p] : 0.0f, dt, &b[p], &a[p], NULL);
}

/* Source scales s = fl32((w64*dt^2)/den_c) for tests of the sparse contract. */
int oracle_source_scales(int ndim, const int64_t* shape, const double* extent, const double* origin,
                         const float* m, const float* damp, double dt, int ns, const double* coords,
                         int64_t* corner, float* s) {
    int nc = 1 << ndim;
    double* w = (double*)malloc(sizeof(double) * (size_t)(ns > 0 ? ns : 1) * nc);
    if (!w) return OR_ENOMEM;
    int st = oracle_sparse(ndim, shape, extent, origin, ns, coords, corner, w);
    if (st == OR_OK) {
        for (int i = 0; i < ns * nc; ++i) {
            if (corner[i] < 0) { s[i] = 0.0f; continue; }
            double den; float bb, aa;
            point_coeffs(m[corner[i]], damp ? damp[corner[i]] : 0.0f, dt, &bb, &aa, &den);
            s[i] = (float)((w[i] * (dt * dt)) / den);
        }
    }
    free(w);
    return st;
}

/* ===========================================================================
 * NEXT-2: the paper's own benchmark operator, 2D (or 3D) diffusion
 *   u_t = nu (u_xx + u_yy)            PAPER.md:732-736 [Evaluation > Examined problem]
 * discretised as in the paper's Devito listing: time_order=1
 * (forward Euler, `solve(eqn, u.forward)`), FD shortcuts u.dx2 + u.dy2 of the
 * given space order, zero padding.  The worked kernel
 * folds nu into the weights (5.0e-1F = nu*1, -1.0F = nu*-2).
 *
 * ORACLE_FP32CANON sequence per point (this build's reading, DESIGN.md §3 Q22):
 *   L = C0*u;  for d = ndim-1..0, j = 1..R: L = fmaf(C[d][j], u_{p-je_d} + u_{p+je_d}, L)
 *   u_next = fmaf(D, L, u)             with D = fl32(nu*dt) (fp64 product, one rounding)
 * ORACLE_FP64CANON: same sequence in fp64 with the same fp32 C, C0, D.
 * ORACLE_FP64EXACT: u_next = u + nu*dt*sum_d sum_j c_|j|/h_d^2 u(p+j e_d) in fp64.
 * u holds the initial field on entry and u^nt on return (float or double by mode).
 * ------------------------------------------------------------------------- */
int oracle_diffusion_run(int mode, int ndim, const int64_t* shape, const double* extent, int space_order,
                         double nu, double dt, int nt, void* u, int nthreads) {
    if (ndim < 2 || ndim > 3) return OR_EINVAL;
    if (space_order < 2 || space_order > 2 * MAXR || (space_order & 1)) return OR_EINVAL;
    if (mode < 0 || mode > 2 || nt < 0) return OR_EINVAL;
    const int R = space_order / 2;
    int64_t N = 1;
    for (int d = 0; d < ndim; ++d) {
        if (shape[d] < R + 1) return OR_EINVAL;
        N *= shape[d];
    }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    float C[3 * (MAXR + 1)], C0;
    double C64[3 * (MAXR + 1)], C064;
    oracle_axis_coeffs(ndim, shape, extent, space_order, C, &C0, C64, &C064);
    const float D = (float)(nu * dt);
    const double D64 = nu * dt;
    size_t esz = (mode == ORACLE_FP32CANON) ? sizeof(float) : sizeof(double);
    void* nxt = malloc(esz * N);
    void* cur = malloc(esz * N);
    if (!nxt || !cur) { free(nxt); free(cur); return OR_ENOMEM; }
    memcpy(cur, u, esz * N);
    for (int step = 0; step < nt; ++step) {
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < N; ++p) {
            int64_t idx[3], q[3];
            int64_t rem = p;
            for (int d = ndim - 1; d >= 0; --d) { idx[d] = rem % shape[d]; rem /= shape[d]; }
            if (mode == ORACLE_FP32CANON) {
                const float* uc = (const float*)cur;
                float L = C0 * uc[p];
                for (int d = ndim - 1; d >= 0; --d)
                    for (int j = 1; j <= R; ++j) {
                        memcpy(q, idx, sizeof(q));
                        q[d] = idx[d] - j;
                        float lo = inside(ndim, shape, q) ? uc[lin_index(ndim, shape, q)] : 0.0f;
                        q[d] = idx[d] + j;
                        float hi = inside(ndim, shape, q) ? uc[lin_index(ndim, shape, q)] : 0.0f;
                        float pair = lo + hi;
                        L = fmaf(C[d * (MAXR + 1) + j], pair, L);
                    }
                ((float*)nxt)[p] = fmaf(D, L, uc[p]);
            } else if (mode == ORACLE_FP64CANON) {
                const double* uc = (const double*)cur;
                double L = (double)C0 * uc[p];
                for (int d = ndim - 1; d >= 0; --d)
                    for (int j = 1; j <= R; ++j) {
                        memcpy(q, idx, sizeof(q));
                        q[d] = idx[d] - j;
                        double lo = inside(ndim, shape, q) ? uc[lin_index(ndim, shape, q)] : 0.0;
                        q[d] = idx[d] + j;
                        double hi = inside(ndim, shape, q) ? uc[lin_index(ndim, shape, q)] : 0.0;
                        L = fma((double)C[d * (MAXR + 1) + j], lo + hi, L);
                    }
                ((double*)nxt)[p] = fma((double)D, L, uc[p]);
            } else {
                const double* uc = (const double*)cur;
                double L = 0.0;
                for (int d = 0; d < ndim; ++d)
                    for (int j = -R; j <= R; ++j) {
                        memcpy(q, idx, sizeof(q));
                        q[d] = idx[d] + j;
                        double v = inside(ndim, shape, q) ? uc[lin_index(ndim, shape, q)] : 0.0;
                        L += C64[d * (MAXR + 1) + (j < 0 ? -j : j)] * v;
                    }
                ((double*)nxt)[p] = uc[p] + D64 * L;
            }
        }
        void* t = cur; cur = nxt; nxt = t;  /* rotation t_k = (time+k) mod 2 */
    }
    memcpy(u, cur, esz * N);
    free(cur); free(nxt);
    return OR_OK;
}

/* ===========================================================================
 * NEXT-3: gradient of the least-squares data misfit by the
 * adjoint-state method -- the "inversion problems" the project exists for
 * (PAPER.md:4, :17, :69, :98 [Plan / Introduction], :248 [Background]).
 * The paper defines no gradient; this build's readings are DESIGN.md §3
 * Q23-Q26:
 *   J(m) = 1/2 sum_{n=0}^{nt-1} sum_r (rec[n][r] - d_obs[n][r])^2
 * for the forward run of oracle_run from zero initial conditions.
 * Differentiating the textbook update (per point p, holding u^n, u^{n-1}):
 *   (m + eta dt/2) u^{n+1} = dt^2 (L u^n + P_s^T q^n) + m (2u^n - u^{n-1}) + (eta dt/2) u^{n-1}
 *   => du^{n+1}_p/dm_p = -(u^{n+1} - 2u^n + u^{n-1})_p / (m_p + eta_p dt/2),
 * and scaling the Lagrange multipliers by dt^2/(m + eta dt/2) turns the
 * adjoint recursion into the SAME damped leapfrog run in reversed time with
 * the residual injected at the receivers like a source:
 *   psi^{-1} = psi^0 = 0,
 *   psi^{k+1} = step(psi^k, psi^{k-1}) + inject(res[nt-1-k] at the receivers),
 *   grad_p = -(1/dt^2) sum_{k=0}^{nt-1} psi^k_p D^n_p,   n = nt-1-k,
 *   D^n = u^{n+1} - 2u^n + u^{n-1}           (u^{-1} = u^0 = 0).
 * Pinned by central finite differences of J (tests/test_oracle_fwi_pins.py),
 * which use only oracle_run -- none of the formulas above.
 * Modes:
 *   FP32CANON: res = fl32(rec - d_obs); D = fl32(fl32(u^{n+1} - 2u^n) + u^{n-1});
 *              G = fmaf(psi^k, D, G) for k = 0..nt-1 from G = 0;
 *              grad = fl32(-(double)G / (dt*dt))
 *   FP64CANON: the same sequence in fp64 (propagations in fp64canon).
 *   FP64EXACT: fp64 textbook propagations, res = rec - (double)d_obs,
 *              grad = -sum_k psi^k D^n / dt^2.
 * J = 0.5 * sum res^2 in fp64 (n-major, r-minor order).
 * The whole forward history is kept (no checkpointing): plain and slow.
 * grad_out, res_out: float (mode 0) or double; res_out may be NULL.
 * ------------------------------------------------------------------------- */
int oracle_fwi_gradient(int mode, int ndim, const int64_t* shape, const double* extent, const double* origin,
                        int space_order, const float* m, const float* damp, double dt, int nt,
                        int ns, const double* src_coords, const float* wavelet,
                        int nr, const double* rec_coords, const float* d_obs,
                        void* grad_out, void* res_out, double* J_out, int nthreads) {
    if (ndim < 2 || ndim > 3 || mode < 0 || mode > 2 || nt < 1 || nr < 1 || !d_obs || !grad_out) return OR_EINVAL;
    int64_t N = 1;
    for (int d = 0; d < ndim; ++d) N *= shape[d];
    const int f32 = mode == ORACLE_FP32CANON;
    const size_t esz = f32 ? sizeof(float) : sizeof(double);
    char* hist = (char*)calloc((size_t)(nt + 2) * N, esz); /* level l at slot l+1, l = -1..nt */
    char* rec = (char*)calloc((size_t)nt * nr, esz);
    char* res = (char*)calloc((size_t)nt * nr, esz);
    char* wadj = (char*)calloc((size_t)nt * nr, esz);
    char* ucur = (char*)calloc((size_t)N, esz);
    char* uprev = (char*)calloc((size_t)N, esz);
    char* G = (char*)calloc((size_t)N, esz);
    int st = OR_OK;
    double J = 0.0;
    if (!hist || !rec || !res || !wadj || !ucur || !uprev || !G) { st = OR_ENOMEM; goto out; }
#define LEVEL(l) (hist + (size_t)((l) + 1) * N * esz)

    /* 1. forward run, one step per call, recording every level */
    for (int n = 0; n < nt; ++n) {
        memcpy(ucur, LEVEL(n), esz * N);
        memcpy(uprev, LEVEL(n - 1), esz * N);
        st = oracle_run_ex(mode, ndim, shape, extent, origin, space_order, m, damp, dt, n, 1, ns, src_coords,
                           wavelet, NULL, nr, rec_coords, rec + (size_t)n * nr * esz, ucur, uprev, nthreads);
        if (st) goto out;
        memcpy(LEVEL(n + 1), ucur, esz * N);
    }

    /* 2. residual, misfit, time-reversed residual as the adjoint "wavelet" */
    for (int n = 0; n < nt; ++n)
        for (int r = 0; r < nr; ++r) {
            size_t i = (size_t)n * nr + r, ir = (size_t)(nt - 1 - n) * nr + r;
            if (f32) {
                float v = ((float*)rec)[i] - d_obs[i];
                ((float*)res)[i] = v;
                ((float*)wadj)[ir] = v;
                J += (double)v * (double)v;
            } else {
                double v = ((double*)rec)[i] - (double)d_obs[i];
                ((double*)res)[i] = v;
                ((double*)wadj)[ir] = v;
                J += v * v;
            }
        }
    J = 0.5 * J;

    /* 3. adjoint run in reversed time with the imaging condition before each step */
    memset(ucur, 0, esz * N);  /* psi^k     */
    memset(uprev, 0, esz * N); /* psi^{k-1} */
    for (int k = 0; k < nt; ++k) {
        const int n = nt - 1 - k;
        const char* u1 = LEVEL(n + 1);
        const char* u0 = LEVEL(n);
        const char* um1 = LEVEL(n - 1);
        for (int64_t p = 0; p < N; ++p) {
            if (f32) {
                float D = (((const float*)u1)[p] - 2.0f * ((const float*)u0)[p]) + ((const float*)um1)[p];
                ((float*)G)[p] = fmaf(((float*)ucur)[p], D, ((float*)G)[p]);
            } else if (mode == ORACLE_FP64CANON) {
                double D = (((const double*)u1)[p] - 2.0 * ((const double*)u0)[p]) + ((const double*)um1)[p];
                ((double*)G)[p] = fma(((double*)ucur)[p], D, ((double*)G)[p]);
            } else {
                double D = ((const double*)u1)[p] - 2.0 * ((const double*)u0)[p] + ((const double*)um1)[p];
                ((double*)G)[p] += ((double*)ucur)[p] * D;
            }
        }
        if (k == nt - 1) break; /* psi^nt pairs with no forward level */
        st = oracle_run_ex(mode, ndim, shape, extent, origin, space_order, m, damp, dt, k, 1, nr, rec_coords,
                           f32 ? (const float*)wadj : NULL, f32 ? NULL : (const double*)wadj, 0, NULL, NULL,
                           ucur, uprev, nthreads);
        if (st) goto out;
    }

    /* 4. gradient = -G / dt^2 */
    {
        const double dt2 = dt * dt;
        for (int64_t p = 0; p < N; ++p) {
            if (f32) ((float*)grad_out)[p] = (float)(-(double)((float*)G)[p] / dt2);
            else ((double*)grad_out)[p] = -((double*)G)[p] / dt2;
        }
    }
    if (res_out) memcpy(res_out, res, esz * (size_t)nt * nr);
    if (J_out) *J_out = J;
#undef LEVEL
out:
    free(hist); free(rec); free(res); free(wadj); free(ucur); free(uprev); free(G);
    return st;
}

/* ===========================================================================
 * Virtual slab decomposition: the same run as
 * oracle_run, mode FP32CANON, computed as `world` slabs of axis 0, each with
 * its own arrays and R = k/2 halo planes on both sides, the way the multi-GPU
 * path decomposes it:
 *   - slab r owns planes [z0_r, z0_r + nz_r): nz_r = n0/world (+1 for the first
 *     n0 % world ranks), contiguous in rank order (aw_slab_partition);
 *   - before every step each slab copies the R outermost owned planes of u^n of
 *     its neighbours into its halo planes (zero beyond the global ends);
 *   - receiver r is read by the slab owning the plane of its base corner i_0;
 *     its +1 corner may lie in that slab's halo (SURVEY §8(e) owner-computes);
 *   - injection entries are applied by the slab owning the corner, in the
 *     global CSR order restricted to its corners;
 *   - traces are summed over slabs (disjoint owners: exact).
 * Decomposition changes no per-point arithmetic, so the result must equal
 * oracle_run bit for bit (tests/test_oracle_pins.py::test_p12_virtual_slabs).
 * The wavefields are returned gathered into the global u_cur/u_prev arrays.
 * ------------------------------------------------------------------------- */
int oracle_run_slabs(int world, int ndim, const int64_t* shape, const double* extent, const double* origin,
                     int space_order, const float* m, const float* damp, double dt, int nt,
                     int ns, const double* src_coords, const float* wavelet,
                     int nr, const double* rec_coords, float* rec_out, float* u_cur, float* u_prev) {
    if (ndim < 2 || ndim > 3 || world < 1 || nt < 0) return OR_EINVAL;
    if (space_order < 2 || space_order > 2 * MAXR || (space_order & 1)) return OR_EINVAL;
    const int R = space_order / 2, nc = 1 << ndim;
    const int64_t n0 = shape[0];
    int64_t per = 1; /* points per plane */
    for (int d = 1; d < ndim; ++d) per *= shape[d];
    if (n0 / world < R) return OR_EINVAL; /* every slab must hold >= R planes */
    float C[3 * (MAXR + 1)], C0;
    oracle_axis_coeffs(ndim, shape, extent, space_order, C, &C0, NULL, NULL);
    int st = OR_OK;
    int64_t N = n0 * per;
    /* global per-point coefficients and sparse setup (the same helpers as oracle_run) */
    float* b = (float*)malloc(sizeof(float) * N);
    float* a = (float*)malloc(sizeof(float) * N);
    int64_t* sc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ns > 0 ? ns : 1) * nc);
    double* sw = (double*)malloc(sizeof(double) * (size_t)(ns > 0 ? ns : 1) * nc);
    int64_t* rc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nr > 0 ? nr : 1) * nc);
    double* rw = (double*)malloc(sizeof(double) * (size_t)(nr > 0 ? nr : 1) * nc);
    inj_entry* inj = (inj_entry*)malloc(sizeof(inj_entry) * (size_t)(ns > 0 ? ns : 1) * nc);
    float* s32 = (float*)malloc(sizeof(float) * (size_t)(ns > 0 ? ns : 1) * nc);
    int64_t* z0 = (int64_t*)malloc(sizeof(int64_t) * world);
    int64_t* nzs = (int64_t*)malloc(sizeof(int64_t) * world);
    float** slot = (float**)calloc((size_t)world * 3, sizeof(float*));
    int ninj = 0;
    if (!b || !a || !sc || !sw || !rc || !rw || !inj || !s32 || !z0 || !nzs || !slot) { st = OR_ENOMEM; goto done; }
    for (int64_t p = 0; p < N; ++p) {
        if (!(m[p] > 0.0f) || !isfinite(m[p])) { st = OR_EINVAL; goto done; }
        point_coeffs(m[p], damp ? damp[p] : 0.0f, dt, &b[p], &a[p], NULL);
    }
    if (ns > 0 && oracle_sparse(ndim, shape, extent, origin, ns, src_coords, sc, sw)) { st = OR_EINVAL; goto done; }
    if (nr > 0 && oracle_sparse(ndim, shape, extent, origin, nr, rec_coords, rc, rw)) { st = OR_EINVAL; goto done; }
    for (int s = 0; s < ns; ++s)
        for (int beta = 0; beta < nc; ++beta) {
            int64_t c = sc[s * nc + beta];
            if (c < 0) continue;
            double den; float bb, aa;
            point_coeffs(m[c], damp ? damp[c] : 0.0f, dt, &bb, &aa, &den);
            s32[s * nc + beta] = (float)((sw[s * nc + beta] * (dt * dt)) / den);
            inj[ninj].key = c; inj[ninj].src = s; inj[ninj].beta = beta;
            ++ninj;
        }
    qsort(inj, (size_t)ninj, sizeof(inj_entry), inj_cmp);
    /* slabs and their arrays: planes [-R, nz+R) of local index, 3 time slots */
    {
        int64_t base = n0 / world, rem = n0 % world;
        for (int r = 0; r < world; ++r) {
            nzs[r] = base + (r < rem ? 1 : 0);
            z0[r] = r * base + (r < rem ? r : rem);
            for (int t = 0; t < 3; ++t) {
                slot[r * 3 + t] = (float*)calloc((size_t)(nzs[r] + 2 * R) * per, sizeof(float));
                if (!slot[r * 3 + t]) { st = OR_ENOMEM; goto done; }
            }
            /* levels -1 (slot 0) and 0 (slot 1): owned planes from the inputs */
            memcpy(slot[r * 3 + 1] + R * per, u_cur + z0[r] * per, sizeof(float) * nzs[r] * per);
            memcpy(slot[r * 3 + 0] + R * per, u_prev + z0[r] * per, sizeof(float) * nzs[r] * per);
        }
    }
    for (int step = 0; step < nt; ++step) {
        const int k = step + 1;
        /* halo exchange of u^n: my halo planes <- the neighbours' R outermost owned planes */
        for (int r = 0; r < world; ++r) {
            float* u = slot[r * 3 + k % 3];
            memset(u, 0, sizeof(float) * R * per);
            memset(u + (R + nzs[r]) * per, 0, sizeof(float) * R * per);
            if (r > 0) {
                const float* lo = slot[(r - 1) * 3 + k % 3];
                memcpy(u, lo + nzs[r - 1] * per, sizeof(float) * R * per); /* its planes [nz-R, nz) */
            }
            if (r + 1 < world) {
                const float* hi = slot[(r + 1) * 3 + k % 3];
                memcpy(u + (R + nzs[r]) * per, hi + R * per, sizeof(float) * R * per); /* its planes [0, R) */
            }
        }
        for (int r = 0; r < world; ++r) {
            const float* u = slot[r * 3 + k % 3];
            const float* um1 = slot[r * 3 + (k - 1) % 3];
            float* un = slot[r * 3 + (k + 1) % 3];
            /* receivers owned by this slab (base corner plane i_0 in [z0, z0+nz)) read u^n */
            for (int q = 0; q < nr; ++q) {
                int64_t c0 = rc[q * nc + 0];
                if (c0 < 0) continue;
                int64_t zb = c0 / per;
                if (zb < z0[r] || zb >= z0[r] + nzs[r]) continue;
                float acc = 0.0f;
                for (int beta = 0; beta < nc; ++beta) {
                    int64_t c = rc[q * nc + beta];
                    if (c < 0) continue;
                    int64_t zl = c / per - z0[r]; /* may be nz (halo plane) */
                    acc = fmaf((float)rw[q * nc + beta], u[(zl + R) * per + c % per], acc);
                }
                rec_out[(int64_t)step * nr + q] += acc;
            }
            /* stencil + update at the owned points, axes d = ndim-1 .. 0 */
            for (int64_t zl = 0; zl < nzs[r]; ++zl)
                for (int64_t i = 0; i < per; ++i) {
                    int64_t idx[3];
                    idx[0] = z0[r] + zl;
                    int64_t rem2 = i;
                    for (int d = ndim - 1; d >= 1; --d) { idx[d] = rem2 % shape[d]; rem2 /= shape[d]; }
                    const int64_t pl = (zl + R) * per + i, pg = (z0[r] + zl) * per + i;
                    float L = C0 * u[pl];
                    for (int d = ndim - 1; d >= 0; --d) {
                        int64_t stride = 1;
                        for (int e = d + 1; e < ndim; ++e) stride *= shape[e];
                        for (int j = 1; j <= R; ++j) {
                            float lo, hi;
                            if (d == 0) { /* halo planes hold the neighbours' values or zeros */
                                lo = u[pl - j * per];
                                hi = u[pl + j * per];
                            } else {
                                lo = idx[d] - j >= 0 ? u[pl - j * stride] : 0.0f;
                                hi = idx[d] + j < shape[d] ? u[pl + j * stride] : 0.0f;
                            }
                            float pair = lo + hi;
                            L = fmaf(C[d * (MAXR + 1) + j], pair, L);
                        }
                    }
                    float t = 2.0f * u[pl] - um1[pl];
                    float w = fmaf(b[pg], L, t);
                    float oma = 1.0f - a[pg];
                    float rr = oma * um1[pl];
                    un[pl] = fmaf(a[pg], w, rr);
                }
            /* injection into owned corners, global CSR order */
            for (int e = 0; e < ninj; ++e) {
                int64_t c = inj[e].key;
                int64_t zl = c / per - z0[r];
                if (zl < 0 || zl >= nzs[r]) continue;
                int s = inj[e].src, beta = inj[e].beta;
                float* v = &un[(zl + R) * per + c % per];
                *v = fmaf(s32[s * nc + beta], wavelet[(int64_t)step * ns + s], *v);
            }
        }
    }
    for (int r = 0; r < world; ++r) {
        memcpy(u_cur + z0[r] * per, slot[r * 3 + (nt + 1) % 3] + R * per, sizeof(float) * nzs[r] * per);
        memcpy(u_prev + z0[r] * per, slot[r * 3 + nt % 3] + R * per, sizeof(float) * nzs[r] * per);
    }
done:
    if (slot) for (int i = 0; i < world * 3; ++i) free(slot[i]);
    free(slot); free(z0); free(nzs);
    free(b); free(a); free(sc); free(sw); free(rc); free(rw); free(inj); free(s32);
    return st;
}
