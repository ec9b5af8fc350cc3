/*
 * idp_oracle.c — CPU restatement of the reference's per-stage IDP Euler update.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker for the CUDA path: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product (paper_2007_00094_b200) never
 * links, imports or falls back to it.
 *
 * It restates, phase by phase and with numpy's exact expression association
 * and reduction order, the single-rank path of
 *   Solver.euler_step      /root/reference/pkg/src/eulerflow/stepper.py:508-610
 * on the reference's padded slot view (stepper.py:163-268, sparsity.py:263-309):
 * rows in global Cuthill-McKee order, slots sorted by CM id, pads (col = row,
 * zero values) up to the global width L.  Pads and the diagonal are processed
 * exactly like the numpy code does (it computes every slot and masks).
 *
 * Parity is pinned: tests/test_oracle_golden.py checks this oracle bit-for-bit
 * against golden vectors produced by the UNMODIFIED reference package with the
 * shared pow (ef_pow.h) installed through physics.set_power_function
 * (tests/golden/make_golden.py).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -pthread).  Rows are
 * independent inside a phase, so the threaded row loops are deterministic.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

#include "../paper_2007_00094_b200/csrc/ef_pow.h"

#define TINY 0x1p-1022 /* np.finfo(np.float64).tiny, limiter.py:40 */
#define TOL_SCALE 1e-10 /* limiter.py:39 */
#define PSI_SIGN (-1.0) /* limiter.py:37 */
#define DENOM_FLOOR 1e-300 /* indicator.py:20 */

enum { OR_OK = 0, OR_ADMISSIBILITY = 1, OR_BAD_STATE = 2, OR_TAU_UNBOUNDED = 3 };

typedef struct {
  double gamma, gm1, gp1_inv, gm1_over_2g, two_g_over_gm1;
} Gas;

typedef struct {
  int64_t n;
  int dim, nvar, L, passes, newton;
  double c_cfl;
  Gas g;
  /* padded view (row-major, CM order) */
  int64_t *cols, *trow, *tslot, *diag, *card;
  uint8_t *valid, *upper, *lower;
  double *c, *cT, *b, *bT, *m_i, *inv_m, *lam;
  /* boundary */
  int64_t n_inflow, n_slip;
  int64_t *inflow, *slip;
  double *slip_n;
  double farfield[5];
  /* work arrays */
  double *U, *U_next, *U0, *f, *eor, *phi, *d, *alpha, *R, *P, *l, *l_next;
  double *rho_min, *rho_max, *phi_min;
  double tau_last;
  int64_t bad_row;
  int nthreads;
} Oracle;

/* ---- numpy scalar semantics ------------------------------------------------ */
static inline double np_max(double a, double b) { return (a >= b || a != a) ? a : b; }
static inline double np_min(double a, double b) { return (a <= b || a != a) ? a : b; }
static inline double np_clip(double x, double lo, double hi) { return np_min(np_max(x, lo), hi); }
static inline double opow(double x, double y) { return ef_pow(x, y); }

/* R1: last-axis sum of length < 8, ((0 + a0) + a1) + ... */
static inline double r1_dot(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int k = 0; k < n; ++k) s += a[k] * b[k];
  return s;
}

/* R2: numpy pairwise sum for 8 <= n <= 128 (8 accumulators, fixed tree). */
static double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i];
    return s;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i;
  for (i = 8; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] += a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += a[i];
  return res;
}

/* physics.internal_energy, physics.py:86-89: E - ((0.5 * |m|^2) / rho) */
static inline double internal_energy(const double* U, int dim) {
  double mm = 0.0;
  for (int a = 0; a < dim; ++a) mm += U[1 + a] * U[1 + a];
  return U[dim + 1] - ((0.5 * mm) / U[0]);
}

/* physics.flux, physics.py:151-163 (f[k*dim + a]) */
static void flux(const double* U, int dim, const Gas* g, double* f) {
  double rho = U[0], E = U[dim + 1];
  double v[3];
  for (int a = 0; a < dim; ++a) v[a] = U[1 + a] / rho;
  double p = g->gm1 * internal_energy(U, dim);
  for (int b = 0; b < dim; ++b) f[0 * dim + b] = U[1 + b];
  for (int a = 0; a < dim; ++a)
    for (int b = 0; b < dim; ++b) f[(1 + a) * dim + b] = v[a] * U[1 + b];
  for (int k = 0; k < dim; ++k) f[(1 + k) * dim + k] += p;
  for (int b = 0; b < dim; ++b) f[(dim + 1) * dim + b] = v[b] * (E + p);
}

/* ---- riemann.py ------------------------------------------------------------- */
typedef struct { double rho, m, E, u, p, c; } Proj;

/* riemann.project, riemann.py:56-69 */
static int project(const double* U, const double* n, int dim, const Gas* g, Proj* o) {
  double rho = U[0], E = U[dim + 1];
  double m_t = 0.0;
  for (int a = 0; a < dim; ++a) m_t += U[1 + a] * n[a];
  double tt = 0.0;
  for (int a = 0; a < dim; ++a) {
    double tg = U[1 + a] - m_t * n[a];
    tt += tg * tg;
  }
  double E_t = E - ((0.5 * tt) / rho);
  double u = m_t / rho;
  double p = g->gm1 * (E_t - (((0.5 * m_t) * m_t) / rho));
  int bad = (rho <= 0.0) || (p <= 0.0);
  o->rho = rho; o->m = m_t; o->E = E_t; o->u = u; o->p = p;
  o->c = sqrt((g->gamma * p) / rho);
  return bad;
}

/* riemann._f_wave, riemann.py:86-90 */
static inline double f_wave(const Proj* S, double p, const Gas* g) {
  if (p >= S->p)
    return (sqrt(2.0) * (p - S->p)) / sqrt(S->rho * (((g->gamma + 1.0) * p) + (g->gm1 * S->p)));
  return (opow(p / S->p, g->gm1_over_2g) - 1.0) * ((2.0 * S->c) / g->gm1);
}

/* riemann._lambda_max_projected, riemann.py:100-109 (+ two_rarefaction_pstar :72-83, psi :93-97) */
static double lambda_max_projected(const Proj* L, const Proj* R, const Gas* g) {
  double p_max = np_max(L->p, R->p);
  double num = (L->c + R->c) - ((0.5 * g->gm1) * (R->u - L->u));
  double den = (L->c * opow(L->p / R->p, -g->gm1_over_2g)) + R->c;
  double base = np_max(num / den, 0.0);
  double p_tr = R->p * opow(base, g->two_g_over_gm1);
  double psi = (f_wave(L, p_max, g) + f_wave(R, p_max, g)) + (R->u - L->u);
  double p_star = (psi < 0.0) ? p_tr : np_min(p_max, p_tr);
  double gp1_over_2g = (g->gamma + 1.0) / (2.0 * g->gamma);
  double x1 = (p_star - L->p) / L->p;
  double x3 = (p_star - R->p) / R->p;
  double lam1 = L->u - (L->c * sqrt(1.0 + (gp1_over_2g * (0.5 * (fabs(x1) + x1)))));
  double lam3 = R->u + (R->c * sqrt(1.0 + (gp1_over_2g * (0.5 * (fabs(x3) + x3)))));
  return np_max(0.5 * (fabs(lam1) - lam1), 0.5 * (fabs(lam3) + lam3));
}

/* riemann.d_ij_low, riemann.py:119-142 (every slot evaluated, as numpy does) */
static double d_ij_low(const double* Ui, const double* Uj, const double* cij, const double* cji,
                       int dim, const Gas* g, int* err) {
  double nij2 = 0.0, nji2 = 0.0;
  for (int a = 0; a < dim; ++a) { nij2 += cij[a] * cij[a]; nji2 += cji[a] * cji[a]; }
  double norm_ij = sqrt(nij2), norm_ji = sqrt(nji2);
  double n_ij[3], n_ji[3];
  for (int a = 0; a < dim; ++a) {
    n_ij[a] = norm_ij > 0.0 ? cij[a] / norm_ij : (a == 0 ? 1.0 : 0.0);
    n_ji[a] = norm_ji > 0.0 ? cji[a] / norm_ji : (a == 0 ? 1.0 : 0.0);
  }
  Proj Li, Rj, Lj, Ri;
  *err |= project(Ui, n_ij, dim, g, &Li);
  *err |= project(Uj, n_ij, dim, g, &Rj);
  double lam_ij = lambda_max_projected(&Li, &Rj, g);
  *err |= project(Uj, n_ji, dim, g, &Lj);
  *err |= project(Ui, n_ji, dim, g, &Ri);
  double lam_ji = lambda_max_projected(&Lj, &Ri, g);
  return np_max(norm_ij > 0.0 ? lam_ij * norm_ij : 0.0, norm_ji > 0.0 ? lam_ji * norm_ji : 0.0);
}

/* ---- limiter.py ------------------------------------------------------------- */
static inline double rho_eps(const double* V, int dim) { /* limiter.py:81-85 */
  double mm = 0.0;
  for (int a = 0; a < dim; ++a) mm += V[1 + a] * V[1 + a];
  return (V[0] * V[dim + 1]) - (0.5 * mm);
}

static inline double psi_at(const double* U, const double* P, double t, double phi_min, int dim,
                            const Gas* g) { /* psi_entropy(U + t P), limiter.py:88-91 */
  double V[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < dim + 2; ++k) V[k] = U[k] + t * P[k];
  return rho_eps(V, dim) - (phi_min * opow(V[0], g->gamma + 1.0));
}

static inline double dpsi_at(const double* U, const double* P, double t, double phi_min, int dim,
                             const Gas* g) { /* dpsi_dt, limiter.py:94-110 */
  double V[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < dim + 2; ++k) V[k] = U[k] + t * P[k];
  double mm = 0.0;
  for (int a = 0; a < dim; ++a) mm += V[1 + a] * P[1 + a];
  return (((P[0] * V[dim + 1]) + (V[0] * P[dim + 1])) - mm) -
         (((phi_min * (g->gamma + 1.0)) * opow(V[0], g->gamma)) * P[0]);
}

/* limiter.limiter_compute, limiter.py:149-193, one lane; quadratic_newton_step :113-146 */
static double limiter_lane(const double* U, const double* P, double rho_min, double rho_max,
                           double phi_min, int max_newton, int dim, const Gas* g) {
  double rho_u = U[0], rho_p = P[0];
  double abs_rho_p = np_max(fabs(rho_p), TINY);
  double t_R = 1.0;
  if (rho_u + t_R * rho_p > rho_max) t_R = fabs(rho_max - rho_u) / abs_rho_p;
  if (rho_u + t_R * rho_p < rho_min) t_R = fabs(rho_min - rho_u) / abs_rho_p;
  t_R = np_clip(t_R, 0.0, 1.0);
  double t_L = 0.0;
  double tol = (TOL_SCALE * fabs(rho_eps(U, dim))) * 1.0;
  for (int it = 0; it < max_newton; ++it) {
    double Psi_R = psi_at(U, P, t_R, phi_min, dim, g);
    if (Psi_R >= 0.0) { t_L = t_R; break; }
    double Psi_L = psi_at(U, P, t_L, phi_min, dim, g);
    if (!(Psi_L > tol)) break;
    double dPsi_L = dpsi_at(U, P, t_L, phi_min, dim, g);
    double dPsi_R = dpsi_at(U, P, t_R, phi_min, dim, g);
    double eps = TINY * (1.0 + t_R);
    double scaling = 1.0 / ((t_R - t_L) + eps);
    double d12 = (Psi_R - Psi_L) * scaling;
    double d112 = (d12 - dPsi_L) * scaling;
    double d122 = (dPsi_R - d12) * scaling;
    double lam_L = np_max((dPsi_L * dPsi_L) - ((4.0 * Psi_L) * d112), 0.0);
    double lam_R = np_max((dPsi_R * dPsi_R) - ((4.0 * Psi_R) * d122), 0.0);
    double den_L = dPsi_L + (PSI_SIGN * sqrt(lam_L));
    double den_R = dPsi_R + (PSI_SIGN * sqrt(lam_R));
    double new_L = fabs(den_L) > eps ? t_L - ((2.0 * Psi_L) / den_L) : t_L;
    double new_R = fabs(den_R) > eps ? t_R - ((2.0 * Psi_R) / den_R) : t_R;
    if (!isfinite(new_L)) new_L = t_L;
    if (!isfinite(new_R)) new_R = t_R;
    new_L = np_clip(new_L, t_L, t_R);
    new_R = np_clip(new_R, t_L, t_R);
    t_L = np_min(new_L, new_R);
    t_R = np_max(new_L, new_R);
  }
  return t_L;
}

/* ---- public API ------------------------------------------------------------- */
#define ALLOC(T, cnt) ((T*)calloc((size_t)(cnt) > 0 ? (size_t)(cnt) : 1, sizeof(T)))
#define COPY(dst, src, T, cnt) do { dst = ALLOC(T, cnt); if (src) memcpy(dst, src, sizeof(T) * (size_t)(cnt)); } while (0)

Oracle* or_create(int64_t n, int dim, int L, const int64_t* cols, const int64_t* card,
                  const double* c, const double* m_slot, const double* m_i, const double* inv_m,
                  const double* gas5, double c_cfl, int passes, int newton,
                  int64_t n_inflow, const int64_t* inflow, const double* farfield,
                  int64_t n_slip, const int64_t* slip, const double* slip_n, int nthreads) {
  Oracle* o = ALLOC(Oracle, 1);
  o->n = n; o->dim = dim; o->nvar = dim + 2; o->L = L;
  o->passes = passes; o->newton = newton; o->c_cfl = c_cfl;
  o->g.gamma = gas5[0]; o->g.gm1 = gas5[1]; o->g.gp1_inv = gas5[2];
  o->g.gm1_over_2g = gas5[3]; o->g.two_g_over_gm1 = gas5[4];
  o->nthreads = nthreads > 0 ? nthreads : 1;
  int64_t NL = n * L;
  int nv = o->nvar;
  COPY(o->cols, cols, int64_t, NL);
  COPY(o->card, card, int64_t, n);
  COPY(o->c, c, double, NL * dim);
  COPY(o->m_i, m_i, double, n);
  COPY(o->inv_m, inv_m, double, n);
  o->trow = ALLOC(int64_t, NL); o->tslot = ALLOC(int64_t, NL);
  o->diag = ALLOC(int64_t, n);
  o->valid = ALLOC(uint8_t, NL); o->upper = ALLOC(uint8_t, NL); o->lower = ALLOC(uint8_t, NL);
  o->cT = ALLOC(double, NL * dim); o->b = ALLOC(double, NL); o->bT = ALLOC(double, NL);
  o->lam = ALLOC(double, n);
  /* padded view: sparsity.py:263-309; masks/lam: stepper.py:211-215; b: :234-236 */
  for (int64_t i = 0; i < n; ++i) {
    o->diag[i] = -1;
    for (int s = 0; s < L; ++s) {
      int64_t p = i * L + s;
      int valid = s < card[i];
      o->valid[p] = (uint8_t)valid;
      if (!valid) o->cols[p] = i;
      if (valid && o->cols[p] == i) o->diag[i] = s;
      o->upper[p] = (uint8_t)(valid && o->cols[p] > i);
      o->lower[p] = (uint8_t)(valid && o->cols[p] < i);
    }
    int64_t den = card[i] - 1 > 1 ? card[i] - 1 : 1;
    o->lam[i] = 1.0 / (double)den;
  }
  for (int64_t i = 0; i < n; ++i) {
    for (int s = 0; s < L; ++s) {
      int64_t p = i * L + s;
      if (!o->valid[p]) { o->trow[p] = i; o->tslot[p] = s; continue; }
      int64_t j = o->cols[p];
      int64_t lo = 0, hi = card[j] - 1, t = -1;
      while (lo <= hi) { /* slots of row j are sorted by column */
        int64_t mid = (lo + hi) / 2, cm = o->cols[j * L + mid];
        if (cm == i) { t = mid; break; }
        if (cm < i) lo = mid + 1; else hi = mid - 1;
      }
      if (t < 0) return NULL; /* pattern not structurally symmetric */
      o->trow[p] = j; o->tslot[p] = t;
    }
  }
  for (int64_t p = 0; p < NL; ++p)
    for (int a = 0; a < dim; ++a)
      o->cT[p * dim + a] = o->c[(o->trow[p] * L + o->tslot[p]) * dim + a];
  for (int64_t i = 0; i < n; ++i)
    for (int s = 0; s < L; ++s) {
      int64_t p = i * L + s;
      double delta = (o->cols[p] == i) ? 1.0 : 0.0;
      double ms = o->valid[p] ? m_slot[p] : 0.0;
      o->b[p] = delta - ms * inv_m[o->cols[p]];
      o->bT[p] = delta - ms * inv_m[i];
    }
  o->n_inflow = n_inflow; o->n_slip = n_slip;
  COPY(o->inflow, inflow, int64_t, n_inflow);
  COPY(o->slip, slip, int64_t, n_slip);
  COPY(o->slip_n, slip_n, double, n_slip * dim);
  for (int k = 0; k < nv; ++k) o->farfield[k] = farfield ? farfield[k] : 0.0;
  o->U = ALLOC(double, n * nv); o->U_next = ALLOC(double, n * nv); o->U0 = ALLOC(double, n * nv);
  o->f = ALLOC(double, n * nv * dim);
  o->eor = ALLOC(double, n); o->phi = ALLOC(double, n); o->alpha = ALLOC(double, n);
  o->d = ALLOC(double, NL); o->R = ALLOC(double, n * nv);
  o->P = ALLOC(double, NL * nv); o->l = ALLOC(double, NL); o->l_next = ALLOC(double, NL);
  o->rho_min = ALLOC(double, n); o->rho_max = ALLOC(double, n); o->phi_min = ALLOC(double, n);
  o->tau_last = NAN;
  o->bad_row = -1;
  return o;
}

void or_destroy(Oracle* o) {
  if (!o) return;
  void* ptrs[] = {o->cols, o->trow, o->tslot, o->diag, o->card, o->valid, o->upper, o->lower,
                  o->c, o->cT, o->b, o->bT, o->m_i, o->inv_m, o->lam, o->inflow, o->slip,
                  o->slip_n, o->U, o->U_next, o->U0, o->f, o->eor, o->phi, o->d, o->alpha,
                  o->R, o->P, o->l, o->l_next, o->rho_min, o->rho_max, o->phi_min};
  for (size_t k = 0; k < sizeof ptrs / sizeof ptrs[0]; ++k) free(ptrs[k]);
  free(o);
}

/* U given in CM row order, AoS (n, nvar) */
void or_set_state(Oracle* o, const double* U) {
  memcpy(o->U, U, sizeof(double) * (size_t)(o->n * o->nvar));
  memcpy(o->U_next, U, sizeof(double) * (size_t)(o->n * o->nvar));
}

void or_get_state(const Oracle* o, double* U) {
  memcpy(U, o->U, sizeof(double) * (size_t)(o->n * o->nvar));
}

/* ---- deterministic row-parallel runner (rows are independent in a phase) ---- */
typedef void (*row_fn)(Oracle* o, int64_t lo, int64_t hi, const double* arg, int* err);
typedef struct { Oracle* o; row_fn fn; const double* arg; int64_t lo, hi; int err; } Job;
static void* job_main(void* p) {
  Job* j = (Job*)p;
  j->fn(j->o, j->lo, j->hi, j->arg, &j->err);
  return NULL;
}
static int run_rows(Oracle* o, row_fn fn, const double* arg) {
  int64_t T = o->nthreads;
  if (T > o->n) T = o->n > 0 ? o->n : 1;
  if (T <= 1) { int e = 0; fn(o, 0, o->n, arg, &e); return e; }
  pthread_t th[256];
  Job jobs[256];
  if (T > 256) T = 256;
  int64_t chunk = (o->n + T - 1) / T;
  int64_t started = 0;
  for (int64_t t = 0; t < T; ++t) {
    int64_t lo = t * chunk, hi = lo + chunk < o->n ? lo + chunk : o->n;
    jobs[t].o = o; jobs[t].fn = fn; jobs[t].arg = arg; jobs[t].lo = lo; jobs[t].hi = hi; jobs[t].err = 0;
    if (lo >= hi) continue;
    pthread_create(&th[t], NULL, job_main, &jobs[t]);
    started = t + 1;
  }
  int err = 0;
  for (int64_t t = 0; t < started; ++t) {
    if (jobs[t].lo >= jobs[t].hi) continue;
    pthread_join(th[t], NULL);
    err |= jobs[t].err;
  }
  return err;
}

/* step0: Solver._k_entropies, stepper.py:399-405 */
static void k_entropies_rows(Oracle* o, int64_t lo, int64_t hi, const double* arg, int* err) {
  const int dim = o->dim, nv = o->nvar;
  (void)arg; (void)err;
  for (int64_t i = lo; i < hi; ++i) {
    const double* U = o->U + i * nv;
    double rho = U[0];
    double eps = internal_energy(U, dim);
    o->eor[i] = opow(rho * eps, o->g.gp1_inv) / rho;
    o->phi[i] = eps * opow(rho, -o->g.gamma);
    flux(U, dim, &o->g, o->f + i * nv * dim);
  }
}

/* step1: Solver._k_viscosity(with_alpha=True), stepper.py:407-425;
 * IndicatorAccumulator.reset/accumulate/result, indicator.py:35-73 */
static void k_viscosity_rows(Oracle* o, int64_t lo, int64_t hi, const double* arg, int* errp) {
  const int dim = o->dim, nv = o->nvar, L = o->L;
  const Gas* g = &o->g;
  int err = 0;
  (void)arg;
  for (int64_t i = lo; i < hi; ++i) {
    const double* Ui = o->U + i * nv;
    for (int s = 0; s < L; ++s) {
      int64_t p = i * L + s;
      const double* Uj = o->U + o->cols[p] * nv;
      double dv = d_ij_low(Ui, Uj, o->c + p * dim, o->cT + p * dim, dim, g, &err);
      o->d[p] = o->upper[p] ? dv : 0.0;
    }
    /* reset: harten_entropy (checked, value unused) + derivative */
    double rho = Ui[0];
    double re = rho * internal_energy(Ui, dim);
    if (!(re > 0.0)) err |= 1;
    (void)opow(re, g->gp1_inv);
    double scale = opow(re, (-g->gamma) * g->gp1_inv) * g->gp1_inv;
    double ep[5];
    ep[0] = scale * Ui[dim + 1];
    for (int a = 0; a < dim; ++a) ep[1 + a] = (-scale) * Ui[1 + a];
    ep[dim + 1] = scale * rho;
    double eor_i = o->eor[i];
    const double* fi = o->f + i * nv * dim;
    double A = 0.0, B[5] = {0, 0, 0, 0, 0};
    for (int s = 0; s < L; ++s) {
      int64_t p = i * L + s;
      int64_t j = o->cols[p];
      const double* Uj = o->U + j * nv;
      const double* cc = o->c + p * dim;
      A += (o->eor[j] - eor_i) * r1_dot(Uj + 1, cc, dim);
      const double* fj = o->f + j * nv * dim;
      for (int k = 0; k < nv; ++k) {
        double t = 0.0;
        for (int a = 0; a < dim; ++a) t += (fj[k * dim + a] - fi[k * dim + a]) * cc[a];
        B[k] += t;
      }
    }
    double eb = 0.0;
    for (int k = 0; k < nv; ++k) eb += ep[k] * B[k];
    double numer = fabs((A - eb) + (eor_i * B[0]));
    double w[5];
    for (int k = 0; k < nv; ++k) w[k] = fabs(ep[k]);
    w[0] = fabs(ep[0] - eor_i);
    double wb = 0.0;
    for (int k = 0; k < nv; ++k) wb += w[k] * fabs(B[k]);
    double denom = fabs(A) + wb;
    double safe = denom > DENOM_FLOOR ? denom : 1.0;
    double al = np_clip(numer / safe, 0.0, 1.0);
    o->alpha[i] = denom > DENOM_FLOOR ? al : 0.0;
  }
  *errp |= err;
}

/* step2: Solver._k_mirror, stepper.py:427-434; tau: :538-548, _tau_local :66-70 */
static void k_mirror_rows(Oracle* o, int64_t lo, int64_t hi, const double* dd_, int* err) {
  const int L = o->L;
  double* dd = (double*)dd_;
  (void)err;
  for (int64_t i = lo; i < hi; ++i) {
    double* row = dd + i * L;
    for (int s = 0; s < L; ++s) {
      int64_t p = i * L + s;
      row[s] = o->lower[p] ? o->d[o->trow[p] * L + o->tslot[p]] : o->d[p];
    }
    double rowsum = np_pairwise_sum(row, L);
    row[o->diag[i]] = -rowsum;
  }
}

static double k_mirror(Oracle* o) {
  const int L = o->L;
  double tau_min = INFINITY;
  double* dd = ALLOC(double, o->n * L);
  run_rows(o, k_mirror_rows, dd);
  memcpy(o->d, dd, sizeof(double) * (size_t)(o->n * L));
  free(dd);
  for (int64_t i = 0; i < o->n; ++i) {
    double dii = o->d[i * L + o->diag[i]];
    if (dii < 0.0) tau_min = np_min(tau_min, o->m_i[i] / (-2.0 * dii));
  }
  return tau_min;
}

/* step3: Solver._k_low_order, stepper.py:436-454 */
static void k_low_order_rows(Oracle* o, int64_t lo, int64_t hi, const double* arg, int* err) {
  const int dim = o->dim, nv = o->nvar, L = o->L;
  const double tau = arg[0];
  (void)err;
  for (int64_t i = lo; i < hi; ++i) {
    const double* Ui = o->U + i * nv;
    const double* fi = o->f + i * nv * dim;
    double sumL[5] = {0, 0, 0, 0, 0}, sumR[5] = {0, 0, 0, 0, 0};
    double rmin = 0, rmax = 0, pmin = 0;
    double ai = o->alpha[i];
    for (int s = 0; s < L; ++s) {
      int64_t p = i * L + s;
      int64_t j = o->cols[p];
      const double* Uj = o->U + j * nv;
      const double* fj = o->f + j * nv * dim;
      const double* cc = o->c + p * dim;
      double dv = o->d[p];
      double dH = dv * (0.5 * (ai + o->alpha[j]));
      double ubar0 = 0;
      for (int k = 0; k < nv; ++k) {
        double dU = Uj[k] - Ui[k];
        double fdc = 0.0;
        for (int a = 0; a < dim; ++a) fdc += (fj[k * dim + a] - fi[k * dim + a]) * cc[a];
        sumL[k] += dv * dU - fdc;
        sumR[k] += dH * dU - fdc;
        if (k == 0) {
          double corr = dv != 0.0 ? fdc / (2.0 * dv) : 0.0;
          ubar0 = (0.5 * (Ui[0] + Uj[0])) - corr;
        }
      }
      if (s == 0) { rmin = ubar0; rmax = ubar0; pmin = o->phi[j]; }
      else { rmin = np_min(rmin, ubar0); rmax = np_max(rmax, ubar0); pmin = np_min(pmin, o->phi[j]); }
    }
    double fac = tau * o->inv_m[i];
    for (int k = 0; k < nv; ++k) {
      o->U_next[i * nv + k] = Ui[k] + fac * sumL[k];
      o->R[i * nv + k] = sumR[k];
    }
    o->rho_min[i] = rmin; o->rho_max[i] = rmax; o->phi_min[i] = pmin;
  }
}

/* step4: Solver._k_correction, stepper.py:456-474 */
static void k_correction_rows(Oracle* o, int64_t lo, int64_t hi, const double* arg, int* err) {
  const int dim = o->dim, nv = o->nvar, L = o->L;
  const double tau = arg[0];
  (void)err;
  for (int64_t i = lo; i < hi; ++i) {
    const double* Ui = o->U + i * nv;
    const double* Ri = o->R + i * nv;
    double ai = o->alpha[i];
    double factor = (tau * o->inv_m[i]) * (double)(o->card[i] - 1);
    for (int s = 0; s < L; ++s) {
      int64_t p = i * L + s;
      int64_t j = o->cols[p];
      double dv = o->d[p];
      double dH = dv * (0.5 * (ai + o->alpha[j]));
      double* P = o->P + p * nv;
      for (int k = 0; k < nv; ++k) {
        double dU = o->U[j * nv + k] - Ui[k];
        double K = ((o->b[p] * o->R[j * nv + k]) - (o->bT[p] * Ri[k])) + ((dH - dv) * dU);
        P[k] = factor * K;
      }
      o->l[p] = limiter_lane(o->U_next + i * nv, P, o->rho_min[i], o->rho_max[i], o->phi_min[i],
                             o->newton, dim, &o->g);
    }
  }
}

/* Solver._k_boundary, stepper.py:493-504.  numpy fancy-index semantics: every
 * slip row is projected from its pre-boundary momentum, then assigned in list
 * order (duplicates: last wins); inflow rows are reset afterwards. */
static void apply_boundary(Oracle* o) {
  const int dim = o->dim, nv = o->nvar;
  double* mom = ALLOC(double, o->n_slip * dim);
  for (int64_t q = 0; q < o->n_slip; ++q) {
    const double* Un = o->U_next + o->slip[q] * nv;
    const double* nr = o->slip_n + q * dim;
    double mn = 0.0;
    for (int a = 0; a < dim; ++a) mn += Un[1 + a] * nr[a];
    for (int a = 0; a < dim; ++a) mom[q * dim + a] = Un[1 + a] - mn * nr[a];
  }
  for (int64_t q = 0; q < o->n_slip; ++q)
    for (int a = 0; a < dim; ++a) o->U_next[o->slip[q] * nv + 1 + a] = mom[q * dim + a];
  free(mom);
  for (int64_t q = 0; q < o->n_inflow; ++q)
    for (int k = 0; k < nv; ++k) o->U_next[o->inflow[q] * nv + k] = o->farfield[k];
}

/* steps 5/6: Solver._k_limited_update, stepper.py:476-491; _k_boundary :493-504 */
static void k_limited_rows(Oracle* o, int64_t lo, int64_t hi, const double* arg, int* err) {
  const int dim = o->dim, nv = o->nvar, L = o->L;
  const int last = arg[0] != 0.0;
  (void)err;
  for (int64_t i = lo; i < hi; ++i) {
    double upd[5] = {0, 0, 0, 0, 0};
    for (int s = 0; s < L; ++s) {
      int64_t p = i * L + s;
      double lT = o->l[o->trow[p] * L + o->tslot[p]];
      double minl = np_min(o->l[p], lT);
      for (int k = 0; k < nv; ++k) upd[k] += minl * o->P[p * nv + k];
    }
    double* Un = o->U_next + i * nv;
    for (int k = 0; k < nv; ++k) Un[k] = Un[k] + o->lam[i] * upd[k];
    if (!last) {
      for (int s = 0; s < L; ++s) {
        int64_t p = i * L + s;
        double lT = o->l[o->trow[p] * L + o->tslot[p]];
        double minl = np_min(o->l[p], lT);
        double* P = o->P + p * nv;
        for (int k = 0; k < nv; ++k) P[k] = P[k] * (1.0 - minl);
        o->l_next[p] = limiter_lane(Un, P, o->rho_min[i], o->rho_max[i], o->phi_min[i],
                                    o->newton, dim, &o->g);
      }
    }
  }
}

static void k_limited_update(Oracle* o, int last) {
  double arg = last ? 1.0 : 0.0;
  run_rows(o, k_limited_rows, &arg);
  if (last) {
    apply_boundary(o);
  } else {
    double* t = o->l; o->l = o->l_next; o->l_next = t;
  }
}

/* Solver._finish_step, stepper.py:612-622 */
static int finish_step(Oracle* o) {
  double* t = o->U; o->U = o->U_next; o->U_next = t;
  for (int64_t i = 0; i < o->n; ++i) {
    const double* U = o->U + i * o->nvar;
    if (!((U[0] > 0.0) && (internal_energy(U, o->dim) > 0.0))) { o->bad_row = i; return OR_BAD_STATE; }
  }
  return OR_OK;
}

/* Solver.euler_step, stepper.py:508-610.  Returns a status; *tau_out = tau used. */
int or_euler_step(Oracle* o, int has_tau, double tau, double tau_max, double* tau_out) {
  run_rows(o, k_entropies_rows, NULL);
  if (run_rows(o, k_viscosity_rows, NULL)) return OR_ADMISSIBILITY;
  double tau_min = k_mirror(o);
  if (!has_tau) {
    if (!isfinite(tau_min)) return OR_TAU_UNBOUNDED;
    double a = o->c_cfl * tau_min;
    tau = (tau_max < a) ? tau_max : a; /* python min(a, tau_max) */
  }
  o->tau_last = tau;
  *tau_out = tau;
  run_rows(o, k_low_order_rows, &tau);
  if (o->passes == 0) {
    apply_boundary(o);
    return finish_step(o);
  }
  run_rows(o, k_correction_rows, &tau);
  for (int p = 0; p < o->passes; ++p) k_limited_update(o, p == o->passes - 1);
  return finish_step(o);
}

/* Solver.ssp_rk3_step, stepper.py:624-636 */
int or_ssp_rk3_step(Oracle* o, int has_tau, double tau, double tau_max, double* tau_out) {
  const int64_t cnt = o->n * o->nvar;
  memcpy(o->U0, o->U, sizeof(double) * (size_t)cnt);
  double t;
  int st = or_euler_step(o, has_tau, tau, tau_max, &t);
  if (st) return st;
  *tau_out = t;
  double t2;
  st = or_euler_step(o, 1, t, INFINITY, &t2);
  if (st) return st;
  for (int64_t q = 0; q < cnt; ++q) o->U[q] = o->U0[q] + 0.25 * (o->U[q] - o->U0[q]);
  st = or_euler_step(o, 1, t, INFINITY, &t2);
  if (st) return st;
  for (int64_t q = 0; q < cnt; ++q) o->U[q] = o->U0[q] + (2.0 / 3.0) * (o->U[q] - o->U0[q]);
  return OR_OK;
}

int64_t or_bad_row(const Oracle* o) { return o->bad_row; }
double or_tau_last(const Oracle* o) { return o->tau_last; }
void or_set_threads(Oracle* o, int nthreads) { o->nthreads = nthreads > 0 ? nthreads : 1; }

/* Intermediates for per-phase parity: 0 d (n*L), 1 alpha (n), 2 R (n*nvar),
 * 3 bounds (n*3: rho_min, rho_max, phi_min), 4 l (n*L, current), 5 eor (n), 6 phi (n),
 * 7 U_next (n*nvar), 8 P (n*L*nvar) */
int or_fetch(const Oracle* o, int which, double* out) {
  const int64_t n = o->n, L = o->L, nv = o->nvar;
  switch (which) {
    case 0: memcpy(out, o->d, sizeof(double) * (size_t)(n * L)); return 0;
    case 1: memcpy(out, o->alpha, sizeof(double) * (size_t)n); return 0;
    case 2: memcpy(out, o->R, sizeof(double) * (size_t)(n * nv)); return 0;
    case 3:
      for (int64_t i = 0; i < n; ++i) {
        out[3 * i] = o->rho_min[i]; out[3 * i + 1] = o->rho_max[i]; out[3 * i + 2] = o->phi_min[i];
      }
      return 0;
    case 4: memcpy(out, o->l, sizeof(double) * (size_t)(n * L)); return 0;
    case 5: memcpy(out, o->eor, sizeof(double) * (size_t)n); return 0;
    case 6: memcpy(out, o->phi, sizeof(double) * (size_t)n); return 0;
    case 7: memcpy(out, o->U_next, sizeof(double) * (size_t)(n * nv)); return 0;
    case 8: memcpy(out, o->P, sizeof(double) * (size_t)(n * L * nv)); return 0;
  }
  return -1;
}

/* host build of the shared pow, installed into the reference by the harness */
void or_pow(const double* x, double y, double* out, int64_t n) {
  for (int64_t q = 0; q < n; ++q) out[q] = ef_pow(x[q], y);
}
void or_pow2(const double* x, const double* y, double* out, int64_t n) {
  for (int64_t q = 0; q < n; ++q) out[q] = ef_pow(x[q], y[q]);
}

/* Function-level checks (riemann.d_ij_low, limiter.limiter_compute) on batches of
 * independent inputs; the tests compare them with the reference's functions and
 * with the device path (ef_eval_dij / ef_eval_limiter). */
void or_eval_dij(int dim, double gamma, double gm1, double gp1_inv, double gm1_over_2g,
                 double two_g_over_gm1, int64_t n, const double* Ui, const double* Uj,
                 const double* cij, const double* cji, double* out, int32_t* err) {
  Gas g = {gamma, gm1, gp1_inv, gm1_over_2g, two_g_over_gm1};
  const int nv = dim + 2;
  for (int64_t q = 0; q < n; ++q) {
    int e = 0;
    out[q] = d_ij_low(Ui + q * nv, Uj + q * nv, cij + q * dim, cji + q * dim, dim, &g, &e);
    err[q] = e;
  }
}

void or_eval_limiter(int dim, double gamma, double gm1, double gp1_inv, double gm1_over_2g,
                     double two_g_over_gm1, int64_t n, const double* U, const double* P,
                     const double* bounds, int newton, double* out) {
  Gas g = {gamma, gm1, gp1_inv, gm1_over_2g, two_g_over_gm1};
  const int nv = dim + 2;
  for (int64_t q = 0; q < n; ++q)
    out[q] = limiter_lane(U + q * nv, P + q * nv, bounds[3 * q], bounds[3 * q + 1], bounds[3 * q + 2],
                          newton, dim, &g);
}
