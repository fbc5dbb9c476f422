/*
 * oracle.c — plain, slow, obviously-correct CPU oracle of the particle half of
 * the implicit-moment PIC cycle (arXiv 2507.20719, iPIC3D).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (libpic, paper_2507_20719_b200/) never links, imports or
 * calls it, and this file includes no header of the product path.
 *
 * fp64 throughout, compiled with -O2 -ffp-contract=off (no FMA contraction, no
 * fast-math) so every operation below is one IEEE-754 rounding in the order
 * written.  One particle at a time, in input order; no blocking, no fusion,
 * no reordering beyond what the equations state.
 *
 * Passages followed (PAPER.md line numbers, /root/reference/PAPER.md):
 *   Eq. 1   PAPER.md:141-145  equations of motion (hot path: gamma == 1)
 *   Eq. 2   PAPER.md:149-165  predictor-corrector mover, fixed-point on v-bar
 *   Eq. 3   PAPER.md:184-187  moments {rho, J, Pi}_g = sum_p q {1, v, vv} W
 *   Alg. 1  PAPER.md:291-334  phase order: mover, then interpolation
 *   §III-B  PAPER.md:235-236  open boundaries: particles leaving are removed
 *   Eq. 5-6 PAPER.md:199-213  susceptibility chi and corrected rho-hat, J-hat
 *                             (NEXT-2, the first consumer of the moments)
 *   §III-B  PAPER.md:232-233  inflow injection of wind particles with a
 *                             prescribed bulk velocity (NEXT-3, reading R28)
 *   §III-B  PAPER.md:238-245  particle control: splitting and pair-wise
 *                             coalescence (NEXT-3, readings R29-R31)
 *   §III-D  PAPER.md:368-372  velocity binning and the Gaussian-mixture fit by
 *                             EM (NEXT-4, readings R32-R33)
 * Readings where the paper is silent or garbled are R1..R23 in DESIGN.md §3
 * (taken from SURVEY.md §8(c)); each use below names its reading.
 *
 * Pins (tests/test_oracle_pins.py) tie every function here to closed forms:
 * free streaming, gyration angle/radius, ExB drift, uniform-E kick, the
 * linear-field worked example, node/cell-centre stencils, global sums,
 * gather/scatter adjointness, lattice loading and exact-rational brute force;
 * the R11 clamp branch of oracle_sample by the closed form of a linear field
 * at the clamped point (test_sample_clamp_branch_linear_field_closed_form).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

/* ---------------------------------------------------------------- types -- */

/* Global grid: cells [0, ncell) per axis, origin 0, Delta = len / ncell.   */
typedef struct {
  int64_t ncell[3];
  double  len[3];
  int32_t bc[3];            /* 0 = periodic, 1 = open                       */
  double  dt, c;
  double  planet_center[3];
  double  planet_radius;    /* 0 = no absorbing body                        */
} oracle_grid;

/* Field window: node-interleaved E,B on global node indices
 * [lo_d, lo_d + n_d) per axis, layout EB[k][j][i][6] = Ex Ey Ez Bx By Bz.
 * Periodic images are replicated by the caller (the window is plain data). */
typedef struct {
  int64_t lo[3];
  int64_t n[3];
  const double *EB;
} oracle_field;

enum { ORACLE_ALIVE = 0, ORACLE_REMOVED = 1, ORACLE_BAD = 2 };

/* ------------------------------------------------------- field sampling -- */

/* Trilinear interpolation W of E and B at position p (R12):
 * xi = (p - lo*Delta)/Delta, i = floor(xi), f = xi - i, weights (1-f, f) per
 * axis, product over axes.  Outside the window xi is clamped to the window
 * (constant extension, R11).  Returns 1 if a clamp happened.                */
int oracle_sample(const oracle_grid *g, const oracle_field *F,
                  const double p[3], double out[6]) {
  int64_t idx[3];
  double f[3];
  int clamped = 0;
  for (int d = 0; d < 3; ++d) {
    double delta = g->len[d] / (double)g->ncell[d];
    double xi = p[d] / delta - (double)F->lo[d];
    double top = (double)(F->n[d] - 1);
    if (!(xi >= 0.0)) { xi = 0.0; clamped = 1; }     /* also catches NaN */
    if (xi > top) { xi = top; clamped = 1; }
    double fl = floor(xi);
    if (fl > top - 1.0) fl = top - 1.0;
    idx[d] = (int64_t)fl;
    f[d] = xi - fl;
  }
  for (int m = 0; m < 6; ++m) out[m] = 0.0;
  for (int c = 0; c < 8; ++c) {
    int bx = c & 1, by = (c >> 1) & 1, bz = (c >> 2) & 1;
    double wx = bx ? f[0] : 1.0 - f[0];
    double wy = by ? f[1] : 1.0 - f[1];
    double wz = bz ? f[2] : 1.0 - f[2];
    double S = wx * wy * wz;
    int64_t i = idx[0] + bx, j = idx[1] + by, k = idx[2] + bz;
    const double *node = F->EB + 6 * ((k * F->n[1] + j) * F->n[0] + i);
    for (int m = 0; m < 6; ++m) out[m] += S * node[m];
  }
  return clamped;
}

/* ------------------------------------------------------------- the mover -- */

/* Boundary treatment after the push (R10, R11, R21).
 * Periodic: one wrap, x >= L -> x - L; x < 0 -> x + L (and L -> 0).
 * Open: outside [0, L) on any open axis, or inside the planet -> removed.   */
static int apply_bc(const oracle_grid *g, double x[3]) {
  int status = ORACLE_ALIVE;
  for (int d = 0; d < 3; ++d) {
    double L = g->len[d];
    if (g->bc[d] == 0) {
      if (x[d] >= L) {
        x[d] = x[d] - L;
      } else if (x[d] < 0.0) {
        x[d] = x[d] + L;
        if (x[d] == L) x[d] = 0.0;
      }
      if (!(x[d] >= 0.0 && x[d] < L)) status = ORACLE_BAD;   /* > one wrap */
    } else {
      if (!(x[d] >= 0.0 && x[d] < L)) {
        if (status == ORACLE_ALIVE) status = ORACLE_REMOVED;
        if (x[d] != x[d]) status = ORACLE_BAD;
      }
    }
  }
  if (status == ORACLE_ALIVE && g->planet_radius > 0.0) {
    double r2 = 0.0;
    for (int d = 0; d < 3; ++d) {
      double dx = x[d] - g->planet_center[d];
      r2 += dx * dx;
    }
    if (r2 < g->planet_radius * g->planet_radius) status = ORACLE_REMOVED;
  }
  return status;
}

/* Eq. 2 in the gamma == 1 limit (R3), one particle:
 *   xb <- xn                                   (R1: first sample at x^n)
 *   repeat n_iter times, no early exit         (R2)
 *     (E,B) <- W(xb)                           (R12)
 *     vt    <- vn + (q/m)(dt/2) E              (Eq. 2 line 3, R7)
 *     a     <- (q/m)(dt/2) B / c   = Omega dt/2 (R8: q signed)
 *     vb    <- (vt + vt x a + (vt.a) a) / (1 + a.a)   (Eq. 2 line 4, D)
 *     xb    <- xn + vb dt/2
 *   x^{n+1} <- xn + vb dt ;  v^{n+1} <- 2 vb - vn     (Eq. 2 lines 1-2)
 *   boundary conditions                                                    */
static int push_one(const oracle_grid *g, const oracle_field *F, double qom,
                    int n_iter, double xn[3], double vn[3]) {
  double ks = qom * (g->dt / 2.0);
  double xb[3] = {xn[0], xn[1], xn[2]};
  double vb[3] = {vn[0], vn[1], vn[2]};
  for (int it = 0; it < n_iter; ++it) {
    double EB[6];
    oracle_sample(g, F, xb, EB);
    double vt[3], a[3];
    for (int d = 0; d < 3; ++d) vt[d] = vn[d] + ks * EB[d];
    for (int d = 0; d < 3; ++d) a[d] = (ks / g->c) * EB[3 + d];
    double cross[3];
    cross[0] = vt[1] * a[2] - vt[2] * a[1];
    cross[1] = vt[2] * a[0] - vt[0] * a[2];
    cross[2] = vt[0] * a[1] - vt[1] * a[0];
    double dot = vt[0] * a[0] + vt[1] * a[1] + vt[2] * a[2];
    double D = 1.0 + (a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    for (int d = 0; d < 3; ++d) vb[d] = (vt[d] + cross[d] + dot * a[d]) / D;
    for (int d = 0; d < 3; ++d) xb[d] = xn[d] + vb[d] * (g->dt / 2.0);
  }
  for (int d = 0; d < 3; ++d) {
    double v_new = 2.0 * vb[d] - vn[d];
    xn[d] = xn[d] + vb[d] * g->dt;
    vn[d] = v_new;
  }
  int status = apply_bc(g, xn);
  for (int d = 0; d < 3; ++d)
    if (!(vn[d] == vn[d]) || isinf(vn[d])) status = ORACLE_BAD;
  return status;
}

/* Eq. 2, relativistic form (NEXT-1), one particle.
 * Velocities v are stored; gamma = 1 / sqrt(1 - |v|^2 / c^2).
 *   gn  <- gamma(vn) ; un <- gn vn ; gt <- gn   (R5: gamma-tilde starts at gamma^n)
 *   xb  <- xn                                    (R1)
 *   repeat n_iter times                          (R2)
 *     (E,B) <- W(xb)                             (R12)
 *     vt    <- gn vn + (q/m)(dt/2) E             (Eq. 2 line 3)
 *     a     <- (dt/(2 gt)) Omega, Omega = (q/(m c)) B          (R8)
 *     D     <- gt (1 + a.a)                      (R6)
 *     vb    <- (vt + vt x a + (vt.a) a) / D      (Eq. 2 line 4; the GC term
 *              with (dt/(2 gt))^2 (vt.Omega) Omega, R4's derived factor)
 *     u1    <- 2 gt vb - gn vn ; g1 <- sqrt(1 + u1.u1 / c^2)   (R5)
 *     gt    <- (gn + g1) / 2
 *     xb    <- xn + vb dt/2
 *   x^{n+1} <- xn + vb dt ; v^{n+1} <- u1 / g1   (Eq. 2 lines 1-2, R5)
 *   boundary conditions.  |vn| >= c makes gn non-finite: ORACLE_BAD (R23). */
static int push_one_rel(const oracle_grid *g, const oracle_field *F, double qom,
                        int n_iter, double xn[3], double vn[3]) {
  double c = g->c;
  double v2 = vn[0] * vn[0] + vn[1] * vn[1] + vn[2] * vn[2];
  double gn = 1.0 / sqrt(1.0 - v2 / (c * c));
  double gt = gn;
  double xb[3] = {xn[0], xn[1], xn[2]};
  double vb[3] = {vn[0], vn[1], vn[2]};
  double u1[3] = {gn * vn[0], gn * vn[1], gn * vn[2]};
  double g1 = gn;
  for (int it = 0; it < n_iter; ++it) {
    double EB[6];
    oracle_sample(g, F, xb, EB);
    double vt[3], a[3];
    for (int d = 0; d < 3; ++d) vt[d] = gn * vn[d] + qom * (g->dt / 2.0) * EB[d];
    for (int d = 0; d < 3; ++d) a[d] = (g->dt / (2.0 * gt)) * ((qom / c) * EB[3 + d]);
    double cross[3];
    cross[0] = vt[1] * a[2] - vt[2] * a[1];
    cross[1] = vt[2] * a[0] - vt[0] * a[2];
    cross[2] = vt[0] * a[1] - vt[1] * a[0];
    double dot = vt[0] * a[0] + vt[1] * a[1] + vt[2] * a[2];
    double D = gt * (1.0 + (a[0] * a[0] + a[1] * a[1] + a[2] * a[2]));
    for (int d = 0; d < 3; ++d) vb[d] = (vt[d] + cross[d] + dot * a[d]) / D;
    for (int d = 0; d < 3; ++d) u1[d] = 2.0 * gt * vb[d] - gn * vn[d];
    g1 = sqrt(1.0 + (u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]) / (c * c));
    gt = (gn + g1) / 2.0;
    for (int d = 0; d < 3; ++d) xb[d] = xn[d] + vb[d] * (g->dt / 2.0);
  }
  for (int d = 0; d < 3; ++d) {
    xn[d] = xn[d] + vb[d] * g->dt;
    vn[d] = u1[d] / g1;
  }
  int status = apply_bc(g, xn);
  for (int d = 0; d < 3; ++d)
    if (!(vn[d] == vn[d]) || isinf(vn[d]) || !(xn[d] == xn[d])) status = ORACLE_BAD;
  return status;
}

/* Mover over np particles of one species (SoA, updated in place).  status[p]
 * on entry: ORACLE_ALIVE particles are pushed, others are skipped.  Returns
 * the number of particles whose status became ORACLE_BAD.                   */
int64_t oracle_mover_ex(const oracle_grid *g, const oracle_field *F, double qom,
                        int n_iter, int relativistic, int64_t np, double *x, double *y,
                        double *z, double *u, double *v, double *w, int8_t *status) {
  int64_t bad = 0;
  for (int64_t p = 0; p < np; ++p) {
    if (status[p] != ORACLE_ALIVE) continue;
    double xn[3] = {x[p], y[p], z[p]};
    double vn[3] = {u[p], v[p], w[p]};
    int s = relativistic ? push_one_rel(g, F, qom, n_iter, xn, vn)
                         : push_one(g, F, qom, n_iter, xn, vn);
    x[p] = xn[0]; y[p] = xn[1]; z[p] = xn[2];
    u[p] = vn[0]; v[p] = vn[1]; w[p] = vn[2];
    status[p] = (int8_t)s;
    if (s == ORACLE_BAD) ++bad;
  }
  return bad;
}

int64_t oracle_mover(const oracle_grid *g, const oracle_field *F, double qom,
                     int n_iter, int64_t np, double *x, double *y, double *z,
                     double *u, double *v, double *w, int8_t *status) {
  return oracle_mover_ex(g, F, qom, n_iter, 0, np, x, y, z, u, v, w, status);
}

/* ----------------------------------------------------------- the moments -- */

/* Number of unique nodes per axis (R18): periodic N (node N == node 0),
 * open N + 1.                                                               */
static int64_t nodes_axis(const oracle_grid *g, int d) {
  return g->bc[d] == 0 ? g->ncell[d] : g->ncell[d] + 1;
}

/* Eq. 3 for one species, over alive particles in input
 * order (R15), into mom[10][nz][ny][nx] on the unique node set (R18):
 *   rho += q S / V ; J += q v S / V ; Pi_ab += q v_a v_b S / V
 * with S the trilinear weight of the corner (R12), V = dx dy dz (R13), q the
 * per-particle charge q_s w_p (R14), Pi in order xx xy xz yy yz zz (R16).
 * absmom (may be NULL) accumulates |each contribution| for the R19 bound.
 * mom/absmom are accumulated into (caller zeroes them).  Returns the number
 * of particles whose stencil left the grid (only possible for bad input).  */
int64_t oracle_moments(const oracle_grid *g, int64_t np, const double *x,
                       const double *y, const double *z, const double *u,
                       const double *v, const double *w, const double *q,
                       const int8_t *status, double *mom, double *absmom) {
  int64_t nn[3] = {nodes_axis(g, 0), nodes_axis(g, 1), nodes_axis(g, 2)};
  int64_t plane = nn[0] * nn[1] * nn[2];
  double delta[3], V = 1.0;
  for (int d = 0; d < 3; ++d) {
    delta[d] = g->len[d] / (double)g->ncell[d];
  }
  V = delta[0] * delta[1] * delta[2];
  int64_t outside = 0;
  for (int64_t p = 0; p < np; ++p) {
    if (status && status[p] != ORACLE_ALIVE) continue;
    double pos[3] = {x[p], y[p], z[p]};
    double vel[3] = {u[p], v[p], w[p]};
    int64_t idx[3];
    double f[3];
    int ok = 1;
    for (int d = 0; d < 3; ++d) {
      double xi = pos[d] / delta[d];
      double fl = floor(xi);
      idx[d] = (int64_t)fl;
      f[d] = xi - fl;
      if (idx[d] < 0 || idx[d] >= g->ncell[d]) ok = 0;
    }
    if (!ok) { ++outside; continue; }
    double val[10];
    val[0] = 1.0;
    val[1] = vel[0]; val[2] = vel[1]; val[3] = vel[2];
    val[4] = vel[0] * vel[0]; val[5] = vel[0] * vel[1]; val[6] = vel[0] * vel[2];
    val[7] = vel[1] * vel[1]; val[8] = vel[1] * vel[2]; val[9] = vel[2] * vel[2];
    for (int c = 0; c < 8; ++c) {
      int bx = c & 1, by = (c >> 1) & 1, bz = (c >> 2) & 1;
      double wx = bx ? f[0] : 1.0 - f[0];
      double wy = by ? f[1] : 1.0 - f[1];
      double wz = bz ? f[2] : 1.0 - f[2];
      double S = wx * wy * wz;
      int64_t i = idx[0] + bx, j = idx[1] + by, k = idx[2] + bz;
      if (g->bc[0] == 0 && i == nn[0]) i = 0;     /* R18 periodic fold */
      if (g->bc[1] == 0 && j == nn[1]) j = 0;
      if (g->bc[2] == 0 && k == nn[2]) k = 0;
      int64_t node = (k * nn[1] + j) * nn[0] + i;
      double qs = q[p] * S / V;
      for (int m = 0; m < 10; ++m) {
        double contrib = qs * val[m];
        mom[m * plane + node] += contrib;
        if (absmom) absmom[m * plane + node] += fabs(contrib);
      }
    }
  }
  return outside;
}

/* ------------------------------------------ all-cores timing build only -- */
#ifdef _OPENMP
#include <omp.h>
/* the oracle timed on all host cores for bench.py's
 * cpu_baseline.  Compiled only into the OpenMP build of this same source
 * (liboracle_omp.so); the parity checker is the single-threaded build.
 * Neither wrapper changes the arithmetic: the mover runs oracle_mover_ex on
 * contiguous particle ranges, one per thread (every particle is independent,
 * so the result is bit-identical); the moments run oracle_moments on the same
 * ranges into per-thread node grids that are then added in thread order (a
 * fixed order: the result equals the sequential sum up to reassociation,
 * within R19).                                                              */
/* every host core, whatever the caller's OpenMP runtime was told (torch sets
 * the process-wide thread count of the shared libgomp) */
int oracle_omp_threads(void) { return omp_get_num_procs(); }

int64_t oracle_mover_par(const oracle_grid *g, const oracle_field *F, double qom, int n_iter, int relativistic,
                         int64_t np, double *x, double *y, double *z, double *u, double *v, double *w,
                         int8_t *status) {
  int64_t bad = 0;
  const int T = oracle_omp_threads();
#pragma omp parallel for num_threads(T) schedule(static, 1) reduction(+ : bad)
  for (int t = 0; t < T; ++t) {
    const int64_t a = np * t / T, b = np * (t + 1) / T;
    bad += oracle_mover_ex(g, F, qom, n_iter, relativistic, b - a, x + a, y + a, z + a, u + a, v + a, w + a,
                           status + a);
  }
  return bad;
}

int64_t oracle_moments_par(const oracle_grid *g, int64_t np, const double *x, const double *y, const double *z,
                           const double *u, const double *v, const double *w, const double *q,
                           const int8_t *status, double *mom) {
  const int64_t nn[3] = {nodes_axis(g, 0), nodes_axis(g, 1), nodes_axis(g, 2)};
  const int64_t plane = nn[0] * nn[1] * nn[2], M = 10 * plane;
  const int T = oracle_omp_threads();
  double **grid = (double **)calloc((size_t)T, sizeof(double *));
  /* node indices each thread touched, per axis (a cell and the next node,
   * periodic wrap included): the merge reads only their product, so a sample
   * that occupies a few planes of a large grid costs no full-grid pass; the
   * per-thread grids are calloc'ed, i.e. untouched pages are never materialised */
  unsigned char **touched = (unsigned char **)calloc((size_t)T, sizeof(unsigned char *));
  const double *pos[3] = {x, y, z};
  int64_t outside = 0;
#pragma omp parallel for num_threads(T) schedule(static, 1) reduction(+ : outside)
  for (int t = 0; t < T; ++t) {
    const int64_t a = np * t / T, b = np * (t + 1) / T;
    grid[t] = (double *)calloc((size_t)M, sizeof(double));
    touched[t] = (unsigned char *)calloc((size_t)(nn[0] + nn[1] + nn[2]), 1);
    outside += oracle_moments(g, b - a, x + a, y + a, z + a, u + a, v + a, w + a, q + a,
                              status ? status + a : NULL, grid[t], NULL);
    unsigned char *tc = touched[t];
    for (int d = 0, o = 0; d < 3; o += (int)nn[d], ++d) {
      const double dl = g->len[d] / (double)g->ncell[d];
      for (int64_t p = a; p < b; ++p) {
        if (status && status[p] != ORACLE_ALIVE) continue;
        int64_t c = (int64_t)floor(pos[d][p] / dl);
        if (c < 0 || c >= g->ncell[d]) continue;
        tc[o + c] = 1;
        tc[o + ((g->bc[d] == 0 && c + 1 == nn[d]) ? 0 : c + 1)] = 1;
      }
    }
  }
  /* merge in thread order (every node adds threads 0, 1, ... in turn) */
  for (int t = 0; t < T; ++t) {
    const unsigned char *tx = touched[t], *ty = tx + nn[0], *tz = ty + nn[1];
#pragma omp parallel for num_threads(T) schedule(static)
    for (int64_t k = 0; k < nn[2]; ++k) {
      if (!tz[k]) continue;
      for (int64_t j = 0; j < nn[1]; ++j) {
        if (!ty[j]) continue;
        for (int64_t i = 0; i < nn[0]; ++i) {
          if (!tx[i]) continue;
          const int64_t node = (k * nn[1] + j) * nn[0] + i;
          for (int m = 0; m < 10; ++m) mom[m * plane + node] += grid[t][m * plane + node];
        }
      }
    }
  }
  for (int t = 0; t < T; ++t) {
    free(grid[t]);
    free(touched[t]);
  }
  free(grid);
  free(touched);
  return outside;
}
#endif

/* Convenience for tests: unique node counts per axis.                      */
void oracle_node_counts(const oracle_grid *g, int64_t out[3]) {
  for (int d = 0; d < 3; ++d) out[d] = nodes_axis(g, d);
}

/* ------------------------------------------- NEXT-2: chi, rho-hat, J-hat -- */

/* d f / d x_axis at node (i,j,k) of a unique-node array f[nz][ny][nx]:
 * second-order central difference, periodic wrap on periodic axes; one-sided
 * first-order difference at the two boundary nodes of an open axis (R27).   */
static double node_diff(const oracle_grid *g, const double *f, const int64_t nn[3], int64_t i,
                        int64_t j, int64_t k, int axis) {
  int64_t c[3] = {i, j, k};
  int64_t n = nn[axis];
  double delta = g->len[axis] / (double)g->ncell[axis];
  int64_t lo[3] = {c[0], c[1], c[2]}, hi[3] = {c[0], c[1], c[2]};
  double h = 2.0 * delta;
  if (g->bc[axis] == 0) {
    lo[axis] = (c[axis] - 1 + n) % n;
    hi[axis] = (c[axis] + 1) % n;
  } else if (c[axis] == 0) {
    hi[axis] = 1;
    h = delta;
  } else if (c[axis] == n - 1) {
    lo[axis] = n - 2;
    h = delta;
  } else {
    lo[axis] = c[axis] - 1;
    hi[axis] = c[axis] + 1;
  }
  double fh = f[(hi[2] * nn[1] + hi[1]) * nn[0] + hi[0]];
  double fl = f[(lo[2] * nn[1] + lo[1]) * nn[0] + lo[0]];
  return (fh - fl) / h;
}

/* R_s(Omega_s dt/2) applied to x: with a = Omega_s dt/2,
 * R x = (x - a x x + (a.x) a) / (1 + a.a).  The printed R omits the scalar
 * 1/(1 + a.a); it is included (R25) so that R is exactly the linear response
 * of the mover's average velocity to E (Eq. 2: vb = R vt), which the pins
 * check against push_one.                                                  */
static void apply_R(const double a[3], const double x[3], double out[3]) {
  double cr[3];
  cr[0] = a[1] * x[2] - a[2] * x[1];
  cr[1] = a[2] * x[0] - a[0] * x[2];
  cr[2] = a[0] * x[1] - a[1] * x[0];
  double dot = a[0] * x[0] + a[1] * x[1] + a[2] * x[2];
  double den = 1.0 + (a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
  for (int d = 0; d < 3; ++d) out[d] = (x[d] - cr[d] + dot * a[d]) / den;
}

/* Eq. 5 and Eq. 6 from the moments of S species (NEXT-2).
 *   mom[s]: species s moments [10][nz][ny][nx] over the unique nodes (after
 *           1/V, the output of oracle_moments); B: node field [nz][ny][nx][3]
 *   chi[9][nz][ny][nx] = sum_s (1/2)(omega_ps dt)^2 R_s        (Eq. 5)
 *       omega_ps^2 = 4 pi rho_s q_s/m_s (rho_s and q_s share their sign, R24)
 *   J_hat[3][...] = sum_s R_s (J_s - (dt/2) div Pi_s)         (Eq. 6, R26: per
 *       species with its own R_s, then summed)
 *   rho_hat[...] = sum_s rho_s - dt div J_hat                 (Eq. 6)
 * Derivatives: node_diff (R27).  Gaussian units, 4 pi explicit.             */
void oracle_implicit_sources(const oracle_grid *g, int n_species, const double *qom,
                             const double *const *mom, const double *B, double *chi,
                             double *rho_hat, double *J_hat) {
  int64_t nn[3] = {nodes_axis(g, 0), nodes_axis(g, 1), nodes_axis(g, 2)};
  int64_t plane = nn[0] * nn[1] * nn[2];
  const double four_pi = 4.0 * 3.14159265358979323846;
  double dt = g->dt;
  for (int64_t m = 0; m < 9 * plane; ++m) chi[m] = 0.0;
  for (int64_t m = 0; m < 3 * plane; ++m) J_hat[m] = 0.0;
  for (int64_t k = 0; k < nn[2]; ++k)
    for (int64_t j = 0; j < nn[1]; ++j)
      for (int64_t i = 0; i < nn[0]; ++i) {
        int64_t node = (k * nn[1] + j) * nn[0] + i;
        for (int s = 0; s < n_species; ++s) {
          const double *ms = mom[s];
          double a[3];
          for (int d = 0; d < 3; ++d) a[d] = (qom[s] * B[3 * node + d] / g->c) * (dt / 2.0);
          double w2 = four_pi * ms[node] * qom[s];
          /* chi_s columns: R_s applied to the unit vectors */
          for (int col = 0; col < 3; ++col) {
            double e[3] = {0.0, 0.0, 0.0}, r[3];
            e[col] = 1.0;
            apply_R(a, e, r);
            for (int row = 0; row < 3; ++row)
              chi[(row * 3 + col) * plane + node] += 0.5 * w2 * dt * dt * r[row];
          }
          /* div Pi_s: (div Pi)_a = sum_b d Pi_ab / d x_b; Pi order xx xy xz yy yz zz */
          static const int pidx[3][3] = {{4, 5, 6}, {5, 7, 8}, {6, 8, 9}};
          double divPi[3];
          for (int ra = 0; ra < 3; ++ra) {
            divPi[ra] = 0.0;
            for (int b = 0; b < 3; ++b)
              divPi[ra] += node_diff(g, ms + pidx[ra][b] * plane, nn, i, j, k, b);
          }
          double x[3], r[3];
          for (int d = 0; d < 3; ++d) x[d] = ms[(1 + d) * plane + node] - (dt / 2.0) * divPi[d];
          apply_R(a, x, r);
          for (int d = 0; d < 3; ++d) J_hat[d * plane + node] += r[d];
        }
      }
  for (int64_t k = 0; k < nn[2]; ++k)
    for (int64_t j = 0; j < nn[1]; ++j)
      for (int64_t i = 0; i < nn[0]; ++i) {
        int64_t node = (k * nn[1] + j) * nn[0] + i;
        double rho = 0.0;
        for (int s = 0; s < n_species; ++s) rho += mom[s][node];
        double divJ = 0.0;
        for (int b = 0; b < 3; ++b) divJ += node_diff(g, J_hat + b * plane, nn, i, j, k, b);
        rho_hat[node] = rho - dt * divJ;
      }
}

/* --------------------------------------------- NEXT-3: inflow injection -- */

/* Philox4x32-10 (Salmon et al., SC'11), the counter-based generator both the
 * oracle and the CUDA path implement (their shared random numbers; pinned by
 * the published known-answer vectors).  c: counter (in/out), k: key.       */
void oracle_philox4x32_10(uint32_t c[4], const uint32_t k_in[2]) {
  uint32_t k0 = k_in[0], k1 = k_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

/* 53-bit uniform in [0, 1) from two words. */
static double u53(uint32_t a, uint32_t b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

/* Draw call `call` of particle k of ghost cell gc: two uniforms. */
static void draw2(uint32_t gc, uint32_t k, uint32_t cycle, uint32_t species, uint32_t call,
                  const uint32_t key[2], double *ua, double *ub) {
  uint32_t c[4] = {gc, k, cycle, (species << 8) | call};
  oracle_philox4x32_10(c, key);
  *ua = u53(c[0], c[1]);
  *ub = u53(c[2], c[3]);
}

/* Inflow injection at the x = 0 face of an open x axis (PAPER.md:232-233,
 * reading R28): in every ghost cell (-1, cy, cz) of the face, ppc particles
 * with uniform positions in the cell and velocities drift + vth * N(0,1)^3
 * (Box-Muller), charge q, id 2^62 | cycle << 40 | species << 37 | (gc ppc + k),
 * gc = cz Ny + cy, are pushed one step with Eq. 2 (push_one / push_one_rel)
 * and kept when they end inside the domain (apply_bc ALIVE); kept particles
 * are appended to the output arrays (at most cap).  Draws: call 0 -> (u0,u1),
 * 1 -> (u2,u3), 2 -> (u4,u5), 3 -> (u6,u7) of Philox(counter {gc, k, cycle,
 * species << 8 | call}, key {seed_lo, seed_hi});
 *   x = (-1 + u0) dx, y = (cy + u1) dy, z = (cz + u2) dz,
 *   (n0, n1) = sqrt(-2 ln(1 - u3)) (cos, sin)(2 pi u4),
 *   n2 = sqrt(-2 ln(1 - u5)) cos(2 pi u6)   (u7 unused).
 * Returns the number appended; -1 if the x axis is not open.                */
int64_t oracle_inject(const oracle_grid *g, const oracle_field *F, int species, double qom, int n_iter,
                      int relativistic, uint32_t seed_lo, uint32_t seed_hi, int64_t cycle, int ppc,
                      double vth, const double drift[3], double q, int64_t cap, double *x, double *y,
                      double *z, double *u, double *v, double *w, double *qo, int64_t *id) {
  if (g->bc[0] != 1) return -1;
  const uint32_t key[2] = {seed_lo, seed_hi};
  double dl[3];
  for (int d = 0; d < 3; ++d) dl[d] = g->len[d] / (double)g->ncell[d];
  const double two_pi = 2.0 * 3.14159265358979323846;
  int64_t n = 0;
  for (int64_t cz = 0; cz < g->ncell[2]; ++cz)
    for (int64_t cy = 0; cy < g->ncell[1]; ++cy) {
      uint32_t gc = (uint32_t)(cz * g->ncell[1] + cy);
      for (int k = 0; k < ppc; ++k) {
        double r[8];
        for (int call = 0; call < 4; ++call)
          draw2(gc, (uint32_t)k, (uint32_t)cycle, (uint32_t)species, (uint32_t)call, key, &r[2 * call],
                &r[2 * call + 1]);
        double xn[3] = {(-1.0 + r[0]) * dl[0], ((double)cy + r[1]) * dl[1], ((double)cz + r[2]) * dl[2]};
        double rad1 = sqrt(-2.0 * log(1.0 - r[3]));
        double rad2 = sqrt(-2.0 * log(1.0 - r[5]));
        double vn[3] = {drift[0] + vth * (rad1 * cos(two_pi * r[4])),
                        drift[1] + vth * (rad1 * sin(two_pi * r[4])),
                        drift[2] + vth * (rad2 * cos(two_pi * r[6]))};
        int st = relativistic ? push_one_rel(g, F, qom, n_iter, xn, vn) : push_one(g, F, qom, n_iter, xn, vn);
        if (st != ORACLE_ALIVE) continue;
        if (n < cap) {
          x[n] = xn[0]; y[n] = xn[1]; z[n] = xn[2];
          u[n] = vn[0]; v[n] = vn[1]; w[n] = vn[2];
          qo[n] = q;
          id[n] = (int64_t)((1ull << 62) | ((uint64_t)cycle << 40) | ((uint64_t)species << 37) |
                            ((uint64_t)gc * (uint64_t)ppc + (uint64_t)k));
        }
        ++n;
      }
    }
  return n;
}

/* ------------------------------------------- NEXT-3: particle control -- */

uint64_t oracle_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* Id of the second child of a split (R30): tagged with bit 61, otherwise a
 * hash of the parent id and the cycle (unique with overwhelming probability). */
int64_t oracle_child_id(int64_t parent, int64_t cycle) {
  uint64_t h = oracle_splitmix64((uint64_t)parent ^ ((uint64_t)cycle << 48) ^ 0x5BD1E995ull);
  return (int64_t)((h & ((1ull << 61) - 1)) | (1ull << 61));
}

/* Splitting ("randomly select particles and split each into
 * multiple particles, adjusting their statistical weights"; reading R30):
 * particle i (ALIVE, i < np) splits iff u0 < p_split, u0 from Philox(counter
 * {id lo, id hi, cycle, species << 8 | 0x80}, key {seed}).  Direction e = n/|n|
 * with n = three Box-Muller normals from the draws 0x80 (u1), 0x81 (u2, u3),
 * 0x82 (u4): n0,n1 = sqrt(-2 ln(1-u1)) (cos, sin)(2 pi u2), n2 = sqrt(-2 ln(1-u3))
 * cos(2 pi u4).  Children at x -/+ eps Delta_d e_d (per axis), each with q/2
 * and the parent's velocity (charge, momentum, energy and charge centroid
 * conserved); the split is skipped if a child would leave the parent's cell.
 * Child 1 keeps the parent's slot and id, child 2 is appended with
 * oracle_child_id.  Returns the new particle count (<= cap).               */
int64_t oracle_split(const oracle_grid *g, int species, int64_t np, int64_t cap, double *x, double *y,
                     double *z, double *u, double *v, double *w, double *q, int64_t *id, int8_t *status,
                     double p_split, double eps, uint32_t seed_lo, uint32_t seed_hi, int64_t cycle) {
  const uint32_t key[2] = {seed_lo, seed_hi};
  const double two_pi = 2.0 * 3.14159265358979323846;
  double dl[3];
  for (int d = 0; d < 3; ++d) dl[d] = g->len[d] / (double)g->ncell[d];
  int64_t n = np;
  for (int64_t i = 0; i < np; ++i) {
    if (status[i] != ORACLE_ALIVE) continue;
    uint64_t uid = (uint64_t)id[i];
    double r[6];
    for (int call = 0; call < 3; ++call) {
      uint32_t c[4] = {(uint32_t)uid, (uint32_t)(uid >> 32), (uint32_t)cycle, ((uint32_t)species << 8) | (0x80u + call)};
      oracle_philox4x32_10(c, key);
      r[2 * call] = u53(c[0], c[1]);
      r[2 * call + 1] = u53(c[2], c[3]);
    }
    if (!(r[0] < p_split)) continue;
    double rad1 = sqrt(-2.0 * log(1.0 - r[1]));
    double rad2 = sqrt(-2.0 * log(1.0 - r[3]));
    double nv[3] = {rad1 * cos(two_pi * r[2]), rad1 * sin(two_pi * r[2]), rad2 * cos(two_pi * r[4])};
    double nrm = sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
    if (!(nrm > 0.0)) continue;
    double pos[3] = {x[i], y[i], z[i]}, a[3], b[3];
    int ok = 1;
    for (int d = 0; d < 3; ++d) {
      double dd = eps * dl[d] * (nv[d] / nrm);
      a[d] = pos[d] - dd;
      b[d] = pos[d] + dd;
      double c0 = floor(pos[d] / dl[d]);
      if (floor(a[d] / dl[d]) != c0 || floor(b[d] / dl[d]) != c0) ok = 0;
    }
    if (!ok || n >= cap) continue;
    double qh = q[i] / 2.0;
    x[n] = b[0]; y[n] = b[1]; z[n] = b[2];
    u[n] = u[i]; v[n] = v[i]; w[n] = w[i];
    q[n] = qh;
    id[n] = oracle_child_id(id[i], cycle);
    status[n] = ORACLE_ALIVE;
    ++n;
    x[i] = a[0]; y[i] = a[1]; z[i] = a[2];
    q[i] = qh;
  }
  return n;
}

/* Coalescence ("pair-wise merging between particles that are
 * close in the phase space by combining their statistical weights"; reading
 * R31).  In every cell with n_c >= 2 ALIVE particles ("in cells
 * with an excessive number of particles"; no size or velocity limit): sort them
 * by the velocity bins (floor(u/dv), floor(v/dv), floor(w/dv)) -- compared as
 * fp64 values, so any finite velocity has a bin -- then by id; scan the sorted
 * list and merge neighbours i, i+1 whose three bins are equal (then continue
 * at i+2) until m_c = floor(frac n_c) merges.  Merge: q = q1 + q2,
 * x = (q1 x1 + q2 x2)/q, v = (q1 v1 + q2 v2)/q per component (charge, momentum
 * and the charge centroid conserved); the particle with the smaller id keeps
 * the result, the other becomes ORACLE_MERGED.  Returns the number of merges. */
enum { ORACLE_MERGED = 3 };
typedef struct { int64_t cell; double bx, by, bz; int64_t id, idx; } coal_key;
static int coal_cmp(const void *pa, const void *pb) {
  const coal_key *a = (const coal_key *)pa, *b = (const coal_key *)pb;
  if (a->cell != b->cell) return a->cell < b->cell ? -1 : 1;
  if (a->bx != b->bx) return a->bx < b->bx ? -1 : 1;
  if (a->by != b->by) return a->by < b->by ? -1 : 1;
  if (a->bz != b->bz) return a->bz < b->bz ? -1 : 1;
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  return 0;
}
int64_t oracle_coalesce(const oracle_grid *g, int64_t np, double *x, double *y, double *z, double *u,
                        double *v, double *w, double *q, int64_t *id, int8_t *status, double dv, double frac) {
  double dl[3];
  for (int d = 0; d < 3; ++d) dl[d] = g->len[d] / (double)g->ncell[d];
  coal_key *k = (coal_key *)malloc(sizeof(coal_key) * (size_t)(np > 0 ? np : 1));
  int64_t m = 0;
  for (int64_t i = 0; i < np; ++i) {
    if (status[i] != ORACLE_ALIVE) continue;
    int64_t cx = (int64_t)floor(x[i] / dl[0]), cy = (int64_t)floor(y[i] / dl[1]), cz = (int64_t)floor(z[i] / dl[2]);
    k[m].cell = (cz * g->ncell[1] + cy) * g->ncell[0] + cx;
    k[m].bx = floor(u[i] / dv);
    k[m].by = floor(v[i] / dv);
    k[m].bz = floor(w[i] / dv);
    k[m].id = id[i];
    k[m].idx = i;
    ++m;
  }
  qsort(k, (size_t)m, sizeof(coal_key), coal_cmp);
  int64_t merges = 0;
  for (int64_t s0 = 0; s0 < m;) {
    int64_t s1 = s0;
    while (s1 < m && k[s1].cell == k[s0].cell) ++s1;
    int64_t nc = s1 - s0;
    if (nc >= 2) {
      int64_t mc = (int64_t)floor(frac * (double)nc), done = 0;
      for (int64_t t = s0; t + 1 < s1 && done < mc;) {
        const coal_key *a = &k[t], *b = &k[t + 1];
        if (a->bx == b->bx && a->by == b->by && a->bz == b->bz) {
          int64_t i1 = a->idx, i2 = b->idx;        /* a has the smaller id */
          double qs = q[i1] + q[i2];
          double nx = (q[i1] * x[i1] + q[i2] * x[i2]) / qs;
          double ny = (q[i1] * y[i1] + q[i2] * y[i2]) / qs;
          double nz = (q[i1] * z[i1] + q[i2] * z[i2]) / qs;
          double nu = (q[i1] * u[i1] + q[i2] * u[i2]) / qs;
          double nv = (q[i1] * v[i1] + q[i2] * v[i2]) / qs;
          double nw = (q[i1] * w[i1] + q[i2] * w[i2]) / qs;
          x[i1] = nx; y[i1] = ny; z[i1] = nz; u[i1] = nu; v[i1] = nv; w[i1] = nw; q[i1] = qs;
          status[i2] = ORACLE_MERGED;
          ++done;
          t += 2;
        } else {
          t += 1;
        }
      }
      merges += done;
    }
    s0 = s1;
  }
  free(k);
  return merges;
}

/* --------------------------------------------------- NEXT-4: GMM fit -- */

/* Velocity binning ("a three-dimensional binning operation in
 * velocity space"; reading R32): B bins per axis over [-vmax, vmax); bin of
 * a component = floor((v + vmax) / (2 vmax) * B) clipped to [0, B-1] (clipped
 * particles counted); weight |q| (the statistical weight).  hist[(bz*B + by)*B
 * + bx] += |q|.  Returns the number of clipped particles.                   */
int64_t oracle_bin_velocities(int64_t np, const double *u, const double *v, const double *w,
                              const double *q, const int8_t *status, int B, double vmax, double *hist) {
  int64_t clipped = 0;
  for (int64_t p = 0; p < np; ++p) {
    if (status && status[p] != ORACLE_ALIVE) continue;
    const double vel[3] = {u[p], v[p], w[p]};
    int64_t b[3];
    int clip = 0;
    for (int d = 0; d < 3; ++d) {
      double t = floor((vel[d] + vmax) / (2.0 * vmax) * (double)B);
      if (t < 0.0) { t = 0.0; clip = 1; }
      if (t > (double)(B - 1)) { t = (double)(B - 1); clip = 1; }
      b[d] = (int64_t)t;
    }
    clipped += clip;
    hist[(b[2] * B + b[1]) * B + b[0]] += fabs(q[p]);
  }
  return clipped;
}

static void inv3(const double S[6], double out[6], double *det) {
  /* symmetric xx xy xz yy yz zz */
  double a = S[0], b = S[1], c = S[2], d = S[3], e = S[4], f = S[5];
  double A = d * f - e * e, Bc = -(b * f - c * e), C = b * e - c * d;
  double D = a * f - c * c, E = -(a * e - b * c), Fz = a * d - b * b;
  double dt = a * A + b * Bc + c * C;
  *det = dt;
  out[0] = A / dt; out[1] = Bc / dt; out[2] = C / dt; out[3] = D / dt; out[4] = E / dt; out[5] = Fz / dt;
}

/* Gaussian-mixture fit by EM on the histogram (reading
 * R33): data = bin centres c_b = -vmax + (b + 1/2) 2 vmax / B with weights
 * hist_b > 0.  Initialisation: mu_1 = centre of the heaviest bin (lowest index
 * on ties), then farthest-point seeding (the occupied bin maximising the
 * squared distance to the nearest chosen centre, lowest index on ties);
 * Sigma_i = the histogram's weighted covariance + eps I; alpha_i = 1/M.
 * Exactly n_em iterations of
 *   E: r_bi = alpha_i N(c_b | mu_i, Sigma_i) / sum_j alpha_j N(c_b | mu_j, Sigma_j)
 *   M: W_i = sum_b h_b r_bi; alpha_i = W_i / W; mu_i = sum_b h_b r_bi c_b / W_i;
 *      Sigma_i = sum_b h_b r_bi (c_b - mu_i)(c_b - mu_i)^T / W_i + eps I,
 * eps = 1e-6 (2 vmax / B)^2.  Covariances as xx xy xz yy yz zz.  Returns 0,
 * or -1 if fewer than M bins are occupied.                                  */
int oracle_fit_gmm(int B, double vmax, const double *hist, int M, int n_em, double *alpha, double *mu,
                   double *sigma) {
  const int64_t nb = (int64_t)B * B * B;
  const double bw = 2.0 * vmax / (double)B;
  const double eps = 1e-6 * bw * bw;
  const double two_pi3 = pow(2.0 * 3.14159265358979323846, 1.5);
  int64_t nocc = 0;
  for (int64_t b = 0; b < nb; ++b) nocc += hist[b] > 0.0;
  if (nocc < M || M < 1) return -1;
  double *cen = (double *)malloc(sizeof(double) * 3 * (size_t)nb);
  double W = 0.0, m1[3] = {0, 0, 0};
  for (int64_t b = 0; b < nb; ++b) {
    int64_t bx = b % B, by = (b / B) % B, bz = b / ((int64_t)B * B);
    cen[3 * b] = -vmax + ((double)bx + 0.5) * bw;
    cen[3 * b + 1] = -vmax + ((double)by + 0.5) * bw;
    cen[3 * b + 2] = -vmax + ((double)bz + 0.5) * bw;
    if (hist[b] > 0.0) {
      W += hist[b];
      for (int d = 0; d < 3; ++d) m1[d] += hist[b] * cen[3 * b + d];
    }
  }
  for (int d = 0; d < 3; ++d) m1[d] /= W;
  double cov[6] = {0, 0, 0, 0, 0, 0};
  static const int ia[6] = {0, 0, 0, 1, 1, 2}, ib[6] = {0, 1, 2, 1, 2, 2};
  for (int64_t b = 0; b < nb; ++b)
    if (hist[b] > 0.0)
      for (int k = 0; k < 6; ++k)
        cov[k] += hist[b] * (cen[3 * b + ia[k]] - m1[ia[k]]) * (cen[3 * b + ib[k]] - m1[ib[k]]);
  for (int k = 0; k < 6; ++k) cov[k] /= W;
  cov[0] += eps; cov[3] += eps; cov[5] += eps;
  /* farthest-point seeding */
  int64_t first = -1;
  for (int64_t b = 0; b < nb; ++b)
    if (hist[b] > 0.0 && (first < 0 || hist[b] > hist[first])) first = b;
  for (int d = 0; d < 3; ++d) mu[d] = cen[3 * first + d];
  for (int i = 1; i < M; ++i) {
    int64_t best = -1;
    double bestd = -1.0;
    for (int64_t b = 0; b < nb; ++b) {
      if (!(hist[b] > 0.0)) continue;
      double dmin = INFINITY;
      for (int j = 0; j < i; ++j) {
        double dd = 0.0;
        for (int d = 0; d < 3; ++d) {
          double t = cen[3 * b + d] - mu[3 * j + d];
          dd += t * t;
        }
        if (dd < dmin) dmin = dd;
      }
      if (dmin > bestd) { bestd = dmin; best = b; }
    }
    for (int d = 0; d < 3; ++d) mu[3 * i + d] = cen[3 * best + d];
  }
  for (int i = 0; i < M; ++i) {
    alpha[i] = 1.0 / (double)M;
    for (int k = 0; k < 6; ++k) sigma[6 * i + k] = cov[k];
  }
  double *r = (double *)malloc(sizeof(double) * (size_t)M);
  double *acc = (double *)malloc(sizeof(double) * (size_t)M * 10);
  for (int it = 0; it < n_em; ++it) {
    double inv[16][6], nrm[16];
    for (int i = 0; i < M; ++i) {
      double det;
      inv3(sigma + 6 * i, inv[i], &det);
      nrm[i] = alpha[i] / (two_pi3 * sqrt(det));
    }
    for (int64_t k = 0; k < (int64_t)M * 10; ++k) acc[k] = 0.0;
    for (int64_t b = 0; b < nb; ++b) {
      if (!(hist[b] > 0.0)) continue;
      double tot = 0.0;
      for (int i = 0; i < M; ++i) {
        double x = cen[3 * b] - mu[3 * i], y = cen[3 * b + 1] - mu[3 * i + 1], z = cen[3 * b + 2] - mu[3 * i + 2];
        const double *A = inv[i];
        double q2 = A[0] * x * x + A[3] * y * y + A[5] * z * z + 2.0 * (A[1] * x * y + A[2] * x * z + A[4] * y * z);
        r[i] = nrm[i] * exp(-0.5 * q2);
        tot += r[i];
      }
      if (!(tot > 0.0)) continue;
      for (int i = 0; i < M; ++i) {
        double wr = hist[b] * (r[i] / tot);
        double *a = acc + 10 * i;
        a[0] += wr;
        for (int d = 0; d < 3; ++d) a[1 + d] += wr * cen[3 * b + d];
        for (int k = 0; k < 6; ++k) a[4 + k] += wr * cen[3 * b + ia[k]] * cen[3 * b + ib[k]];
      }
    }
    for (int i = 0; i < M; ++i) {
      const double *a = acc + 10 * i;
      if (!(a[0] > 0.0)) continue;   /* an empty component keeps its parameters */
      alpha[i] = a[0] / W;
      for (int d = 0; d < 3; ++d) mu[3 * i + d] = a[1 + d] / a[0];
      for (int k = 0; k < 6; ++k)
        sigma[6 * i + k] = a[4 + k] / a[0] - mu[3 * i + ia[k]] * mu[3 * i + ib[k]] + ((ia[k] == ib[k]) ? eps : 0.0);
    }
  }
  free(r);
  free(acc);
  free(cen);
  return 0;
}
