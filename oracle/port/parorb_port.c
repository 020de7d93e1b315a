/* parorb_port.c — CPU restatement of the reference hot path (TEST INFRASTRUCTURE
 * ONLY; see parorb_port.h). Citations are to /root/reference/proj. */
#include "parorb_port.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.141592653589793238462643383279502884;

/* ---------------------------------------------------------------- numeric */

/* include/parorb/numeric.hpp:12-23 — blocked pairwise tree, leaf 256. */
static double pw_dot(int64_t n, const double* a, const double* b) {
  if (n <= 256) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
  }
  const int64_t half = n / 2;
  return pw_dot(half, a, b) + pw_dot(n - half, a + half, b + half);
}
static double pw_sum(int64_t n, const double* a) {
  if (n <= 256) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += a[i];
    return acc;
  }
  const int64_t half = n / 2;
  return pw_sum(half, a) + pw_sum(n - half, a + half);
}
static double pw_abs_sum(int64_t n, const double* a) {
  if (n <= 256) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += fabs(a[i]);
    return acc;
  }
  const int64_t half = n / 2;
  return pw_abs_sum(half, a) + pw_abs_sum(n - half, a + half);
}
/* sum_q v[q] * u[q] * u[q]  (energy.cpp:274-279) */
static double pw_vuu(int64_t n, const double* v, const double* u) {
  if (n <= 256) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += v[i] * u[i] * u[i];
    return acc;
  }
  const int64_t half = n / 2;
  return pw_vuu(half, v, u) + pw_vuu(n - half, v + half, u + half);
}
/* BB products, optimizer.cpp:386-397 */
static double pw_diff_sq(int64_t n, const double* a, const double* b) {
  if (n <= 256) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double s = a[i] - b[i];
      acc += s * s;
    }
    return acc;
  }
  const int64_t half = n / 2;
  return pw_diff_sq(half, a, b) + pw_diff_sq(n - half, a + half, b + half);
}
static double pw_diff_prod(int64_t n, const double* a, const double* b, const double* c,
                           const double* d) {
  if (n <= 256) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += (a[i] - b[i]) * (c[i] - d[i]);
    return acc;
  }
  const int64_t half = n / 2;
  return pw_diff_prod(half, a, b, c, d) + pw_diff_prod(n - half, a + half, b + half, c + half, d + half);
}

double pp_pairwise_dot(int64_t n, const double* a, const double* b) { return pw_dot(n, a, b); }
double pp_pairwise_sum(int64_t n, const double* a) { return pw_sum(n, a); }

static double inner(const pp_grid* g, const double* f, const double* h) {
  return g->w * pw_dot(g->ng, f, h); /* grid.cpp:126-129 */
}

/* ------------------------------------------------------------------- grid */

/* grid.cpp:11-41 */
int pp_grid_init(pp_grid* g, int dim, const int64_t* n, const double* ext) {
  if (dim < 1 || dim > 3) return PP_EINVAL;
  memset(g, 0, sizeof *g);
  g->dim = dim;
  g->ng = 1;
  for (int a = 0; a < dim; ++a) {
    if (!(ext[a] > 0.0) || n[a] < 1) return PP_EINVAL;
    g->n[a] = n[a];
    g->ext[a] = ext[a];
    g->h[a] = ext[a] / (double)(n[a] + 1);
    g->ng *= n[a];
  }
  g->w = 1.0;
  for (int a = 0; a < dim; ++a) g->w *= g->h[a];
  return PP_OK;
}

/* grid.cpp:94-122: three axis passes accumulated into a zeroed dst. */
void pp_laplacian(const pp_grid* g, const double* src, double* dst) {
  memset(dst, 0, sizeof(double) * (size_t)g->ng);
  for (int axis = 0; axis < g->dim; ++axis) {
    const int64_t n = g->n[axis];
    int64_t outer = 1, inn = 1;
    for (int k = 0; k < axis; ++k) outer *= g->n[k];
    for (int k = axis + 1; k < g->dim; ++k) inn *= g->n[k];
    const double inv_h2 = 1.0 / (g->h[axis] * g->h[axis]);
    for (int64_t o = 0; o < outer; ++o) {
      const int64_t base = o * n * inn;
      for (int64_t in = 0; in < inn; ++in) {
        for (int64_t i = 0; i < n; ++i) {
          const int64_t idx = base + i * inn + in;
          const double left = i > 0 ? src[idx - inn] : 0.0;
          const double right = i + 1 < n ? src[idx + inn] : 0.0;
          dst[idx] += (left - 2.0 * src[idx] + right) * inv_h2;
        }
      }
    }
  }
}

static void coords(const pp_grid* g, int64_t flat, double* xyz) { /* grid.cpp:63-69 */
  for (int a = g->dim - 1; a >= 0; --a) {
    const int64_t n = g->n[a];
    xyz[a] = (double)(flat % n + 1) * g->h[a];
    flat /= n;
  }
}

/* ----------------------------------------------------------------- energy */

/* energy.cpp:78-99 */
void pp_external_potential(const pp_grid* g, const pp_atom* atoms, int natoms, double* v) {
  double xyz[3];
  for (int64_t p = 0; p < g->ng; ++p) {
    if (natoms == 0) { v[p] = 0.0; continue; }
    coords(g, p, xyz);
    double acc = 0.0;
    for (int k = 0; k < natoms; ++k) {
      double r2 = atoms[k].softening * atoms[k].softening;
      for (int a = 0; a < g->dim; ++a) {
        const double dx = xyz[a] - atoms[k].pos[a];
        r2 += dx * dx;
      }
      acc -= atoms[k].charge / sqrt(r2);
    }
    v[p] = acc;
  }
}

/* energy.cpp:67-76; occupation != 1 is the closed-shell extension (gate B). */
void pp_density(const pp_grid* g, int n, const double* u, double occupation, double* rho) {
  memset(rho, 0, sizeof(double) * (size_t)g->ng);
  for (int i = 0; i < n; ++i) {
    const double* src = u + (int64_t)i * g->ng;
    for (int64_t p = 0; p < g->ng; ++p) rho[p] += src[p] * src[p];
  }
  if (occupation != 1.0)
    for (int64_t p = 0; p < g->ng; ++p) rho[p] *= occupation;
}

/* energy.cpp:105-143: plain CG on -lap v = b, x0 = 0, rel. tol 1e-10,
 * <= 20000 iterations per restart, <= 3 restarts with a true-residual check. */
static int poisson_solve(const pp_grid* g, const double* b, double* x, int* iters) {
  const int64_t ng = g->ng;
  memset(x, 0, sizeof(double) * (size_t)ng);
  const double b_norm = sqrt(pw_dot(ng, b, b));
  if (b_norm == 0.0) return PP_OK;
  double* r = malloc(sizeof(double) * (size_t)ng);
  double* p = malloc(sizeof(double) * (size_t)ng);
  double* ap = malloc(sizeof(double) * (size_t)ng);
  int rc = PP_ESOLVER;
  memcpy(r, b, sizeof(double) * (size_t)ng);
  for (int restart = 0; restart <= 3; ++restart) {
    memcpy(p, r, sizeof(double) * (size_t)ng);
    double rr = pw_dot(ng, r, r);
    for (int it = 0; it < 20000; ++it) {
      if (sqrt(rr) <= 1e-10 * b_norm) break;
      pp_laplacian(g, p, ap);
      for (int64_t i = 0; i < ng; ++i) ap[i] = -ap[i];
      const double pap = pw_dot(ng, p, ap);
      if (!(pap > 0.0)) { rc = PP_ESOLVER; goto done; }
      const double alpha = rr / pap;
      for (int64_t i = 0; i < ng; ++i) x[i] += alpha * p[i];
      const double malpha = -alpha;
      for (int64_t i = 0; i < ng; ++i) r[i] += malpha * ap[i];
      const double rr_new = pw_dot(ng, r, r);
      const double beta = rr_new / rr;
      rr = rr_new;
      for (int64_t i = 0; i < ng; ++i) p[i] = r[i] + beta * p[i];
      if (iters) ++*iters;
    }
    pp_laplacian(g, x, ap);
    for (int64_t i = 0; i < ng; ++i) ap[i] = -ap[i];
    memcpy(r, b, sizeof(double) * (size_t)ng);
    for (int64_t i = 0; i < ng; ++i) r[i] += -1.0 * ap[i];
    if (sqrt(pw_dot(ng, r, r)) <= 1e-10 * b_norm) { rc = PP_OK; goto done; }
  }
done:
  free(r); free(p); free(ap);
  return rc;
}

/* energy.cpp:197-210 (3D Poisson mode only; the kernel mode is 1D/2D) */
int pp_hartree(const pp_grid* g, const double* rho, double* vh, int* cg_iters) {
  for (int64_t p = 0; p < g->ng; ++p)
    if (rho[p] < 0.0) return PP_EINVAL;
  if (g->dim != 3) return PP_EINVAL;
  double* b = malloc(sizeof(double) * (size_t)g->ng);
  const double four_pi = 4.0 * kPi;
  for (int64_t p = 0; p < g->ng; ++p) b[p] = rho[p] * four_pi;
  const int rc = poisson_solve(g, b, vh, cg_iters);
  free(b);
  return rc;
}

/* energy.cpp:18,212-226 */
static double dirac_cx(void) { return 0.75 * cbrt(3.0 / kPi); }
int pp_xc_energy_density(int64_t ng, const double* rho, double* eps) {
  const double cx = dirac_cx();
  for (int64_t i = 0; i < ng; ++i) {
    if (rho[i] < 0.0) return PP_EINVAL;
    eps[i] = -cx * cbrt(rho[i]);
  }
  return PP_OK;
}
int pp_xc_potential(int64_t ng, const double* rho, double* v) {
  const int rc = pp_xc_energy_density(ng, rho, v);
  const double f = 4.0 / 3.0;
  for (int64_t i = 0; i < ng; ++i) v[i] *= f;
  return rc;
}

/* energy.cpp:228-246 */
int pp_build_hamiltonian(const pp_grid* g, int n, const double* u, const double* v_ext,
                         int hartree, int xc, double occupation, pp_state* s) {
  const int64_t ng = g->ng;
  pp_density(g, n, u, occupation, s->rho);
  int rc = PP_OK;
  s->cg_iters = 0;
  if (hartree) {
    rc = pp_hartree(g, s->rho, s->v_h, &s->cg_iters);
    if (rc) return rc;
  } else {
    memset(s->v_h, 0, sizeof(double) * (size_t)ng);
  }
  if (xc) {
    rc = pp_xc_potential(ng, s->rho, s->v_xc);
    if (rc) return rc;
  } else {
    memset(s->v_xc, 0, sizeof(double) * (size_t)ng);
  }
  for (int64_t i = 0; i < ng; ++i) s->v_local[i] = v_ext[i] + (s->v_h[i] + s->v_xc[i]);
  return PP_OK;
}

/* energy.cpp:248-265 */
void pp_apply_hamiltonian(const pp_grid* g, const double* v, int n, const double* u,
                          double* hu) {
  for (int i = 0; i < n; ++i) {
    const double* uu = u + (int64_t)i * g->ng;
    double* h = hu + (int64_t)i * g->ng;
    pp_laplacian(g, uu, h);
    for (int64_t p = 0; p < g->ng; ++p) h[p] = -0.5 * h[p] + v[p] * uu[p];
  }
}

/* energy.cpp:267-280 */
double pp_kinetic_term(const pp_grid* g, const double* u) {
  double* lap = malloc(sizeof(double) * (size_t)g->ng);
  pp_laplacian(g, u, lap);
  const double k = -0.5 * inner(g, lap, u);
  free(lap);
  return k;
}
double pp_potential_term(const pp_grid* g, const double* v, const double* u) {
  return g->w * pw_vuu(g->ng, v, u);
}

/* energy.cpp:282-314. Occupation scales the per-orbital sums (gate B). */
void pp_total_energy(const pp_grid* g, int n, const double* u, const double* v_ext,
                     const pp_state* s, int hartree, int xc, double occupation, double* out5,
                     double* kin_each, double* ext_each) {
  double* kin = kin_each ? kin_each : malloc(sizeof(double) * (size_t)n);
  double* ext = ext_each ? ext_each : malloc(sizeof(double) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    kin[i] = pp_kinetic_term(g, u + (int64_t)i * g->ng);
    ext[i] = pp_potential_term(g, v_ext, u + (int64_t)i * g->ng);
    if (occupation != 1.0) { kin[i] *= occupation; ext[i] *= occupation; }
  }
  double kinetic = 0.0, external = 0.0, eh = 0.0, exc = 0.0;
  for (int i = 0; i < n; ++i) kinetic += kin[i];
  for (int i = 0; i < n; ++i) external += ext[i];
  if (hartree) eh = 0.5 * inner(g, s->v_h, s->rho);
  if (xc) {
    double* eps = malloc(sizeof(double) * (size_t)g->ng);
    pp_xc_energy_density(g->ng, s->rho, eps);
    exc = inner(g, eps, s->rho);
    free(eps);
  }
  out5[0] = kinetic;
  out5[1] = external;
  out5[2] = eh;
  out5[3] = exc;
  out5[4] = kinetic + external + eh + exc;
  if (!kin_each) free(kin);
  if (!ext_each) free(ext);
}

/* --------------------------------------------------------------- manifold */

/* manifold.cpp:41-61 */
void pp_gram(const pp_grid* g, int n, const double* psi, const double* phi, int same,
             double* gm) {
  const int64_t ng = g->ng;
  if (same) {
    for (int i = 0; i < n; ++i)
      for (int j = i; j < n; ++j) {
        gm[i * n + j] = inner(g, psi + i * ng, phi + j * ng);
        gm[j * n + i] = gm[i * n + j];
      }
    return;
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) gm[i * n + j] = inner(g, psi + i * ng, phi + j * ng);
}

/* manifold.cpp:67-85: out_i = sum_k in_k m(k, i), zero coefficients skipped. */
void pp_mix(int64_t ng, int n, const double* in, const double* m, double* out) {
  for (int i = 0; i < n; ++i) {
    double* dst = out + (int64_t)i * ng;
    memset(dst, 0, sizeof(double) * (size_t)ng);
    for (int k = 0; k < n; ++k) {
      const double c = m[k * n + i];
      if (c == 0.0) continue;
      const double* src = in + (int64_t)k * ng;
      for (int64_t p = 0; p < ng; ++p) dst[p] += c * src[p];
    }
  }
}

/* LLT exactly as the oracle's clean-room Eigen subset computes it
 * (oracle/eigen_subset/Eigen/Cholesky); l row-major lower. */
static int llt(int n, const double* a, double* l) {
  memcpy(l, a, sizeof(double) * (size_t)n * (size_t)n);
  for (int j = 0; j < n; ++j) {
    double d = l[j * n + j];
    for (int k = 0; k < j; ++k) d -= l[j * n + k] * l[j * n + k];
    if (!(d > 0.0)) return -1;
    const double ljj = sqrt(d);
    l[j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = l[i * n + j];
      for (int k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
      l[i * n + j] = s / ljj;
    }
  }
  return 0;
}

/* manifold.cpp:97-114: out = in * L^{-T}; 0 on success, -1 on rejection. */
static int cholesky_pass(const pp_grid* g, int n, const double* in, const double* gm,
                         double* out, double* cond) {
  double* l = malloc(sizeof(double) * (size_t)n * (size_t)n);
  double* x = calloc((size_t)n * (size_t)n, sizeof(double));
  int rc = -1;
  if (llt(n, gm, l) != 0) goto done;
  double pmin = l[0], pmax = l[0];
  for (int i = 1; i < n; ++i) {
    if (l[i * n + i] < pmin) pmin = l[i * n + i];
    if (l[i * n + i] > pmax) pmax = l[i * n + i];
  }
  if (!(pmin > 0.0) || !isfinite(pmax) || pmin * pmin < 1e-10 * pmax * pmax) goto done;
  if (cond) *cond = (pmax / pmin) * (pmax / pmin);
  /* X = L^{-1} by forward substitution on I, column by column. */
  for (int c = 0; c < n; ++c)
    for (int i = 0; i < n; ++i) {
      double acc = i == c ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) acc -= l[i * n + k] * x[k * n + c];
      x[i * n + c] = acc / l[i * n + i];
    }
  /* M = X^T: M(k, i) = X(i, k) */
  double* m = malloc(sizeof(double) * (size_t)n * (size_t)n);
  for (int k = 0; k < n; ++k)
    for (int i = 0; i < n; ++i) m[k * n + i] = x[i * n + k];
  pp_mix(g->ng, n, in, m, out);
  free(m);
  rc = 0;
done:
  free(l);
  free(x);
  return rc;
}

/* Cyclic Jacobi eigensolver, ascending; evecs columns (row-major storage). */
int pp_syev(int n, const double* a_in, double* evals, double* v) {
  double* a = malloc(sizeof(double) * (size_t)n * (size_t)n);
  memcpy(a, a_in, sizeof(double) * (size_t)n * (size_t)n);
  for (int i = 0; i < n * n; ++i) v[i] = 0.0;
  for (int i = 0; i < n; ++i) v[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += a[i * n + j] * a[i * n + j];
        if (i != j) off += a[i * n + j] * a[i * n + j];
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (apq == 0.0) continue;
        const double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = c * akp - s * akq;
          a[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = c * apk - s * aqk;
          a[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = c * vkp - s * vkq;
          v[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  /* sort ascending (insertion sort on columns) */
  for (int i = 0; i < n; ++i) evals[i] = a[i * n + i];
  for (int i = 1; i < n; ++i) {
    for (int j = i; j > 0 && evals[j - 1] > evals[j]; --j) {
      const double t = evals[j]; evals[j] = evals[j - 1]; evals[j - 1] = t;
      for (int k = 0; k < n; ++k) {
        const double x = v[k * n + j]; v[k * n + j] = v[k * n + j - 1]; v[k * n + j - 1] = x;
      }
    }
  }
  free(a);
  return PP_OK;
}

/* manifold.cpp:118-132 */
static int symmetric_fallback(const pp_grid* g, int n, const double* in, const double* g0,
                              double* out) {
  double* s = malloc(sizeof(double) * (size_t)n * (size_t)n);
  double* q = malloc(sizeof(double) * (size_t)n * (size_t)n);
  double* lam = malloc(sizeof(double) * (size_t)n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) s[i * n + j] = 0.5 * (g0[i * n + j] + g0[j * n + i]);
  pp_syev(n, s, lam, q);
  const double lmax = lam[n - 1];
  int rc = PP_OK;
  if (!(lmax > 0.0) || !isfinite(lmax) || lam[0] < 1e-12 * lmax) {
    rc = PP_EDEGENERATE;
  } else {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double acc = 0.0;
        for (int k = 0; k < n; ++k) acc += q[i * n + k] * (1.0 / sqrt(lam[k])) * q[j * n + k];
        s[i * n + j] = acc;
      }
    pp_mix(g->ng, n, in, s, out);
  }
  free(s); free(q); free(lam);
  return rc;
}

static double max_dev_identity(int n, const double* gm) {
  double dev = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double v = fabs(gm[i * n + j] - (i == j ? 1.0 : 0.0));
      if (v > dev || isnan(v)) dev = v;
    }
  return dev;
}

/* manifold.cpp:136-169 */
int pp_orthonormalize(const pp_grid* g, int n, const double* in, int measure, double* out,
                      double* pre_gram, double* post_dev, int* used_fallback) {
  const size_t nn = (size_t)n * (size_t)n;
  double* g0 = pre_gram ? pre_gram : malloc(sizeof(double) * nn);
  pp_gram(g, n, in, in, 1, g0);
  double cond = INFINITY;
  int rc = PP_OK;
  if (used_fallback) *used_fallback = 0;
  if (cholesky_pass(g, n, in, g0, out, &cond) != 0) {
    rc = symmetric_fallback(g, n, in, g0, out);
    if (used_fallback) *used_fallback = 1;
    cond = INFINITY;
    if (rc) goto done;
  }
  if (!measure && cond <= 1e2) {
    if (post_dev) *post_dev = -1.0;
    goto done;
  }
  {
    double* g2 = malloc(sizeof(double) * nn);
    pp_gram(g, n, out, out, 1, g2);
    double dev = max_dev_identity(n, g2);
    if (!(dev <= 1e-12)) {
      double* rep = malloc(sizeof(double) * (size_t)n * (size_t)g->ng);
      if (cholesky_pass(g, n, out, g2, rep, NULL) != 0) {
        rc = PP_EDEGENERATE;
      } else {
        memcpy(out, rep, sizeof(double) * (size_t)n * (size_t)g->ng);
        pp_gram(g, n, out, out, 1, g2);
        dev = max_dev_identity(n, g2);
      }
      free(rep);
    }
    if (post_dev) *post_dev = dev;
    free(g2);
  }
done:
  if (!pre_gram) free(g0);
  return rc;
}

/* manifold.cpp:204-216 */
void pp_diagonal_residuals(const pp_grid* g, int n, const double* u, const double* hu,
                           double* z, double* sigma_diag) {
  for (int i = 0; i < n; ++i) {
    const double* a = hu + (int64_t)i * g->ng;
    const double* b = u + (int64_t)i * g->ng;
    const double s = inner(g, a, b);
    if (sigma_diag) sigma_diag[i] = s;
    const double ms = -s;
    double* d = z + (int64_t)i * g->ng;
    for (int64_t p = 0; p < g->ng; ++p) d[p] = a[p] + ms * b[p];
  }
}

/* manifold.cpp:181-202 (+ optimizer.cpp:474-476 norm accumulation) */
static int stiefel_dirs(const pp_grid* g, int n, const double* u, const double* hu,
                        double* dirs, double* sigma_out) {
  const size_t nn = (size_t)n * (size_t)n;
  double* sg = sigma_out ? sigma_out : malloc(sizeof(double) * nn);
  pp_gram(g, n, hu, u, 0, sg);
  double asym = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double v = fabs(sg[i * n + j] - sg[j * n + i]);
      if (v > asym) asym = v;
    }
  int rc = PP_OK;
  if (asym > 1e-10) {
    rc = PP_EINVAL;
  } else {
    for (int i = 0; i < n; ++i) {
      double* d = dirs + (int64_t)i * g->ng;
      memcpy(d, hu + (int64_t)i * g->ng, sizeof(double) * (size_t)g->ng);
      for (int k = 0; k < n; ++k) {
        const double c = sg[k * n + i];
        const double* src = u + (int64_t)k * g->ng;
        for (int64_t p = 0; p < g->ng; ++p) d[p] -= c * src[p];
      }
    }
  }
  if (!sigma_out) free(sg);
  return rc;
}

int pp_stiefel_gradient_norm2(const pp_grid* g, int n, const double* u, const double* hu,
                              double* norm2, double* sigma) {
  double* d = malloc(sizeof(double) * (size_t)n * (size_t)g->ng);
  int rc = stiefel_dirs(g, n, u, hu, d, sigma);
  if (rc == PP_OK) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += inner(g, d + (int64_t)i * g->ng, d + (int64_t)i * g->ng);
    *norm2 = acc;
  }
  free(d);
  return rc;
}

/* manifold.cpp:218-247 */
int pp_subspace_rotate(int n, const double* sigma, double* gamma, double* p) {
  double* s = malloc(sizeof(double) * (size_t)n * (size_t)n);
  double asym = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double v = fabs(sigma[i * n + j] - sigma[j * n + i]);
      if (v > asym) asym = v;
      s[i * n + j] = 0.5 * (sigma[i * n + j] + sigma[j * n + i]);
    }
  if (asym > 1e-8) { free(s); return PP_EINVAL; }
  pp_syev(n, s, gamma, p);
  for (int j = 0; j < n; ++j) {
    double scale = 0.0;
    for (int i = 0; i < n; ++i) if (fabs(p[i * n + j]) > scale) scale = fabs(p[i * n + j]);
    for (int i = 0; i < n; ++i) {
      if (fabs(p[i * n + j]) > 1e-12 * scale) {
        if (p[i * n + j] < 0.0)
          for (int k = 0; k < n; ++k) p[k * n + j] = -p[k * n + j];
        break;
      }
    }
  }
  free(s);
  return PP_OK;
}

/* ------------------------------------------------------------------- rng */

/* mt19937_64 (the C++ standard engine, restated) + rng.hpp:13-41 */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt_seed(mt64* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
  m->idx = 312;
}
static uint64_t mt_next(mt64* m) {
  if (m->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (m->mt[i] & 0xFFFFFFFF80000000ULL) | (m->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
    }
    m->idx = 0;
  }
  uint64_t y = m->mt[m->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}
static double mt_uniform(mt64* m) { return (double)(mt_next(m) >> 11) * 0x1.0p-53; }

void pp_rng_normals(uint64_t seed, int64_t count, double* out) {
  mt64 m;
  mt_seed(&m, seed);
  int have = 0;
  double spare = 0.0;
  for (int64_t k = 0; k < count; ++k) {
    if (have) { have = 0; out[k] = spare; continue; }
    double u1 = mt_uniform(&m);
    while (u1 == 0.0) u1 = mt_uniform(&m);
    const double r = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * kPi * mt_uniform(&m);
    spare = r * sin(theta);
    have = 1;
    out[k] = r * cos(theta);
  }
}

/* ------------------------------------------------------------- optimizer */

void pp_default_params(pp_params* p) { /* optimizer.hpp:22-46 */
  p->algorithm = PP_ALG_OPT_PAR_MOD;
  p->bb_variant = PP_BB1;
  p->bb_trace_abs = PP_TRACE_DIAG_ABS;
  p->convergence_mode = PP_CONV_GRAD_NORM;
  p->rho1 = 1e-4;
  p->delta = 0.1;
  p->eta = 0.85;
  p->n_diag = 100;
  p->n_org = 1;
  p->max_inner = 10000;
  p->max_backtracks = 20;
  p->tau_min = 1e-10;
  p->tau_max = 1e3;
  p->grad_tol = 1e-6;
  p->mean_abs_tol = 5e-9;
  p->energy_tol = 1e-13;
  p->verify_orthonormality = 1;
}

static double clamp_tau(double raw, const pp_params* p) { /* optimizer.cpp:25-28 */
  if (!isfinite(raw)) return p->tau_max;
  return raw < p->tau_min ? p->tau_min : (raw > p->tau_max ? p->tau_max : raw);
}
static int use_bb1(int v, int iter) { /* :30-34 */
  if (v == PP_BB1) return 1;
  if (v == PP_BB2) return 0;
  return iter % 2 == 0;
}

typedef struct {
  const pp_grid* g;
  int n;
  const double* v_ext;
  int hartree, xc;
  double occ;
} ctx_t;

typedef struct {
  pp_state st;
  double* buf;
} state_slot;

static void state_alloc(state_slot* s, int64_t ng) {
  s->buf = calloc((size_t)ng * 4, sizeof(double));
  s->st.rho = s->buf;
  s->st.v_h = s->buf + ng;
  s->st.v_xc = s->buf + 2 * ng;
  s->st.v_local = s->buf + 3 * ng;
  s->st.cg_iters = 0;
}
static void state_copy(state_slot* dst, const state_slot* src, int64_t ng) {
  if (dst->buf == src->buf) return;
  memcpy(dst->buf, src->buf, sizeof(double) * (size_t)ng * 4);
}
static void state_swap(state_slot* a, state_slot* b) {
  state_slot t = *a; *a = *b; *b = t;
}

/* InnerLoop::run, optimizer.cpp:322-579, and finalize :581-597. */
int pp_solve(const pp_grid* g, int n, const double* v_ext, int hartree, int xc,
             double occupation, const pp_params* p, const double* u0, pp_result* r) {
  const int64_t ng = g->ng;
  const size_t bsz = sizeof(double) * (size_t)n * (size_t)ng;
  const size_t nn = (size_t)n * (size_t)n;
  const int nonlinear = hartree || xc;
  const int n_org = p->algorithm == PP_ALG_OPT_PAR_MOD ? p->n_org : 1;
  const int full_grad = p->algorithm == PP_ALG_OPTM_QR;
  const int grad_style = p->convergence_mode == PP_CONV_GRAD_NORM ||
                         p->convergence_mode == PP_CONV_MEAN_ABS;
  const double wq = g->w;
  int rc = PP_OK;

  r->n_records = r->n_accepted = 0;
  r->cg_iters_total = 0;
  r->message[0] = 0;
  r->outcome = PP_OUT_MAX_ITERATIONS;

  /* run_single_level checks, optimizer.cpp:599-606 */
  if (!(p->rho1 > 0) || !(p->delta > 0 && p->delta < 1) || !(p->eta >= 0 && p->eta < 1) ||
      p->n_diag < 0 || p->n_org < 1 || p->max_inner < 1 || p->max_backtracks < 0 ||
      !(p->tau_min > 0) || !(p->tau_max >= p->tau_min) || r->cap < p->max_inner) {
    snprintf(r->message, sizeof r->message, "invalid optimizer parameters");
    return PP_EINVAL;
  }
  double* w = malloc(bsz);
  double* hw = malloc(bsz);
  double* z = malloc(bsz);
  double* prev_w = malloc(bsz);
  double* prev_z = malloc(bsz);
  double* trial = malloc(bsz);
  double* orth_w = malloc(bsz);
  double* rec_w = malloc(bsz);
  double* tmp = malloc(bsz);
  double* g0 = malloc(sizeof(double) * nn);
  double* pre = malloc(sizeof(double) * nn);
  double* sig = malloc(sizeof(double) * nn);
  double* gam = malloc(sizeof(double) * (size_t)n);
  double* pm = malloc(sizeof(double) * nn);
  double* kin_each = malloc(sizeof(double) * (size_t)n);
  double* ext_each = malloc(sizeof(double) * (size_t)n);
  double* orth_e = malloc(sizeof(double) * (size_t)(p->max_inner + 2));
  int n_orth_e = 0;
  state_slot cur, tri, rec;
  state_alloc(&cur, ng);
  state_alloc(&tri, ng);
  state_alloc(&rec, ng);

  memcpy(w, u0, bsz);
  pp_gram(g, n, w, w, 1, g0);
  if (max_dev_identity(n, g0) > 1e-8) {
    snprintf(r->message, sizeof r->message, "solver: initial orbital set is not orthonormal");
    rc = PP_EINVAL;
    goto cleanup;
  }

#define MAKE_STATE(slot, u)                                                            \
  do {                                                                                 \
    if (nonlinear || !fixed_built) {                                                   \
      rc = pp_build_hamiltonian(g, n, (u), v_ext, hartree, xc, occupation, &(slot).st); \
      if (rc) { snprintf(r->message, sizeof r->message, "build_hamiltonian failed"); goto cleanup; } \
      r->cg_iters_total += (slot).st.cg_iters;                                         \
      if (!nonlinear) { fixed_built = 1; state_copy(&cur, &(slot), ng);                \
        state_copy(&tri, &(slot), ng); state_copy(&rec, &(slot), ng); }                \
    }                                                                                  \
  } while (0)

  int fixed_built = 0;
  double e5[5];
  MAKE_STATE(cur, w);
  pp_apply_hamiltonian(g, cur.st.v_local, n, w, hw);
  pp_total_energy(g, n, w, v_ext, &cur.st, hartree, xc, occupation, e5, kin_each, ext_each);
  if (!isfinite(e5[4])) {
    snprintf(r->message, sizeof r->message, "non-finite total energy at the level start");
    r->outcome = PP_OUT_NUMERICAL_FAILURE;
    goto finalize;
  }
  r->e_kinetic = e5[0]; r->e_external = e5[1]; r->e_hartree = e5[2]; r->e_xc = e5[3];
  r->e_total = e5[4];

  double nm_c = e5[4], nm_q = 1.0;
  orth_e[n_orth_e++] = e5[4];
  int history_valid = 0, last_rotation_iter = 0, steps_until_orth = 0, converged = 0;
  memcpy(rec_w, w, bsz);
  state_copy(&rec, &cur, ng);
  int failed_searches = 0;
  double last_accepted_tau = 0.0;

  for (int l = 0; l < p->max_inner && !converged; ++l) {
    const int orth_iter = steps_until_orth == 0;
    const int need_full = orth_iter && grad_style;
    /* compute_directions, optimizer.cpp:265-320 */
    double znorm2 = 0.0, grad_norm = -1.0, mean_abs = -1.0;
    if (full_grad) {
      rc = stiefel_dirs(g, n, w, hw, z, NULL);
      if (rc) { snprintf(r->message, sizeof r->message, "stiefel_gradient: <(HU)^T U> is not symmetric"); goto cleanup; }
      for (int i = 0; i < n; ++i) znorm2 += inner(g, z + i * ng, z + i * ng);
      grad_norm = sqrt(znorm2 > 0.0 ? znorm2 : 0.0);
      if (p->convergence_mode == PP_CONV_MEAN_ABS && need_full) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += pw_abs_sum(ng, z + i * ng);
        mean_abs = acc / ((double)n * (double)ng);
      }
    } else {
      pp_diagonal_residuals(g, n, w, hw, z, NULL);
      for (int i = 0; i < n; ++i) znorm2 += inner(g, z + i * ng, z + i * ng);
      if (need_full) {
        rc = stiefel_dirs(g, n, w, hw, tmp, NULL);
        if (rc) { snprintf(r->message, sizeof r->message, "stiefel_gradient: <(HU)^T U> is not symmetric"); goto cleanup; }
        double acc = 0.0, abs_acc = 0.0;
        for (int i = 0; i < n; ++i) {
          acc += inner(g, tmp + i * ng, tmp + i * ng);
          if (p->convergence_mode == PP_CONV_MEAN_ABS) abs_acc += pw_abs_sum(ng, tmp + i * ng);
        }
        grad_norm = sqrt(acc > 0.0 ? acc : 0.0);
        if (p->convergence_mode == PP_CONV_MEAN_ABS) mean_abs = abs_acc / ((double)n * (double)ng);
      }
    }
    if (orth_iter && grad_style) {
      int conv = 0;
      if (p->convergence_mode == PP_CONV_GRAD_NORM) conv = grad_norm >= 0.0 && grad_norm < p->grad_tol;
      else conv = mean_abs >= 0.0 && mean_abs < p->mean_abs_tol;
      if (conv) { converged = 1; break; }
    }
    if (znorm2 == 0.0) { converged = 1; break; }

    double tau_raw;
    if (history_valid) { /* optimizer.cpp:376-411 */
      double tr_ss = 0.0, tr_yy = 0.0, sy_abs = 0.0, sy_tr = 0.0;
      for (int i = 0; i < n; ++i) {
        const double* wv = w + i * ng; const double* wp = prev_w + i * ng;
        const double* zv = z + i * ng; const double* zp = prev_z + i * ng;
        const double ss = wq * pw_diff_sq(ng, wv, wp);
        const double sy = wq * pw_diff_prod(ng, wv, wp, zv, zp);
        const double yy = wq * pw_diff_sq(ng, zv, zp);
        tr_ss += ss; tr_yy += yy; sy_abs += fabs(sy); sy_tr += sy;
      }
      const double tr_abs_sy = p->bb_trace_abs == PP_TRACE_DIAG_ABS ? sy_abs : fabs(sy_tr);
      const double raw = use_bb1(p->bb_variant, l) ? tr_ss / tr_abs_sy : tr_abs_sy / tr_yy;
      tau_raw = clamp_tau(raw, p);
    } else {
      const double inv = 1.0 / sqrt(znorm2);
      tau_raw = clamp_tau(p->tau_max < inv ? p->tau_max : inv, p);
    }

    pp_record rc_ = {0};
    rc_.level = 0;
    rc_.iter = l;
    rc_.grad_norm = grad_norm >= 0.0 ? grad_norm : sqrt(znorm2 > 0.0 ? znorm2 : 0.0);

    if (!orth_iter) { /* raw step, optimizer.cpp:419-444 */
      double tau = tau_raw;
      if (last_accepted_tau > 0.0 && 5.0 * last_accepted_tau < tau) tau = 5.0 * last_accepted_tau;
      const double mt = -tau;
      for (int64_t q = 0; q < (int64_t)n * ng; ++q) trial[q] = w[q] + mt * z[q];
      { double* t = prev_w; prev_w = w; w = trial; trial = t; }
      { double* t = prev_z; prev_z = z; z = t; }
      history_valid = 1;
      MAKE_STATE(cur, w);
      pp_apply_hamiltonian(g, cur.st.v_local, n, w, hw);
      --steps_until_orth;
      rc_.tau = tau;
      rc_.energy = orth_e[n_orth_e - 1];
    } else { /* backtracked orthogonalization step, :446-561 */
      int accepted = 0, s = 0, used_fb = 0;
      double tau = 0.0, dev = 0.0;
      double te[5] = {0};
      for (s = 0; s <= p->max_backtracks; ++s) {
        tau = tau_raw * pow(p->delta, s);
        if (s > 0 && tau < p->tau_min) break;
        const double mt = -tau;
        for (int64_t q = 0; q < (int64_t)n * ng; ++q) trial[q] = w[q] + mt * z[q];
        const int orc = pp_orthonormalize(g, n, trial, p->verify_orthonormality, orth_w, pre,
                                          &dev, &used_fb);
        if (orc == PP_EDEGENERATE) continue;
        MAKE_STATE(tri, orth_w);
        pp_total_energy(g, n, orth_w, v_ext, &tri.st, hartree, xc, occupation, te, kin_each, ext_each);
        if (isfinite(te[4]) && te[4] <= nm_c - p->rho1 * tau * znorm2) { accepted = 1; break; }
      }
      if (!accepted) {
        if (++failed_searches > 8) {
          snprintf(r->message, sizeof r->message,
                   "line search stagnated at level %d iteration %d (C = %.17g)", 0, l, nm_c);
          r->outcome = PP_OUT_STAGNATION;
          goto finalize;
        }
        memcpy(w, rec_w, bsz);
        state_copy(&cur, &rec, ng);
        pp_apply_hamiltonian(g, cur.st.v_local, n, w, hw);
        history_valid = 0;
        steps_until_orth = 0;
        continue;
      }
      failed_searches = 0;
      const double c_before = nm_c, q_before = nm_q;
      nm_q = p->eta * q_before + 1.0;
      nm_c = (p->eta * q_before * c_before + te[4]) / nm_q;
      if (r->accepted) {
        double* a = r->accepted + 9 * r->n_accepted;
        a[0] = 0; a[1] = l; a[2] = te[4]; a[3] = c_before; a[4] = nm_c; a[5] = q_before;
        a[6] = nm_q; a[7] = tau; a[8] = znorm2;
      }
      r->n_accepted++;
      if (te[4] > nm_c + 1e-9 * (1.0 + fabs(te[4]))) {
        snprintf(r->message, sizeof r->message, "nonmonotone ledger violated (C < E after update)");
        r->outcome = PP_OUT_NUMERICAL_FAILURE;
        goto finalize;
      }
      { double* t = prev_w; prev_w = w; w = orth_w; orth_w = t; }
      { double* t = prev_z; prev_z = z; z = t; }
      state_swap(&cur, &tri);
      history_valid = 1;
      last_accepted_tau = tau;
      pp_apply_hamiltonian(g, cur.st.v_local, n, w, hw);
      r->e_kinetic = te[0]; r->e_external = te[1]; r->e_hartree = te[2]; r->e_xc = te[3];
      r->e_total = te[4];
      orth_e[n_orth_e++] = te[4];
      double offd = 0.0;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
          if (i != j && fabs(pre[i * n + j]) > offd) offd = fabs(pre[i * n + j]);
      rc_.did_orth = 1;
      rc_.tau = tau;
      rc_.backtracks = s;
      rc_.offdiag_max = offd;
      rc_.energy = te[4];
      steps_until_orth = n_org - 1;
      if (p->n_diag > 0 && (l + 1 - last_rotation_iter) >= p->n_diag && !full_grad) {
        pp_gram(g, n, hw, w, 0, sig);
        if (pp_subspace_rotate(n, sig, gam, pm) != PP_OK) {
          snprintf(r->message, sizeof r->message, "subspace_rotate: Sigma asymmetry exceeds tolerance");
          rc = PP_EINVAL;
          goto cleanup;
        }
        pp_mix(ng, n, w, pm, tmp);
        memcpy(w, tmp, bsz);
        pp_mix(ng, n, hw, pm, tmp);
        memcpy(hw, tmp, bsz);
        last_rotation_iter = l + 1;
        rc_.did_diag = 1;
        history_valid = 0;
      }
      memcpy(rec_w, w, bsz);
      state_copy(&rec, &cur, ng);
      if (r->sigma_eigs) { /* trace: eig(<(HW)^T W>) at the accepted iterate */
        pp_gram(g, n, hw, w, 0, sig);
        if (pp_subspace_rotate(n, sig, gam, pm) == PP_OK)
          memcpy(r->sigma_eigs + (size_t)r->n_records * (size_t)n, gam, sizeof(double) * (size_t)n);
      }
      if (p->convergence_mode == PP_CONV_ENERGY_CHANGE && n_orth_e >= 4) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) {
          const double e_new = orth_e[n_orth_e - 1 - k], e_old = orth_e[n_orth_e - 2 - k];
          acc += fabs(e_old - e_new) / (fabs(e_old) + 1.0) / (double)(n_org > 1 ? n_org : 1);
        }
        if (acc / 3.0 < p->energy_tol) converged = 1;
      }
    }
    r->records[r->n_records++] = rc_;
  }
  r->outcome = converged ? PP_OUT_CONVERGED : PP_OUT_MAX_ITERATIONS;

finalize: /* optimizer.cpp:581-597 */
  MAKE_STATE(cur, w);
  pp_apply_hamiltonian(g, cur.st.v_local, n, w, hw);
  {
    double gn2 = 0.0;
    rc = pp_stiefel_gradient_norm2(g, n, w, hw, &gn2, NULL);
    if (rc) { snprintf(r->message, sizeof r->message, "stiefel_gradient: <(HU)^T U> is not symmetric"); goto cleanup; }
    r->final_grad_norm = sqrt(gn2 > 0.0 ? gn2 : 0.0);
  }
  if (r->w_out) memcpy(r->w_out, w, bsz);

cleanup:
#undef MAKE_STATE
  free(w); free(hw); free(z); free(prev_w); free(prev_z); free(trial); free(orth_w);
  free(rec_w); free(tmp); free(g0); free(pre); free(sig); free(gam); free(pm);
  free(kin_each); free(ext_each); free(orth_e);
  free(cur.buf); free(tri.buf); free(rec.buf);
  return rc;
}
