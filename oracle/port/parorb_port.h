/* parorb_port — CPU restatement of the reference's hot path in plain C.
 *
 * TEST INFRASTRUCTURE ONLY: this is the parity oracle. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it, and only as the checker or the timed CPU baseline — never as
 * the product path. Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj). Floating-point operation order
 * follows the reference so that, compiled with -ffp-contract=off, results
 * match the unmodified reference (oracle/_ref) bit for bit except where the
 * reference calls Eigen (Cholesky / eigensolver), where they agree to
 * round-off.
 *
 * Layout: an orbital block is orbital-major, u[i * ng + p], p lexicographic
 * with the last axis fastest (include/parorb/grid.hpp:11-14). N x N matrices
 * are row-major, m[i * n + j] = M(i, j).
 */
#ifndef PARORB_PORT_H
#define PARORB_PORT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int dim;
  int64_t n[3];
  double ext[3];
  double h[3];
  double w;  /* quadrature weight */
  int64_t ng;
} pp_grid;

typedef struct {
  double pos[3];
  double charge;
  double softening;
} pp_atom;

enum { PP_OK = 0, PP_EINVAL = 1, PP_EDEGENERATE = 2, PP_ESOLVER = 3, PP_ESTAGNATION = 4 };
enum { PP_ALG_OPTM_QR = 0, PP_ALG_OPT_PAR = 1, PP_ALG_OPT_PAR_MOD = 2 };
enum { PP_BB1 = 0, PP_BB2 = 1, PP_BB_ALTERNATE = 2 };
enum { PP_TRACE_DIAG_ABS = 0, PP_TRACE_ABS_TRACE = 1 };
enum { PP_CONV_GRAD_NORM = 0, PP_CONV_MEAN_ABS = 1, PP_CONV_ENERGY_CHANGE = 2 };
enum { PP_OUT_CONVERGED = 0, PP_OUT_MAX_ITERATIONS = 1, PP_OUT_STAGNATION = 2,
       PP_OUT_NUMERICAL_FAILURE = 3 };

/* OptimizerParams, include/parorb/optimizer.hpp:22-46 */
typedef struct {
  int algorithm, bb_variant, bb_trace_abs, convergence_mode;
  double rho1, delta, eta;
  int n_diag, n_org, max_inner, max_backtracks;
  double tau_min, tau_max, grad_tol, mean_abs_tol, energy_tol;
  int verify_orthonormality;
} pp_params;

/* IterationRecord, optimizer.hpp:61-72 (wall_ms omitted) */
typedef struct {
  int level, iter;
  double energy, grad_norm, tau;
  int backtracks, did_orth, did_diag;
  double offdiag_max;
} pp_record;

typedef struct {
  /* caller-provided capacities/buffers */
  int cap;                  /* >= max_inner */
  pp_record* records;       /* cap */
  double* accepted;         /* cap * 9: level, iter, E, c_b, c_a, q_b, q_a, tau, znorm2 */
  double* sigma_eigs;       /* optional cap * n: eig(<(HW)^T W>) after each accepted step */
  double* w_out;            /* n * ng final orbitals */
  /* outputs */
  int n_records, n_accepted, outcome, cg_iters_total;
  double e_kinetic, e_external, e_hartree, e_xc, e_total;
  double final_grad_norm;
  char message[200];
} pp_result;

void pp_default_params(pp_params* p);
int pp_grid_init(pp_grid* g, int dim, const int64_t* n, const double* ext);

/* numeric.hpp:12-34 */
double pp_pairwise_dot(int64_t n, const double* a, const double* b);
double pp_pairwise_sum(int64_t n, const double* a);
/* grid.cpp:94-122 */
void pp_laplacian(const pp_grid* g, const double* f, double* out);
/* energy.cpp:78-99 */
void pp_external_potential(const pp_grid* g, const pp_atom* atoms, int natoms, double* v);
/* energy.cpp:67-76 (occupation 1 = unmodified reference) */
void pp_density(const pp_grid* g, int n, const double* u, double occupation, double* rho);
/* energy.cpp:105-143 + 197-210; returns PP_OK or PP_ESOLVER / PP_EINVAL */
int pp_hartree(const pp_grid* g, const double* rho, double* vh, int* cg_iters);
/* energy.cpp:212-226 */
int pp_xc_energy_density(int64_t ng, const double* rho, double* eps);
int pp_xc_potential(int64_t ng, const double* rho, double* v);
/* energy.cpp:248-257 */
void pp_apply_hamiltonian(const pp_grid* g, const double* v_local, int n, const double* u,
                          double* hu);
/* energy.cpp:267-280 */
double pp_kinetic_term(const pp_grid* g, const double* u);
double pp_potential_term(const pp_grid* g, const double* v, const double* u);

/* Hamiltonian state, energy.hpp:41-50 / energy.cpp:228-246 */
typedef struct {
  double *rho, *v_h, *v_xc, *v_local;
  int cg_iters;
} pp_state;
int pp_build_hamiltonian(const pp_grid* g, int n, const double* u, const double* v_ext,
                         int hartree, int xc, double occupation, pp_state* s);
/* energy.cpp:282-314; out5 = kinetic, external, hartree, xc, total */
void pp_total_energy(const pp_grid* g, int n, const double* u, const double* v_ext,
                     const pp_state* s, int hartree, int xc, double occupation, double* out5,
                     double* kin_each, double* ext_each);

/* manifold.cpp:41-61 (same != 0: symmetric fill) */
void pp_gram(const pp_grid* g, int n, const double* psi, const double* phi, int same,
             double* gm);
/* manifold.cpp:67-85 */
void pp_mix(int64_t ng, int n, const double* in, const double* m, double* out);
/* manifold.cpp:136-169; returns PP_OK or PP_EDEGENERATE */
int pp_orthonormalize(const pp_grid* g, int n, const double* in, int measure, double* out,
                      double* pre_gram, double* post_dev, int* used_fallback);
/* manifold.cpp:204-216 */
void pp_diagonal_residuals(const pp_grid* g, int n, const double* u, const double* hu,
                           double* z, double* sigma_diag);
/* manifold.cpp:181-202: gradient squared norm sum_i <D_i, D_i>; PP_EINVAL on asymmetry */
int pp_stiefel_gradient_norm2(const pp_grid* g, int n, const double* u, const double* hu,
                              double* norm2, double* sigma);
/* symmetric eigensolver for n x n row-major (cyclic Jacobi), ascending */
int pp_syev(int n, const double* a, double* evals, double* evecs_rowmajor);
/* manifold.cpp:218-247: gamma ascending and P (row-major) with the sign rule */
int pp_subspace_rotate(int n, const double* sigma, double* gamma, double* p);

/* optimizer.cpp:599-629 (run_single_level -> InnerLoop::run -> finalize) */
int pp_solve(const pp_grid* g, int n, const double* v_ext, int hartree, int xc,
             double occupation, const pp_params* p, const double* u0, pp_result* r);

/* rng.hpp:13-41 + tests/problems.hpp:59-68 (normals only; caller orthonormalizes) */
void pp_rng_normals(uint64_t seed, int64_t count, double* out);

#ifdef __cplusplus
}
#endif
#endif
