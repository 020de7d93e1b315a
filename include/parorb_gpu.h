/* parorb_gpu.h — C ABI of the B200-native hot path of arXiv 1510.07230.
 *
 * The reference (`parorb`, /root/reference/proj) exposes its hot path as C++
 * free functions over host `Field` vectors (include/parorb/grid.hpp:62-81,
 * energy.hpp:61-93, manifold.hpp:26-80) driven by the solver entry points
 * opt_par_inner / opt_par_mod_inner / optm_qr_solve (optimizer.hpp:153-161).
 * This header is the drop-in boundary for that path: plain C types, host
 * pointers and sizes, no CUDA or torch types. Device data stays resident in
 * an engine (one per GPU / rank); blocks are addressed by integer handles.
 *
 * Layout contract (same as the reference's Field, grid.hpp:11-14):
 *   - grid points p are lexicographic with the last axis fastest;
 *   - an orbital block is orbital-major, host[i * ng_local + p];
 *   - N x N matrices are row-major, m[i * n + j] = M(i, j);
 *   - a rank owns the planes [z0, z0 + nz) of axis 0 (slab decomposition).
 *
 * Errors: every call returns PO_OK (0) or a PO_E* code; po_last_error()
 * returns the message. The codes map one-to-one onto the reference's
 * exception classes (errors.hpp:10-45): PO_EINVAL -> InvalidArgument,
 * PO_EDEGENERATE -> DegenerateSetError, PO_ESOLVER -> SolverError,
 * PO_ESTAGNATION -> StagnationError. PO_ECUDA / PO_ENCCL / PO_ENOMEM are
 * device-side failures with no reference counterpart.
 *
 * Threading: one host thread per engine; calls are stream-ordered and not
 * re-entrant. Calls returning host scalars or matrices synchronise the
 * engine's stream. With size > 1 every rank must issue the same call
 * sequence (collectives are inside the calls).
 */
#ifndef PARORB_GPU_H
#define PARORB_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PO_ABI_VERSION 3  /* 2: po_result gained checkpoints / drift_iterations; po_stiefel_gradient_d; 3: po_direction_sums */

enum po_status {
  PO_OK = 0,
  PO_EINVAL = 1,
  PO_EDEGENERATE = 2,
  PO_ESOLVER = 3,
  PO_ESTAGNATION = 4,
  PO_ECUDA = 5,
  PO_ENCCL = 6,
  PO_ENOMEM = 7
};

/* Fields held by an engine (local slab, ng_local doubles each).
 * energy.hpp:41-50 HamiltonianState + Problem::v_ext. */
enum po_field { PO_VEXT = 0, PO_RHO = 1, PO_VH = 2, PO_VXC = 3, PO_VLOCAL = 4 };

/* Communicator kinds for multi-rank engines. */
enum po_comm_kind {
  PO_COMM_NONE = 0,    /* single rank */
  PO_COMM_NCCL = 1,    /* handle = 128-byte ncclUniqueId, one process per GPU */
  PO_COMM_THREADS = 2  /* in-process ranks sharing one po_thread_group (tests) */
};

typedef struct po_engine po_engine;
typedef struct po_thread_group po_thread_group;

typedef struct {
  int64_t n[3];      /* interior points per axis (3D only on this path) */
  double extent[3];  /* box side lengths, bohr */
} po_grid_desc;

typedef struct {
  int rank;
  int size;
  int kind;              /* po_comm_kind */
  const void* handle;    /* PO_COMM_NCCL: ncclUniqueId bytes; PO_COMM_THREADS: po_thread_group* */
  int device;            /* CUDA device ordinal (-1: current) */
} po_dist_desc;

/* ------------------------------------------------------------ lifecycle */

int po_abi_version(void);
/* grid.cpp:11-41 (Grid) + energy.cpp:34-60 (Problem). occupation = 1 is the
 * unmodified reference (energy.cpp:67-76); 2 is closed shell. dist may be NULL. */
int po_create(const po_grid_desc* grid, int n_orbitals, double occupation,
              const po_dist_desc* dist, po_engine** out);
int po_destroy(po_engine* e);
const char* po_last_error(const po_engine* e);
/* Local slab of this rank: first plane and plane count along axis 0. */
/* The engine's slab decomposition along axis 0 (host only; no GPU needed):
 * rank r of `size` owns planes [z0, z0 + nz), nz = n0 / size (+1 for the first
 * n0 % size ranks); its halo planes come from lo_peer / hi_peer (-1 at the
 * global boundary, where the Dirichlet zero applies, grid.cpp:109-119). */
int po_slab_plan(int64_t n0, int size, int rank, int64_t* z0, int64_t* nz, int* lo_peer,
                 int* hi_peer);
int po_local_slab(const po_engine* e, int64_t* z0, int64_t* nz, int64_t* ng_local);
/* Total device bytes an engine with these parameters needs for the solver
 * (before allocation); lets callers report "does not fit" instead of failing. */
int64_t po_solver_bytes(const po_grid_desc* grid, int n_orbitals, int size);
/* Default stream the engine launches on (cudaStream_t), for event timing. */
void* po_stream(po_engine* e);
int po_synchronize(po_engine* e);

/* In-process multi-rank group (PO_COMM_THREADS). */
int po_thread_group_create(int size, po_thread_group** out);
int po_thread_group_destroy(po_thread_group* g);

/* ------------------------------------------------------ data movement */

int po_alloc_block(po_engine* e, int* block);   /* N x ng_local, zero-filled */
int po_free_block(po_engine* e, int block);
int po_upload_block(po_engine* e, int block, const double* host);
int po_download_block(po_engine* e, int block, double* host);
int po_copy_block(po_engine* e, int dst, int src);
int po_set_field(po_engine* e, int field, const double* host);
int po_get_field(po_engine* e, int field, double* host);
/* Build V_ext on the device from softened-Coulomb atoms (energy.cpp:78-99).
 * atoms: natoms x {x, y, z, Z, a}. */
int po_external_potential(po_engine* e, const double* atoms, int natoms);
/* Smooth local potential sum_k A_k exp(-|r-c_k|^2 / (2 w_k^2)) (BASELINE C5).
 * wells: nwells x {cx, cy, cz, A, w}; written into V_ext. */
int po_gaussian_potential(po_engine* e, const double* wells, int nwells);
/* i.i.d. N(0,1) block from parorb::Rng(seed) (rng.hpp:13-41), orbital-major,
 * exactly the reference's bits; generated on the host for this rank's slab. */
int po_random_block(po_engine* e, int block, uint64_t seed);
/* i.i.d. N(0,1) block filled ON THE DEVICE from a counter hash of (seed, global
 * point, orbital): independent of the slab decomposition, NOT the reference's
 * Rng bits — for measurement blocks too large for the host draw (C5). */
int po_fill_normal(po_engine* e, int block, uint64_t seed);
/* optimizer.cpp:156-197 initialize_orbitals: Gaussians centred on the atoms
 * (x, y, z, Z, a per atom, cycled over the orbitals; the box centre without
 * atoms) with widths ~ U(0.5, 2) and 1e-2 U(-1, 1) noise from Rng(seed +
 * attempt), orthonormalised; up to 5 attempts. Result in block w. */
int po_initialize_orbitals(po_engine* e, const double* atoms, int natoms, uint64_t seed, int w);
/* grid.cpp:137-149 refine_uniform: n -> 2n + 1 per axis, same extents. */
int po_refine_grid(const po_grid_desc* grid, po_grid_desc* fine);
/* grid.cpp:151-203 prolongate, every orbital of block cblock (engine coarse)
 * into block fblock of engine fine (its grid = po_refine_grid of the coarse
 * one); bitwise the reference's values. Single-rank engines. */
int po_prolongate(po_engine* coarse, int cblock, po_engine* fine, int fblock);

/* ------------------------------------------------------------ operators */

/* energy.cpp:228-246 build_hamiltonian: rho -> v_H (Poisson CG) -> v_xc ->
 * v_local, from block u. Outputs E_H = 1/2 <v_H, rho>, E_xc = <eps_xc, rho>,
 * and the CG iteration count (any may be NULL). */
int po_build_hamiltonian(po_engine* e, int u, int hartree, int xc, double* e_hartree,
                         double* e_xc, int* cg_iters);
/* energy.cpp:248-265 apply_hamiltonian (batched) fused with the per-orbital
 * reductions sigma_ii = <Hu_i, u_i> (manifold.cpp:211), kinetic -1/2<lap u_i,
 * u_i> and external <V_ext u_i, u_i> (energy.cpp:267-280). out may be -1 (no
 * store); any host array may be NULL. Occupation is NOT applied to kin/ext. */
int po_apply_hamiltonian(po_engine* e, int u, int out, double* sigma_diag, double* kinetic,
                         double* external);
/* energy.cpp:282-314 total_energy from the state last built; out5 =
 * kinetic, external, hartree, xc, total. */
int po_total_energy(po_engine* e, int u, int hartree, int xc, double* out5);
/* grid.cpp:94-122 apply_laplacian on every orbital of a block. */
int po_laplacian(po_engine* e, int u, int out);
/* manifold.cpp:41-61 gram: G(i,j) = <a_i, b_j>; a == b uses the symmetric path. */
int po_gram(po_engine* e, int a, int b, double* g_host);
/* Gram of the fused trial point a + s b (no trial block written), symmetric. */
int po_gram_lincomb(po_engine* e, int a, double s, int b, double* g_host);
/* manifold.cpp:67-85 mix: out_i = sum_k in_k M(k, i). */
int po_mix(po_engine* e, int in, const double* m_host, int out);
/* manifold.cpp:136-169 orthonormalize_with_gram (Cholesky-QR on the device,
 * symmetric-eigen fallback, CholeskyQR2 repair). pre_gram may be NULL. */
int po_orthonormalize(po_engine* e, int in, int out, int measure, double* pre_gram,
                      double* post_deviation, int* used_fallback);
/* manifold.cpp:204-216 diagonal_residuals: z_i = hu_i - sigma_ii u_i. */
int po_diagonal_residuals(po_engine* e, int u, int hu, int z, double* sigma_diag,
                          double* z_norm2);
/* manifold.cpp:181-202 stiefel_gradient: sigma = <(HU)^T U> and, per orbital,
 * <D_i, D_i> with D = HU - U Sigma. PO_EINVAL if max|Sigma - Sigma^T| > 1e-10. */
int po_stiefel_gradient(po_engine* e, int u, int hu, double* sigma_host, double* d_norm2);
/* The same with the gradient block itself (StiefelGradient::directions,
 * manifold.hpp:47-54): D = HU - U Sigma written to block d (d != u, hu). */
int po_stiefel_gradient_d(po_engine* e, int u, int hu, int d, double* sigma_host,
                          double* d_norm2);
/* manifold.cpp:218-247 subspace_rotate: gamma ascending, P (row-major) with the
 * sign rule, w <- W P in place. */
int po_subspace_rotate(po_engine* e, int w, const double* sigma_host, double* gamma,
                       double* p_host);
/* grid.cpp:219-228 linear_combination, block-wise: out = a + s * b. */
int po_linear_combination(po_engine* e, int a, double s, int b, int out);
/* optimizer.cpp:376-397 per-orbital BB products (weighted). */
int po_bb_products(po_engine* e, int w, int w_prev, int z, int z_prev, double* ss,
                   double* sy, double* yy);

/* The direction step of one iteration as the solver runs it (optimizer.cpp:265-320 with
 * manifold.cpp:204-216, and the BB products of optimizer.cpp:386-397), the direction
 * z_i = HU_i - sigma_ii U_i never stored: sigma_ii = <hu_i, u_i>, ||z_i||^2 and — with a
 * history (u_prev, hu_prev >= 0, sigma_prev the previous iterate's sigma_ii) — <s_i, s_i>,
 * <s_i, y_i>, <y_i, y_i> for s = u - u_prev, y = z - z_prev, z_prev = hu_prev - sigma_prev u_prev.
 * sigma_full (row-major N x N, may be null) receives <(HU)^T U> (manifold.cpp:183). For
 * N > 64 all of it is ONE pass (the Sigma Gram carries the sums); smaller N take the Gram
 * and a streaming pass. Host outputs of length N; any may be null. */
int po_direction_sums(po_engine* e, int u, int hu, int u_prev, int hu_prev, const double* sigma_prev,
                      double* sigma_diag, double* sigma_full, double* zz, double* ss, double* sy,
                      double* yy);

/* -------------------------------------------------------------- solver */

enum { PO_ALG_OPTM_QR = 0, PO_ALG_OPT_PAR = 1, PO_ALG_OPT_PAR_MOD = 2 };
enum { PO_BB1 = 0, PO_BB2 = 1, PO_BB_ALTERNATE = 2 };
enum { PO_TRACE_DIAG_ABS = 0, PO_TRACE_ABS_TRACE = 1 };
enum { PO_CONV_GRAD_NORM = 0, PO_CONV_MEAN_ABS = 1, PO_CONV_ENERGY_CHANGE = 2 };
/* Hartree solve of -lap v = 4 pi rho (energy.cpp:105-143). All three stop on
 * the reference's criterion ||b - A x|| <= 1e-10 ||b||, checked with the
 * 7-point stencil; they differ only in the start point of the CG iteration. */
enum {
  PO_POISSON_CG = 0,       /* x0 = 0: the reference's algorithm */
  PO_POISSON_CG_WARM = 1,  /* x0 = previous v_H */
  PO_POISSON_DST = 2       /* x0 = fast-diagonalisation (DST-I) solve; CG verifies/refines */
};
enum { PO_OUT_CONVERGED = 0, PO_OUT_MAX_ITERATIONS = 1, PO_OUT_STAGNATION = 2,
       PO_OUT_NUMERICAL_FAILURE = 3 };

/* OptimizerParams, optimizer.hpp:22-46 (same fields, same defaults). */
typedef struct {
  int algorithm, bb_variant, bb_trace_abs, convergence_mode;
  double rho1, delta, eta;
  int n_diag, n_org, max_inner, max_backtracks;
  double tau_min, tau_max, grad_tol, mean_abs_tol, energy_tol;
  int verify_orthonormality;
  int hartree, xc;          /* Problem::hartree_enabled / xc_enabled */
  int trace_sigma_eigs;     /* record eig(<(HW)^T W>) after every accepted step */
  int poisson_solver;       /* PO_POISSON_* (default PO_POISSON_DST) */
  int outer_levels;         /* optimizer.hpp:39 (po_solve_levels) */
  uint64_t seed;            /* optimizer.hpp:40 initialize_orbitals seed (po_solve_levels) */
} po_params;

/* IterationRecord, optimizer.hpp:61-72. */
typedef struct {
  int level, iter;
  double energy, grad_norm, tau;
  int backtracks, did_orth, did_diag;
  double offdiag_max;
  double wall_ms;
} po_record;

typedef struct {
  int cap;                 /* capacity of records / accepted / sigma_eigs rows */
  po_record* records;
  double* accepted;        /* cap x 9: level, iter, E, C_before, C_after, Q_b, Q_a, tau, znorm2 */
  double* sigma_eigs;      /* cap x N or NULL */
  int n_records, n_accepted, outcome;
  int64_t cg_iters_total;
  double e_kinetic, e_external, e_hartree, e_xc, e_total;
  double final_grad_norm;
  double wall_seconds, par_seconds, sync_seconds;
  char message[200];
  /* SolveResult::checkpoints (optimizer.hpp:87-93, filled at optimizer.cpp:535-538):
   * one row per accepted orthogonalization step, cap x 5 = level, iter,
   * offdiag_max, diag_deviation_max, orth_deviation (-1 when not measured);
   * NULL to skip. n_checkpoints counts every step (rows beyond cap dropped). */
  double* checkpoints;
  int n_checkpoints;
  /* SolveResult::drift_iterations (optimizer.cpp:539: offdiag_max > 0.5), cap
   * entries or NULL; n_drift counts every flag. */
  int* drift_iterations;
  int n_drift;
} po_result;

void po_default_params(po_params* p);

/* Iterator form of the same loop (one InnerLoop iteration per step), for
 * callers that interleave their own work or time iterations individually.
 * create = InnerLoop set-up (initial state, energy; optimizer.cpp:358-372);
 * step = one iteration l (:374-576), *more = 0 once the loop has ended;
 * current = handle of the block holding the current iterate W;
 * finish = remaining iterations + finalize (:581-597), W copied into the
 * block given to create. The po_result is filled progressively. */
typedef struct po_solver po_solver;
int po_solver_create(po_engine* e, const po_params* p, int w, po_result* r, po_solver** out);
int po_solver_step(po_solver* s, int* more);
int po_solver_current(po_solver* s, int* block);
int po_solver_finish(po_solver* s);
int po_solver_destroy(po_solver* s);
/* Kernel launches issued by the library so far (process-wide). */
long long po_launch_count(void);

/* ------------------------------------------------- measurement helpers */

/* Enqueue ONE hot-path kernel on the engine stream without synchronising, so
 * a caller can bracket it with CUDA events on po_stream() (roofline timing,
 * BASELINE config 5 microbenchmarks). M for the mix ops is the matrix set by
 * po_set_matrix. */
enum {
  PO_OP_HAMILTONIAN = 0, /* out = H a (+ reductions), uses the default state's v_local */
  PO_OP_GRAM_SYM = 1,    /* G = <a^T a> (symmetric path) */
  PO_OP_GRAM = 2,        /* G = <a^T b> */
  PO_OP_MIX = 3,         /* out = a M */
  PO_OP_MIX_UPPER = 4,   /* out = a M, M upper triangular (the U L^{-T} rotation) */
  PO_OP_DENSITY_XC = 5,  /* rho, v_xc, 4 pi rho from block a */
  PO_OP_POISSON = 6,     /* CG solve on the last density (default state) */
  PO_OP_CHOLESKY = 7,    /* device Cholesky + L^{-T} of the last Gram */
  PO_OP_LAPLACIAN = 8,   /* out = lap a */
  PO_OP_GRAM_TRIAL = 9,  /* G = <(a - 0.3 b)^T (a - 0.3 b)> (the line-search trial Gram) */
  PO_OP_ROTATION = 10,   /* out = (a - 0.3 b) M, M = last Cholesky's L^{-T} (upper) */
  PO_OP_DIRECTIONS = 11, /* fused directions: W = a, HW = b, history (a, b), Sigma = last Gram */
  PO_OP_ROTATION_FUSED = 12, /* rotation + verification Gram + density/xc (default state) */
  PO_OP_ROTATION_IMPLICIT = 13, /* out = (a - 0.3 z) M with z = b - sigma a implicit (b = HW; N > 64) */
  PO_OP_GRAM_DENSITY = 15, /* G = <a^T a> + rho, 4 pi rho of block a in the same pass (64 < N <= 128) */
  PO_OP_GRAM_SIGMA_BB = 14, /* G = <a^T b> (a = HW, b = W) + the directions' ||z||^2 / BB sums (N > 64) */
  PO_OP_HAMILTONIAN_VARIANT = 100  /* + v: H a design-space variants (measurement builds only:
                                      make VARIANTS=1; else PO_EINVAL) */
};
int po_enqueue(po_engine* e, int op, int a, int b, int out);
int po_set_matrix(po_engine* e, const double* m_host);
/* Poisson solver used by po_build_hamiltonian / po_enqueue(PO_OP_POISSON). */
int po_set_poisson_solver(po_engine* e, int mode);
/* 128-byte NCCL unique id for PO_COMM_NCCL (rank 0 creates, caller broadcasts). */
int po_nccl_unique_id(void* out128);
/* optimizer.cpp:599-613 run_single_level: u0 (orthonormal, block handle) is
 * iterated in place — on return block w holds the final orbitals. */
int po_solve(po_engine* e, const po_params* p, int w, po_result* r);
/* The same on host buffers (N x ng_local, orbital-major): w_in uploaded, the
 * final orbitals written to w_out — the download overlaps the finalize pass. */
int po_solve_host(po_engine* e, const po_params* p, const double* w_in, double* w_out,
                  po_result* r);
/* optimizer.cpp:638-669 solve: initialize_orbitals(p->seed) on grid0 (atoms as
 * in po_external_potential), then p->outer_levels levels — from the second on,
 * refine_uniform + prolongate + orthonormalize — one InnerLoop each (records
 * carry the level), early stop on stagnation / numerical failure, finalize on
 * the last grid. Returns the final engine (caller po_destroy's it; also on
 * error, for po_last_error) and the block holding the final orbitals. */
int po_solve_levels(const po_grid_desc* grid0, int n_orbitals, double occupation,
                    const double* atoms, int natoms, const po_params* p, po_result* r,
                    po_engine** out_engine, int* out_block);
/* driver.cpp:131-142 log row "level,iter,energy,grad_norm,tau,backtracks,did_orth,
 * did_diag,offdiag_max,wall_ms" (no newline); returns the length or -1. */
int po_format_log_row(const po_record* rec, char* buf, int len);
/* driver.cpp:152-165 write_log (header + every log_every-th row + each level's last);
 * driver.cpp:199-215 write_reduction (final level, orthonormalisation steps). */
int po_write_log(const char* path, const po_record* recs, int n, int log_every);
int po_write_reduction(const char* path, const po_record* recs, int n, double e_min);

#ifdef __cplusplus
}
#endif
#endif
