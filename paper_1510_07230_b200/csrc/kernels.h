// Host-side launchers of the parorb sm_100a kernels (internal to libparorb_b200).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace po {

// Number of kernel launches issued by this library (bench evidence of GPU work).
void count_launch();
long long launch_count();

// ---------------------------------------------------------------- stencil.cu
// Batched H u (energy.cpp:248-265) fused with the per-orbital reductions
// sigma_ii, <lap u_i, u_i>, <V_ext u_i, u_i> (energy.cpp:267-280). Partials:
// [3][N][nblk], raw (unweighted) sums. hu may be null (reductions only).
int hamiltonian_nblk(const SlabGeom& g);
void launch_hamiltonian(const SlabGeom& g, int N, const double* u, const double* halo_lo,
                        const double* halo_hi, const double* v_local, const double* v_ext,
                        double* hu, double* partials, cudaStream_t s);
// v2: register-queue z-march, shuffle/smem neighbours; v_ext may be null (no
// external partials). Partials [3][N][hamiltonian2_nblk].
int hamiltonian2_nblk(const SlabGeom& g);
void launch_hamiltonian2(const SlabGeom& g, int N, const double* u, const double* halo_lo,
                         const double* halo_hi, const double* v_local, const double* v_ext,
                         double* hu, double* partials, cudaStream_t s);
// Slab H u with the halo exchange overlapped: interior planes 1 .. nz-2 (no
// halo needed) and, once the neighbours' planes arrived, planes 0 and nz-1;
// both fill one partials layout of hamiltonian_split_nblk columns (nz >= 3).
bool hamiltonian_split_ok(const SlabGeom& g);
int hamiltonian_split_nblk(const SlabGeom& g);
void launch_hamiltonian_interior(const SlabGeom& g, int N, const double* u, const double* v_local,
                                 const double* v_ext, double* hu, double* partials, cudaStream_t s);
void launch_hamiltonian_boundary(const SlabGeom& g, int N, const double* u, const double* halo_lo,
                                 const double* halo_hi, const double* v_local, const double* v_ext,
                                 double* hu, double* partials, cudaStream_t s);
#ifdef PO_MEASUREMENT_VARIANTS  // make VARIANTS=1 (measurement-only H u variants)
int launch_hamiltonian_variant(int v, const SlabGeom& g, int N, const double* u,
                               const double* v_local, const double* v_ext, double* hu,
                               double* partials, cudaStream_t s);
#endif
// Plain 7-point Dirichlet Laplacian of every orbital (grid.cpp:94-122).
void launch_laplacian(const SlabGeom& g, int N, const double* u, const double* halo_lo,
                      const double* halo_hi, double* out, cudaStream_t s);

// ----------------------------------------------------------------- fields.cu
int points_nblk(const SlabGeom& g);
// CTAs per orbital of the per-orbital streaming kernels (partials row length).
int per_orbital_nblk(const SlabGeom& g, int N);
// rho = f sum_i u_i^2 (energy.cpp:67-76); v_xc, eps (energy.cpp:212-226);
// b = 4 pi rho written at b (may be null). Partials [2][nblk]: sum eps*rho, sum v_ext*rho
// (v_ext may be null).
void launch_density_xc(const SlabGeom& g, int N, const double* u, double occupation, int xc,
                       double* rho, double* v_xc, double* b, const double* v_ext, double* partials,
                       cudaStream_t s, const double* guard = nullptr);
// v_local = v_ext + (v_h + v_xc) (energy.cpp:241-244); partials [1][nblk]: sum v_h*rho.
// xc_here >= 0: v_xc formed here from rho (Dirac when 1, zero when 0) and partials
// [3][nblk]: sum eps*rho, sum v_ext*rho, sum v_h*rho.
void launch_vlocal(const SlabGeom& g, const double* v_ext, const double* v_h_src, double* v_h,
                   double* v_xc, const double* rho, double* v_local, double* partials,
                   cudaStream_t s, int xc_here = -1, const double* bfull = nullptr,
                   const double* xfull = nullptr, int* cg_out = nullptr);
// z_i = hu_i - sigma_ii u_i (manifold.cpp:204-216); partials [1][N][nblk]: sum z^2.
void launch_residual_diag(const SlabGeom& g, int N, const double* u, const double* hu,
                          const double* sigma_diag, double* z, double* partials, cudaStream_t s);
// residual + BB products in one pass; partials [4][N][nblk]: zz, ss, sy, yy (raw).
void launch_residual_bb(const SlabGeom& g, int N, const double* u, const double* hu,
                        const double* sigma_diag, const double* up, const double* zp, double* z,
                        double* partials, cudaStream_t s);
// The elementwise directions pass (N > 64 with ||D||^2 from the Grams): z = fma(-sigma, u, hu)
// (written only if z != null), partials [4][N][nblk]: zz, ss, sy, yy (raw) against
// (up, z_prev), z_prev = fma(-sig_prev, up, xp) when sig_prev else xp; no history when
// up is null (row 0 only). Returns nblk.
int launch_residual_bb_stream(const SlabGeom& g, int N, const double* u, const double* hu,
                              const double* sigma_diag, const double* up, const double* xp,
                              const double* sig_prev, double* z, double* partials, cudaStream_t s);
// BB products (optimizer.cpp:386-397); partials [3][N][nblk]: ss, sy, yy (raw).
void launch_bb(const SlabGeom& g, int N, const double* w, const double* wp, const double* z,
               const double* zp, double* partials, cudaStream_t s);
// out = a + s * b over a whole block (grid.cpp:219-228).
void launch_z_from_hw(const SlabGeom& g, int N, const double* w, const double* hw,
                      const double* sig, double* z, cudaStream_t s);
void launch_lincomb(const SlabGeom& g, int N, const double* a, double sc, const double* b,
                    double* out, cudaStream_t s);
// Per-orbital sum of |x| (mean-abs convergence, optimizer.cpp:446-458): partials [1][N][nblk].
void launch_abs_sum(const SlabGeom& g, int N, const double* x, double* partials, cudaStream_t s);
// out[r] = scale * sum_b partials[r * nblk + b], fixed order (deterministic).
void launch_reduce_rows(const double* partials, int rows, int nblk, double scale, double* out,
                        cudaStream_t s, const double* guard = nullptr);
// ngroups (<= 3) consecutive groups of grp rows, group q scaled by scales[q], one launch.
// (rows > grp * ngroups: the rows past the groups take the last scale.)
void launch_reduce_rows_grouped(const double* partials, int grp, int ngroups, int nblk,
                                const double* scales, double* out, cudaStream_t s, int rows = 0);
// V_ext from softened-Coulomb atoms (energy.cpp:78-99) / Gaussian wells (C5).
void launch_external_potential(const SlabGeom& g, const double* h3, const double* atoms,
                               int natoms, int gaussian, double* v, cudaStream_t s);
// Pack plane `plane_idx` of every orbital into dst[N][plane] (halo send buffers).
void launch_pack_plane(const SlabGeom& g, int N, const double* u, int64_t plane_idx,
                       double* dst, cudaStream_t s);

// ------------------------------------------------------------------ dmma.cu
// Split-K tall-skinny Gram on the FP64 tensor cores (mma.sync f64):
// G(i,j) = w * sum_p (A + sa Ab)_i[p] (B + sb Bb)_j[p]. Ab/Bb may be null.
// sym: A == B (and Ab == Bb, sa == sb); only upper tiles are computed and
// G is mirrored exactly (manifold.cpp:45-53). G: device N x N row-major.
size_t gram_workspace_doubles(const SlabGeom& g, int N);
void launch_gram(const SlabGeom& g, int N, const double* A, const double* Ab, double sa,
                 const double* B, const double* Bb, double sb, int sym, double* ws,
                 double* G, cudaStream_t s, const double* guard = nullptr);
// Column mixing on the FP64 tensor cores (manifold.cpp:67-85):
// out_i = alpha * sum_k (A + sa Ab)_k M(k, i) + beta * C_i. M device row-major.
// upper: M is upper triangular (skip zero k-blocks). out may be null; norms
// (may be null) receives partials [N][nblk] of sum_p out_i[p]^2.
int mix_nblk(const SlabGeom& g);
int mix_nblk_max(const SlabGeom& g);  // partials buffer sizing (any mix path)
// zsig (nullable, large-N TMA paths only): Ab is HW and the second source is the
// implicit direction z = HW - zsig_k W (rebuilt per element with the FMA the
// directions pass uses); -2 when no path can take it.
int launch_mix(const SlabGeom& g, int N, const double* A, const double* Ab, double sa,
                const double* M, double alpha, const double* C, double beta, int upper,
                double* out, double* norms, cudaStream_t s, const double* guard = nullptr,
                const double* zsig = nullptr);

// dmma_tma.cu: 2D tensor-map TMA versions of the small-N Gram / mix (false / -1
// when unavailable: no driver entry point or N out of range).
bool tma2d_available();
// once per kernel: max-shared carveout + dynamic shared-memory limit (bytes may be 0)
void set_smem(const void* k, int bytes);
// G2 != null with sym = 0: the same pass also writes G2 = w A^T A (symmetric).
// diag (optional): G's diagonal also written there (one launch for the reduction).
bool launch_gram_tma(int N, int64_t ld, int sym, const double* A, const double* Ab, double sa,
                     const double* B, const double* Bb, double sb, double* ws, double* G, double w,
                     cudaStream_t s, const double* guard, double* G2 = nullptr,
                     double* diag = nullptr);
// Trial Gram of W - tau Z from the iteration's Grams, Z = HW - W diag(sigma):
//   G0 = G_WW - tau (W^T Z + Z^T W) + tau^2 Z^T Z with W^T Z = Sigma^T - G_WW diag(sigma),
//   Z^T Z = G_HH - Sigma diag(sigma) - diag(sigma) Sigma^T + diag(sigma) G_WW diag(sigma)
// (Sigma_ij = <HW_i, W_j>). Exactly symmetric.
void launch_trial_gram(int N, const double* gww, const double* sigma, const double* ghh,
                       double tau, double* G0, cudaStream_t s, const double* tau_dev = nullptr);
// Barzilai-Borwein step on the device (optimizer.cpp:25-41, 376-411), same
// sequential sums as the host mirror: out[0] = tau_raw, out[1] = -tau_raw,
// out[2] = sum_i zz_i. zz/ss/sy/yy are per-orbital rows (ss/sy/yy unused
// without history).
void launch_bb_tau(int N, const double* zz, const double* ss, const double* sy, const double* yy,
                   int history, int use_bb1, int trace_abs_diag, double tau_min, double tau_max,
                   double* out, cudaStream_t s);
// Large-N (N > 48) Gram: 128x128 (or 64x64) orbital tiles x point splits,
// one 16-point 2D box per source per stage; returns false when unavailable.
size_t gram_big_workspace_doubles(int64_t ld, int N);
// rho (nullable): with one source, sym and 64 < N <= 128 (one diagonal tile) the
// Gram also writes the density occ sum_i A_i^2 (+ 4 pi rho into bvec) of the
// ngl points; false (nothing launched) where that is unavailable
// bbl (N > 64, A = HW, B = W, non-symmetric): the Gram also does the
// elementwise half of compute_directions (||z_i||^2 and, with wp / xp, the BB
// products; z = HW - sig W implicit) — partials [4][N][nsplit]: zz, ss, sy, yy.
struct GramBB {
  const double* sig;   // sigma_i (device, N): the H u pass's <HW_i, W_i>
  const double* sigp;  // previous sigma when xp is the previous HW, null when xp is a stored Z_prev
  const double* wp;    // W_prev (null: no history, only ||z||^2)
  const double* xp;    // HW_prev or Z_prev
  double* partials;
  int nsplit;          // out: partial columns per (sum, orbital)
};
bool launch_gram_big(int N, int64_t ld, int sym, const double* A, const double* Ab, double sa,
                     const double* B, const double* Bb, double sb, double* ws, size_t ws_doubles,
                     double* G, double w, cudaStream_t s, const double* guard, double* rho = nullptr,
                     double* bvec = nullptr, double occ = 1.0, int64_t ngl = 0, GramBB* bbl = nullptr);
// Fused compute_directions + BB products for N <= 48 (one pass over W, HW
// [, WP, ZP]): writes Z = HW - diag(sig) W and per-orbital partial rows
// [zz | dd | ss | sy | yy] (dd = ||HW - W Sigma||^2 when Sigma != null; the
// last three only with WP/ZP). Returns the partials row length, -1 if N is
// out of range or 2D TMA is unavailable.
// Line-search rotation W~ = (A + sa Ab) M (M upper) fused with the
// verification Gram G = w W~^T W~ (written to G) and the density / Dirac xc of
// W~ (rho, v_xc, 4 pi rho into bvec when non-null, partial rows [<eps,rho> |
// <V_ext,rho>] x grid in dpart). N <= 48; returns the partials row length or -1.
int launch_rotate_fused(int N, int64_t ld, int64_t ngl, const double* A, const double* Ab,
                        double sa, const double* M, double* out, double* ws, double* G, double w,
                        double occ, int xc, double* rho, double* vxc, double* bvec,
                        const double* vext, double* dpart, cudaStream_t s,
                        const double* sa_dev = nullptr, const double* zsig = nullptr);
// zsig (rotate_fused): Ab is HW and the direction is z = HW - zsig W, rebuilt in
// the kernel. Directions: Z may be null (z not stored); psig: ZP is the previous
// HW and the previous z is HWP - psig WP; sig_out receives the sigma used.
int launch_directions(int N, int64_t ld, int64_t ngl, const double* W, const double* HW,
                      const double* WP, const double* ZP, const double* Sigma, const double* sig,
                      double* Z, double* partials, cudaStream_t s, const double* psig = nullptr,
                      double* sig_out = nullptr);
int launch_mix_tma(int N, int64_t ld, int64_t ngl, const double* A, const double* Ab, double sa,
                   const double* M, double alpha, const double* C, double beta, int upper,
                   double* out, double* norms, cudaStream_t s, const double* guard);
// Large-N (N > 64) mix: persistent 128-point x 128-orbital DMMA tiles fed by
// 2D TMA (A, Ab and a padded M^T). Same contract as launch_mix; returns the
// norm-partials row length (= mix_nblk) or -1 when unavailable.
int launch_mix_big(int N, int64_t ld, int64_t ngl, const double* A, const double* Ab, double sa,
                   const double* M, double alpha, const double* C, double beta, int upper,
                   double* out, double* norms, cudaStream_t s, const double* guard,
                   const double* zsig = nullptr);
// compute_directions for N > 64 (dir_big_kernel): partial rows [zz | dd | ss | sy | yy]
// x n_pt. History (WP != null): XP_ is HW_prev with sig_prev (implicit z_prev =
// HW_prev - sig_prev W_prev) or a stored Z_prev (sig_prev null). Z null: z stays
// implicit; sig_save (nullable) receives sig for the next iteration's z_prev.
int launch_directions_big(int N, int64_t ld, int64_t ngl, const double* W, const double* HW,
                          const double* WP, const double* XP_, const double* sig_prev,
                          const double* Sigma, const double* sig, double* Z, double* sig_save,
                          double* partials, cudaStream_t s);
// Batched left-multiply out_b = S X_b for X_b = rows [N][ld] at A + b * bstride
// (valid row length ngl; ld multiple of 32, padding zero). DST transforms.
void launch_mix_batched(int N, int64_t ld, int64_t ngl, int batch, int64_t bstride,
                        const double* A, const double* M, double* out, cudaStream_t s);

// ----------------------------------------------------------------- dense.cu
// Cholesky G = L L^T (lower) and M = L^{-T} (upper, row-major M[k*N+i]),
// following manifold.cpp:97-114. stats: {pmin, pmax, cond, ok}.
void launch_cholesky_inv(int N, const double* G, double* Lscratch, double* M, double* stats,
                         cudaStream_t s, const double* guard = nullptr);
// Arguments of the device-side BB step (launch_bb_tau), for fusing it into a later kernel.
struct BBArgs {
  int N;
  const double *zz, *ss, *sy, *yy;
  int history, use_bb1, trace_abs_diag;
  double tau_min, tau_max;
  double* out;
};
// trial_gram + matrix_stats(G0) + Cholesky / L^{-T} of G0 in one launch (N <= 128); with bb
// the BB step runs first in the same kernel and tau comes from it (out[0]):
// G0 of W - tau Z from G_WW, Sigma, G_HH (tau from tau_dev when non-null) into G0,
// its statistics into mstats, then as launch_cholesky_inv. false when unavailable.
bool launch_trial_cholesky(int N, const double* gww, const double* sigma, const double* ghh,
                           double tau, const double* tau_dev, double* G0, double* mstats, double* M,
                           double* stats, cudaStream_t s, const BBArgs* bb = nullptr);
// Device-side decisions of manifold.cpp:147-167 without a host round trip:
// out[0] = 1 if the repair pass runs ((measure || cond > 100) && dev > 1e-12),
// from the pass-1 Cholesky stats and the verification-Gram stats.
void launch_qr2_decision(const double* chol_stats, const double* gram2_stats, int measure,
                         double* out, cudaStream_t s);
// dst = src (n doubles) if guard is null or *guard != 0
void launch_copy_guarded(double* dst, const double* src, int64_t n, const double* guard,
                         cudaStream_t s);
// Symmetric eigensolver (parallel cyclic Jacobi) on 1/2 (A + A^T):
// evals ascending, evecs column j in evecs[i*N + j]; sign rule of
// manifold.cpp:233-241 applied when sign_rule != 0. stats: {asym, ok}.
void launch_syev(int N, const double* A, double* work, double* evals, double* evecs,
                 int sign_rule, double* stats, cudaStream_t s);
// M = Q diag(lam^{-1/2}) Q^T (manifold.cpp:128-130); stats: {lam_min, lam_max, ok}.
void launch_inv_sqrt_from_eig(int N, const double* evals, const double* evecs, double* M,
                              double* stats, cudaStream_t s);
// max |G - I| (manifold.cpp:158) and max |S - S^T|, offdiag / diag deviation
// (manifold.cpp:249-259): out {dev, asym, offdiag_max, diag_dev_max}.
void launch_matrix_stats(int N, const double* G, double* out, cudaStream_t s,
                         const double* guard = nullptr);
// out[i] = M(i, i)
void launch_copy_diag(int N, const double* M, double* out, cudaStream_t s);
// ||D_i||^2 of D = HW - W Sigma from Sigma, G_WW, G_HH (dd) with a rounding bound
// (err); sig_save (nullable) <- sig (dense.cu dnorm_grams_kernel)
void launch_dnorm_grams(int N, const double* S, const double* Gww, const double* Ghh, double* dd,
                        double* err, const double* sig, double* sig_save, cudaStream_t s);

// ------------------------------------------------------------------ rng.cu
// parorb::Rng(seed) normals (rng.hpp:13-41) drawn orbital-major over the full
// grid (tests/problems.hpp:59-68); keeps points [offset, offset+count) of each
// of the N orbitals: out[i * count + k].
// i.i.d. N(0,1) device fill from a counter hash of (seed, global point, orbital)
// — measurement blocks (C5), not the reference's Rng bits; padding untouched
void launch_fill_normal(const SlabGeom& g, int N, int64_t ng_full, uint64_t seed, double* out,
                        cudaStream_t s);
void rng_normals_slab(uint64_t seed, int N, int64_t ng_full, int64_t offset, int64_t count,
                      double* out);

// --------------------------------------------------------------- poisson.cu
struct CgResult {
  int status;      // 0 ok, 3 solver error
  int iters;       // CG iterations over all restarts
  double bnorm;
};
// -lap x = b (Dirichlet) by CG on the full grid, x0 = 0 or warm (x holds the
// guess), rel. tol 1e-10, <= 20000 its x <= 4 passes (energy.cpp:105-143).
// One cooperative persistent kernel; work: ws >= 5 * ng doubles + scratch.
size_t cg_workspace_doubles(int64_t ng);
// Fast-diagonalisation Poisson solve (DST-I along each axis as FP64 tensor-core
// left-multiplies): x = A^{-1} b to round-off, used as the CG start point.
struct DstPoisson {
  int64_t n0 = 0, n1 = 0, n2 = 0, n1p = 0, n2p = 0, len = 0;
  double* S[3] = {};     // DST-I matrices sin(pi (j+1)(k+1)/(n+1))
  double* lam = nullptr; // [n0 + n1 + n2] eigenvalues of -lap_h per axis
  double* scale = nullptr;  // [n0][n1][n2] c / (lam0 + lam1 + lam2), precomputed once
  double* t0 = nullptr;  // workspaces (len doubles each)
  double* t1 = nullptr;
  double norm = 1.0;
  void init(int64_t n0, int64_t n1, int64_t n2, const double h[3]);
  void release();
  void solve(const double* b, double* x, cudaStream_t s);
};
// initialize_orbitals (optimizer.cpp:156-197): u_i = exp(-|x - c_i|^2 / (2 w_i^2)) + noise_i
// (centers [N][3], widths [N] on the device; noise is a block with stride ld).
void rng_init_noise_slab(uint64_t seed, int N, int64_t ng_full, int64_t offset, int64_t count,
                         double* widths, double* noise);
void launch_init_orbitals(const SlabGeom& g, int N, const double* h3, const double* centers,
                          const double* widths, double* u, cudaStream_t s);
// prolongate (grid.cpp:151-203) of every orbital of a block: coarse n_a -> fine 2 n_a + 1,
// separable linear interpolation with linear extrapolation past the ends, axes 0, 1, 2.
void launch_prolongate(int N, const int64_t nc[3], int64_t ldc, const double* C,
                       const int64_t nf[3], int64_t ldf, double* F, cudaStream_t s);
// three-kernel DST solve (axis-0 GEMM, per-plane shared-memory kernel, axis-0
// GEMM) for grids up to 128 points per axis; false when unsupported.
bool dst_fused_supported(int64_t n0, int64_t n1, int64_t n2);
bool launch_dst_fused(const DstPoisson& d, const double* b, double* x, cudaStream_t s);
void launch_cg(int64_t n0, int64_t n1, int64_t n2, const double ih2[3], const double* b,
               double* x, int warm, double* ws, unsigned* bar, int* out_i, double* out_d,
               cudaStream_t s);
int cg_grid_blocks();

}  // namespace po
