// Host C++ mirror of the reference solver loop over device-resident blocks.
//
// Restates InnerLoop::run (optimizer.cpp:322-579), finalize (:581-597) and
// run_single_level (:599-613) decision for decision — tau clamps (:25-28), BB
// variants and the tr|.| reading (:30-41, :376-411), the raw-step growth cap
// (:419-444), the delta^s search with the tau_min break (:455-484), recovery
// from the last orthonormalised iterate (:485-508), the C/Q ledger (:509-521),
// checkpoints / drift flags (:535-539) and the n_diag subspace rotation
// (:550-561) — while every field / block operation runs on the GPU. Per
// line-search trial the device pipeline is:
//   Gram(W - tau Z)  ->  Cholesky + L^{-T} (device)  ->  (W - tau Z) L^{-T}
//   [-> Gram -> CholeskyQR2 repair]  ->  rho, v_xc  ->  Poisson CG  ->  v_local
//   ->  H W~ with fused sigma / kinetic / external reductions
// and the trial's H W~ becomes the next iteration's HW when it is accepted, so
// the reference's separate total_energy Laplacians and apply_hamiltonian pass
// collapse into one stencil pass.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <memory>
#include <thread>
#include <utility>
#include <vector>

#include "engine.h"

namespace po {

namespace {

using Clock = std::chrono::steady_clock;
using BRef = std::shared_ptr<int>;
using SRef = std::shared_ptr<DevState>;

struct BlockPool {
  Engine& E;
  std::vector<int> free_;
  explicit BlockPool(Engine& e) : E(e) {}
  ~BlockPool() {  // back to the engine's cache: the next solve allocates nothing
    for (int h : free_) E.give_block(h);
  }
  void reserve(int n) {  // allocate up front: no cudaMalloc inside the iteration loop
    while ((int)free_.size() < n) free_.push_back(E.take_block());
  }
  BRef get() {
    int h;
    if (!free_.empty()) {
      h = free_.back();
      free_.pop_back();
    } else {
      h = E.take_block();
    }
    return BRef(new int(h), [this](int* p) {
      free_.push_back(*p);
      delete p;
    });
  }
};

struct StatePool {
  Engine& E;
  std::vector<DevState*> free_;
  explicit StatePool(Engine& e) : E(e) {}
  ~StatePool() {
    for (DevState* s : free_) E.give_state(s);
  }
  void reserve(int n) {
    while ((int)free_.size() < n) free_.push_back(E.take_state());
  }
  SRef get() {
    DevState* s;
    if (!free_.empty()) {
      s = free_.back();
      free_.pop_back();
    } else {
      s = E.take_state();
    }
    return SRef(s, [this](DevState* p) { free_.push_back(p); });
  }
};

double clamp_tau(double raw, const po_params& p) {  // optimizer.cpp:25-28
  if (!std::isfinite(raw)) return p.tau_max;
  return std::min(std::max(raw, p.tau_min), p.tau_max);
}

bool use_bb1(int v, int iter) {  // optimizer.cpp:30-34
  if (v == PO_BB1) return true;
  if (v == PO_BB2) return false;
  return iter % 2 == 0;
}

}  // namespace

struct OrthOut {
  double post_dev = 0.0;
  double offdiag_max = 0.0;  // near_identity_from_gram(pre_gram), manifold.cpp:249-259
  double diag_dev_max = 0.0;
  bool fallback = false;
  bool reported = true;  // post_dev is reported (else -1: verification skipped, manifold.cpp:150)
};

// manifold.cpp:136-169 on the device. in = A + sa * Ab (Ab may be null).
// Returns false on DegenerateSetError. pre-Gram stays in E.dmat[0].
bool orthonormalize_dev(Engine& E, const double* A, const double* Ab, double sa, double* out,
                        const std::function<double*()>& scratch, bool measure, OrthOut& o) {
  double* sc = E.scal();
  E.gram(A, Ab, sa, A, Ab, sa, 1, E.dmat[0]);
  launch_matrix_stats(E.N, E.dmat[0], sc + Engine::S_MSTAT, E.s);
  launch_cholesky_inv(E.N, E.dmat[0], E.chol_L, E.dmat[1], sc + Engine::S_CHOL, E.s);
  E.fetch(E.off_scal(), 64);
  const double* hs = E.hvec + E.off_scal();
  o.offdiag_max = hs[Engine::S_MSTAT + 2];
  o.diag_dev_max = hs[Engine::S_MSTAT + 3];
  double cond = std::numeric_limits<double>::infinity();
  int upper = 1;
  o.fallback = false;
  if (hs[Engine::S_CHOL + 3] != 1.0) {
    // symmetric_fallback, manifold.cpp:118-132
    launch_syev(E.N, E.dmat[0], E.syev_work, E.dmat[6], E.dmat[5], 0, sc + Engine::S_EIG, E.s);
    launch_inv_sqrt_from_eig(E.N, E.dmat[6], E.dmat[5], E.dmat[1], sc + Engine::S_INVS, E.s);
    E.fetch(E.off_scal(), 64);
    if (hs[Engine::S_INVS + 2] != 1.0) return false;
    upper = 0;
    o.fallback = true;
  } else {
    cond = hs[Engine::S_CHOL + 2];
  }
  E.mix(A, Ab, sa, E.dmat[1], 1.0, nullptr, 0.0, upper, out, nullptr);
  if (!measure && cond <= 1e2) {
    o.post_dev = -1.0;
    return true;
  }
  E.gram(out, nullptr, 0.0, out, nullptr, 0.0, 1, E.dmat[2]);
  launch_matrix_stats(E.N, E.dmat[2], sc + Engine::S_MSTAT2, E.s);
  E.fetch(E.off_scal(), 64);
  double dev = hs[Engine::S_MSTAT2];
  if (!(dev <= 1e-12)) {  // CholeskyQR2 repair pass
    launch_cholesky_inv(E.N, E.dmat[2], E.chol_L, E.dmat[3], sc + Engine::S_CHOL, E.s);
    E.fetch(E.off_scal(), 64);
    if (hs[Engine::S_CHOL + 3] != 1.0) return false;
    double* tmp = scratch();
    E.mix(out, nullptr, 0.0, E.dmat[3], 1.0, nullptr, 0.0, 1, tmp, nullptr);
    PO_CUDA(cudaMemcpyAsync(out, tmp, sizeof(double) * E.N * E.g.ld, cudaMemcpyDeviceToDevice,
                            E.s));
    E.gram(out, nullptr, 0.0, out, nullptr, 0.0, 1, E.dmat[2]);
    launch_matrix_stats(E.N, E.dmat[2], sc + Engine::S_MSTAT2, E.s);
    E.fetch(E.off_scal(), 64);
    dev = hs[Engine::S_MSTAT2];
  }
  o.post_dev = dev;
  return true;
}

// Asynchronous form of manifold.cpp:136-169 for the line search: pass 1
// (Gram -> Cholesky -> rotation -> verification Gram) is enqueued assuming the
// Cholesky succeeds, with no host round trip before the trial's energy. Whether
// the CholeskyQR2 repair is due ((measure || cond > 100) && dev > 1e-12) is
// decided on the host from the trial's single readback (orth_outcome); the
// repair itself (rare: dev is ~1e-15 for the well-conditioned trial Grams of a
// line search) then runs synchronously (orth_repair) and the trial's state and
// H W~ are rebuilt. A failed pass-1 Cholesky is redone with the symmetric-eigen
// fallback (orthonormalize_dev).
bool orth_enqueue(Engine& E, const double* A, const double* Ab, double sa, double* out,
                  bool measure, DevState* st = nullptr, int hartree = 0, int xc = 0,
                  bool g0_from_grams = false, const double* tau_dev = nullptr,
                  const BBArgs* bb = nullptr, const double* zsig = nullptr) {
  (void)measure;
  double* sc = E.scal();
  // zsig: Ab is HW and the direction z = HW - zsig W is implicit; only the
  // Grams-based trial Gram and the TMA rotations (fused small-N / large-N
  // tiles) can take it (callers check)
  if (zsig && !(g0_from_grams && st && tma2d_available() && (E.N <= 48 || E.N > 64)))
    throw Error(PO_EINVAL, "implicit direction outside the TMA trial paths");
  // G0 of W - tau Z from G_WW (dmat[8]), Sigma (dmat[4]), G_HH (dmat[7]), its stats and
  // its Cholesky in one launch where possible
  if (!(g0_from_grams &&
        launch_trial_cholesky(E.N, E.dmat[8], E.dmat[4], E.dmat[7], -sa, tau_dev, E.dmat[0],
                              sc + Engine::S_MSTAT, E.dmat[1], sc + Engine::S_CHOL, E.s, bb))) {
    if (bb)  // the BB step as its own launch (the fused form is unavailable)
      launch_bb_tau(bb->N, bb->zz, bb->ss, bb->sy, bb->yy, bb->history, bb->use_bb1,
                    bb->trace_abs_diag, bb->tau_min, bb->tau_max, bb->out, E.s);
    if (g0_from_grams)
      launch_trial_gram(E.N, E.dmat[8], E.dmat[4], E.dmat[7], -sa, E.dmat[0], E.s, tau_dev);
    else
      E.gram(A, Ab, sa, A, Ab, sa, 1, E.dmat[0]);
    launch_matrix_stats(E.N, E.dmat[0], sc + Engine::S_MSTAT, E.s);
    launch_cholesky_inv(E.N, E.dmat[0], E.chol_L, E.dmat[1], sc + Engine::S_CHOL, E.s);
  }
  bool fused = false;
  if (st && E.N <= 48 && tma2d_available()) {
    // rotation + verification Gram + density/xc of the rotated block in one pass
    // (xc = -1: the rotation writes rho and 4 pi rho only; v_xc, E_xc and E_ext
    // come from the v_local pass of build_state(density_done))
    (void)xc;
    const int nb = launch_rotate_fused(E.N, E.g.ld, E.g.ngl, A, Ab, sa, E.dmat[1], out, E.gram_ws,
                                       E.dmat[2], E.g.w, E.occ, -1, st->rho, st->v_xc,
                                       E.density_b_target(hartree), E.v_ext, E.partials, E.s,
                                       tau_dev ? tau_dev + 1 : nullptr, zsig);
    if (nb >= 0) {
      if (E.size > 1) E.comm->allreduce_sum(E.dmat[2], (size_t)E.N * E.N, E.s);
      fused = true;
    }
  }
  if (!fused) {
    if (tau_dev) throw Error(PO_EINVAL, "device-side trial scale needs the fused rotation");
    E.mix(A, Ab, sa, E.dmat[1], 1.0, nullptr, 0.0, 1, out, nullptr, nullptr, zsig);
    // 64 < N <= 128: the verification Gram of the rotated block also writes its
    // density and 4 pi rho (xc and the energies come from the v_local pass)
    if (st && E.gram_density(out, E.dmat[2], st->rho, E.density_b_target(hartree)))
      fused = true;
    else
      E.gram(out, nullptr, 0.0, out, nullptr, 0.0, 1, E.dmat[2]);
  }
  launch_matrix_stats(E.N, E.dmat[2], sc + Engine::S_MSTAT2, E.s);
  return fused;
}

// 0 ok, 1 pass-1 Cholesky rejected (caller redoes the trial with the fallback),
// 3 the CholeskyQR2 repair is due (caller runs orth_repair).
int orth_outcome(const Engine& E, bool measure, OrthOut& o, bool g0_rebuilt) {
  const double* hs = E.hvec + E.off_scal();
  o.offdiag_max = hs[Engine::S_MSTAT + 2];
  o.diag_dev_max = hs[Engine::S_MSTAT + 3];
  o.fallback = false;
  if (hs[Engine::S_CHOL + 3] != 1.0) return 1;
  // manifold.cpp:150: verification unless !measure && cond <= 1e2; :159 repair iff !(dev <= 1e-12)
  const bool verify = measure || !(hs[Engine::S_CHOL + 2] <= 1e2);
  const double dev = hs[Engine::S_MSTAT2];
  o.post_dev = verify ? dev : -1.0;
  o.reported = verify;
  static const bool force = std::getenv("PO_FORCE_QR2") != nullptr;  // test hook: exercise the repair
  // The reference skips the check for a well-conditioned exact Gram. A G0
  // rebuilt from the iteration's Grams (G_WW - tau (W^T Z + Z^T W) + tau^2 Z^T Z)
  // carries cancellation the exact Gram does not, so the rotation's own G2
  // statistics (already read back) are always checked there; the reported
  // deviation stays -1 as in the reference.
  return (verify || g0_rebuilt) && (force || !(dev <= 1e-12)) ? 3 : 0;
}

// CholeskyQR2 second pass on block out (manifold.cpp:159-166), synchronously;
// false on a rejected repair Cholesky (DegenerateSetError).
bool orth_repair(Engine& E, double* out, double* tmp, OrthOut& o) {
  double* sc = E.scal();
  launch_cholesky_inv(E.N, E.dmat[2], E.chol_L, E.dmat[3], sc + Engine::S_CHOL2, E.s);
  E.fetch(E.off_scal(), 64);
  if (E.hvec[E.off_scal() + Engine::S_CHOL2 + 3] != 1.0) return false;
  E.mix(out, nullptr, 0.0, E.dmat[3], 1.0, nullptr, 0.0, 1, tmp, nullptr);
  PO_CUDA(cudaMemcpyAsync(out, tmp, sizeof(double) * E.N * E.g.ld, cudaMemcpyDeviceToDevice, E.s));
  E.gram(out, nullptr, 0.0, out, nullptr, 0.0, 1, E.dmat[2]);
  launch_matrix_stats(E.N, E.dmat[2], sc + Engine::S_MSTAT2, E.s);
  E.fetch(E.off_scal(), 64);
  o.post_dev = o.reported ? E.hvec[E.off_scal() + Engine::S_MSTAT2] : -1.0;
  return true;
}

namespace {

struct Solver {
  Engine& E;
  const po_params& p;
  po_result* r;
  BlockPool pool;
  StatePool spool;
  bool nonlinear;
  SRef fixed_state;
  bool have_prev_solve = false;

  // InnerLoop::run state (optimizer.cpp:358-372), kept across step() calls
  BRef w, hw, prev_w, prev_z, recovery_w;
  // Implicit directions (fused small-N path, every iteration orthonormalised):
  // z = HW - sigma W is never stored; the rotation rebuilds it from HW and the
  // next iteration's BB products from the previous HW (prev_hw) with the sigma
  // row saved in dvec zsig slot prev_zslot. Any other consumer materialises it.
  BRef prev_hw;
  bool prev_zv = false;
  int prev_zslot = 0;
  SRef state, recovery_state;
  double nm_c = 0.0, nm_q = 1.0;
  std::vector<double> orth_energies;
  bool history_valid = false, converged = false, finished = false;
  bool sig_valid = true;  // dvec sigma row belongs to (w, hw)
  // trial Grams from the iteration's Grams (no pass over W - tau Z): G_WW of the
  // iterate in dmat[8] (the accepted trial's verification Gram), G_HH in dmat[7]
  bool gww_valid = false, ghh_fresh = false;
  int last_rotation_iter = 0, steps_until_orth = 0, failed_searches = 0, l = 0;
  double last_accepted_tau = 0.0;
  int n_org = 1;
  bool full_grad = false, grad_style = true, mean_abs = false;
  double ngd = 1.0;

  Solver(Engine& e, const po_params& pp, po_result* rr, int lvl = 0)
      : E(e), p(pp), r(rr), pool(e), spool(e), nonlinear(pp.hartree || pp.xc), level(lvl) {}
  int level = 0;  // outer refinement level (optimizer.cpp:654-664)

  double* P(const BRef& b) { return E.blk(*b); }

  SRef make_state(const BRef& u) {  // optimizer.cpp:224-229
    SRef st = enqueue_state(u);
    if (!st_fresh) return st;
    E.fetch_all();
    finish(st);
    return st;
  }

  // enqueue build_hamiltonian(u) without waiting; finish() after the next fetch
  bool st_fresh = false;
  SRef enqueue_state(const BRef& u, SRef pre = SRef(), bool density_done = false) {
    st_fresh = false;
    if (!nonlinear && fixed_state) return fixed_state;
    SRef st = pre ? pre : spool.get();
    E.poisson_solver = p.poisson_solver;
    E.build_state(P(u), p.hartree, p.xc, st.get(), have_prev_solve, density_done);
    if (p.hartree) have_prev_solve = true;
    if (!nonlinear) fixed_state = st;
    st_fresh = true;
    return st;
  }
  void finish(const SRef& st) {  // after a fetch covering the state build
    E.state_results(st.get());
    r->cg_iters_total += st->cg_iters;
  }

  // apply H and return the energy breakdown (energy.cpp:282-314) of u
  // Nonlinear problems take E_ext = w <V_ext, rho> from the state built from u
  // (energy.cpp:286-291 summed over orbitals); linear ones reuse a fixed state,
  // so the stencil pass reduces <V_ext u_i, u_i> per orbital instead.
  EnergyParts apply_and_energy(const BRef& u, const BRef& hu, const DevState& st) {
    E.apply_h(P(u), hu ? P(hu) : nullptr, st.v_local, !nonlinear);
    E.fetch(0, (size_t)3 * E.N);
    return energy_from_fetch(st);
  }
  EnergyParts energy_from_fetch(const DevState& st) {
    EnergyParts e;
    for (int i = 0; i < E.N; ++i) e.kinetic += E.occ * E.hvec[E.off_kin() + i];
    if (nonlinear) {
      e.external = st.e_ext;
    } else {
      for (int i = 0; i < E.N; ++i) e.external += E.occ * E.hvec[E.off_ext() + i];
    }
    e.hartree = p.hartree ? st.e_hartree : 0.0;
    e.xc = p.xc ? st.e_xc : 0.0;
    e.total = e.kinetic + e.external + e.hartree + e.xc;
    return e;
  }

  void set_energy(const EnergyParts& e) {
    r->e_kinetic = e.kinetic;
    r->e_external = e.external;
    r->e_hartree = e.hartree;
    r->e_xc = e.xc;
    r->e_total = e.total;
  }

  int fail(int outcome, const char* msg) {
    std::snprintf(r->message, sizeof r->message, "%s", msg);
    r->outcome = outcome;
    return outcome;
  }

  // Sigma = <(HW)^T W> into dmat[4]; max asymmetry into S_SYM+1
  void sigma(const BRef& w, const BRef& hw) {
    E.gram(P(hw), nullptr, 0.0, P(w), nullptr, 0.0, 0, E.dmat[4]);
    launch_matrix_stats(E.N, E.dmat[4], E.scal() + Engine::S_SYM, E.s);
  }

  // Sigma and G_HH = w (HW)^T HW in one pass (small N); false if unavailable
  bool sigma_dual(const BRef& w, const BRef& hw) {
    // sigma_ii comes out of the same reduction launch (no copy_diag) on one rank
    if (!launch_gram_tma(E.N, E.g.ld, 0, P(hw), nullptr, 0.0, P(w), nullptr, 0.0, E.gram_ws,
                         E.dmat[4], E.g.w, E.s, nullptr, E.dmat[7],
                         E.size == 1 ? E.dvec + E.off_sig() : nullptr))
      return false;
    if (E.size > 1) {
      E.comm->allreduce_sum(E.dmat[4], (size_t)E.N * E.N, E.s);
      E.comm->allreduce_sum(E.dmat[7], (size_t)E.N * E.N, E.s);
    }
    launch_matrix_stats(E.N, E.dmat[4], E.scal() + Engine::S_SYM, E.s);
    return true;
  }

  void trace_eigs(const BRef& w, const BRef& hw) {
    if (!p.trace_sigma_eigs || !r->sigma_eigs) return;
    sigma(w, hw);
    launch_syev(E.N, E.dmat[4], E.syev_work, E.dmat[6], E.dmat[5], 1, E.scal() + Engine::S_EIG,
                E.s);
    PO_CUDA(cudaMemcpyAsync(E.hmat, E.dmat[6], sizeof(double) * E.N, cudaMemcpyDeviceToHost, E.s));
    E.sync();
    std::memcpy(r->sigma_eigs + (size_t)r->n_records * E.N, E.hmat, sizeof(double) * E.N);
  }

  // Phase 1 of an iteration (directions + the speculative first trial), enqueued
  // either at the start of step() or already at the end of the previous step,
  // so the GPU never waits for the host between iterations
  struct Phase1 {
    bool valid = false;
    Clock::time_point t0;
    bool orth_iter = false, need_full = false, fused = false;
    bool zv = false;  // z implicit (see prev_hw); zsig slot zslot
    bool bigdir = false;  // the directions ran on the N > 64 passes (z may be implicit)
    bool dd_grams = false;  // ||D_i||^2 came from the Grams (checked at the readback)
    int zslot = 0;
    BRef z, dscratch;
    struct {
      BRef wt, rep, hwt;
      SRef pre, tstate;
      bool on = false;
    } spec;
  };
  Phase1 ph1;
  void enqueue_phase1(int iter);  // iter: the iteration these directions belong to
  const double* zsig(int slot) { return E.dvec + E.off_zsig(slot); }
  // write out an implicit direction (block of hw - sigma w)
  BRef materialize_z(const BRef& wb, const BRef& hwb, int slot) {
    BRef zb = pool.get();
    launch_z_from_hw(E.g, E.N, P(wb), P(hwb), zsig(slot), P(zb), E.s);
    return zb;
  }
  void materialize_prev_z() {
    if (!prev_zv) return;
    prev_z = materialize_z(prev_w, prev_hw, prev_zslot);
    prev_zv = false;
    prev_hw.reset();
  }
  void prefetch_next() {
    if (!ph1.valid && !finished && !converged && l < p.max_inner) enqueue_phase1(l);
  }

  void init(const BRef& w0);
  bool step();  // one InnerLoop iteration; false once the loop has ended
};

void Solver::init(const BRef& w0) {
  const int n = E.N;
  n_org = p.algorithm == PO_ALG_OPT_PAR_MOD ? p.n_org : 1;
  full_grad = p.algorithm == PO_ALG_OPTM_QR;
  grad_style = p.convergence_mode == PO_CONV_GRAD_NORM || p.convergence_mode == PO_CONV_MEAN_ABS;
  mean_abs = p.convergence_mode == PO_CONV_MEAN_ABS;
  ngd = (double)E.g.n0 * (double)E.g.n1 * (double)E.g.n2;
  (void)n;
  // live blocks at most: w, hw, z, prev_w, prev_z, recovery, trial w/hw/scratch
  // (+ rotation / mean-abs scratch); states: current, trial, recovery, spare
  pool.reserve(p.n_diag > 0 || mean_abs ? 11 : 9);
  spool.reserve(4);
  E.sync();
  w = w0;
  state = make_state(w);
  hw = pool.get();
  const EnergyParts e0 = apply_and_energy(w, hw, *state);
  if (!std::isfinite(e0.total)) {
    fail(PO_OUT_NUMERICAL_FAILURE, "non-finite total energy at the level start");
    finished = true;
    return;
  }
  set_energy(e0);
  nm_c = e0.total;
  nm_q = 1.0;
  orth_energies.assign(1, e0.total);
  recovery_w = w;
  recovery_state = state;
  if (tma2d_available()) {
    E.gram(P(w), nullptr, 0.0, P(w), nullptr, 0.0, 1, E.dmat[8]);
    gww_valid = true;
  }
}

void Solver::enqueue_phase1(int iter) {
  const int n = E.N;
  Phase1& ph = ph1;
  ph = Phase1();
  ph.valid = true;
  ph.t0 = Clock::now();
  const bool orth_iter = ph.orth_iter = steps_until_orth == 0;
  const bool need_full = ph.need_full = orth_iter && grad_style;

    // ---- compute_directions, optimizer.cpp:265-320
    BRef& z = ph.z;
    BRef& dscratch = ph.dscratch;
    const int onb = per_orbital_nblk(E.g, n);
    bool& fused = ph.fused;
    bool bb_done = false;
    ghh_fresh = false;  // G_HH (dmat[7]) belongs to this iteration's HW only
    static const bool zfree_env = !std::getenv("PO_ZFREE") || std::atoi(std::getenv("PO_ZFREE")) != 0;
    const bool fused_dir = !full_grad && !(mean_abs && need_full) && n <= 48 && tma2d_available();
    // N > 64: dir_big_kernel (z implicit or stored, z_prev implicit or stored)
    // (every rank runs it on its slab: the partial sums and the Grams are all-reduced)
    static const bool big_dir_sharded =
        !std::getenv("PO_BIG_DIR_SHARDED") || std::atoi(std::getenv("PO_BIG_DIR_SHARDED")) != 0;
    const bool big_dir = !fused_dir && !full_grad && need_full && !mean_abs &&
                         (E.size == 1 || big_dir_sharded) && n > 64 && tma2d_available();
    // implicit z: only where every consumer is the fused rotation of a trial
    // whose Gram comes from the iteration's Grams (nonlinear, orthonormalised
    // every iteration); the rare other consumers materialise it
    ph.zslot = prev_zv ? prev_zslot ^ 1 : 0;
    if (!fused_dir && !big_dir) materialize_prev_z();
    if (fused_dir) {
      // one pass: z, ||z||^2, ||HW - W Sigma||^2 and the BB products
      if (need_full || !sig_valid) {
        ghh_fresh = gww_valid && sigma_dual(w, hw);
        if (!ghh_fresh) sigma(w, hw);
        if (!ghh_fresh || E.size > 1) launch_copy_diag(n, E.dmat[4], E.dvec + E.off_sig(), E.s);
      }
      ph.zv = zfree_env && orth_iter && n_org == 1 && nonlinear && gww_valid && ghh_fresh;
      if (!ph.zv) {
        z = pool.get();
        materialize_prev_z();  // a stored z pairs with a stored previous z
      }
      const int nb = launch_directions(
          n, E.g.ld, E.g.ngl, P(w), P(hw), history_valid ? P(prev_w) : nullptr,
          history_valid ? (prev_zv ? P(prev_hw) : P(prev_z)) : nullptr,
          need_full ? E.dmat[4] : nullptr, E.dvec + E.off_sig(), ph.zv ? nullptr : P(z), E.partials,
          E.s, history_valid && prev_zv ? zsig(prev_zslot) : nullptr,
          ph.zv ? E.dvec + E.off_zsig(ph.zslot) : nullptr);
      if (nb < 0 && ph.zv) throw Error(PO_EINVAL, "fused directions unavailable for an implicit z");
      if (nb < 0) materialize_prev_z();
      if (nb >= 0) {
        E.reduce_rows(E.partials, (history_valid ? 5 : 2) * n, nb, E.g.w, E.dvec + E.off_zz(), true);
        fused = true;
      }
    }
    if (big_dir)  // z stays implicit where every consumer can rebuild it (see the fused path)
      ph.zv = zfree_env && orth_iter && n_org == 1 && nonlinear && gww_valid;
    if (!z && !ph.zv) z = pool.get();
    if (fused) {
    } else if (full_grad) {
      sigma(w, hw);
      E.mix(P(w), nullptr, 0.0, E.dmat[4], -1.0, P(hw), 1.0, 0, P(z), E.dvec + E.off_dd());
      if (mean_abs && need_full) {
        launch_abs_sum(E.g, n, P(z), E.partials, E.s);
        E.reduce_rows(E.partials, n, onb, 1.0, E.dvec + E.off_abs(), true);
      }
    } else {
      static const bool dd_grams_env =
          !std::getenv("PO_DNORM_GRAMS") || std::atoi(std::getenv("PO_DNORM_GRAMS")) != 0;
      // N > 64 with z implicit and ||D||^2 from the Grams: the elementwise
      // half of the directions (||z||^2, BB products) rides on the Sigma Gram,
      // with sigma_i from the H u pass (dvec sigma row) — no pass of its own
      int bb_nb = -1;
      if (need_full || !sig_valid) {
        if (big_dir && ph.zv && dd_grams_env && gww_valid && sig_valid && tma2d_available()) {
          GramBB gb{E.dvec + E.off_sig(),
                    history_valid && prev_zv ? zsig(prev_zslot) : nullptr,
                    history_valid ? P(prev_w) : nullptr,
                    history_valid ? (prev_zv ? P(prev_hw) : P(prev_z)) : nullptr,
                    E.partials, 0};
          if (E.gram_sigma_bb(P(hw), P(w), E.dmat[4], &gb)) {
            launch_matrix_stats(E.N, E.dmat[4], E.scal() + Engine::S_SYM, E.s);
            bb_nb = gb.nsplit;
          }
        }
        if (bb_nb < 0) sigma(w, hw);
        if (gww_valid) {
          // G_HH = w (HW)^T HW: the line search's trial Grams then come from
          // G_WW, Sigma and G_HH (launch_trial_gram) instead of a two-source
          // pass over W - tau Z per trial
          E.gram(P(hw), nullptr, 0.0, P(hw), nullptr, 0.0, 1, E.dmat[7]);
          ghh_fresh = true;
        }
        if (bb_nb < 0) launch_copy_diag(n, E.dmat[4], E.dvec + E.off_sig(), E.s);
      }
      int dnb = -1;
      bool stream_done = false;
      if (big_dir) {
        if (ph.zv && !ghh_fresh) {  // the trial Grams need G_HH: no implicit z without it
          ph.zv = false;
          z = pool.get();
        }
        const double* xprev =
            history_valid ? (prev_zv ? P(prev_hw) : P(prev_z)) : nullptr;
        const double* sprev = history_valid && prev_zv ? zsig(prev_zslot) : nullptr;
        double* zsave = ph.zv ? E.dvec + E.off_zsig(ph.zslot) : nullptr;
        if (dd_grams_env && gww_valid && ghh_fresh && tma2d_available()) {
          // ||D_i||^2 from Sigma, G_WW, G_HH (checked against its rounding bound at
          // the readback; the direct pass when it is not provably accurate) and
          // the elementwise half — z, ||z||^2, BB products — as one streaming pass
          launch_dnorm_grams(n, E.dmat[4], E.dmat[8], E.dmat[7], E.dvec + E.off_dd(),
                             E.dvec + E.off_abs(), E.dvec + E.off_sig(), zsave, E.s);
          const int nb = bb_nb >= 0 ? bb_nb
                                    : launch_residual_bb_stream(
                                          E.g, n, P(w), P(hw), E.dvec + E.off_sig(),
                                          history_valid ? P(prev_w) : nullptr, xprev, sprev,
                                          ph.zv ? nullptr : P(z), E.partials, E.s);
          E.reduce_rows(E.partials, n, nb, E.g.w, E.dvec + E.off_zz(), true);
          if (history_valid)
            E.reduce_rows(E.partials + (size_t)n * nb, 3 * n, nb, E.g.w, E.dvec + E.off_ss(), true);
          ph.dd_grams = true;
          stream_done = true;
          bb_done = history_valid;
        } else {
          // z (implicit or stored), ||z||^2, ||HW - W Sigma||^2 and the BB products
          // against (W_prev, z_prev) in one TMA pass (dir_big_kernel)
          dnb = launch_directions_big(n, E.g.ld, E.g.ngl, P(w), P(hw),
                                      history_valid ? P(prev_w) : nullptr, xprev, sprev, E.dmat[4],
                                      E.dvec + E.off_sig(), ph.zv ? nullptr : P(z), zsave,
                                      E.partials, E.s);
          if (dnb < 0) {  // unavailable: the stored-direction passes below
            if (ph.zv) {
              ph.zv = false;
              z = pool.get();
            }
            materialize_prev_z();
          }
        }
        ph.bigdir = stream_done || dnb >= 0;
      }
      if (stream_done) {
      } else if (dnb >= 0) {
        E.reduce_rows(E.partials, (history_valid ? 5 : 2) * n, dnb, E.g.w, E.dvec + E.off_zz(), true);
        bb_done = history_valid;
      } else if (history_valid) {  // z, ||z||^2 and the BB products in one pass
        launch_residual_bb(E.g, n, P(w), P(hw), E.dvec + E.off_sig(), P(prev_w), P(prev_z), P(z),
                           E.partials, E.s);
        E.reduce_rows(E.partials, n, onb, E.g.w, E.dvec + E.off_zz(), true);
        E.reduce_rows(E.partials + (size_t)n * onb, 3 * n, onb, E.g.w, E.dvec + E.off_ss(), true);
        bb_done = true;
      } else {
        launch_residual_diag(E.g, n, P(w), P(hw), E.dvec + E.off_sig(), P(z), E.partials, E.s);
        E.reduce_rows(E.partials, n, onb, E.g.w, E.dvec + E.off_zz(), true);
      }
      if (need_full && dnb < 0 && !stream_done) {
        if (mean_abs) dscratch = pool.get();
        E.mix(P(w), nullptr, 0.0, E.dmat[4], -1.0, P(hw), 1.0, 0, dscratch ? P(dscratch) : nullptr,
              E.dvec + E.off_dd());
        if (mean_abs) {
          launch_abs_sum(E.g, n, P(dscratch), E.partials, E.s);
          E.reduce_rows(E.partials, n, onb, 1.0, E.dvec + E.off_abs(), true);
        }
      }
    }
    if (history_valid && !fused && !bb_done) {
      launch_bb(E.g, n, P(w), P(prev_w), P(z), P(prev_z), E.partials, E.s);
      E.reduce_rows(E.partials, 3 * n, onb, E.g.w, E.dvec + E.off_ss(), true);
    }
    // First trial of an orthonormalisation iteration without a host round trip:
    // the BB step is taken on the device (bb_tau_kernel, the host's sums in the
    // host's order) and the trial pipeline reads tau from there. The host then
    // reads the directions and the trial together; a converged / failing
    // iteration simply discards the speculative trial.
    auto& spec = ph.spec;
    if (ph.zv && !(orth_iter && (fused || ph.bigdir) && gww_valid && ghh_fresh && nonlinear)) {
      z = materialize_z(w, hw, ph.zslot);  // no fused first trial: write z out
      ph.zv = false;
    }
    if (orth_iter && fused && gww_valid && ghh_fresh && nonlinear && E.N <= 48 &&
        tma2d_available()) {
      double* st_tau = E.scal() + Engine::S_TAU;
      // the BB step runs inside the trial's Cholesky launch (orth_enqueue)
      const BBArgs bb{n, E.dvec + E.off_zz(), E.dvec + E.off_ss(), E.dvec + E.off_sy(),
                      E.dvec + E.off_yy(), history_valid ? 1 : 0,
                      use_bb1(p.bb_variant, iter) ? 1 : 0,
                      p.bb_trace_abs == PO_TRACE_DIAG_ABS ? 1 : 0, p.tau_min, p.tau_max, st_tau};
      spec.wt = pool.get();
      spec.rep = pool.get();
      spec.pre = spool.get();
      const bool dens = orth_enqueue(E, P(w), ph.zv ? P(hw) : P(z), 0.0, P(spec.wt),
                                     p.verify_orthonormality != 0, spec.pre.get(), p.hartree,
                                     p.xc, true, st_tau, &bb, ph.zv ? zsig(ph.zslot) : nullptr);
      spec.tstate = enqueue_state(spec.wt, spec.pre, dens);
      spec.hwt = pool.get();
      E.apply_h(P(spec.wt), P(spec.hwt), spec.tstate->v_local, false);
      spec.on = true;
    }
}

bool Solver::step() {
  const int n = E.N;
  if (finished) return false;
  if (!(l < p.max_inner && !converged)) {
    r->outcome = converged ? PO_OUT_CONVERGED : PO_OUT_MAX_ITERATIONS;
    finished = true;
    return false;
  }
  {
    if (!ph1.valid) enqueue_phase1(l);
    Phase1 ph = std::move(ph1);
    ph1 = Phase1();
    const auto t0 = ph.t0;
    const bool orth_iter = ph.orth_iter;
    const bool need_full = ph.need_full;
    BRef z = ph.z;
    bool zv = ph.zv;
    const int zslot = ph.zslot;
    auto need_z = [&]() {  // a consumer that reads z itself
      if (zv) {
        z = materialize_z(w, hw, zslot);
        zv = false;
      }
    };
    BRef dscratch = ph.dscratch;
    const bool fused = ph.fused;
    auto& spec = ph.spec;
    (void)dscratch;
    E.fetch_all();
    const double* hv = E.hvec;
    if (ph.dd_grams) {
      // ||D||^2 from the Grams is used only when provably accurate: its rounding
      // bound below 1e-8 of the value, and the gradient far from grad_tol (the
      // convergence decision cannot flip); else the direct pass over the blocks
      double sdd = 0.0, serr = 0.0;
      for (int i = 0; i < n; ++i) {
        sdd += hv[E.off_dd() + i];
        serr += hv[E.off_abs() + i];
      }
      static const bool dbg = std::getenv("PO_DEBUG_DD") != nullptr;
      if (dbg) std::fprintf(stderr, "dd_grams: sum dd %.17g sum err %.6g\n", sdd, serr);
      if (!(sdd >= 1e8 * serr && sdd >= 100.0 * p.grad_tol * p.grad_tol)) {
        E.mix(P(w), nullptr, 0.0, E.dmat[4], -1.0, P(hw), 1.0, 0, nullptr, E.dvec + E.off_dd());
        E.fetch_all();
      }
    }
    if ((full_grad || need_full) && hv[E.off_scal() + Engine::S_SYM + 1] > 1e-10)
      throw Error(PO_EINVAL, "stiefel_gradient: <(HU)^T U> is not symmetric; inconsistent H or U");
    double znorm2 = 0.0, grad_norm = -1.0, mean_abs_v = -1.0;
    if (full_grad) {
      for (int i = 0; i < n; ++i) znorm2 += hv[E.off_dd() + i];
      grad_norm = std::sqrt(std::max(0.0, znorm2));
      if (mean_abs && need_full) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += hv[E.off_abs() + i];
        mean_abs_v = acc / ((double)n * ngd);
      }
    } else {
      for (int i = 0; i < n; ++i) znorm2 += hv[E.off_zz() + i];
      if (need_full) {
        double acc = 0.0, abs_acc = 0.0;
        for (int i = 0; i < n; ++i) {
          acc += hv[E.off_dd() + i];
          if (mean_abs) abs_acc += hv[E.off_abs() + i];
        }
        grad_norm = std::sqrt(std::max(0.0, acc));
        if (mean_abs) mean_abs_v = abs_acc / ((double)n * ngd);
      }
    }
    if (orth_iter && grad_style) {  // check_convergence, optimizer.cpp:126-148
      const bool conv = p.convergence_mode == PO_CONV_GRAD_NORM
                            ? (grad_norm >= 0.0 && grad_norm < p.grad_tol)
                            : (mean_abs_v >= 0.0 && mean_abs_v < p.mean_abs_tol);
      if (conv) {
        converged = true;
        r->outcome = PO_OUT_CONVERGED;
        finished = true;
        return false;
      }
    }
    if (znorm2 == 0.0) {
      converged = true;
      r->outcome = PO_OUT_CONVERGED;
      finished = true;
      return false;
    }

    // ---- BB step, optimizer.cpp:376-411
    double tau_raw;
    if (history_valid) {
      double tr_ss = 0.0, tr_yy = 0.0, sy_abs = 0.0, sy_tr = 0.0;
      for (int i = 0; i < n; ++i) {
        tr_ss += hv[E.off_ss() + i];
        tr_yy += hv[E.off_yy() + i];
        sy_abs += std::abs(hv[E.off_sy() + i]);
        sy_tr += hv[E.off_sy() + i];
      }
      const double tr_abs_sy = p.bb_trace_abs == PO_TRACE_DIAG_ABS ? sy_abs : std::abs(sy_tr);
      const double raw = use_bb1(p.bb_variant, l) ? tr_ss / tr_abs_sy : tr_abs_sy / tr_yy;
      tau_raw = clamp_tau(raw, p);
    } else {
      tau_raw = clamp_tau(std::min(p.tau_max, 1.0 / std::sqrt(znorm2)), p);
    }
    if (spec.on) tau_raw = hv[E.off_scal() + Engine::S_TAU];  // the value the trial used

    po_record rec{};
    rec.level = level;
    rec.iter = l;
    rec.grad_norm = grad_norm >= 0.0 ? grad_norm : std::sqrt(std::max(0.0, znorm2));

    if (!orth_iter) {  // raw step, optimizer.cpp:419-444
      double tau = tau_raw;
      if (last_accepted_tau > 0.0) tau = std::min(tau, 5.0 * last_accepted_tau);
      BRef wn = pool.get();
      need_z();
      launch_lincomb(E.g, n, P(w), -tau, P(z), P(wn), E.s);
      prev_w = w;
      prev_z = z;
      prev_zv = false;
      prev_hw.reset();
      w = wn;
      history_valid = true;
      gww_valid = false;  // a raw step leaves the manifold
      state = enqueue_state(w);
      BRef hn = pool.get();
      E.apply_h(P(w), P(hn), state->v_local, false);
      E.fetch_all();
      if (st_fresh) finish(state);
      hw = hn;
      sig_valid = true;
      --steps_until_orth;
      rec.tau = tau;
      rec.energy = orth_energies.back();
    } else {  // backtracked orthogonalization step, optimizer.cpp:446-541
      bool accepted = false;
      int s = 0;
      double tau = 0.0;
      OrthOut orth;
      BRef wt, hwt;
      SRef tstate;
      EnergyParts te;
      bool sync_orth = false;  // the accepted trial went through orthonormalize_dev
      bool trial_g0g = false;  // the trial's G0 was rebuilt from the iteration's Grams
      for (s = 0; s <= p.max_backtracks; ++s) {
        sync_orth = false;
        tau = tau_raw * std::pow(p.delta, s);
        if (s > 0 && tau < p.tau_min) break;
        BRef rep;
        if (s == 0 && spec.on) {  // enqueued and read back with the directions
          wt = spec.wt;
          rep = spec.rep;
          tstate = spec.tstate;
          hwt = spec.hwt;
          spec = {};
          trial_g0g = true;
        } else {
          wt = pool.get();
          rep = pool.get();
          // one device pipeline per trial, one readback (energy + decisions)
          SRef pre = nonlinear ? spool.get() : SRef();
          const bool g0g = gww_valid && ghh_fresh;
          trial_g0g = g0g;
          if (!(g0g && nonlinear)) need_z();
          const bool dens = orth_enqueue(E, P(w), zv ? P(hw) : P(z), -tau, P(wt),
                                         p.verify_orthonormality != 0, pre.get(), p.hartree, p.xc,
                                         g0g, nullptr, nullptr, zv ? zsig(zslot) : nullptr);
          tstate = enqueue_state(wt, pre, dens);
          hwt = pool.get();
          E.apply_h(P(wt), P(hwt), tstate->v_local, !nonlinear);
          E.fetch_all();
        }
        const int oc = orth_outcome(E, p.verify_orthonormality != 0, orth, trial_g0g);
        if (oc == 3) {  // CholeskyQR2 repair (rare): redo the trial's tail on the repaired block
          if (!orth_repair(E, P(wt), P(rep), orth)) continue;  // DegenerateSetError -> NaN energy
          sync_orth = false;
          tstate = make_state(wt);
          te = apply_and_energy(wt, hwt, *tstate);
        } else if (oc == 1) {  // pass-1 Cholesky rejected: symmetric fallback, synchronously
          auto scratch = [&]() -> double* { return P(rep); };
          need_z();
          if (!orthonormalize_dev(E, P(w), P(z), -tau, P(wt), scratch,
                                  p.verify_orthonormality != 0, orth))
            continue;
          sync_orth = true;
          tstate = make_state(wt);
          te = apply_and_energy(wt, hwt, *tstate);
        } else {
          if (st_fresh) finish(tstate);
          if (!tstate->poisson_ok) {  // DST solve missed the CG criterion: CG from it, then redo H
            E.force_cg_verify = true;
            enqueue_state(wt, tstate, true);
            E.force_cg_verify = false;
            E.fetch_all();
            finish(tstate);
            te = apply_and_energy(wt, hwt, *tstate);
          } else {
            te = energy_from_fetch(*tstate);
          }
        }
        if (std::isfinite(te.total) && te.total <= nm_c - p.rho1 * tau * znorm2) {
          accepted = true;
          break;
        }
      }
      if (!accepted) {  // recovery, optimizer.cpp:485-508
        if (++failed_searches > 8) {
          char buf[200];
          std::snprintf(buf, sizeof buf,
                        "line search stagnated at level %d iteration %d (%d trials, C = %.17g)", level,
                        l, s, nm_c);
          fail(PO_OUT_STAGNATION, buf);
          finished = true;
          return false;
        }
        w = recovery_w;
        state = recovery_state;
        BRef hn = pool.get();
        E.apply_h(P(w), P(hn), state->v_local, false);
        hw = hn;
        sig_valid = true;
        gww_valid = false;
        history_valid = false;
        prev_w.reset();
        prev_z.reset();
        prev_hw.reset();
        prev_zv = false;
        steps_until_orth = 0;
        ++l;
        prefetch_next();
        return true;  // no record for a failed search (optimizer.cpp:485-508)
      }
      failed_searches = 0;
      const double c_before = nm_c, q_before = nm_q;
      nm_q = p.eta * q_before + 1.0;
      nm_c = (p.eta * q_before * c_before + te.total) / nm_q;
      if (r->accepted && r->n_accepted < r->cap) {
        double* a = r->accepted + 9 * (size_t)r->n_accepted;
        const double v[9] = {(double)level, (double)l, te.total, c_before, nm_c, q_before, nm_q, tau, znorm2};
        std::memcpy(a, v, sizeof v);
      }
      r->n_accepted++;
      if (te.total > nm_c + 1e-9 * (1.0 + std::abs(te.total)))
      {
        fail(PO_OUT_NUMERICAL_FAILURE, "nonmonotone ledger violated (C < E after update)");
        finished = true;
        return false;
      }
      prev_w = w;
      prev_z = z;
      prev_zv = zv;
      prev_zslot = zslot;
      prev_hw = zv ? hw : BRef();
      w = wt;
      state = tstate;
      hw = hwt;
      sig_valid = true;
      history_valid = true;
      last_accepted_tau = tau;
      // the accepted trial's verification Gram (post-repair if repaired) is G_WW of w
      gww_valid = !sync_orth && tma2d_available();
      if (gww_valid) std::swap(E.dmat[8], E.dmat[2]);  // no copy: exchange the buffers
      steps_until_orth = n_org - 1;
      const bool rotation_due =
          p.n_diag > 0 && (l + 1 - last_rotation_iter) >= p.n_diag && !full_grad;
      // the next iteration's directions + first trial go to the GPU now; the
      // bookkeeping below overlaps with them
      if (!rotation_due && l + 1 < p.max_inner) enqueue_phase1(l + 1);
      set_energy(te);
      orth_energies.push_back(te.total);
      rec.did_orth = 1;
      rec.tau = tau;
      rec.backtracks = s;
      rec.offdiag_max = orth.offdiag_max;
      // SolveResult::checkpoints / drift_iterations, optimizer.cpp:535-539
      if (r->checkpoints && r->n_checkpoints < r->cap) {
        double* c = r->checkpoints + 5 * (size_t)r->n_checkpoints;
        const double v[5] = {(double)level, (double)l, orth.offdiag_max, orth.diag_dev_max, orth.post_dev};
        std::memcpy(c, v, sizeof v);
      }
      r->n_checkpoints++;
      if (orth.offdiag_max > 0.5) {
        if (r->drift_iterations && r->n_drift < r->cap) r->drift_iterations[r->n_drift] = l;
        r->n_drift++;
      }
      rec.energy = te.total;
      steps_until_orth = n_org - 1;
      if (p.n_diag > 0 && (l + 1 - last_rotation_iter) >= p.n_diag && !full_grad) {
        // subspace diagonalization, optimizer.cpp:550-561 / manifold.cpp:218-247
        sigma(w, hw);
        launch_syev(n, E.dmat[4], E.syev_work, E.dmat[6], E.dmat[5], 1, E.scal() + Engine::S_EIG,
                    E.s);
        E.fetch(E.off_scal(), 64);
        if (E.hvec[E.off_scal() + Engine::S_EIG] > 1e-8)
          throw Error(PO_EINVAL, "subspace_rotate: Sigma asymmetry exceeds tolerance");
        BRef wr = pool.get(), hr = pool.get();
        E.mix(P(w), nullptr, 0.0, E.dmat[5], 1.0, nullptr, 0.0, 0, P(wr), nullptr);
        E.mix(P(hw), nullptr, 0.0, E.dmat[5], 1.0, nullptr, 0.0, 0, P(hr), nullptr);
        w = wr;
        hw = hr;
        last_rotation_iter = l + 1;
        rec.did_diag = 1;
        history_valid = false;
        sig_valid = false;
        gww_valid = false;
        prev_w.reset();
        prev_z.reset();
        prev_hw.reset();
        prev_zv = false;
      }
      recovery_w = w;
      recovery_state = state;
      trace_eigs(w, hw);
      if (p.convergence_mode == PO_CONV_ENERGY_CHANGE && orth_energies.size() >= 4) {
        double acc = 0.0;
        const size_t m = orth_energies.size();
        for (size_t k = 0; k < 3; ++k) {
          const double e_new = orth_energies[m - 1 - k], e_old = orth_energies[m - 2 - k];
          acc += std::abs(e_old - e_new) / (std::abs(e_old) + 1.0) / (double)std::max(1, n_org);
        }
        if (acc / 3.0 < p.energy_tol) converged = true;
      }
    }
    if (!ph1.valid) E.sync();  // else the next iteration is already running on the stream
    rec.wall_ms = 1e3 * std::chrono::duration<double>(Clock::now() - t0).count();
    if (r->n_records < r->cap) r->records[r->n_records] = rec;
    r->n_records++;
  }
  ++l;
  prefetch_next();
  return true;
}

}  // namespace

}  // namespace po

using po::Engine;
using po::Error;

extern "C" {

void po_default_params(po_params* p) {  // optimizer.hpp:22-46
  std::memset(p, 0, sizeof *p);
  p->algorithm = PO_ALG_OPT_PAR_MOD;
  p->bb_variant = PO_BB1;
  p->bb_trace_abs = PO_TRACE_DIAG_ABS;
  p->convergence_mode = PO_CONV_GRAD_NORM;
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
  p->hartree = 1;
  p->xc = 1;
  p->trace_sigma_eigs = 0;
  p->poisson_solver = PO_POISSON_DST;
  p->outer_levels = 1;
  p->seed = 1;
}

int po_orthonormalize(po_engine* h, int in, int out, int measure, double* pre_gram,
                      double* post_deviation, int* used_fallback) {
  if (!h || !h->e) return PO_EINVAL;
  Engine& E = *h->e;
  try {
    if (in == out) throw Error(PO_EINVAL, "orthonormalize: in and out must differ");
    int tmp = -1;
    auto scratch = [&]() -> double* {
      tmp = E.alloc_block();
      return E.blk(tmp);
    };
    po::OrthOut o;
    const bool ok = po::orthonormalize_dev(E, E.blk(in), nullptr, 0.0, E.blk(out), scratch,
                                           measure != 0, o);
    if (tmp >= 0) E.free_block(tmp);
    if (pre_gram) {
      PO_CUDA(cudaMemcpyAsync(E.hmat, E.dmat[0], sizeof(double) * E.N * E.N,
                              cudaMemcpyDeviceToHost, E.s));
      E.sync();
      std::memcpy(pre_gram, E.hmat, sizeof(double) * E.N * E.N);
    }
    if (!ok) throw Error(PO_EDEGENERATE, "orthonormalize: orbital set is numerically rank deficient");
    if (post_deviation) *post_deviation = o.post_dev;
    if (used_fallback) *used_fallback = o.fallback ? 1 : 0;
    E.sync();
  } catch (const Error& ex) {
    h->err = ex.what();
    return ex.code;
  } catch (const std::exception& ex) {
    h->err = ex.what();
    return PO_EINVAL;
  }
  return PO_OK;
}

static void validate_params(const po_params* p) {  // OptimizerParams::validate, optimizer.cpp:43-58
  if (!(p->rho1 > 0.0)) throw Error(PO_EINVAL, "optimizer: rho1 must be positive");
  if (!(p->delta > 0.0 && p->delta < 1.0)) throw Error(PO_EINVAL, "optimizer: delta must lie in (0, 1)");
  if (!(p->eta >= 0.0 && p->eta < 1.0)) throw Error(PO_EINVAL, "optimizer: eta must lie in [0, 1)");
  if (p->n_diag < 0) throw Error(PO_EINVAL, "optimizer: n_diag must be >= 0 (0 disables)");
  if (p->n_org < 1) throw Error(PO_EINVAL, "optimizer: n_org must be >= 1");
  if (p->max_inner < 1) throw Error(PO_EINVAL, "optimizer: max_inner must be >= 1");
  if (p->max_backtracks < 0) throw Error(PO_EINVAL, "optimizer: max_backtracks must be >= 0");
  if (!(p->tau_min > 0.0) || !(p->tau_max >= p->tau_min))
    throw Error(PO_EINVAL, "optimizer: require 0 < tau_min <= tau_max");
  if (!(p->grad_tol > 0.0)) throw Error(PO_EINVAL, "optimizer: grad_tol must be positive");
  if (!(p->mean_abs_tol > 0.0)) throw Error(PO_EINVAL, "optimizer: mean_abs_tol must be positive");
  if (!(p->energy_tol > 0.0)) throw Error(PO_EINVAL, "optimizer: energy_tol must be positive");
  if (p->outer_levels < 1) throw Error(PO_EINVAL, "optimizer: outer_levels must be >= 1");
}

static void reset_result(po_result* r) {
  r->n_records = r->n_accepted = 0;
  r->n_checkpoints = r->n_drift = 0;
  r->par_seconds = r->sync_seconds = 0.0;
  r->cg_iters_total = 0;
  r->message[0] = 0;
  r->outcome = PO_OUT_MAX_ITERATIONS;
  r->e_kinetic = r->e_external = r->e_hartree = r->e_xc = r->e_total = 0.0;
  r->final_grad_norm = 0.0;
}

// PhaseTimer mirror (parallel.hpp:55-86, SolveResult::par/sync_seconds filled at
// optimizer.cpp:594-595): every orbital-parallel phase runs on the device, so
// par_seconds is the wall time the host spent waiting on the device pipeline
// (Engine::wait_seconds: stream syncs + readback spins) and sync_seconds the
// rest of the call (host-side control, launches, checks); par + sync = wall.
static void set_phase_times(po_result* r, double wall, double waited) {
  r->wall_seconds = wall;
  r->par_seconds = std::min(wall, std::max(0.0, waited));
  r->sync_seconds = wall - r->par_seconds;
}

// One InnerLoop level on block w_handle (iterated in place).
static void run_level(Engine& E, const po_params* p, int w_handle, po_result* r, int level) {
  po::Solver S(E, *p, r, level);
  std::shared_ptr<int> w(new int(w_handle), [](int* q) { delete q; });
  S.init(w);
  while (S.step()) {
  }
  w = S.w;
  if (*w != w_handle)
    PO_CUDA(cudaMemcpyAsync(E.blk(w_handle), E.blk(*w), sizeof(double) * E.N * E.g.ld,
                            cudaMemcpyDeviceToDevice, E.s));
  E.sync();
}

// finalize, optimizer.cpp:581-597: full Stiefel gradient norm at the final iterate
static void finalize_grad(Engine& E, const po_params* p, int w_handle, po_result* r) {
  po::Solver S(E, *p, r);
  std::shared_ptr<int> w(new int(w_handle), [](int* q) { delete q; });
  po::SRef st = S.make_state(w);
  po::BRef hw = S.pool.get();
  E.apply_h(E.blk(*w), E.blk(*hw), st->v_local, false);
  S.sigma(w, hw);
  E.mix(E.blk(*w), nullptr, 0.0, E.dmat[4], -1.0, E.blk(*hw), 1.0, 0, nullptr,
        E.dvec + E.off_dd());
  E.fetch_all();
  if (E.hvec[E.off_scal() + Engine::S_SYM + 1] > 1e-10)
    throw Error(PO_EINVAL, "stiefel_gradient: <(HU)^T U> is not symmetric; inconsistent H or U");
  double acc = 0.0;
  for (int i = 0; i < E.N; ++i) acc += E.hvec[E.off_dd() + i];
  r->final_grad_norm = std::sqrt(std::max(0.0, acc));
  E.sync();
}

int po_solve(po_engine* h, const po_params* p, int w_handle, po_result* r) {
  if (!h || !h->e || !p || !r) return PO_EINVAL;
  Engine& E = *h->e;
  const auto t0 = std::chrono::steady_clock::now();
  const double wait0 = po::host_wait_seconds();
  reset_result(r);
  try {
    validate_params(p);
    // run_single_level: u0 must be orthonormal (optimizer.cpp:601-603)
    E.gram(E.blk(w_handle), nullptr, 0.0, E.blk(w_handle), nullptr, 0.0, 1, E.dmat[2]);
    po::launch_matrix_stats(E.N, E.dmat[2], E.scal() + Engine::S_MSTAT2, E.s);
    E.fetch(E.off_scal(), 64);
    if (E.hvec[E.off_scal() + Engine::S_MSTAT2] > 1e-8)
      throw Error(PO_EINVAL, "solver: initial orbital set is not orthonormal");
    run_level(E, p, w_handle, r, 0);
    finalize_grad(E, p, w_handle, r);
  } catch (const Error& ex) {
    h->err = ex.what();
    std::snprintf(r->message, sizeof r->message, "%s", ex.what());
    return ex.code;
  } catch (const std::exception& ex) {
    h->err = ex.what();
    return PO_EINVAL;
  }
  set_phase_times(r, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                  po::host_wait_seconds() - wait0);
  return PO_OK;
}

// po_solve on host buffers: W uploaded, iterated, and downloaded on a side
// stream while the finalize kernels (which only read W) run — the drop-in's
// whole reference-facing call in one entry.
int po_solve_host(po_engine* h, const po_params* p, const double* w_in, double* w_out,
                  po_result* r) {
  if (!h || !h->e || !p || !r || !w_in || !w_out) return PO_EINVAL;
  Engine& E = *h->e;
  const auto t0 = std::chrono::steady_clock::now();
  const double wait0 = po::host_wait_seconds();
  reset_result(r);
  int w_handle = -1;
  cudaStream_t side = nullptr;
  cudaEvent_t ev = nullptr;
  try {
    validate_params(p);
    w_handle = E.take_block();
    E.upload_host(E.blk(w_handle), w_in, E.s);  // pageable input: pinned chunk pipeline
    E.gram(E.blk(w_handle), nullptr, 0.0, E.blk(w_handle), nullptr, 0.0, 1, E.dmat[2]);
    po::launch_matrix_stats(E.N, E.dmat[2], E.scal() + Engine::S_MSTAT2, E.s);
    E.fetch(E.off_scal(), 64);
    if (E.hvec[E.off_scal() + Engine::S_MSTAT2] > 1e-8)
      throw Error(PO_EINVAL, "solver: initial orbital set is not orthonormal");
    run_level(E, p, w_handle, r, 0);
    PO_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    PO_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    PO_CUDA(cudaEventRecord(ev, E.s));
    PO_CUDA(cudaStreamWaitEvent(side, ev, 0));
    // the download (a host thread drives the staging pipeline for pageable
    // output) overlaps the finalize pass, which only reads W
    std::exception_ptr dl_err;
    std::thread dl([&] {
      try {
        E.download_host(w_out, E.blk(w_handle), side);
      } catch (...) {
        dl_err = std::current_exception();
      }
    });
    try {
      finalize_grad(E, p, w_handle, r);
    } catch (...) {
      dl.join();
      throw;
    }
    dl.join();
    if (dl_err) std::rethrow_exception(dl_err);
  } catch (const Error& ex) {
    if (side) cudaStreamSynchronize(side);
    if (side) cudaStreamDestroy(side);
    if (ev) cudaEventDestroy(ev);
    if (w_handle >= 0) E.give_block(w_handle);
    h->err = ex.what();
    std::snprintf(r->message, sizeof r->message, "%s", ex.what());
    return ex.code;
  }
  cudaStreamDestroy(side);
  cudaEventDestroy(ev);
  E.give_block(w_handle);
  set_phase_times(r, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                  po::host_wait_seconds() - wait0);
  return PO_OK;
}

// optimizer.cpp:638-669 solve: initialize_orbitals on level 0, then per level
// refine_uniform + prolongate + orthonormalize (level > 0) and one InnerLoop;
// stops early on stagnation / numerical failure; finalize on the last grid.
int po_solve_levels(const po_grid_desc* grid0, int n_orbitals, double occupation,
                    const double* atoms, int natoms, const po_params* p, po_result* r,
                    po_engine** out_engine, int* out_block) {
  if (!grid0 || !p || !r || !out_engine || !out_block) return PO_EINVAL;
  *out_engine = nullptr;
  *out_block = -1;
  const auto t0 = std::chrono::steady_clock::now();
  const double wait0 = po::host_wait_seconds();
  reset_result(r);
  po_engine* cur = nullptr;
  int w = -1;
  auto fail = [&](int code, const std::string& msg) {
    std::snprintf(r->message, sizeof r->message, "%s", msg.c_str());
    if (cur) {
      cur->err = msg;
      *out_engine = cur;  // caller reads po_last_error, then po_destroy
    }
    return code;
  };
  try {
    validate_params(p);
    po_grid_desc g = *grid0;
    int rc = po_create(&g, n_orbitals, occupation, nullptr, &cur);
    if (rc != PO_OK) return fail(rc, cur ? cur->err : "po_create failed");
    if ((rc = po_external_potential(cur, atoms, natoms)) != PO_OK) return fail(rc, cur->err);
    if ((rc = po_alloc_block(cur, &w)) != PO_OK) return fail(rc, cur->err);
    if ((rc = po_initialize_orbitals(cur, atoms, natoms, p->seed, w)) != PO_OK)
      return fail(rc, cur->err);
    for (int level = 0; level < p->outer_levels; ++level) {
      if (level > 0) {
        po_grid_desc fg;
        if ((rc = po_refine_grid(&g, &fg)) != PO_OK) return fail(rc, "refine_uniform: invalid grid");
        po_engine* fine = nullptr;
        rc = po_create(&fg, n_orbitals, occupation, nullptr, &fine);
        if (rc != PO_OK) {
          const std::string m = fine ? fine->err : "po_create failed";
          po_destroy(fine);
          return fail(rc, m);
        }
        int fw = -1, raw = -1;
        if ((rc = po_external_potential(fine, atoms, natoms)) != PO_OK ||
            (rc = po_alloc_block(fine, &raw)) != PO_OK || (rc = po_alloc_block(fine, &fw)) != PO_OK ||
            (rc = po_prolongate(cur, w, fine, raw)) != PO_OK ||
            (rc = po_orthonormalize(fine, raw, fw, 1, nullptr, nullptr, nullptr)) != PO_OK) {
          const std::string m = fine->err;
          po_destroy(fine);
          return fail(rc, m);
        }
        po_free_block(fine, raw);
        po_destroy(cur);
        cur = fine;
        w = fw;
        g = fg;
      }
      run_level(*cur->e, p, w, r, level);
      if (r->outcome == PO_OUT_STAGNATION || r->outcome == PO_OUT_NUMERICAL_FAILURE) break;
    }
    finalize_grad(*cur->e, p, w, r);
  } catch (const Error& ex) {
    return fail(ex.code, ex.what());
  } catch (const std::exception& ex) {
    return fail(PO_EINVAL, ex.what());
  }
  set_phase_times(r, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                  po::host_wait_seconds() - wait0);
  *out_engine = cur;
  *out_block = w;
  return PO_OK;
}

struct po_solver {
  po_engine* h;
  po_params p;
  po::Solver* S;
  std::shared_ptr<int> w_user;
  int w_handle;
  std::chrono::steady_clock::time_point t0;
  double wait0;  // Engine::wait_seconds at create (PhaseTimer mirror)
};

static int solver_error(po_engine* h, po_result* r, const std::exception& ex, int code) {
  h->err = ex.what();
  if (r) std::snprintf(r->message, sizeof r->message, "%s", ex.what());
  return code;
}

int po_solver_create(po_engine* h, const po_params* p, int w_handle, po_result* r,
                     po_solver** out) {
  if (!h || !h->e || !p || !r || !out) return PO_EINVAL;
  Engine& E = *h->e;
  *out = nullptr;
  reset_result(r);
  auto* sv = new po_solver{h, *p, nullptr, nullptr, w_handle, std::chrono::steady_clock::now(),
                           po::host_wait_seconds()};
  try {
    E.blk(w_handle);
    sv->S = new po::Solver(E, sv->p, r);
    sv->w_user = std::shared_ptr<int>(new int(w_handle), [](int* q) { delete q; });
    sv->S->init(sv->w_user);
  } catch (const Error& ex) {
    delete sv->S;
    delete sv;
    return solver_error(h, r, ex, ex.code);
  } catch (const std::exception& ex) {
    delete sv->S;
    delete sv;
    return solver_error(h, r, ex, PO_EINVAL);
  }
  *out = sv;
  return PO_OK;
}

int po_solver_step(po_solver* sv, int* more) {
  if (!sv || !sv->S) return PO_EINVAL;
  try {
    const bool m = sv->S->step();
    if (more) *more = m ? 1 : 0;
  } catch (const Error& ex) {
    return solver_error(sv->h, sv->S->r, ex, ex.code);
  } catch (const std::exception& ex) {
    return solver_error(sv->h, sv->S->r, ex, PO_EINVAL);
  }
  return PO_OK;
}

int po_solver_current(po_solver* sv, int* block) {
  if (!sv || !sv->S || !block || !sv->S->w) return PO_EINVAL;
  *block = *sv->S->w;
  return PO_OK;
}

int po_solver_finish(po_solver* sv) {
  if (!sv || !sv->S) return PO_EINVAL;
  Engine& E = *sv->h->e;
  po::Solver& S = *sv->S;
  po_result* r = S.r;
  try {
    while (S.step()) {
    }
    po::SRef st = S.make_state(S.w);
    po::BRef hw = S.pool.get();
    E.apply_h(E.blk(*S.w), E.blk(*hw), st->v_local, false);
    S.sigma(S.w, hw);
    E.mix(E.blk(*S.w), nullptr, 0.0, E.dmat[4], -1.0, E.blk(*hw), 1.0, 0, nullptr,
          E.dvec + E.off_dd());
    E.fetch_all();
    if (E.hvec[E.off_scal() + Engine::S_SYM + 1] > 1e-10)
      throw Error(PO_EINVAL, "stiefel_gradient: <(HU)^T U> is not symmetric; inconsistent H or U");
    double acc = 0.0;
    for (int i = 0; i < E.N; ++i) acc += E.hvec[E.off_dd() + i];
    r->final_grad_norm = std::sqrt(std::max(0.0, acc));
    if (*S.w != sv->w_handle)
      PO_CUDA(cudaMemcpyAsync(E.blk(sv->w_handle), E.blk(*S.w), sizeof(double) * E.N * E.g.ld,
                              cudaMemcpyDeviceToDevice, E.s));
    E.sync();
    set_phase_times(r, std::chrono::duration<double>(std::chrono::steady_clock::now() - sv->t0).count(),
                    po::host_wait_seconds() - sv->wait0);
  } catch (const Error& ex) {
    return solver_error(sv->h, r, ex, ex.code);
  } catch (const std::exception& ex) {
    return solver_error(sv->h, r, ex, PO_EINVAL);
  }
  return PO_OK;
}

int po_solver_destroy(po_solver* sv) {
  if (!sv) return PO_OK;
  delete sv->S;
  delete sv;
  return PO_OK;
}

}  // extern "C"
