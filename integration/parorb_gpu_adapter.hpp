// parorb_gpu_adapter.hpp — reference-side drop-in for the B200 hot path.
//
// A maintainer of the reference (parorb, /root/reference/proj) adds this header
// and links libparorb_b200.so; call sites of opt_par_inner / opt_par_mod_inner /
// optm_qr_solve (include/parorb/optimizer.hpp:153-161) switch to parorb::gpu::*
// with identical arguments and get the reference's SolveResult back. Only the C
// ABI (include/parorb_gpu.h) is used: no CUDA or torch types cross the boundary.
#pragma once

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "parorb/energy.hpp"
#include "parorb/errors.hpp"
#include "parorb/optimizer.hpp"
#include "parorb_gpu.h"

namespace parorb::gpu {

namespace detail {

// errors.hpp:10-45 <- po_status
inline void check(int rc, po_engine* e) {
  if (rc == PO_OK) return;
  const std::string msg = e ? po_last_error(e) : "po_create failed";
  switch (rc) {
    case PO_EINVAL: throw InvalidArgument(msg);
    case PO_EDEGENERATE: throw DegenerateSetError(msg);
    case PO_ESOLVER: throw SolverError(msg);
    case PO_ESTAGNATION: throw StagnationError(msg, {});
    default: throw std::runtime_error("parorb_gpu: " + msg);
  }
}

struct EngineDeleter {
  void operator()(po_engine* e) const { po_destroy(e); }
};

inline po_params to_params(const OptimizerParams& p, Algorithm alg, const Problem& prob) {
  po_params q;
  po_default_params(&q);
  q.algorithm = alg == Algorithm::kOptmQr ? PO_ALG_OPTM_QR
                : alg == Algorithm::kOptPar ? PO_ALG_OPT_PAR
                                            : PO_ALG_OPT_PAR_MOD;
  q.bb_variant = p.bb_variant == BbVariant::kBb1 ? PO_BB1
                 : p.bb_variant == BbVariant::kBb2 ? PO_BB2
                                                   : PO_BB_ALTERNATE;
  q.bb_trace_abs = p.bb_trace_abs == BbTraceAbs::kDiagAbs ? PO_TRACE_DIAG_ABS : PO_TRACE_ABS_TRACE;
  q.convergence_mode = p.convergence_mode == ConvergenceMode::kGradNorm ? PO_CONV_GRAD_NORM
                       : p.convergence_mode == ConvergenceMode::kMeanAbs ? PO_CONV_MEAN_ABS
                                                                         : PO_CONV_ENERGY_CHANGE;
  q.rho1 = p.rho1;
  q.delta = p.delta;
  q.eta = p.eta;
  q.n_diag = p.n_diag;
  q.n_org = p.n_org;
  q.max_inner = p.max_inner;
  q.max_backtracks = p.max_backtracks;
  q.tau_min = p.tau_min;
  q.tau_max = p.tau_max;
  q.grad_tol = p.grad_tol;
  q.mean_abs_tol = p.mean_abs_tol;
  q.energy_tol = p.energy_tol;
  q.verify_orthonormality = p.verify_orthonormality ? 1 : 0;
  q.hartree = prob.hartree_enabled ? 1 : 0;
  q.xc = prob.xc_enabled ? 1 : 0;
  q.outer_levels = p.outer_levels;
  q.seed = p.seed;
  return q;
}

// Host-side output arrays of one po_result (records, accepted steps,
// checkpoints, drift flags), sized for `cap` rows.
struct ResultBuffers {
  std::vector<po_record> recs;
  std::vector<double> acc, ckpt;
  std::vector<int> drift;
  po_result r{};
  explicit ResultBuffers(std::size_t cap) : recs(cap), acc(9 * cap), ckpt(5 * cap), drift(cap) {
    r.cap = static_cast<int>(cap);
    r.records = recs.data();
    r.accepted = acc.data();
    r.checkpoints = ckpt.data();
    r.drift_iterations = drift.data();
  }
};

// po_result -> the reference's SolveResult fields (optimizer.hpp:98-112)
inline void fill_result(SolveResult& out, const ResultBuffers& b) {
  const po_result& r = b.r;
  const std::vector<po_record>& recs = b.recs;
  const std::vector<double>& acc = b.acc;
  out.energy = EnergyBreakdown{r.e_kinetic, r.e_external, r.e_hartree, r.e_xc, r.e_total};
  out.outcome = static_cast<SolveOutcome>(r.outcome);  // same enumerator order
  out.message = r.message;
  for (int k = 0; k < r.n_records && k < r.cap; ++k) {
    const po_record& x = recs[k];
    out.records.push_back(IterationRecord{x.level, x.iter, x.energy, x.grad_norm, x.tau,
                                          x.backtracks, x.did_orth != 0, x.did_diag != 0,
                                          x.offdiag_max, x.wall_ms});
  }
  for (int k = 0; k < r.n_accepted && k < r.cap; ++k) {
    const double* a = acc.data() + 9 * k;
    out.accepted_steps.push_back(AcceptedStep{static_cast<int>(a[0]), static_cast<int>(a[1]), a[2],
                                              a[3], a[4], a[5], a[6], a[7], a[8]});
  }
  // OrthCheckpoint per orthogonalization step and the drift flags (optimizer.cpp:535-539)
  for (int k = 0; k < r.n_checkpoints && k < r.cap; ++k) {
    const double* c = b.ckpt.data() + 5 * k;
    out.checkpoints.push_back(
        OrthCheckpoint{static_cast<int>(c[0]), static_cast<int>(c[1]), c[2], c[3], c[4]});
  }
  for (int k = 0; k < r.n_drift && k < r.cap; ++k) out.drift_iterations.push_back(b.drift[k]);
  out.iterations_total = static_cast<int>(out.records.size());
  out.final_grad_norm = r.final_grad_norm;
  out.wall_seconds = r.wall_seconds;
  out.par_seconds = r.par_seconds;  // PhaseTimer buckets (optimizer.cpp:594-595)
  out.sync_seconds = r.sync_seconds;
}

inline SolveResult run(const OrbitalSet& u0, const Problem& prob, const OptimizerParams& params,
                       Algorithm alg) {
  params.validate();
  const Grid& g = *prob.grid;
  if (g.dimension() != 3) throw InvalidArgument("parorb_gpu: 3D grids only");
  po_grid_desc gd;
  for (int a = 0; a < 3; ++a) {
    gd.n[a] = g.points(a);
    gd.extent[a] = g.extent(a);
  }
  po_engine* raw = nullptr;
  const int rc = po_create(&gd, u0.n(), 1.0, nullptr, &raw);
  std::unique_ptr<po_engine, EngineDeleter> e(raw);
  check(rc, raw);
  check(po_set_field(raw, PO_VEXT, prob.v_ext.values.data()), raw);  // Problem::v_ext
  const std::int64_t ng = g.num_points();
  std::vector<double> host(static_cast<std::size_t>(u0.n() * ng));
  for (int i = 0; i < u0.n(); ++i)
    std::memcpy(host.data() + i * ng, u0.orbitals[i].values.data(), sizeof(double) * ng);
  const po_params q = to_params(params, alg, prob);
  ResultBuffers rb(static_cast<std::size_t>(q.max_inner) + 1);
  // upload, InnerLoop, finalize with the final download overlapped: one call
  // (pageable std::vector memory: po_solve_host stages it through pinned chunks)
  check(po_solve_host(raw, &q, host.data(), host.data(), &rb.r), raw);

  SolveResult out;  // optimizer.hpp:98-112
  std::vector<Field> fields;
  for (int i = 0; i < u0.n(); ++i) {
    Field f = make_field(prob.grid);
    std::memcpy(f.values.data(), host.data() + i * ng, sizeof(double) * ng);
    fields.push_back(std::move(f));
  }
  out.orbitals = OrbitalSet{std::move(fields)};
  fill_result(out, rb);
  return out;
}

}  // namespace detail

// Drop-ins for optimizer.hpp:153-161 (same signatures minus the Executor).
inline SolveResult optm_qr_solve(const OrbitalSet& u0, const Problem& p, const OptimizerParams& q) {
  return detail::run(u0, p, q, Algorithm::kOptmQr);
}
inline SolveResult opt_par_inner(const OrbitalSet& u0, const Problem& p, const OptimizerParams& q) {
  return detail::run(u0, p, q, Algorithm::kOptPar);
}
inline SolveResult opt_par_mod_inner(const OrbitalSet& u0, const Problem& p,
                                     const OptimizerParams& q) {
  return detail::run(u0, p, q, Algorithm::kOptParMod);
}

// Drop-in for optimizer.hpp:163-167 solve (initialize_orbitals + outer levels).
inline SolveResult solve(const Problem& level0, const OptimizerParams& params) {
  params.validate();
  const Grid& g = *level0.grid;
  if (g.dimension() != 3) throw InvalidArgument("parorb_gpu: 3D grids only");
  po_grid_desc gd;
  for (int a = 0; a < 3; ++a) {
    gd.n[a] = g.points(a);
    gd.extent[a] = g.extent(a);
  }
  std::vector<double> atoms;
  for (const Atom& at : level0.atoms) {
    atoms.insert(atoms.end(), {at.position[0], at.position[1], at.position[2], at.charge,
                               at.softening});
  }
  const po_params q = detail::to_params(params, params.algorithm, level0);
  detail::ResultBuffers rb(static_cast<std::size_t>(q.max_inner) * q.outer_levels + 1);
  po_engine* raw = nullptr;
  int w = -1;
  const int rc = po_solve_levels(&gd, level0.n_orbitals, 1.0, atoms.data(),
                                 static_cast<int>(level0.atoms.size()), &q, &rb.r, &raw, &w);
  std::unique_ptr<po_engine, detail::EngineDeleter> e(raw);
  detail::check(rc, raw);
  // the final grid: refine_uniform applied outer_levels - 1 times (grid.cpp:137-149)
  GridPtr grid = level0.grid;
  for (int l = 1; l < params.outer_levels; ++l) grid = refine_uniform(*grid);
  const std::int64_t ng = grid->num_points();
  std::vector<double> host(static_cast<std::size_t>(level0.n_orbitals * ng));
  detail::check(po_download_block(raw, w, host.data()), raw);
  SolveResult out;
  std::vector<Field> fields;
  for (int i = 0; i < level0.n_orbitals; ++i) {
    Field f = make_field(grid);
    std::memcpy(f.values.data(), host.data() + i * ng, sizeof(double) * ng);
    fields.push_back(std::move(f));
  }
  out.orbitals = OrbitalSet{std::move(fields)};
  detail::fill_result(out, rb);
  return out;
}

}  // namespace parorb::gpu
