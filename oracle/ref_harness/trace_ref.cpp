// trace_ref — TEST INFRASTRUCTURE ONLY (oracle side, never shipped or timed as
// the product). Drives the UNMODIFIED reference library (built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/) through its
// public C++ API and dumps results as raw little-endian float64 files so the
// Python tests can pin the C restatement (oracle/port) and the CUDA path.
//
//   trace_ref solve <spec.json> <outdir>   run opt_par_inner / opt_par_mod_inner /
//                                           optm_qr_solve (optimizer.hpp:153-161)
//   trace_ref ops   <spec.json> <outdir>   one evaluation of every hot-path
//                                           operator on the start block (full
//                                           arrays, or reduced with "sketch")
//   trace_ref orth  <spec.json> <outdir>   orthonormalize_with_gram of the start
//   trace_ref levels / prolong             solve (optimizer.cpp:638-669) /
//                                           refine_uniform + prolongate
//
// Spec keys: n[3], extent[3], atoms[[x,y,z,Z,a]...], n_orbitals, hartree, xc,
// start{kind: random_orthonormal|initialize|file, seed, path}, algorithm,
// params{...OptimizerParams fields...}, threads.
#include <json.hpp>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <thread>
#include <string>
#include <vector>

#include "parorb/driver.hpp"
#include "parorb/energy.hpp"
#include "parorb/errors.hpp"
#include "parorb/grid.hpp"
#include "parorb/manifold.hpp"
#include "parorb/numeric.hpp"
#include "parorb/optimizer.hpp"
#include "parorb/parallel.hpp"
#include "parorb/rng.hpp"
#include "problems.hpp"  // reference test helper: testing::random_orthonormal

using json = nlohmann::json;
using namespace parorb;

namespace {

void write_bin(const std::string& path, const double* p, std::size_t n) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot write " + path);
  f.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(n * sizeof(double)));
}

void write_vec(const std::string& path, const std::vector<double>& v) {
  write_bin(path, v.data(), v.size());
}

void write_field(const std::string& path, const Field& f) { write_vec(path, f.values); }

void write_set(const std::string& path, const FieldSet& s) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot write " + path);
  for (const Field& x : s) {
    f.write(reinterpret_cast<const char*>(x.values.data()),
            static_cast<std::streamsize>(x.values.size() * sizeof(double)));
  }
}

void write_mat(const std::string& path, const Eigen::MatrixXd& m) {
  // row-major dump: entry (i, j) at i * cols + j
  std::vector<double> v(static_cast<std::size_t>(m.rows() * m.cols()));
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index j = 0; j < m.cols(); ++j) v[i * m.cols() + j] = m(i, j);
  write_vec(path, v);
}

std::vector<double> read_bin(const std::string& path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) throw IoError("cannot read " + path);
  const auto bytes = static_cast<std::size_t>(f.tellg());
  std::vector<double> v(bytes / sizeof(double));
  f.seekg(0);
  f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(bytes));
  return v;
}

// ---- size-independent fingerprints of large blocks (C3 / C4-grid fixtures)
//
// A block B (N x N_g, orbital-major) is reduced to
//   S = sqrt(w) * B X          (N x m), X(p, a) = +-1 Rademacher signs from a
//                               splitmix64 hash of (seed, p * m + a)
//   rows at K sampled points    p_j = (j * 2654435761) mod N_g
// The sign rule is restated bit-for-bit in tests/helpers.py (sketch_signs).
// For two orthonormal sets, X^T P X = S^T G^-1 S, so the off-diagonal entries
// of the difference of the two m x m matrices estimate ||P1 - P2||_F without
// either side holding the other's block (tests/helpers.py:sketch_projector_distance).
struct Sketch {
  int m = 0;
  std::uint64_t seed = 0;
  int samples = 0;
};

inline double sketch_sign(std::uint64_t seed, std::uint64_t key) {
  std::uint64_t z = seed ^ (key * 0xD1B54A32D192ED03ull);
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (z >> 63) ? -1.0 : 1.0;
}

std::vector<double> sketch_block(const FieldSet& s, const Sketch& k, double weight) {
  const std::size_t n = s.size();
  const std::size_t ng = s.empty() ? 0 : s[0].values.size();
  const std::size_t m = static_cast<std::size_t>(k.m);
  std::vector<double> out(n * m, 0.0);
  const std::size_t chunk = 2048;
  std::vector<double> x(chunk * m);
  for (std::size_t p0 = 0; p0 < ng; p0 += chunk) {
    const std::size_t np = std::min(chunk, ng - p0);
    for (std::size_t p = 0; p < np; ++p)
      for (std::size_t a = 0; a < m; ++a) x[p * m + a] = sketch_sign(k.seed, (p0 + p) * m + a);
    std::vector<std::thread> pool;
    const std::size_t nt = std::max<std::size_t>(1, std::min<std::size_t>(n, 8));
    for (std::size_t t = 0; t < nt; ++t) {
      pool.emplace_back([&, t] {
        for (std::size_t i = t; i < n; i += nt) {
          const double* u = s[i].values.data() + p0;
          double* o = out.data() + i * m;
          for (std::size_t p = 0; p < np; ++p) {
            const double v = u[p];
            const double* xr = x.data() + p * m;
            for (std::size_t a = 0; a < m; ++a) o[a] += v * xr[a];
          }
        }
      });
    }
    for (auto& th : pool) th.join();
  }
  const double sw = std::sqrt(weight);
  for (double& v : out) v *= sw;
  return out;
}

std::vector<std::int64_t> sample_points(std::int64_t ng, int k) {
  std::vector<std::int64_t> p(static_cast<std::size_t>(k));
  for (int j = 0; j < k; ++j)
    p[static_cast<std::size_t>(j)] =
        static_cast<std::int64_t>((static_cast<unsigned __int128>(j) * 2654435761ull) % ng);
  return p;
}

std::vector<double> sample_block(const FieldSet& s, const std::vector<std::int64_t>& pts) {
  std::vector<double> out;
  out.reserve(s.size() * pts.size());
  for (const Field& f : s)
    for (std::int64_t p : pts) out.push_back(f.values[static_cast<std::size_t>(p)]);
  return out;
}

std::vector<double> sample_field(const Field& f, const std::vector<std::int64_t>& pts) {
  std::vector<double> out;
  for (std::int64_t p : pts) out.push_back(f.values[static_cast<std::size_t>(p)]);
  return out;
}

// sum and sum of squares of a field, long double accumulation (fixture norms)
std::vector<double> field_norms(const Field& f) {
  long double s = 0.0L, q = 0.0L;
  for (double v : f.values) {
    s += v;
    q += static_cast<long double>(v) * v;
  }
  return {static_cast<double>(s), static_cast<double>(q)};
}

struct Setup {
  Problem problem;
  OrbitalSet u0;
  OptimizerParams params;
  std::string algorithm = "opt_par";
  int threads = 1;
  Sketch sketch;
  bool write_final_w = true;
};

Setup load(const std::string& spec_path) {
  std::ifstream in(spec_path);
  if (!in) throw IoError("cannot open spec " + spec_path);
  json j = json::parse(in);
  Setup s;
  const int dim = static_cast<int>(j["n"].size());
  std::vector<double> ext = j["extent"].get<std::vector<double>>();
  std::vector<std::int64_t> pts = j["n"].get<std::vector<std::int64_t>>();
  GridPtr g = build_grid(dim, ext, pts);
  AtomList atoms;
  for (const auto& a : j.value("atoms", json::array())) {
    Atom at;
    for (int k = 0; k < dim; ++k) at.position[k] = a[k].get<double>();
    at.charge = a[3].get<double>();
    at.softening = a[4].get<double>();
    atoms.push_back(at);
  }
  const int n = j["n_orbitals"].get<int>();
  const bool hartree = j.value("hartree", false);
  const bool xc = j.value("xc", false);
  const HartreeMode mode = dim == 3 ? HartreeMode::kPoisson : HartreeMode::kKernel;
  s.problem = make_problem(g, atoms, n, hartree, xc, mode);

  const json st = j.value("start", json{{"kind", "random_orthonormal"}, {"seed", 42}});
  const std::string kind = st.value("kind", "random_orthonormal");
  const std::uint64_t seed = st.value("seed", 42ull);
  if (kind == "random_orthonormal") {
    s.u0 = testing::random_orthonormal(g, n, seed);
  } else if (kind == "initialize") {
    s.u0 = initialize_orbitals(g, atoms, n, seed);
  } else if (kind == "file") {
    std::vector<double> v = read_bin(st["path"].get<std::string>());
    const std::int64_t ng = g->num_points();
    if (static_cast<std::int64_t>(v.size()) != ng * n) throw InvalidArgument("start file size");
    std::vector<Field> fields;
    for (int i = 0; i < n; ++i) {
      Field f = make_field(g);
      std::copy(v.begin() + i * ng, v.begin() + (i + 1) * ng, f.values.begin());
      fields.push_back(std::move(f));
    }
    s.u0 = make_orbital_set(std::move(fields));
    if (st.value("orthonormalize", false)) s.u0 = orthonormalize(s.u0);
  } else {
    throw InvalidArgument("unknown start kind " + kind);
  }

  const json p = j.value("params", json::object());
  OptimizerParams& q = s.params;
  q.max_inner = p.value("max_inner", q.max_inner);
  q.n_org = p.value("n_org", q.n_org);
  q.n_diag = p.value("n_diag", q.n_diag);
  q.max_backtracks = p.value("max_backtracks", q.max_backtracks);
  q.rho1 = p.value("rho1", q.rho1);
  q.delta = p.value("delta", q.delta);
  q.eta = p.value("eta", q.eta);
  q.tau_min = p.value("tau_min", q.tau_min);
  q.tau_max = p.value("tau_max", q.tau_max);
  q.grad_tol = p.value("grad_tol", q.grad_tol);
  q.mean_abs_tol = p.value("mean_abs_tol", q.mean_abs_tol);
  q.energy_tol = p.value("energy_tol", q.energy_tol);
  q.verify_orthonormality = p.value("verify_orthonormality", q.verify_orthonormality);
  q.outer_levels = p.value("outer_levels", q.outer_levels);
  q.seed = p.value("seed", q.seed);
  const std::string bb = p.value("bb_variant", "bb1");
  q.bb_variant = bb == "bb2" ? BbVariant::kBb2 : bb == "alternate" ? BbVariant::kAlternate : BbVariant::kBb1;
  q.bb_trace_abs = p.value("bb_trace_abs", "diag_abs") == "abs_trace" ? BbTraceAbs::kAbsTrace
                                                                      : BbTraceAbs::kDiagAbs;
  const std::string cm = p.value("convergence_mode", "grad_norm");
  q.convergence_mode = cm == "mean_abs" ? ConvergenceMode::kMeanAbs
                       : cm == "energy_change" ? ConvergenceMode::kEnergyChange
                                               : ConvergenceMode::kGradNorm;
  s.algorithm = j.value("algorithm", "opt_par");
  s.threads = j.value("threads", 1);
  if (j.contains("sketch")) {
    const json& k = j["sketch"];
    s.sketch.m = k.value("m", 64);
    s.sketch.seed = k.value("seed", 7ull);
    s.sketch.samples = k.value("samples", 1024);
  }
  s.write_final_w = j.value("write_final_w", true);
  return s;
}

const char* outcome_name(SolveOutcome o) {
  switch (o) {
    case SolveOutcome::kConverged: return "converged";
    case SolveOutcome::kMaxIterations: return "max_iterations";
    case SolveOutcome::kStagnation: return "stagnation";
    case SolveOutcome::kNumericalFailure: return "numerical_failure";
  }
  return "?";
}

json energy_json(const EnergyBreakdown& e) {
  return json{{"kinetic", e.kinetic}, {"external", e.external}, {"hartree", e.hartree},
              {"xc", e.xc}, {"total", e.total}};
}

int cmd_solve(const Setup& s, const std::string& out) {
  Executor ex(s.threads);
  write_set(out + "/u0.bin", s.u0.orbitals);
  const auto t0 = std::chrono::steady_clock::now();
  SolveResult r;
  if (s.algorithm == "opt_par") r = opt_par_inner(s.u0, s.problem, s.params, ex);
  else if (s.algorithm == "opt_par_mod") r = opt_par_mod_inner(s.u0, s.problem, s.params, ex);
  else if (s.algorithm == "optm_qr") r = optm_qr_solve(s.u0, s.problem, s.params, ex);
  else throw InvalidArgument("unknown algorithm " + s.algorithm);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

  {
    std::ofstream f(out + "/records.csv");
    f << log_header() << '\n';
    for (const IterationRecord& rec : r.records) f << format_log_row(rec) << '\n';
  }
  {
    std::ofstream f(out + "/accepted.csv");
    f << "level,iter,energy,c_before,c_after,q_before,q_after,tau,znorm2\n";
    char buf[512];
    for (const AcceptedStep& a : r.accepted_steps) {
      std::snprintf(buf, sizeof buf, "%d,%d,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g\n",
                    a.level, a.iter, a.energy, a.c_before, a.c_after, a.q_before, a.q_after,
                    a.tau, a.znorm2);
      f << buf;
    }
  }
  {
    std::ofstream f(out + "/checkpoints.csv");
    f << "level,iter,offdiag_max,diag_deviation_max,orth_deviation\n";
    char buf[256];
    for (const OrthCheckpoint& c : r.checkpoints) {
      std::snprintf(buf, sizeof buf, "%d,%d,%.17g,%.17g,%.17g\n", c.level, c.iter,
                    c.offdiag_max, c.diag_deviation_max, c.orth_deviation);
      f << buf;
    }
  }
  if (s.write_final_w) write_set(out + "/final_w.bin", r.orbitals.orbitals);
  // Orbital eigenvalues at the final iterate: eig(Sigma), Sigma = <(HW)^T W>.
  HamiltonianState st = build_hamiltonian(r.orbitals, s.problem);
  FieldSet hw = apply_hamiltonian(st, r.orbitals, ex);
  GramMatrix sigma = gram(hw, r.orbitals.orbitals);
  SubspaceRotation rot = subspace_rotate(r.orbitals, sigma);
  std::vector<double> gam(static_cast<std::size_t>(rot.gamma.size()));
  for (std::size_t i = 0; i < gam.size(); ++i) gam[i] = rot.gamma(static_cast<Eigen::Index>(i));
  write_vec(out + "/final_eig.bin", gam);
  if (s.sketch.m > 0) {
    const double wq = r.orbitals.grid().quadrature_weight();
    write_vec(out + "/final_sketch.bin", sketch_block(r.orbitals.orbitals, s.sketch, wq));
    write_mat(out + "/final_gram.bin", gram(r.orbitals, r.orbitals));
  }

  json sum{{"outcome", outcome_name(r.outcome)},
           {"message", r.message},
           {"energy", energy_json(r.energy)},
           {"iterations_total", r.iterations_total},
           {"final_grad_norm", r.final_grad_norm},
           {"wall_seconds", r.wall_seconds},
           {"wall_seconds_outer", wall},
           {"par_seconds", r.par_seconds},
           {"sync_seconds", r.sync_seconds},
           {"threads", s.threads},
           {"drift_iterations", r.drift_iterations}};
  std::ofstream(out + "/summary.json") << sum.dump(1) << '\n';
  return 0;
}

int cmd_ops(const Setup& s, const std::string& out) {
  Executor ex(s.threads);
  const OrbitalSet& w = s.u0;
  const double wq = w.grid().quadrature_weight();
  // Full arrays, or (s.sketch.m > 0) the reduced fingerprints for shapes whose
  // blocks are too large to commit (C3, the C4 grid): fields at sampled points
  // + sum / sum of squares, blocks as sampled rows + a Rademacher sketch.
  const bool reduced = s.sketch.m > 0;
  const std::vector<std::int64_t> pts =
      reduced ? sample_points(w.grid().num_points(), s.sketch.samples) : std::vector<std::int64_t>{};
  auto put_field = [&](const std::string& name, const Field& f) {
    if (!reduced) return write_field(out + "/" + name + ".bin", f);
    write_vec(out + "/" + name + "_samples.bin", sample_field(f, pts));
    write_vec(out + "/" + name + "_norms.bin", field_norms(f));
  };
  auto put_set = [&](const std::string& name, const FieldSet& b) {
    if (!reduced) return write_set(out + "/" + name + ".bin", b);
    write_vec(out + "/" + name + "_rows.bin", sample_block(b, pts));
    write_vec(out + "/" + name + "_sketch.bin", sketch_block(b, s.sketch, wq));
  };
  if (!reduced) write_set(out + "/u0.bin", w.orbitals);
  else put_set("u0", w.orbitals);
  put_field("v_ext", s.problem.v_ext);
  HamiltonianState st = build_hamiltonian(w, s.problem);
  put_field("rho", st.density);
  put_field("v_h", st.v_hartree);
  put_field("v_xc", st.v_xc);
  put_field("v_local", st.v_local);
  put_field("eps_xc", xc_energy_density(st.density));
  FieldSet hw = apply_hamiltonian(st, w, ex);
  put_set("hw", hw);
  std::vector<double> kin, ext;
  for (const Field& f : w.orbitals) {
    kin.push_back(kinetic_term(f));
    ext.push_back(potential_term(s.problem.v_ext, f));
  }
  write_vec(out + "/kin.bin", kin);
  write_vec(out + "/ext.bin", ext);
  EnergyBreakdown e = total_energy(w, st, ex);
  write_mat(out + "/gram_ww.bin", gram(w, w));
  GramMatrix sigma = gram(hw, w.orbitals);
  write_mat(out + "/sigma.bin", sigma);
  DiagonalResiduals dr = diagonal_residuals(w, hw, ex);
  put_set("z", dr.directions);
  write_vec(out + "/sigma_diag.bin", dr.sigma_diag);
  StiefelGradient sg = stiefel_gradient(w, hw, ex);
  double gn = 0.0;
  std::vector<double> dnorm2;
  for (const Field& f : sg.directions) {
    const double d2 = inner_product(f, f);
    dnorm2.push_back(d2);
    gn += d2;
  }
  write_vec(out + "/d_norm2.bin", dnorm2);
  if (reduced) put_set("d", sg.directions);
  // Trial step + orthonormalization, as in one line-search trial.
  const double tau = 0.3;
  std::vector<Field> trial;
  for (int i = 0; i < w.n(); ++i) trial.push_back(linear_combination(w.orbitals[i], -tau, dr.directions[i]));
  OrthResult orth = orthonormalize_with_gram(OrbitalSet{trial}, true);
  put_set("orth_w", orth.w.orbitals);
  write_mat(out + "/orth_pre_gram.bin", orth.pre_gram);
  if (reduced) write_mat(out + "/orth_gram.bin", gram(orth.w, orth.w));
  HamiltonianState st2 = build_hamiltonian(orth.w, s.problem);
  EnergyBreakdown e2 = total_energy(orth.w, st2, ex);
  SubspaceRotation rot = subspace_rotate(w, sigma);
  std::vector<double> gam;
  for (Eigen::Index i = 0; i < rot.gamma.size(); ++i) gam.push_back(rot.gamma(i));
  write_vec(out + "/sigma_eig.bin", gam);
  json sum{{"energy", energy_json(e)},
           {"trial_tau", tau},
           {"trial_energy", energy_json(e2)},
           {"orth_post_deviation", orth.post_deviation},
           {"grad_norm", std::sqrt(gn)},
           {"weight", wq},
           {"reduced", reduced}};
  std::ofstream(out + "/ops.json") << sum.dump(1) << '\n';
  return 0;
}

// The reference's multi-level solve (optimizer.cpp:638-669) from its own
// initialize_orbitals(params.seed): records, final orbitals and summary.
int cmd_levels(const Setup& s, const std::string& out) {
  Executor ex(s.threads);
  OptimizerParams q = s.params;
  q.algorithm = s.algorithm == "opt_par" ? Algorithm::kOptPar
                : s.algorithm == "optm_qr" ? Algorithm::kOptmQr
                                           : Algorithm::kOptParMod;
  SolveResult r = solve(s.problem, q, ex);
  {
    std::ofstream f(out + "/records.csv");
    f << log_header() << '\n';
    for (const IterationRecord& rec : r.records) f << format_log_row(rec) << '\n';
  }
  write_set(out + "/final_w.bin", r.orbitals.orbitals);
  json sum{{"outcome", outcome_name(r.outcome)},
           {"message", r.message},
           {"energy", energy_json(r.energy)},
           {"iterations_total", r.iterations_total},
           {"final_grad_norm", r.final_grad_norm},
           {"final_points", r.orbitals.grid().num_points()}};
  std::ofstream(out + "/summary.json") << sum.dump(1) << '\n';
  return 0;
}

// orthonormalize_with_gram (manifold.cpp:136-169) of the start block as given
// (start kind "file" without "orthonormalize"): the symmetric-eigen fallback
// fixture (manifold.cpp:118-132) on an ill-conditioned, full-rank set.
int cmd_orth(const Setup& s, const std::string& out) {
  OrthResult o = orthonormalize_with_gram(s.u0, true);
  write_set(out + "/orth_w.bin", o.w.orbitals);
  write_mat(out + "/pre_gram.bin", o.pre_gram);
  json sum{{"post_deviation", o.post_deviation}};
  std::ofstream(out + "/orth.json") << sum.dump(1) << '\n';
  return 0;
}

// refine_uniform + prolongate (grid.cpp:137-212) of the start orbitals
int cmd_prolong(const Setup& s, const std::string& out) {
  GridPtr fine = refine_uniform(s.u0.grid());
  FieldSet p;
  for (const Field& f : s.u0.orbitals) p.push_back(prolongate(f, fine));
  write_set(out + "/u0.bin", s.u0.orbitals);
  write_set(out + "/prolong.bin", p);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 4) {
    std::fprintf(stderr, "usage: trace_ref solve|ops|levels|prolong|orth <spec.json> <outdir>\n");
    return 1;
  }
  try {
    const std::string cmd = argv[1];
    Setup s = load(argv[2]);
    if (cmd == "solve") return cmd_solve(s, argv[3]);
    if (cmd == "ops") return cmd_ops(s, argv[3]);
    if (cmd == "levels") return cmd_levels(s, argv[3]);
    if (cmd == "prolong") return cmd_prolong(s, argv[3]);
    if (cmd == "orth") return cmd_orth(s, argv[3]);
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "trace_ref: %s\n", e.what());
    return 3;
  }
}
