// dropin_demo — the reference's own API on both sides of the boundary.
// Builds a Problem with the UNMODIFIED reference library, starts from the
// reference's testing::random_orthonormal, runs parorb::opt_par_mod_inner
// (CPU reference) and parorb::gpu::opt_par_mod_inner (this repo, via the C
// ABI) and compares the IterationRecord energies. Exit 0 iff every iteration
// agrees within 1e-6 Ha. Built by oracle/Makefile (target dropin) because it
// links the reference; the binary is test infrastructure.
//   dropin_demo [n_points=16] [n_orbitals=4] [iterations=12]
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "parorb/energy.hpp"
#include "parorb/optimizer.hpp"
#include "parorb_gpu_adapter.hpp"
#include "problems.hpp"

int main(int argc, char** argv) {
  using namespace parorb;
  const int n = argc > 1 ? std::atoi(argv[1]) : 16;
  const int norb = argc > 2 ? std::atoi(argv[2]) : 4;
  const int iters = argc > 3 ? std::atoi(argv[3]) : 12;
  const int levels = argc > 4 ? std::atoi(argv[4]) : 1;  // > 1: the multi-level solve()
  const double L = n >= 64 ? 20.0 : 8.0;
  const double ext[] = {L, L, L};
  const std::int64_t pts[] = {n, n, n};
  GridPtr g = build_grid(3, ext, pts);
  AtomList atoms(3);
  const double c = L / 2;
  atoms[0].position = {c, c, c};
  atoms[0].charge = 8.0;
  atoms[1].position = {c + 1.43, c + 1.11, c};
  atoms[2].position = {c - 1.43, c + 1.11, c};
  Problem p = make_problem(g, atoms, norb, true, true, HartreeMode::kPoisson);
  OrbitalSet u0 = testing::random_orthonormal(g, norb, 42);
  OptimizerParams params;
  params.max_inner = iters;
  params.outer_levels = levels;
  params.seed = 7;
  Executor ex(1);
  SolveResult cpu = levels > 1 ? solve(p, params, ex) : opt_par_mod_inner(u0, p, params, ex);
  SolveResult gpu = levels > 1 ? gpu::solve(p, params) : gpu::opt_par_mod_inner(u0, p, params);
  double worst = 0.0;
  const std::size_t m = std::min(cpu.records.size(), gpu.records.size());
  for (std::size_t k = 0; k < m; ++k) {
    const double d = std::abs(cpu.records[k].energy - gpu.records[k].energy);
    worst = std::max(worst, d);
    std::printf("level %d iter %3d  E_ref % .15f  E_gpu % .15f  |dE| %.2e  backtracks %d/%d\n",
                cpu.records[k].level, cpu.records[k].iter, cpu.records[k].energy, gpu.records[k].energy, d,
                cpu.records[k].backtracks, gpu.records[k].backtracks);
  }
  const bool ok = cpu.records.size() == gpu.records.size() && worst < 1e-6 &&
                  std::abs(cpu.energy.total - gpu.energy.total) < 1e-6;
  std::printf("records %zu/%zu  final E_ref %.15f  E_gpu %.15f  max|dE| %.3e  wall ref %.3f s gpu %.3f s  %s\n",
              cpu.records.size(), gpu.records.size(), cpu.energy.total, gpu.energy.total, worst,
              cpu.wall_seconds, gpu.wall_seconds, ok ? "OK" : "MISMATCH");
  return ok ? 0 : 1;
}
