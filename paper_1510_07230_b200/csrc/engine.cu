// Engine (device-resident rank state) and the operator-level C ABI
// (include/parorb_gpu.h). Each po_* operator mirrors one reference function
// (cited in the header); all arithmetic runs in the sm_100a kernels — there is
// no host compute path.
#include <chrono>
#include <dlfcn.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <vector>

#include <cstdlib>

#include "engine.h"

namespace po {

bool pdl_on() {
  static const bool on = !getenv("PO_PDL") || atoi(getenv("PO_PDL")) != 0;
  return on;
}


namespace {
__global__ void copy_diag_kernel(int N, const double* __restrict__ M, double* __restrict__ out) {
  PO_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) out[i] = M[(int64_t)i * N + i];
}
}  // namespace

void launch_copy_diag(int N, const double* M, double* out, cudaStream_t s) {
  ::po::count_launch();
  launch_pdl(copy_diag_kernel, dim3((N + 255) / 256), dim3(256), 0, s, N, M, out);
}

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }

static int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

Engine::Engine(const po_grid_desc* grid, int n, double occupation, const po_dist_desc* dist) {
  if (!grid) throw Error(PO_EINVAL, "null grid");
  for (int a = 0; a < 3; ++a) {
    if (grid->n[a] < 1) throw Error(PO_EINVAL, "grid: points_per_axis must be >= 1");
    if (!(grid->extent[a] > 0.0) || !std::isfinite(grid->extent[a]))
      throw Error(PO_EINVAL, "grid: extents must be positive and finite");
  }
  if (n < 1) throw Error(PO_EINVAL, "make_problem: n_orbitals must be >= 1");
  if (!(occupation > 0.0)) throw Error(PO_EINVAL, "occupation must be positive");
  N = n;
  occ = occupation;
  if (dist && dist->device >= 0) PO_CUDA(cudaSetDevice(dist->device));
  comm = make_comm(dist);
  rank = comm->rank;
  size = comm->size;

  g.n0 = grid->n[0];
  g.n1 = grid->n[1];
  g.n2 = grid->n[2];
  if (g.n0 < size) throw Error(PO_EINVAL, "fewer axis-0 planes than ranks");
  if ((int64_t)n > g.n0 * g.n1 * g.n2)
    throw Error(PO_EINVAL, "make_problem: more orbitals than grid points");
  const int64_t base = g.n0 / size, rem = g.n0 % size;
  int lo_peer, hi_peer;
  po_slab_plan(g.n0, size, rank, &g.z0, &g.nz, &lo_peer, &hi_peer);
  g.plane = g.n1 * g.n2;
  g.ngl = g.nz * g.plane;
  g.ld = round_up(g.ngl, 32);
  if (const char* e = getenv("PO_LD_PAD")) g.ld += round_up(atoi(e), 32);  // measurement
  g.w = 1.0;
  for (int a = 0; a < 3; ++a) {
    ext[a] = grid->extent[a];
    h[a] = grid->extent[a] / (double)(grid->n[a] + 1);  // grid.cpp:33
    g.ih2[a] = 1.0 / (h[a] * h[a]);
    g.w *= h[a];
  }
  ng_full = g.n0 * g.n1 * g.n2;
  max_slab_points = (base + (rem ? 1 : 0)) * g.plane;

  PO_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t fb = sizeof(double) * (size_t)g.ngl;
  PO_CUDA(cudaMalloc(&v_ext, fb));
  PO_CUDA(cudaMemsetAsync(v_ext, 0, fb, s));
  def_state_ = new_state();

  size_t pc = 0;
  auto upd = [&](size_t v) { pc = v > pc ? v : pc; };
  upd((size_t)3 * N * hamiltonian_nblk(g));
  upd((size_t)3 * N * hamiltonian2_nblk(g));
  if (hamiltonian_split_ok(g)) upd((size_t)3 * N * hamiltonian_split_nblk(g));
  upd((size_t)5 * N * mix_nblk_max(g));  // fused directions: 5 partial rows
  upd((size_t)4 * N * per_orbital_nblk(g, N));  // residual + BB rows
  upd((size_t)4 * N * 512);  // the same rows from the Sigma Gram's splits (at most one wave of CTAs)
  upd((size_t)2 * points_nblk(g));
  partials_cap = pc;
  PO_CUDA(cudaMalloc(&partials, pc * sizeof(double)));
  PO_CUDA(cudaMalloc(&gram_ws, gram_workspace_doubles(g, N) * sizeof(double)));
  PO_CUDA(cudaMalloc(&dvec, dvec_len() * sizeof(double)));
  PO_CUDA(cudaMemsetAsync(dvec, 0, dvec_len() * sizeof(double), s));
  PO_CUDA(cudaHostAlloc(&hvec, dvec_len() * sizeof(double), cudaHostAllocMapped));
  PO_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hvec_dev), hvec, 0));
  PO_CUDA(cudaHostAlloc(&hflag, sizeof(unsigned long long), cudaHostAllocMapped));
  PO_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hflag_dev), hflag, 0));
  *hflag = 0;
  const size_t nn = (size_t)N * N * sizeof(double);
  for (auto& m : dmat) PO_CUDA(cudaMalloc(&m, nn));
  PO_CUDA(cudaMalloc(&chol_L, nn));
  PO_CUDA(cudaMalloc(&syev_work, nn));
  PO_CUDA(cudaMallocHost(&hmat, nn));
  if (size > 1) {
    const size_t hb = (size_t)N * g.plane * sizeof(double);
    PO_CUDA(cudaMalloc(&halo_lo, hb));
    PO_CUDA(cudaMalloc(&halo_hi, hb));
    PO_CUDA(cudaMalloc(&send_lo, hb));
    PO_CUDA(cudaMalloc(&send_hi, hb));
    PO_CUDA(cudaMemsetAsync(halo_lo, 0, hb, s));
    PO_CUDA(cudaMemsetAsync(halo_hi, 0, hb, s));
    PO_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    PO_CUDA(cudaEventCreateWithFlags(&ev_pack, cudaEventDisableTiming));
    PO_CUDA(cudaEventCreateWithFlags(&ev_halo, cudaEventDisableTiming));
  }
  // replicated full-grid Poisson buffers (+ gather staging for size > 1)
  // [full grid | size x max_slab gather staging | max_slab local send slab]
  const size_t full = (size_t)ng_full + (size > 1 ? (size_t)(size + 1) * max_slab_points : 0);
  PO_CUDA(cudaMalloc(&cg_b, full * sizeof(double)));
  PO_CUDA(cudaMalloc(&cg_x, (size_t)ng_full * sizeof(double)));
  PO_CUDA(cudaMemsetAsync(cg_x, 0, (size_t)ng_full * sizeof(double), s));
  PO_CUDA(cudaMalloc(&cg_ws, cg_workspace_doubles(ng_full) * sizeof(double)));
  PO_CUDA(cudaMalloc(&cg_bar, 4 * sizeof(unsigned)));
  PO_CUDA(cudaMalloc(&cg_out_i, 4 * sizeof(int)));
  PO_CUDA(cudaMalloc(&cg_out_d, 4 * sizeof(double)));
  PO_CUDA(cudaHostAlloc(&h_cg_i, 4 * sizeof(int), cudaHostAllocMapped));
  PO_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_cg_i_dev), h_cg_i, 0));
  std::memset(h_cg_i, 0, 4 * sizeof(int));
  PO_CUDA(cudaMallocHost(&h_cg_d, 4 * sizeof(double)));
  PO_CUDA(cudaMemsetAsync(cg_out_i, 0, 4 * sizeof(int), s));
  PO_CUDA(cudaMemsetAsync(cg_out_d, 0, 4 * sizeof(double), s));
  sync();
  dst.init(g.n0, g.n1, g.n2, h);
  PO_CUDA(cudaGetLastError());
}

Engine::~Engine() {
  free_staging();
  if (s) cudaStreamSynchronize(s);
  for (double* b : blocks_)
    if (b) cudaFree(b);
  for (DevState* st : states_) {
    if (!st) continue;
    cudaFree(st->rho);
    cudaFree(st->v_h);
    cudaFree(st->v_xc);
    cudaFree(st->v_local);
    delete st;
  }
  double* bufs[] = {v_ext, partials, gram_ws, dvec, chol_L, syev_work, halo_lo, halo_hi,
                    send_lo, send_hi, cg_b, cg_x, cg_ws, cg_out_d};
  for (double* p : bufs)
    if (p) cudaFree(p);
  for (double* m : dmat)
    if (m) cudaFree(m);
  if (cg_bar) cudaFree(cg_bar);
  if (cg_out_i) cudaFree(cg_out_i);
  if (hvec) cudaFreeHost(hvec);
  if (hmat) cudaFreeHost(hmat);
  if (h_cg_i) cudaFreeHost(h_cg_i);
  if (hflag) cudaFreeHost(hflag);
  if (h_cg_d) cudaFreeHost(h_cg_d);
  dst.release();
  comm.reset();
  if (cs) cudaStreamSynchronize(cs);
  if (ev_pack) cudaEventDestroy(ev_pack);
  if (ev_halo) cudaEventDestroy(ev_halo);
  if (cs) cudaStreamDestroy(cs);
  if (s) cudaStreamDestroy(s);
}

// Spin on the stream instead of a blocking wait: the solver's per-trial
// readback is on the critical path and blocking-sync wake-up jitter dominated
// the iteration time on the host side.
namespace {
thread_local double t_host_wait = 0.0;  // seconds this thread spent waiting on a device
struct WaitClock {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  ~WaitClock() {
    t_host_wait += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
};
}  // namespace

double host_wait_seconds() { return t_host_wait; }

void Engine::sync() {
  PO_CUDA(cudaGetLastError());
  WaitClock wc;
  cudaError_t e;
  while ((e = cudaStreamQuery(s)) == cudaErrorNotReady) {
  }
  if (e != cudaSuccess) throw Error(PO_ECUDA, std::string("stream: ") + cudaGetErrorString(e));
}

int Engine::alloc_block() {
  double* p = nullptr;
  const size_t bytes = sizeof(double) * (size_t)N * (size_t)g.ld;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(PO_ENOMEM, std::string("block allocation failed: ") + cudaGetErrorString(e));
  }
  PO_CUDA(cudaMemsetAsync(p, 0, bytes, s));  // padding stays zero forever
  for (size_t i = 0; i < blocks_.size(); ++i)
    if (!blocks_[i]) {
      blocks_[i] = p;
      return (int)i;
    }
  blocks_.push_back(p);
  return (int)blocks_.size() - 1;
}

void Engine::free_block(int b) {
  double* p = blk(b);
  PO_CUDA(cudaStreamSynchronize(s));
  PO_CUDA(cudaFree(p));
  blocks_[b] = nullptr;
}

double* Engine::blk(int b) const {
  if (b < 0 || b >= (int)blocks_.size() || !blocks_[b]) throw Error(PO_EINVAL, "invalid block handle");
  return blocks_[b];
}

void Engine::zero_block(int b) {
  PO_CUDA(cudaMemsetAsync(blk(b), 0, sizeof(double) * (size_t)N * g.ld, s));
}

DevState* Engine::new_state() {
  auto* st = new DevState;
  const size_t fb = sizeof(double) * (size_t)g.ngl;
  PO_CUDA(cudaMalloc(&st->rho, fb));
  PO_CUDA(cudaMalloc(&st->v_h, fb));
  PO_CUDA(cudaMalloc(&st->v_xc, fb));
  PO_CUDA(cudaMalloc(&st->v_local, fb));
  for (double* p : {st->rho, st->v_h, st->v_xc, st->v_local}) PO_CUDA(cudaMemsetAsync(p, 0, fb, s));
  states_.push_back(st);
  return st;
}

void Engine::free_state(DevState* st) {
  for (auto& x : states_)
    if (x == st) {
      PO_CUDA(cudaStreamSynchronize(s));
      cudaFree(st->rho);
      cudaFree(st->v_h);
      cudaFree(st->v_xc);
      cudaFree(st->v_local);
      delete st;
      x = nullptr;
    }
}

// Readback without the copy engine: one small kernel stores the scalars (and
// the Poisson status) straight into mapped pinned memory, then a sequence flag;
// the host spins on the flag (a cudaMemcpyAsync D2H + stream query costs
// 7-9 us of copy-engine latency plus the polling interval per readback).
__global__ void publish_kernel(const double* __restrict__ src, double* dst, int n,
                               const int* __restrict__ isrc, int* idst,
                               volatile unsigned long long* flag, unsigned long long seq) {
  PO_PDL_ENTRY();
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  if (threadIdx.x < 2) idst[threadIdx.x] = isrc[threadIdx.x];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    *flag = seq;
    __threadfence_system();
  }
}

void Engine::fetch(size_t off, size_t n) {
  PO_CUDA(cudaGetLastError());
  const unsigned long long seq = ++pub_seq;
  ::po::count_launch();
  launch_pdl(publish_kernel, dim3(1), dim3(256), 0, s, dvec + off, hvec_dev + off, (int)n, cg_out_i, h_cg_i_dev,
                                   hflag_dev, seq);
  PO_CUDA(cudaGetLastError());
  WaitClock wc;
  volatile unsigned long long* f = hflag;
  for (unsigned spins = 1; *f != seq; ++spins) {
    if ((spins & 1023u) == 0) {  // surface stream errors instead of spinning forever
      const cudaError_t e = cudaStreamQuery(s);
      if (e != cudaSuccess && e != cudaErrorNotReady)
        throw Error(PO_ECUDA, std::string("stream: ") + cudaGetErrorString(e));
      if (e == cudaSuccess && *f != seq) break;
    }
  }
  if (*f != seq) sync();
  std::atomic_thread_fence(std::memory_order_acquire);
}

void Engine::reduce_rows(const double* parts, int rows, int nblk, double scale, double* out,
                         bool allreduce) {
  launch_reduce_rows(parts, rows, nblk, scale, out, s);
  if (allreduce && size > 1) comm->allreduce_sum(out, (size_t)rows, s);
}

// energy.cpp:228-246
void Engine::poisson(int warm_ok) {
  if (poisson_solver == PO_POISSON_DST) {
    dst.solve(cg_b, cg_x, s);
    launch_cg(g.n0, g.n1, g.n2, g.ih2, cg_b, cg_x, 1, cg_ws, cg_bar, cg_out_i, cg_out_d, s);
  } else {
    const int warm = poisson_solver == PO_POISSON_CG_WARM && warm_ok;
    launch_cg(g.n0, g.n1, g.n2, g.ih2, cg_b, cg_x, warm, cg_ws, cg_bar, cg_out_i, cg_out_d, s);
  }
}

void Engine::build_state(const double* u, int hartree, int xc, DevState* st, int warm_ok,
                         bool density_done) {
  double* b_local = density_b_target(hartree);
  const int pn = points_nblk(g);
  static const int defer_env = getenv("PO_POISSON_DEFER") ? atoi(getenv("PO_POISSON_DEFER")) : 1;
  // a line-search trial's DST solve is checked by the v_local pass instead of the
  // CG verification kernel; a failed check (never seen: the DST solve is exact to
  // round-off) is repaired by the solver with CG (Solver::repair_poisson)
  const bool defer = defer_env && density_done && hartree && poisson_solver == PO_POISSON_DST &&
                     !force_cg_verify;
  if (!density_done) {  // else: rho and 4 pi rho came from the rotation; v_xc, E_xc, E_ext below
    launch_density_xc(g, N, u, occ, xc, st->rho, st->v_xc, b_local, v_ext, partials, s);
    launch_reduce_rows(partials, 2, pn, g.w, scal() + S_EXC, s);  // E_xc = <eps, rho>, E_ext
  }
  if (hartree) {
    if (size > 1) {
      comm->allgather(b_local, cg_b + ng_full, (size_t)max_slab_points, s);
      // compact rank slabs (uneven split) into the full grid
      const int64_t base = g.n0 / size, rem = g.n0 % size;
      int64_t z = 0;
      for (int r = 0; r < size; ++r) {
        const int64_t nz = base + (r < rem ? 1 : 0);
        PO_CUDA(cudaMemcpyAsync(cg_b + z * g.plane, cg_b + ng_full + (int64_t)r * max_slab_points,
                                sizeof(double) * nz * g.plane, cudaMemcpyDeviceToDevice, s));
        z += nz;
      }
    }
    if (defer)
      dst.solve(cg_b, cg_x, s);  // the CG-criterion check rides on the v_local pass below
    else
      poisson(warm_ok);
  } else {
    PO_CUDA(cudaMemsetAsync(cg_out_i, 0, 2 * sizeof(int), s));
  }
  st->poisson_deferred = defer;
  st->poisson_ok = true;
  // v_H slab copied out of the Poisson solution by the same pass that forms v_local
  launch_vlocal(g, v_ext, hartree ? cg_x + g.z0 * g.plane : nullptr, st->v_h, st->v_xc, st->rho,
               st->v_local, partials, s, density_done ? (xc ? 1 : 0) : -1, defer ? cg_b : nullptr,
               defer ? cg_x : nullptr, defer ? cg_out_i : nullptr);
  if (density_done) {  // E_xc = w <eps, rho>, E_ext = w <V_ext, rho>, E_H = 1/2 w <v_H, rho>
    // (+ with the deferred check: |r|^2, |b|^2 at scale w/2 in S_EH + 1, S_EH + 2)
    const double sc[3] = {g.w, g.w, 0.5 * g.w};
    launch_reduce_rows_grouped(partials, 1, 3, pn, sc, scal() + S_EXC, s, defer ? 5 : 3);
  } else {
    launch_reduce_rows(partials, 1, pn, 0.5 * g.w, scal() + S_EH, s);  // E_H = 1/2 <v_H, rho>
  }
  if (size > 1) comm->allreduce_sum(scal() + S_EXC, defer ? 5 : 3, s);  // S_EXC..S_EH (+ check)
  PO_CUDA(cudaGetLastError());
  if (!xc) PO_CUDA(cudaMemsetAsync(scal() + S_EXC, 0, sizeof(double), s));
  if (!hartree) PO_CUDA(cudaMemsetAsync(scal() + S_EH, 0, sizeof(double), s));
}

void Engine::finish_state(DevState* st) {
  fetch_all();
  state_results(st);
}

void Engine::state_results(DevState* st) {
  if (h_cg_i[0] != 0) throw Error(PO_ESOLVER, "poisson: CG did not reach the requested residual");
  st->cg_iters = h_cg_i[1];
  if (st->poisson_deferred) {  // energy.cpp:120-142 criterion, from the v_local pass's sums
    static const bool force = std::getenv("PO_FORCE_POISSON_REPAIR") != nullptr;  // test hook
    const double rr = hvec[off_scal() + S_EH + 1], bb = hvec[off_scal() + S_EH + 2];
    st->poisson_ok = !force && std::sqrt(rr) <= 1e-10 * std::sqrt(bb);
  }
  st->e_xc = hvec[off_scal() + S_EXC];
  st->e_hartree = hvec[off_scal() + S_EH];
  st->e_ext = hvec[off_scal() + S_EEXT];
}

void Engine::halo_exchange(const double* u) {
  if (size <= 1) return;
  launch_pack_plane(g, N, u, 0, send_lo, s);
  launch_pack_plane(g, N, u, g.nz - 1, send_hi, s);
  comm->halo(send_lo, send_hi, halo_lo, halo_hi, (size_t)N * g.plane, s);
}

void Engine::apply_h(const double* u, double* out, const double* v_local, bool with_ext) {
  const double* lo = (size > 1 && rank > 0) ? halo_lo : nullptr;
  const double* hi = (size > 1 && rank + 1 < size) ? halo_hi : nullptr;
  const double* ve = with_ext ? v_ext : nullptr;
  static const bool overlap = !std::getenv("PO_HALO_OVERLAP") || std::atoi(std::getenv("PO_HALO_OVERLAP"));
  int nb;
  if (size > 1 && overlap && hamiltonian_split_ok(g)) {
    // grid.cpp:109-119's axis-0 taps across ranks: the boundary planes go out on
    // the comm stream while s computes planes 1 .. nz-2 (no remote tap), then
    // planes 0 and nz-1 with the received neighbours
    launch_pack_plane(g, N, u, 0, send_lo, s);
    launch_pack_plane(g, N, u, g.nz - 1, send_hi, s);
    PO_CUDA(cudaEventRecord(ev_pack, s));
    PO_CUDA(cudaStreamWaitEvent(cs, ev_pack, 0));
    launch_hamiltonian_interior(g, N, u, v_local, ve, out, partials, s);
    comm->halo(send_lo, send_hi, halo_lo, halo_hi, (size_t)N * g.plane, cs);
    PO_CUDA(cudaEventRecord(ev_halo, cs));
    PO_CUDA(cudaStreamWaitEvent(s, ev_halo, 0));
    launch_hamiltonian_boundary(g, N, u, lo, hi, v_local, ve, out, partials, s);
    nb = hamiltonian_split_nblk(g);
  } else {
    halo_exchange(u);
    launch_hamiltonian2(g, N, u, lo, hi, v_local, ve, out, partials, s);
    nb = hamiltonian2_nblk(g);
  }
  // sigma_ii (w), kinetic (-w/2), external (w): one launch over the consecutive rows
  const double sc[3] = {g.w, -0.5 * g.w, g.w};
  launch_reduce_rows_grouped(partials, N, with_ext ? 3 : 2, nb, sc, dvec + off_sig(), s);
  if (size > 1) comm->allreduce_sum(dvec + off_sig(), (size_t)(with_ext ? 3 : 2) * N, s);
}

void Engine::gram(const double* A, const double* Ab, double sa, const double* B, const double* Bb,
                  double sb, int sym, double* Gdev, const double* guard) {
  launch_gram(g, N, A, Ab, sa, B, Bb, sb, sym, gram_ws, Gdev, s, guard);
  if (size > 1) comm->allreduce_sum(Gdev, (size_t)N * N, s);
}

bool Engine::gram_density(const double* A, double* Gdev, double* rho, double* bvec) {
  static const bool off = std::getenv("PO_NO_GRAM_DENSITY") != nullptr;  // measurement switch
  if (off || N <= 64 || N > 128 || !tma2d_available()) return false;
  if (!launch_gram_big(N, g.ld, 1, A, nullptr, 0.0, A, nullptr, 0.0, gram_ws,
                       gram_workspace_doubles(g, N), Gdev, g.w, s, nullptr, rho, bvec, occ, g.ngl))
    return false;
  if (size > 1) comm->allreduce_sum(Gdev, (size_t)N * N, s);
  return true;
}

bool Engine::gram_sigma_bb(const double* hw, const double* w, double* Gdev, GramBB* bb) {
  if (N <= 64 || !tma2d_available()) return false;
  if (!launch_gram_big(N, g.ld, 0, hw, nullptr, 0.0, w, nullptr, 0.0, gram_ws,
                       gram_workspace_doubles(g, N), Gdev, g.w, s, nullptr, nullptr, nullptr, 1.0, 0, bb))
    return false;
  if (size > 1) comm->allreduce_sum(Gdev, (size_t)N * N, s);  // (the sums' partials: reduce_rows)
  return true;
}

void Engine::mix(const double* A, const double* Ab, double sa, const double* M, double alpha,
                 const double* C, double beta, int upper, double* out, double* norm_rows,
                 const double* guard, const double* zsig) {
  const int nb = launch_mix(g, N, A, Ab, sa, M, alpha, C, beta, upper, out,
                            norm_rows ? partials : nullptr, s, guard, zsig);
  if (nb == -2) throw Error(PO_EINVAL, "mix: implicit direction unavailable on this path");
  if (norm_rows) reduce_rows(partials, N, nb, g.w, norm_rows, true);
}

}  // namespace po

// ============================================================== C ABI ====

using po::Engine;
using po::Error;

#define API_TRY try {
#define API_CATCH(h)                                   \
  }                                                    \
  catch (const po::Error& ex) {                        \
    if (h) (h)->err = ex.what();                       \
    return ex.code;                                    \
  }                                                    \
  catch (const std::exception& ex) {                   \
    if (h) (h)->err = ex.what();                       \
    return PO_EINVAL;                                  \
  }                                                    \
  return PO_OK;

#define ENGINE_OR_EINVAL(h) \
  if (!(h) || !(h)->e) return PO_EINVAL; \
  Engine& E = *(h)->e;

extern "C" {

int po_abi_version(void) { return PO_ABI_VERSION; }

long long po_launch_count(void) { return po::launch_count(); }

int po_create(const po_grid_desc* grid, int n_orbitals, double occupation,
              const po_dist_desc* dist, po_engine** out) {
  if (!out) return PO_EINVAL;
  *out = nullptr;
  auto* h = new po_engine{nullptr, {}};
  try {
    h->e = new Engine(grid, n_orbitals, occupation, dist);
  } catch (const Error& ex) {
    h->err = ex.what();
    *out = h;  // caller can read po_last_error, then po_destroy
    return ex.code;
  }
  *out = h;
  return PO_OK;
}

int po_destroy(po_engine* h) {
  if (!h) return PO_OK;
  delete h->e;
  delete h;
  return PO_OK;
}

const char* po_last_error(const po_engine* h) { return h ? h->err.c_str() : "null engine"; }

int po_slab_plan(int64_t n0, int size, int rank, int64_t* z0, int64_t* nz, int* lo_peer,
                 int* hi_peer) {
  if (size < 1 || rank < 0 || rank >= size || n0 < size) return PO_EINVAL;
  const int64_t base = n0 / size, rem = n0 % size;
  if (nz) *nz = base + (rank < rem ? 1 : 0);
  if (z0) *z0 = rank * base + (rank < rem ? rank : rem);
  if (lo_peer) *lo_peer = rank > 0 ? rank - 1 : -1;          // sends it plane z0 - 1
  if (hi_peer) *hi_peer = rank + 1 < size ? rank + 1 : -1;  // sends it plane z0 + nz
  return PO_OK;
}

int po_local_slab(const po_engine* h, int64_t* z0, int64_t* nz, int64_t* ngl) {
  if (!h || !h->e) return PO_EINVAL;
  if (z0) *z0 = h->e->g.z0;
  if (nz) *nz = h->e->g.nz;
  if (ngl) *ngl = h->e->g.ngl;
  return PO_OK;
}

int64_t po_solver_bytes(const po_grid_desc* grid, int n, int size) {
  if (!grid || n < 1 || size < 1) return -1;
  const int64_t ng = grid->n[0] * grid->n[1] * grid->n[2];
  const int64_t nzmax = (grid->n[0] + size - 1) / size;
  const int64_t ngl = nzmax * grid->n[1] * grid->n[2];
  const int64_t ld = (ngl + 31) / 32 * 32;
  const int64_t block = (int64_t)n * ld * 8;
  // W HW Z WP ZP WT HWT WT2 REC(+ shared) + scratch: ~10 blocks worst case
  const int64_t fields = 8 * ngl * 8 * 3 + 7 * ng * 8;
  return 10 * block + fields + (int64_t)n * n * 8 * 12;
}

void* po_stream(po_engine* h) { return (h && h->e) ? (void*)h->e->s : nullptr; }

int po_synchronize(po_engine* h) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  E.sync();
  API_CATCH(h)
}

int po_alloc_block(po_engine* h, int* block) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  *block = E.alloc_block();
  API_CATCH(h)
}

int po_free_block(po_engine* h, int block) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  E.free_block(block);
  API_CATCH(h)
}

int po_upload_block(po_engine* h, int block, const double* host) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  if (!host) throw Error(PO_EINVAL, "upload_block: null host buffer");
  E.upload_host(E.blk(block), host, E.s);  // pageable buffers: pinned chunk pipeline (staging.cu)
  E.sync();
  API_CATCH(h)
}

int po_download_block(po_engine* h, int block, double* host) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  if (!host) throw Error(PO_EINVAL, "download_block: null host buffer");
  E.download_host(host, E.blk(block), E.s);
  API_CATCH(h)
}

int po_copy_block(po_engine* h, int dst, int src) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  PO_CUDA(cudaMemcpyAsync(E.blk(dst), E.blk(src), sizeof(double) * E.N * E.g.ld,
                          cudaMemcpyDeviceToDevice, E.s));
  API_CATCH(h)
}

static double* field_ptr(Engine& E, int f) {
  po::DevState* st = E.default_state();
  switch (f) {
    case PO_VEXT: return E.v_ext;
    case PO_RHO: return st->rho;
    case PO_VH: return st->v_h;
    case PO_VXC: return st->v_xc;
    case PO_VLOCAL: return st->v_local;
  }
  throw Error(PO_EINVAL, "unknown field");
}

int po_set_field(po_engine* h, int field, const double* host) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  PO_CUDA(cudaMemcpyAsync(field_ptr(E, field), host, sizeof(double) * E.g.ngl,
                          cudaMemcpyHostToDevice, E.s));
  E.sync();
  API_CATCH(h)
}

int po_get_field(po_engine* h, int field, double* host) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  PO_CUDA(cudaMemcpyAsync(host, field_ptr(E, field), sizeof(double) * E.g.ngl,
                          cudaMemcpyDeviceToHost, E.s));
  E.sync();
  API_CATCH(h)
}

static int set_potential(po_engine* h, const double* atoms, int n, int gaussian) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  if (n < 0 || (n > 0 && !atoms)) throw Error(PO_EINVAL, "invalid atom list");
  for (int a = 0; a < n && !gaussian; ++a) {
    const double* q = atoms + 5 * a;
    if (!(q[3] > 0.0)) throw Error(PO_EINVAL, "make_problem: atom charge must be positive");
    if (!(q[4] > 0.0)) throw Error(PO_EINVAL, "make_problem: atom softening must be positive");
    for (int d = 0; d < 3; ++d)
      if (!(q[d] >= 0.0) || !(q[d] <= E.ext[d]))
        throw Error(PO_EINVAL, "make_problem: atom position outside the grid box");
  }
  double* d = nullptr;
  if (n > 0) {
    PO_CUDA(cudaMalloc(&d, sizeof(double) * 5 * n));
    PO_CUDA(cudaMemcpyAsync(d, atoms, sizeof(double) * 5 * n, cudaMemcpyHostToDevice, E.s));
  }
  po::launch_external_potential(E.g, E.h, d, n, gaussian, E.v_ext, E.s);
  E.sync();
  if (d) cudaFree(d);
  API_CATCH(h)
}

int po_external_potential(po_engine* h, const double* atoms, int natoms) {
  return set_potential(h, atoms, natoms, 0);
}

int po_gaussian_potential(po_engine* h, const double* wells, int nwells) {
  return set_potential(h, wells, nwells, 1);
}

int po_random_block(po_engine* h, int block, uint64_t seed) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  // The reference draws orbital-major over the whole grid (tests/problems.hpp:59-68);
  // this rank keeps the values of its slab.
  std::vector<double> host((size_t)E.N * E.g.ngl);
  po::rng_normals_slab(seed, E.N, E.ng_full, E.g.z0 * E.g.plane, E.g.ngl, host.data());
  PO_CUDA(cudaMemcpy2DAsync(E.blk(block), E.g.ld * 8, host.data(), E.g.ngl * 8, E.g.ngl * 8, E.N,
                            cudaMemcpyHostToDevice, E.s));
  E.sync();
  API_CATCH(h)
}

int po_fill_normal(po_engine* h, int block, uint64_t seed) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  po::launch_fill_normal(E.g, E.N, E.ng_full, seed, E.blk(block), E.s);
  E.sync();
  API_CATCH(h)
}

// optimizer.cpp:156-197: Gaussians at the atoms (cycled; the box centre without
// atoms), widths and 1e-2 uniform noise from Rng(seed + attempt), orthonormalised
// (manifold.cpp:171), retried with the next derived seed on a rank-deficient set.
int po_initialize_orbitals(po_engine* h, const double* atoms, int natoms, uint64_t seed, int w) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  if (natoms < 0 || (natoms > 0 && !atoms)) throw Error(PO_EINVAL, "invalid atom list");
  if ((int64_t)E.N > E.ng_full)
    throw Error(PO_EINVAL, "initialize_orbitals: more orbitals than grid points");
  std::vector<double> centers(3 * (size_t)E.N);
  for (int i = 0; i < E.N; ++i)
    for (int d = 0; d < 3; ++d)
      centers[3 * i + d] = natoms > 0 ? atoms[5 * (i % natoms) + d] : 0.5 * E.ext[d];
  double* dc = nullptr;
  double* dw = nullptr;
  PO_CUDA(cudaMalloc(&dc, sizeof(double) * 3 * E.N));
  PO_CUDA(cudaMalloc(&dw, sizeof(double) * E.N));
  PO_CUDA(cudaMemcpy(dc, centers.data(), sizeof(double) * 3 * E.N, cudaMemcpyHostToDevice));
  std::vector<double> widths(E.N);
  std::vector<double> noise((size_t)E.N * E.g.ngl);
  const int raw = E.alloc_block();
  bool done = false;
  try {
    for (int attempt = 0; attempt < 5 && !done; ++attempt) {
      po::rng_init_noise_slab(seed + (uint64_t)attempt, E.N, E.ng_full, E.g.z0 * E.g.plane,
                              E.g.ngl, widths.data(), noise.data());
      PO_CUDA(cudaMemcpyAsync(dw, widths.data(), sizeof(double) * E.N, cudaMemcpyHostToDevice,
                              E.s));
      PO_CUDA(cudaMemcpy2DAsync(E.blk(raw), E.g.ld * 8, noise.data(), E.g.ngl * 8, E.g.ngl * 8,
                                E.N, cudaMemcpyHostToDevice, E.s));
      po::launch_init_orbitals(E.g, E.N, E.h, dc, dw, E.blk(raw), E.s);
      E.sync();
      const int rc = po_orthonormalize(h, raw, w, 1, nullptr, nullptr, nullptr);
      if (rc == PO_OK) done = true;
      else if (rc != PO_EDEGENERATE) throw Error(rc, h->err);
    }
  } catch (...) {
    E.free_block(raw);
    cudaFree(dc);
    cudaFree(dw);
    throw;
  }
  E.free_block(raw);
  cudaFree(dc);
  cudaFree(dw);
  if (!done) throw Error(PO_EDEGENERATE, "initialize_orbitals: no full-rank start in 5 attempts");
  API_CATCH(h)
}

// grid.cpp:137-149
int po_refine_grid(const po_grid_desc* g, po_grid_desc* fine) {
  if (!g || !fine) return PO_EINVAL;
  for (int a = 0; a < 3; ++a) {
    if (g->n[a] < 1 || g->n[a] > (INT64_MAX - 1) / 2) return PO_EINVAL;
    fine->n[a] = 2 * g->n[a] + 1;
    fine->extent[a] = g->extent[a];
  }
  return PO_OK;
}

// grid.cpp:151-203 on every orbital of a block (single-rank engines)
int po_prolongate(po_engine* coarse, int cblock, po_engine* fine, int fblock) {
  if (!coarse || !coarse->e || !fine || !fine->e) return PO_EINVAL;
  Engine& C = *coarse->e;
  Engine& F = *fine->e;
  try {
    if (C.size != 1 || F.size != 1)
      throw Error(PO_EINVAL, "prolongate: sharded engines are not supported");
    if (C.N != F.N) throw Error(PO_EINVAL, "prolongate: orbital counts differ");
    const int64_t nc[3] = {C.g.n0, C.g.n1, C.g.n2}, nf[3] = {F.g.n0, F.g.n1, F.g.n2};
    for (int a = 0; a < 3; ++a)
      if (nf[a] != 2 * nc[a] + 1 || F.ext[a] != C.ext[a])
        throw Error(PO_EINVAL, "prolongate: grids are not in refinement relation");
    C.sync();
    po::launch_prolongate(C.N, nc, C.g.ld, C.blk(cblock), nf, F.g.ld, F.blk(fblock), F.s);
    F.sync();
  } catch (const Error& ex) {
    fine->err = ex.what();
    return ex.code;
  }
  return PO_OK;
}

int po_build_hamiltonian(po_engine* h, int u, int hartree, int xc, double* e_hartree,
                         double* e_xc, int* cg_iters) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  po::DevState* st = E.default_state();
  E.build_state(E.blk(u), hartree, xc, st, 0);
  E.finish_state(st);
  if (e_hartree) *e_hartree = st->e_hartree;
  if (e_xc) *e_xc = st->e_xc;
  if (cg_iters) *cg_iters = st->cg_iters;
  API_CATCH(h)
}

int po_apply_hamiltonian(po_engine* h, int u, int out, double* sigma, double* kin, double* ext) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  E.apply_h(E.blk(u), out >= 0 ? E.blk(out) : nullptr, E.default_state()->v_local);
  E.fetch(0, (size_t)3 * E.N);
  if (sigma) std::memcpy(sigma, E.hvec + E.off_sig(), sizeof(double) * E.N);
  if (kin) std::memcpy(kin, E.hvec + E.off_kin(), sizeof(double) * E.N);
  if (ext) std::memcpy(ext, E.hvec + E.off_ext(), sizeof(double) * E.N);
  API_CATCH(h)
}

int po_total_energy(po_engine* h, int u, int hartree, int xc, double* out5) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  po::DevState* st = E.default_state();
  E.apply_h(E.blk(u), nullptr, st->v_local);
  E.fetch(0, (size_t)3 * E.N);
  double kin = 0.0, ext = 0.0;
  for (int i = 0; i < E.N; ++i) kin += E.occ * E.hvec[E.off_kin() + i];
  for (int i = 0; i < E.N; ++i) ext += E.occ * E.hvec[E.off_ext() + i];
  out5[0] = kin;
  out5[1] = ext;
  out5[2] = hartree ? st->e_hartree : 0.0;
  out5[3] = xc ? st->e_xc : 0.0;
  out5[4] = out5[0] + out5[1] + out5[2] + out5[3];
  API_CATCH(h)
}

int po_laplacian(po_engine* h, int u, int out) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  E.halo_exchange(E.blk(u));
  const double* lo = (E.size > 1 && E.rank > 0) ? E.halo_lo : nullptr;
  const double* hi = (E.size > 1 && E.rank + 1 < E.size) ? E.halo_hi : nullptr;
  po::launch_laplacian(E.g, E.N, E.blk(u), lo, hi, E.blk(out), E.s);
  E.sync();
  API_CATCH(h)
}

static void fetch_matrix(Engine& E, const double* dm, double* host) {
  PO_CUDA(cudaMemcpyAsync(E.hmat, dm, sizeof(double) * E.N * E.N, cudaMemcpyDeviceToHost, E.s));
  E.sync();
  std::memcpy(host, E.hmat, sizeof(double) * E.N * E.N);
}

static void put_matrix(Engine& E, const double* host, double* dm) {
  std::memcpy(E.hmat, host, sizeof(double) * E.N * E.N);
  PO_CUDA(cudaMemcpyAsync(dm, E.hmat, sizeof(double) * E.N * E.N, cudaMemcpyHostToDevice, E.s));
  E.sync();
}

int po_gram(po_engine* h, int a, int b, double* g_host) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  E.gram(E.blk(a), nullptr, 0.0, E.blk(b), nullptr, 0.0, a == b, E.dmat[6]);
  fetch_matrix(E, E.dmat[6], g_host);
  API_CATCH(h)
}

int po_mix(po_engine* h, int in, const double* m_host, int out) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  if (in == out) throw Error(PO_EINVAL, "mix: in and out must differ");
  put_matrix(E, m_host, E.dmat[6]);
  E.mix(E.blk(in), nullptr, 0.0, E.dmat[6], 1.0, nullptr, 0.0, 0, E.blk(out), nullptr);
  E.sync();
  API_CATCH(h)
}

int po_linear_combination(po_engine* h, int a, double sc, int b, int out) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  po::launch_lincomb(E.g, E.N, E.blk(a), sc, E.blk(b), E.blk(out), E.s);
  E.sync();
  API_CATCH(h)
}

int po_bb_products(po_engine* h, int w, int wp, int z, int zp, double* ss, double* sy,
                   double* yy) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  const int nb = po::per_orbital_nblk(E.g, E.N);
  po::launch_bb(E.g, E.N, E.blk(w), E.blk(wp), E.blk(z), E.blk(zp), E.partials, E.s);
  E.reduce_rows(E.partials, 3 * E.N, nb, E.g.w, E.dvec + E.off_ss(), true);
  E.fetch(E.off_ss(), (size_t)3 * E.N);
  if (ss) std::memcpy(ss, E.hvec + E.off_ss(), sizeof(double) * E.N);
  if (sy) std::memcpy(sy, E.hvec + E.off_sy(), sizeof(double) * E.N);
  if (yy) std::memcpy(yy, E.hvec + E.off_yy(), sizeof(double) * E.N);
  API_CATCH(h)
}

int po_direction_sums(po_engine* h, int u, int hu, int u_prev, int hu_prev, const double* sigma_prev,
                      double* sigma_diag, double* sigma_full, double* zz, double* ss, double* sy,
                      double* yy) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  const bool hist = u_prev >= 0 && hu_prev >= 0;
  if (hist && !sigma_prev) throw Error(PO_EINVAL, "direction_sums: a history needs sigma_prev");
  const int onb = po::per_orbital_nblk(E.g, E.N);
  // sigma_ii = <hu_i, u_i> (the s*y product of the BB kernel with zero "previous" blocks)
  po::launch_bb(E.g, E.N, E.blk(hu), nullptr, E.blk(u), nullptr, E.partials, E.s);
  E.reduce_rows(E.partials + (size_t)E.N * onb, E.N, onb, E.g.w, E.dvec + E.off_sig(), true);
  double* sp = E.dvec + E.off_zsig(0);
  if (hist) {
    std::memcpy(E.hmat, sigma_prev, sizeof(double) * E.N);
    PO_CUDA(cudaMemcpyAsync(sp, E.hmat, sizeof(double) * E.N, cudaMemcpyHostToDevice, E.s));
  }
  po::GramBB gb{E.dvec + E.off_sig(), hist ? sp : nullptr, hist ? E.blk(u_prev) : nullptr,
                hist ? E.blk(hu_prev) : nullptr, E.partials, 0};
  int nb;
  if (E.gram_sigma_bb(E.blk(hu), E.blk(u), E.dmat[4], &gb)) {
    nb = gb.nsplit;
  } else {
    E.gram(E.blk(hu), nullptr, 0.0, E.blk(u), nullptr, 0.0, 0, E.dmat[4]);
    nb = po::launch_residual_bb_stream(E.g, E.N, E.blk(u), E.blk(hu), E.dvec + E.off_sig(),
                                       hist ? E.blk(u_prev) : nullptr, hist ? E.blk(hu_prev) : nullptr,
                                       hist ? sp : nullptr, nullptr, E.partials, E.s);
  }
  E.reduce_rows(E.partials, E.N, nb, E.g.w, E.dvec + E.off_zz(), true);
  if (hist) E.reduce_rows(E.partials + (size_t)E.N * nb, 3 * E.N, nb, E.g.w, E.dvec + E.off_ss(), true);
  E.fetch_all();
  if (sigma_full) fetch_matrix(E, E.dmat[4], sigma_full);
  if (sigma_diag) std::memcpy(sigma_diag, E.hvec + E.off_sig(), sizeof(double) * E.N);
  if (zz) std::memcpy(zz, E.hvec + E.off_zz(), sizeof(double) * E.N);
  if (hist) {
    if (ss) std::memcpy(ss, E.hvec + E.off_ss(), sizeof(double) * E.N);
    if (sy) std::memcpy(sy, E.hvec + E.off_sy(), sizeof(double) * E.N);
    if (yy) std::memcpy(yy, E.hvec + E.off_yy(), sizeof(double) * E.N);
  }
  API_CATCH(h)
}

int po_diagonal_residuals(po_engine* h, int u, int hu, int z, double* sigma, double* znorm2) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  const int nb = po::per_orbital_nblk(E.g, E.N);
  // sigma_ii = <hu_i, u_i>: the s*y product of the BB kernel with zero "previous" blocks
  po::launch_bb(E.g, E.N, E.blk(hu), nullptr, E.blk(u), nullptr, E.partials, E.s);
  E.reduce_rows(E.partials + (size_t)E.N * nb, E.N, nb, E.g.w, E.dvec + E.off_sig(), true);
  po::launch_residual_diag(E.g, E.N, E.blk(u), E.blk(hu), E.dvec + E.off_sig(), E.blk(z),
                           E.partials, E.s);
  E.reduce_rows(E.partials, E.N, nb, E.g.w, E.dvec + E.off_zz(), true);
  E.fetch(0, E.off_dd());
  if (sigma) std::memcpy(sigma, E.hvec + E.off_sig(), sizeof(double) * E.N);
  if (znorm2) std::memcpy(znorm2, E.hvec + E.off_zz(), sizeof(double) * E.N);
  API_CATCH(h)
}

int po_stiefel_gradient(po_engine* h, int u, int hu, double* sigma_host, double* dnorm2) {
  return po_stiefel_gradient_d(h, u, hu, -1, sigma_host, dnorm2);
}

int po_stiefel_gradient_d(po_engine* h, int u, int hu, int d, double* sigma_host, double* dnorm2) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  if (d >= 0 && (d == u || d == hu)) throw Error(PO_EINVAL, "stiefel_gradient: D must not alias U or HU");
  double* dout = d >= 0 ? E.blk(d) : nullptr;
  E.gram(E.blk(hu), nullptr, 0.0, E.blk(u), nullptr, 0.0, 0, E.dmat[4]);
  po::launch_matrix_stats(E.N, E.dmat[4], E.scal() + Engine::S_SYM, E.s);
  E.mix(E.blk(u), nullptr, 0.0, E.dmat[4], -1.0, E.blk(hu), 1.0, 0, dout, E.dvec + E.off_dd());
  E.fetch_all();
  if (sigma_host) fetch_matrix(E, E.dmat[4], sigma_host);
  if (dnorm2) std::memcpy(dnorm2, E.hvec + E.off_dd(), sizeof(double) * E.N);
  if (E.hvec[E.off_scal() + Engine::S_SYM + 1] > 1e-10)
    throw Error(PO_EINVAL, "stiefel_gradient: <(HU)^T U> is not symmetric; inconsistent H or U");
  API_CATCH(h)
}

int po_subspace_rotate(po_engine* h, int w, const double* sigma_host, double* gamma,
                       double* p_host) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  put_matrix(E, sigma_host, E.dmat[4]);
  po::launch_syev(E.N, E.dmat[4], E.syev_work, E.dmat[6], E.dmat[5], 1, E.scal() + Engine::S_EIG,
                  E.s);
  E.fetch(E.off_scal(), 64);
  if (E.hvec[E.off_scal() + Engine::S_EIG] > 1e-8)
    throw Error(PO_EINVAL, "subspace_rotate: Sigma asymmetry exceeds tolerance");
  int tmp = E.alloc_block();
  E.mix(E.blk(w), nullptr, 0.0, E.dmat[5], 1.0, nullptr, 0.0, 0, E.blk(tmp), nullptr);
  PO_CUDA(cudaMemcpyAsync(E.blk(w), E.blk(tmp), sizeof(double) * E.N * E.g.ld,
                          cudaMemcpyDeviceToDevice, E.s));
  E.free_block(tmp);
  if (gamma) {
    PO_CUDA(cudaMemcpyAsync(E.hmat, E.dmat[6], sizeof(double) * E.N, cudaMemcpyDeviceToHost, E.s));
    E.sync();
    std::memcpy(gamma, E.hmat, sizeof(double) * E.N);
  }
  if (p_host) fetch_matrix(E, E.dmat[5], p_host);
  E.sync();
  API_CATCH(h)
}

}  // extern "C"

extern "C" int po_set_matrix(po_engine* h, const double* m_host) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  put_matrix(E, m_host, E.dmat[1]);
  API_CATCH(h)
}

extern "C" int po_enqueue(po_engine* h, int op, int a, int b, int out) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  po::DevState* st = E.default_state();
  switch (op) {
    case PO_OP_HAMILTONIAN:
      po::launch_hamiltonian2(E.g, E.N, E.blk(a), nullptr, nullptr, st->v_local, nullptr,
                              out >= 0 ? E.blk(out) : nullptr, E.partials, E.s);
      break;
    case PO_OP_GRAM_SYM:
      po::launch_gram(E.g, E.N, E.blk(a), nullptr, 0.0, E.blk(a), nullptr, 0.0, 1, E.gram_ws,
                      E.dmat[0], E.s);
      break;
    case PO_OP_GRAM:
      po::launch_gram(E.g, E.N, E.blk(a), nullptr, 0.0, E.blk(b), nullptr, 0.0, 0, E.gram_ws,
                      E.dmat[0], E.s);
      break;
    case PO_OP_MIX:
    case PO_OP_MIX_UPPER:
      po::launch_mix(E.g, E.N, E.blk(a), nullptr, 0.0, E.dmat[1], 1.0, nullptr, 0.0,
                     op == PO_OP_MIX_UPPER, E.blk(out), nullptr, E.s);
      break;
    case PO_OP_DENSITY_XC:
      po::launch_density_xc(E.g, E.N, E.blk(a), E.occ, 1, st->rho, st->v_xc,
                            E.cg_b + E.g.z0 * E.g.plane, E.v_ext, E.partials, E.s);
      break;
    case PO_OP_POISSON:
      E.poisson(0);
      break;
    case PO_OP_CHOLESKY:
      po::launch_cholesky_inv(E.N, E.dmat[0], E.chol_L, E.dmat[1], E.scal() + Engine::S_CHOL, E.s);
      break;
    case PO_OP_LAPLACIAN:
      po::launch_laplacian(E.g, E.N, E.blk(a), nullptr, nullptr, E.blk(out), E.s);
      break;
    case PO_OP_GRAM_TRIAL:
      po::launch_gram(E.g, E.N, E.blk(a), E.blk(b), -0.3, E.blk(a), E.blk(b), -0.3, 1, E.gram_ws,
                      E.dmat[0], E.s);
      break;
    case PO_OP_ROTATION:
      po::launch_mix(E.g, E.N, E.blk(a), E.blk(b), -0.3, E.dmat[1], 1.0, nullptr, 0.0, 1,
                     E.blk(out), nullptr, E.s);
      break;
    case PO_OP_ROTATION_FUSED:
      // the iteration's form: b is HW and z = HW - sigma W is implicit (sigma row:
      // dvec), rho and 4 pi rho only (v_xc and the energies belong to v_local)
      if (po::launch_rotate_fused(E.N, E.g.ld, E.g.ngl, E.blk(a), E.blk(b), -0.3, E.dmat[1],
                                  E.blk(out), E.gram_ws, E.dmat[2], E.g.w, E.occ, -1, st->rho,
                                  st->v_xc, E.density_b_target(1), E.v_ext, E.partials, E.s,
                                  nullptr, E.dvec + E.off_sig()) < 0)
        throw Error(PO_EINVAL, "fused rotation unavailable for this N");
      break;
    case PO_OP_DIRECTIONS:
      // the iteration's form: z implicit (not stored), previous z from the previous
      // HW (here b again) and sigma row; out is not written
      (void)out;
      if ((E.N > 64 ? po::launch_directions_big(E.N, E.g.ld, E.g.ngl, E.blk(a), E.blk(b), E.blk(a),
                                                E.blk(b), E.dvec, E.dmat[0], E.dvec, nullptr,
                                                E.dvec + E.off_zsig(0), E.partials, E.s)
                    : po::launch_directions(E.N, E.g.ld, E.g.ngl, E.blk(a), E.blk(b), E.blk(a),
                                            E.blk(b), E.dmat[0], E.dvec, nullptr, E.partials, E.s,
                                            E.dvec, E.dvec + E.off_zsig(0))) < 0)
        throw Error(PO_EINVAL, "directions kernel unavailable for this N");
      break;
    case PO_OP_GRAM_SIGMA_BB: {
      // the iteration's Sigma Gram (a = HW, b = W) carrying ||z||^2 and the BB
      // products (history: the same blocks, previous z implicit); N > 64
      po::GramBB gb{E.dvec + E.off_sig(), E.dvec + E.off_sig(), E.blk(b), E.blk(a), E.partials, 0};
      if (!E.gram_sigma_bb(E.blk(a), E.blk(b), E.dmat[0], &gb))
        throw Error(PO_EINVAL, "Sigma Gram with fused directions unavailable for this N");
      E.reduce_rows(E.partials, E.N, gb.nsplit, E.g.w, E.dvec + E.off_zz(), true);
      E.reduce_rows(E.partials + (size_t)E.N * gb.nsplit, 3 * E.N, gb.nsplit, E.g.w, E.dvec + E.off_ss(), true);
      break;
    }
    case PO_OP_GRAM_DENSITY:
      // the trial's verification Gram that also writes rho and 4 pi rho (64 < N <= 128)
      if (!E.gram_density(E.blk(a), E.dmat[0], st->rho, E.density_b_target(1)))
        throw Error(PO_EINVAL, "Gram with fused density unavailable for this N");
      break;
    case PO_OP_ROTATION_IMPLICIT:
      // the large-N trial rotation: b is HW, z = HW - sigma W rebuilt per element
      if (po::launch_mix(E.g, E.N, E.blk(a), E.blk(b), -0.3, E.dmat[1], 1.0, nullptr, 0.0, 1,
                         E.blk(out), nullptr, E.s, nullptr, E.dvec + E.off_sig()) < 0)
        throw Error(PO_EINVAL, "implicit rotation unavailable for this N");
      break;
    default:
#ifdef PO_MEASUREMENT_VARIANTS  // make VARIANTS=1: the H u design-space probes (tools/hu_*.py)
      if (op >= PO_OP_HAMILTONIAN_VARIANT &&
          po::launch_hamiltonian_variant(op - PO_OP_HAMILTONIAN_VARIANT, E.g, E.N, E.blk(a),
                                         st->v_local, E.v_ext, out >= 0 ? E.blk(out) : nullptr,
                                         E.partials, E.s) == 0)
        break;
#endif
      throw Error(PO_EINVAL, "unknown op");
  }
  PO_CUDA(cudaGetLastError());
  API_CATCH(h)
}

extern "C" int po_set_poisson_solver(po_engine* h, int mode) {
  ENGINE_OR_EINVAL(h);
  if (mode < PO_POISSON_CG || mode > PO_POISSON_DST) return PO_EINVAL;
  E.poisson_solver = mode;
  return PO_OK;
}

extern "C" int po_nccl_unique_id(void* out128) {
  if (!out128) return PO_EINVAL;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return PO_ENCCL;
  auto fn = (int (*)(void*))dlsym(lib, "ncclGetUniqueId");
  if (!fn) return PO_ENCCL;
  return fn(out128) == 0 ? PO_OK : PO_ENCCL;
}

// Gram of the fused trial point (a + s b), symmetric path — the line-search
// Gram of optimizer.cpp:459-463 + manifold.cpp:138 without materialising the
// trial block. Exposed for parity tests of the fused load.
extern "C" int po_gram_lincomb(po_engine* h, int a, double sc, int b, double* g_host) {
  ENGINE_OR_EINVAL(h);
  API_TRY
  E.gram(E.blk(a), E.blk(b), sc, E.blk(a), E.blk(b), sc, 1, E.dmat[6]);
  fetch_matrix(E, E.dmat[6], g_host);
  API_CATCH(h)
}
