// po_engine: device-resident state of one rank (one GPU) and the host-side
// orchestration of the hot-path kernels. Internal C++ API used by the C ABI
// (engine.cu) and the InnerLoop mirror (solver.cu).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/parorb_gpu.h"
#include "kernels.h"

namespace po {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PO_CUDA(x)                                                                      \
  do {                                                                                  \
    cudaError_t _e = (x);                                                               \
    if (_e != cudaSuccess)                                                              \
      throw ::po::Error(PO_ECUDA, std::string(#x ": ") + cudaGetErrorString(_e));      \
  } while (0)

// Collectives between the ranks of one job (slab decomposition).
struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  // in-place sum over ranks of n doubles on the device; identical result on all ranks
  virtual void allreduce_sum(double* d, size_t n, cudaStream_t s) = 0;
  // recv[r * n + k] = send_r[k]
  virtual void allgather(const double* send, double* recv, size_t n, cudaStream_t s) = 0;
  // exchange one plane block with the axis-0 neighbours: send_lo -> rank-1's recv_hi,
  // send_hi -> rank+1's recv_lo (n doubles each)
  virtual void halo(const double* send_lo, const double* send_hi, double* recv_lo,
                    double* recv_hi, size_t n, cudaStream_t s) = 0;
};
std::unique_ptr<Comm> make_comm(const po_dist_desc* d);

// A built Hamiltonian state (HamiltonianState, energy.hpp:41-50) on the device.
struct DevState {
  double* rho = nullptr;
  double* v_h = nullptr;   // local slab
  double* v_xc = nullptr;
  double* v_local = nullptr;
  double* vh_full = nullptr;  // full-grid v_H (warm start / replicated solve)
  double e_hartree = 0.0, e_xc = 0.0;
  double e_ext = 0.0;  // w <V_ext, rho> (= sum_i f <V_ext u_i, u_i>)
  int cg_iters = 0;
  // DST solve whose CG-criterion check (||b - A x|| <= 1e-10 ||b||, energy.cpp:120-142)
  // rode on the v_local pass; poisson_ok is known after the readback (state_results)
  bool poisson_deferred = false, poisson_ok = true;
};

struct EnergyParts {  // EnergyBreakdown, energy.hpp:52-58
  double kinetic = 0, external = 0, hartree = 0, xc = 0, total = 0;
};

class Engine {
 public:
  Engine(const po_grid_desc* grid, int n, double occupation, const po_dist_desc* dist);
  ~Engine();

  SlabGeom g;
  int N;
  double occ;
  double h[3], ext[3];
  int rank = 0, size = 1;
  cudaStream_t s = nullptr;
  // size > 1: the halo exchange runs on cs while s computes the interior planes
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
  std::unique_ptr<Comm> comm;
  std::string err;

  // ---- blocks (handles)
  int alloc_block();
  void free_block(int b);
  // solver scratch kept across solves (no cudaMalloc in a warm po_solve)
  int take_block() {
    if (spare_blocks_.empty()) return alloc_block();
    const int b = spare_blocks_.back();
    spare_blocks_.pop_back();
    return b;
  }
  void give_block(int b) { spare_blocks_.push_back(b); }
  double* blk(int b) const;
  void zero_block(int b);

  // ---- states
  DevState* new_state();
  void free_state(DevState* st);
  DevState* take_state() {
    if (spare_states_.empty()) return new_state();
    DevState* st = spare_states_.back();
    spare_states_.pop_back();
    return st;
  }
  void give_state(DevState* st) { spare_states_.push_back(st); }
  DevState* default_state() { return def_state_; }
  double* v_ext = nullptr;

  // ---- operators (device-side results land in dvec_ regions; see *_result)
  // density -> Poisson -> xc -> v_local; returns after queueing; results via sync_state
  void build_state(const double* u, int hartree, int xc, DevState* st, int warm_ok,
                   bool density_done = false);
  // where build_state puts 4 pi rho for the Poisson solve (null without Hartree)
  double* density_b_target(int hartree) {
    if (!hartree) return nullptr;
    return size > 1 ? cg_b + ng_full + (int64_t)size * max_slab_points : cg_b + g.z0 * g.plane;
  }
  void poisson(int warm_ok);  // cg_b -> cg_x with the selected solver
  // CG outcome + E_H / E_xc of the last build (synchronises)
  void finish_state(DevState* st);
  // H u with fused reductions (sigma, kin, ext), scaled, into dvec rows
  // with_ext: also per-orbital <V_ext u_i, u_i> (else E_ext comes from the state)
  void apply_h(const double* u, double* out, const double* v_local, bool with_ext = true);
  void halo_exchange(const double* u);
  void gram(const double* A, const double* Ab, double sa, const double* B, const double* Bb,
            double sb, int sym, double* Gdev, const double* guard = nullptr);
  // symmetric Gram of A that also writes A's density rho (+ 4 pi rho into bvec);
  // false (nothing enqueued) where the fused form is unavailable
  bool gram_density(const double* A, double* Gdev, double* rho, double* bvec);
  // Sigma = w (HW)^T W with the elementwise half of compute_directions fused
  // (N > 64; all-reduced over the ranks); false if unavailable (nothing launched)
  bool gram_sigma_bb(const double* hw, const double* w, double* Gdev, GramBB* bb);
  void mix(const double* A, const double* Ab, double sa, const double* M, double alpha,
           const double* C, double beta, int upper, double* out, double* norm_rows,
           const double* guard = nullptr, const double* zsig = nullptr);
  // CG outcome + E_H / E_xc / E_ext of the last build from the last fetch (no sync)
  void state_results(DevState* st);
  void reduce_rows(const double* partials, int rows, int nblk, double scale, double* out,
                   bool allreduce);

  // device scratch
  double* partials = nullptr;
  size_t partials_cap = 0;
  double* gram_ws = nullptr;
  double* dvec = nullptr;      // small device vector scratch (kDvec doubles)
  double* hvec = nullptr;      // pinned, device-mapped mirror of dvec
  double* hvec_dev = nullptr;  // its device alias (written by the publish kernel)
  unsigned long long* hflag = nullptr;      // mapped: sequence number of the last publish
  unsigned long long* hflag_dev = nullptr;
  int* h_cg_i_dev = nullptr;
  unsigned long long pub_seq = 0;
  double* dmat[10] = {};       // N x N device matrices ([7] G_HH, [8] G_WW of the iterate)
  double* hmat = nullptr;      // pinned N x N host
  // host <-> device block transfers (staging.cu): pinned buffers go straight to
  // the copy engine, pageable ones through two pinned chunks filled / drained by
  // several host threads while the other chunk is in flight
  static constexpr size_t kStageBytes = size_t(32) << 20;
  double* stage_h[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  void ensure_staging();
  void free_staging();
  int host_threads() const;
  void upload_host(double* dev, const double* host, cudaStream_t st);    // async for pinned
  void download_host(double* host, const double* dev, cudaStream_t st);  // returns when complete
  double* chol_L = nullptr;    // N x N scratch
  double* syev_work = nullptr;
  double* halo_lo = nullptr;   // recv planes (N x plane) or null
  double* halo_hi = nullptr;
  double* send_lo = nullptr;
  double* send_hi = nullptr;
  // Poisson (full grid, replicated across ranks)
  double* cg_b = nullptr;
  double* cg_x = nullptr;
  double* cg_ws = nullptr;
  unsigned* cg_bar = nullptr;
  int* cg_out_i = nullptr;     // device {status, iters}
  double* cg_out_d = nullptr;  // device {bnorm, relres}
  int* h_cg_i = nullptr;       // pinned
  double* h_cg_d = nullptr;
  int64_t ng_full = 0;
  DstPoisson dst;
  int poisson_solver = PO_POISSON_DST;
  int64_t max_slab_points = 0;

  // dvec layout (offsets in doubles); N-length rows
  size_t off_sig() const { return 0; }
  size_t off_kin() const { return (size_t)N; }
  size_t off_ext() const { return 2 * (size_t)N; }
  size_t off_zz() const { return 3 * (size_t)N; }
  size_t off_dd() const { return 4 * (size_t)N; }
  size_t off_ss() const { return 5 * (size_t)N; }
  size_t off_sy() const { return 6 * (size_t)N; }
  size_t off_yy() const { return 7 * (size_t)N; }
  size_t off_abs() const { return 8 * (size_t)N; }
  size_t off_scal() const { return 9 * (size_t)N; }  // 64 scalars
  // two sigma rows an implicit direction z = HW - sigma W was built from (solver)
  size_t off_zsig(int k) const { return 9 * (size_t)N + 64 + (size_t)k * N; }
  size_t dvec_len() const { return 11 * (size_t)N + 64; }
  // scalar slots
  enum { S_EXC = 0, S_EEXT = 1, S_EH = 2, S_CHOL = 8, S_EIG = 12, S_INVS = 16, S_MSTAT = 20,
         S_MSTAT2 = 24, S_SYM = 28, S_QR2 = 32, S_CHOL2 = 36,
         S_TAU = 40 /* [0] tau_raw, [1] -tau_raw (trial scale), [2] znorm2 */ };
  double* scal() { return dvec + off_scal(); }
  // copy n doubles of dvec starting at off into hvec (same offsets) and synchronise
  bool force_cg_verify = false;  // build_state: run the CG verification kernel (no deferral)
  void fetch(size_t off, size_t n);
  void fetch_all() { fetch(0, dvec_len()); }
  void sync();

 private:
  std::vector<double*> blocks_;
  std::vector<DevState*> states_;
  DevState* def_state_ = nullptr;
  std::vector<int> spare_blocks_;
  std::vector<DevState*> spare_states_;
};

}  // namespace po

namespace po {
// wall seconds the calling thread has spent blocked on device work (Engine::sync /
// Engine::fetch): the par_seconds bucket of the PhaseTimer mirror (solver.cu)
double host_wait_seconds();
}  // namespace po

struct po_engine {
  po::Engine* e;
  std::string err;
};
