// Host <-> device block transfers for the drop-in's host-buffer entry points
// (po_solve_host, po_upload_block / po_download_block).
//
// The reference's callers hold orbitals in pageable std::vector memory
// (Field.values, grid.hpp:48-51). A plain cudaMemcpy from pageable memory is
// staged by the driver through a small bounce buffer, one chunk at a time with
// a single CPU thread. Pinned (page-locked / cudaHostRegister'ed) buffers go
// straight to the copy engine. For pageable buffers the engine keeps two
// pinned staging chunks and pipelines them: while the copy engine moves chunk
// k, several host threads fill (or drain) chunk k + 1, so PCIe and the host
// memcpy overlap. The block layout on the device is pitched (ld), on the host
// dense (ngl): pieces never cross an orbital row.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "engine.h"

namespace po {

namespace {

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice ||
         a.type == cudaMemoryTypeManaged;
}

// dst[0:n) = src[0:n) with up to `threads` host threads
void parallel_copy(void* dst, const void* src, size_t bytes, int threads) {
  const size_t min_slice = size_t(2) << 20;
  int t = (int)std::min<size_t>((size_t)threads, std::max<size_t>(1, bytes / min_slice));
  if (t <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> pool;
  const size_t slice = (bytes / (size_t)t + 63) & ~size_t(63);
  for (int k = 0; k < t; ++k) {
    const size_t a = (size_t)k * slice;
    if (a >= bytes) break;
    const size_t n = std::min(slice, bytes - a);
    pool.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, n);
    });
  }
  for (auto& th : pool) th.join();
}

struct Piece {
  int row;
  int64_t off, len;  // doubles within the row
};

std::vector<Piece> pieces_of(int N, int64_t ngl, int64_t chunk_doubles) {
  std::vector<Piece> v;
  for (int i = 0; i < N; ++i)
    for (int64_t o = 0; o < ngl; o += chunk_doubles) v.push_back({i, o, std::min(chunk_doubles, ngl - o)});
  return v;
}

}  // namespace

void Engine::ensure_staging() {
  if (stage_h[0]) return;
  for (int b = 0; b < 2; ++b) {
    PO_CUDA(cudaMallocHost(&stage_h[b], kStageBytes));
    PO_CUDA(cudaEventCreateWithFlags(&stage_ev[b], cudaEventDisableTiming));
  }
}

void Engine::free_staging() {
  for (int b = 0; b < 2; ++b) {
    if (stage_ev[b]) cudaEventDestroy(stage_ev[b]);
    if (stage_h[b]) cudaFreeHost(stage_h[b]);
    stage_ev[b] = nullptr;
    stage_h[b] = nullptr;
  }
}

int Engine::host_threads() const {
  static const int forced = std::getenv("PO_HOST_THREADS") ? std::atoi(std::getenv("PO_HOST_THREADS")) : 0;
  if (forced > 0) return forced;
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(8u, hc ? hc / 2 : 1u));
}

// host (N x ngl, dense) -> device block (N x ld, pitched), on stream st
void Engine::upload_host(double* dev, const double* host, cudaStream_t st) {
  if (is_pinned(host)) {
    PO_CUDA(cudaMemcpy2DAsync(dev, g.ld * 8, host, g.ngl * 8, g.ngl * 8, N, cudaMemcpyHostToDevice, st));
    return;
  }
  ensure_staging();
  const int nt = host_threads();
  const auto ps = pieces_of(N, g.ngl, (int64_t)(kStageBytes / 8));
  for (size_t k = 0; k < ps.size(); ++k) {
    const int b = (int)(k & 1);
    PO_CUDA(cudaEventSynchronize(stage_ev[b]));  // the copy engine is done with this chunk
    const Piece& p = ps[k];
    parallel_copy(stage_h[b], host + (int64_t)p.row * g.ngl + p.off, (size_t)p.len * 8, nt);
    PO_CUDA(cudaMemcpyAsync(dev + (int64_t)p.row * g.ld + p.off, stage_h[b], (size_t)p.len * 8,
                            cudaMemcpyHostToDevice, st));
    PO_CUDA(cudaEventRecord(stage_ev[b], st));
  }
}

// device block -> host, on stream st; returns when the host buffer is complete
void Engine::download_host(double* host, const double* dev, cudaStream_t st) {
  if (is_pinned(host)) {
    PO_CUDA(cudaMemcpy2DAsync(host, g.ngl * 8, dev, g.ld * 8, g.ngl * 8, N, cudaMemcpyDeviceToHost, st));
    PO_CUDA(cudaStreamSynchronize(st));
    return;
  }
  ensure_staging();
  const int nt = host_threads();
  const auto ps = pieces_of(N, g.ngl, (int64_t)(kStageBytes / 8));
  auto issue = [&](size_t k) {
    const Piece& p = ps[k];
    const int b = (int)(k & 1);
    PO_CUDA(cudaMemcpyAsync(stage_h[b], dev + (int64_t)p.row * g.ld + p.off, (size_t)p.len * 8,
                            cudaMemcpyDeviceToHost, st));
    PO_CUDA(cudaEventRecord(stage_ev[b], st));
  };
  if (!ps.empty()) issue(0);
  for (size_t k = 0; k < ps.size(); ++k) {
    if (k + 1 < ps.size()) issue(k + 1);  // the next chunk moves while this one is drained
    const int b = (int)(k & 1);
    PO_CUDA(cudaEventSynchronize(stage_ev[b]));
    const Piece& p = ps[k];
    parallel_copy(host + (int64_t)p.row * g.ngl + p.off, stage_h[b], (size_t)p.len * 8, nt);
  }
}

}  // namespace po
