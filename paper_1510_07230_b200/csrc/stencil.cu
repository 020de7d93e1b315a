// Batched Kohn-Sham Hamiltonian apply on B200 (sm_100a).
//
// Replaces the reference's per-orbital CPU loop apply_hamiltonian
// (energy.cpp:248-265 -> grid.cpp:94-122 three axis passes) and the energy
// terms kinetic_term / potential_term (energy.cpp:267-280), which the
// reference evaluates with a second Laplacian per orbital.
//
// Design: one CTA = a 32 x 8 column tile of the (axis1, axis2) plane of ONE
// orbital, marching along axis 0 over a z-chunk with a 3-register sliding
// window (u[z-1], u[z], u[z+1]), so each orbital value is read from HBM once;
// the x/y neighbours of the current plane are re-reads that hit L1. The
// local potential planes are shared by all orbitals and stay L2-resident.
// Per point: read u (8 B), write Hu (8 B); v_local/v_ext come from L2.
// The three reductions (sigma_ii, <lap u,u>, <v_ext u,u>) are warp-shuffle
// + smem block sums written as deterministic per-CTA partials.
#include "kernels.h"

namespace po {

namespace {

constexpr int TX = 32, TY = 8;
constexpr int ZCHUNK = 16;

struct HGrid {
  int ntx, nty, nzc;
};

HGrid hgrid(const SlabGeom& g) {
  HGrid h;
  h.ntx = (int)((g.n2 + TX - 1) / TX);
  h.nty = (int)((g.n1 + TY - 1) / TY);
  h.nzc = (int)((g.nz + ZCHUNK - 1) / ZCHUNK);
  return h;
}

// MODE 0: Hu + reductions; MODE 1: Laplacian only (store lap).
template <int MODE>
__global__ void __launch_bounds__(TX * TY) hamiltonian_kernel(
    SlabGeom g, int N, int ntx, const double* __restrict__ u, const double* __restrict__ halo_lo,
    const double* __restrict__ halo_hi, const double* __restrict__ vloc,
    const double* __restrict__ vext, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double red[3 * 32];
  const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
  const int64_t x = (int64_t)tx * TX + threadIdx.x;
  const int64_t y = (int64_t)ty * TY + threadIdx.y;
  const int i = blockIdx.z;
  const bool active = x < g.n2 && y < g.n1;
  const int64_t zs = (int64_t)blockIdx.y * ZCHUNK;
  const int64_t ze = min(zs + (int64_t)ZCHUNK, g.nz);
  const int64_t plane = g.plane;
  const double* ui = u + (int64_t)i * g.ld;
  double* oi = out ? out + (int64_t)i * g.ld : nullptr;
  const int64_t col = y * g.n2 + x;
  const double ih0 = g.ih2[0], ih1 = g.ih2[1], ih2 = g.ih2[2];
  double acc[3] = {0.0, 0.0, 0.0};
  if (active) {
    double zm;
    if (zs > 0) zm = __ldg(ui + (zs - 1) * plane + col);
    else zm = halo_lo ? __ldg(halo_lo + (int64_t)i * plane + col) : 0.0;
    double c = __ldg(ui + zs * plane + col);
    for (int64_t z = zs; z < ze; ++z) {
      const int64_t idx = z * plane + col;
      double zp;
      if (z + 1 < g.nz) zp = __ldg(ui + idx + plane);
      else zp = halo_hi ? __ldg(halo_hi + (int64_t)i * plane + col) : 0.0;
      const double xm = x > 0 ? __ldg(ui + idx - 1) : 0.0;
      const double xp = x + 1 < g.n2 ? __ldg(ui + idx + 1) : 0.0;
      const double ym = y > 0 ? __ldg(ui + idx - g.n2) : 0.0;
      const double yp = y + 1 < g.n1 ? __ldg(ui + idx + g.n2) : 0.0;
      // axis order 0, 1, 2 as the reference accumulates its passes
      const double lap = ((zm - 2.0 * c + zp) * ih0 + (ym - 2.0 * c + yp) * ih1) +
                         (xm - 2.0 * c + xp) * ih2;
      if (MODE == 0) {
        const double h = -0.5 * lap + __ldg(vloc + idx) * c;
        if (oi) oi[idx] = h;
        acc[0] += h * c;
        acc[1] += lap * c;
        acc[2] += __ldg(vext + idx) * c * c;
      } else {
        oi[idx] = lap;
      }
      zm = c;
      c = zp;
    }
  }
  if (MODE == 0) {
    block_sum<3>(acc, red);
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      const int nblk = gridDim.x * gridDim.y;
      const int b = blockIdx.x + gridDim.x * blockIdx.y;
#pragma unroll
      for (int q = 0; q < 3; ++q) partials[((int64_t)q * N + i) * nblk + b] = acc[q];
    }
  }
}

}  // namespace

int hamiltonian_nblk(const SlabGeom& g) {
  HGrid h = hgrid(g);
  return h.ntx * h.nty * h.nzc;
}

void launch_hamiltonian(const SlabGeom& g, int N, const double* u, const double* halo_lo,
                        const double* halo_hi, const double* v_local, const double* v_ext,
                        double* hu, double* partials, cudaStream_t s) {
  HGrid h = hgrid(g);
  dim3 grid(h.ntx * h.nty, h.nzc, N), block(TX, TY);
  ::po::count_launch();
  hamiltonian_kernel<0><<<grid, block, 0, s>>>(g, N, h.ntx, u, halo_lo, halo_hi, v_local, v_ext,
                                               hu, partials);
}

void launch_laplacian(const SlabGeom& g, int N, const double* u, const double* halo_lo,
                      const double* halo_hi, double* out, cudaStream_t s) {
  HGrid h = hgrid(g);
  dim3 grid(h.ntx * h.nty, h.nzc, N), block(TX, TY);
  ::po::count_launch();
  hamiltonian_kernel<1><<<grid, block, 0, s>>>(g, N, h.ntx, u, halo_lo, halo_hi, nullptr, nullptr,
                                               out, nullptr);
}

}  // namespace po
