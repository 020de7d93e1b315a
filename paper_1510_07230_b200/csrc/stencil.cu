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

// ---------------------------------------------------------------- v2
// Same math, barrier-free and with deep memory-level parallelism: each thread
// owns one (y, x) column and processes its z-range in groups of ZG planes.
// For a group it issues ALL loads up front — own column z..z+ZG (the z-1 value
// is carried), the y-1 / y+1 columns (L1/L2 hits: neighbouring warps stream
// them), v_local (L2) and, when EXT, v_ext — then computes the ZG points.
// x-neighbours come from warp shuffles (lane 0 / 31 load the tile edge).
// Per orbital.point from HBM: one load, one store. EXT = per-orbital
// <V_ext u, u> partials (C ABI / linear problems); the nonlinear solver takes
// E_ext = w <V_ext, rho> from the density kernel instead.
constexpr int ZG = 4;        // planes per load group
constexpr int ZCHUNK2 = 32;  // planes per CTA

template <bool EXT>
__global__ void __launch_bounds__(TX * TY, 3) hamiltonian2_kernel(
    SlabGeom g, int N, int ntx, const double* __restrict__ u, const double* __restrict__ halo_lo,
    const double* __restrict__ halo_hi, const double* __restrict__ vloc,
    const double* __restrict__ vext, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double red[3 * 32];
  const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
  const int lane = threadIdx.x;
  const int64_t x = (int64_t)tx * TX + lane;
  const int64_t y = (int64_t)ty * TY + threadIdx.y;
  const bool active = x < g.n2 && y < g.n1;
  const int i = blockIdx.z;
  const int64_t zs = (int64_t)blockIdx.y * ZCHUNK2;
  const int64_t ze = min(zs + (int64_t)ZCHUNK2, g.nz);
  const int64_t plane = g.plane;
  const double* ui = u + (int64_t)i * g.ld;
  double* oi = out ? out + (int64_t)i * g.ld : nullptr;
  const int64_t col = y * g.n2 + x;
  const double ih0 = g.ih2[0], ih1 = g.ih2[1], ih2 = g.ih2[2];
  const bool has_ym = active && y > 0, has_yp = active && y + 1 < g.n1;
  const bool has_xm = active && x > 0, has_xp = active && x + 1 < g.n2;

  auto at = [&](int64_t z, int64_t c) -> double {  // u at (plane z, column c), halos/zero outside
    if (z < 0) return halo_lo ? __ldg(halo_lo + (int64_t)i * plane + c) : 0.0;
    if (z >= g.nz) return halo_hi ? __ldg(halo_hi + (int64_t)i * plane + c) : 0.0;
    return __ldg(ui + z * plane + c);
  };
  double zm = active ? at(zs - 1, col) : 0.0;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t z0 = zs; z0 < ze; z0 += ZG) {
    double cz[ZG + 1], ym[ZG], yp[ZG], v[ZG], ve[ZG], xe[ZG];
#pragma unroll
    for (int k = 0; k <= ZG; ++k) {
      const int64_t z = z0 + k;
      cz[k] = (active && z <= ze) ? at(z, col) : 0.0;  // plane ze = last point's z+1 neighbour
    }
#pragma unroll
    for (int k = 0; k < ZG; ++k) {
      const int64_t z = z0 + k;
      const bool in = z < ze;
      ym[k] = (in && has_ym) ? __ldg(ui + z * plane + col - g.n2) : 0.0;
      yp[k] = (in && has_yp) ? __ldg(ui + z * plane + col + g.n2) : 0.0;
      v[k] = (in && active) ? __ldg(vloc + z * plane + col) : 0.0;
      if (EXT) ve[k] = (in && active) ? __ldg(vext + z * plane + col) : 0.0;
      // tile-edge x neighbours (lane 0 needs x-1, lane 31 needs x+1)
      xe[k] = 0.0;
      if (in && lane == 0 && has_xm) xe[k] = __ldg(ui + z * plane + col - 1);
      if (in && lane == TX - 1 && has_xp) xe[k] = __ldg(ui + z * plane + col + 1);
    }
#pragma unroll
    for (int k = 0; k < ZG; ++k) {
      const int64_t z = z0 + k;
      if (z >= ze) break;
      const double c = cz[k];
      double xm = __shfl_up_sync(0xffffffffu, c, 1);
      double xp = __shfl_down_sync(0xffffffffu, c, 1);
      if (lane == 0) xm = xe[k];
      if (lane == TX - 1) xp = xe[k];
      if (!has_xp) xp = 0.0;
      if (!has_xm) xm = 0.0;
      if (active) {
        const double lap = ((zm - 2.0 * c + cz[k + 1]) * ih0 + (ym[k] - 2.0 * c + yp[k]) * ih1) +
                           (xm - 2.0 * c + xp) * ih2;
        const double h = -0.5 * lap + v[k] * c;
        if (oi) oi[z * plane + col] = h;
        acc[0] += h * c;
        acc[1] += lap * c;
        if (EXT) acc[2] += ve[k] * c * c;
      }
      zm = c;
    }
  }
  block_sum<3>(acc, &red[0]);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    const int nblk = gridDim.x * gridDim.y;
    const int b = blockIdx.x + gridDim.x * blockIdx.y;
#pragma unroll
    for (int q = 0; q < 3; ++q) partials[((int64_t)q * N + i) * nblk + b] = acc[q];
  }
}

}  // namespace

int hamiltonian2_nblk(const SlabGeom& g) {
  HGrid h = hgrid(g);
  return h.ntx * h.nty * (int)((g.nz + ZCHUNK2 - 1) / ZCHUNK2);
}

void launch_hamiltonian2(const SlabGeom& g, int N, const double* u, const double* halo_lo,
                         const double* halo_hi, const double* v_local, const double* v_ext,
                         double* hu, double* partials, cudaStream_t s) {
  HGrid h = hgrid(g);
  dim3 grid(h.ntx * h.nty, (unsigned)((g.nz + ZCHUNK2 - 1) / ZCHUNK2), N), block(TX, TY);
  ::po::count_launch();
  if (v_ext)
    hamiltonian2_kernel<true><<<grid, block, 0, s>>>(g, N, h.ntx, u, halo_lo, halo_hi, v_local,
                                                     v_ext, hu, partials);
  else
    hamiltonian2_kernel<false><<<grid, block, 0, s>>>(g, N, h.ntx, u, halo_lo, halo_hi, v_local,
                                                      nullptr, hu, partials);
}

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
