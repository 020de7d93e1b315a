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
constexpr int ZCHUNK2 = 32;  // planes per CTA

template <bool EXT, int ZG, int MINB>
__global__ void __launch_bounds__(TX * TY, MINB) hamiltonian2_kernel(
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

constexpr int MAXJ = 8;  // row-length bound of the full-row kernels: n2 <= 32 * MAXJ

#ifdef PO_MEASUREMENT_VARIANTS
// ---------------------------------------------------------------- v3
// Full-row tiles: a CTA owns TY whole x-rows (rows y0..y0+7 of a plane are one
// contiguous TY*n2*8-byte chunk) for a z-range of one orbital; each thread holds
// the J = ceil(n2/32) columns x = lane + 32 j of its row, so all x-neighbours
// come from shuffles (chunk boundaries via lane-0/31 broadcasts) and every
// plane is streamed as large contiguous pieces. y-neighbours are __ldg (L1:
// the adjacent warps stream those rows).

template <int J, bool EXT>
__global__ void __launch_bounds__(TX * TY, 2) hamiltonian3_kernel(
    SlabGeom g, int N, const double* __restrict__ u, const double* __restrict__ halo_lo,
    const double* __restrict__ halo_hi, const double* __restrict__ vloc,
    const double* __restrict__ vext, double* __restrict__ out, double* __restrict__ partials) {
  __shared__ double red[3 * 32];
  const int lane = threadIdx.x;
  const int64_t y = (int64_t)blockIdx.x * TY + threadIdx.y;
  const bool yin = y < g.n1;
  const int i = blockIdx.z;
  const int64_t zs = (int64_t)blockIdx.y * ZCHUNK2;
  const int64_t ze = min(zs + (int64_t)ZCHUNK2, g.nz);
  const int64_t plane = g.plane;
  const double* ui = u + (int64_t)i * g.ld;
  double* oi = out ? out + (int64_t)i * g.ld : nullptr;
  const double ih0 = g.ih2[0], ih1 = g.ih2[1], ih2 = g.ih2[2];
  const bool has_ym = yin && y > 0, has_yp = yin && y + 1 < g.n1;
  bool xin[J];
  int64_t col[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int64_t x = lane + 32 * j;
    xin[j] = yin && x < g.n2;
    col[j] = y * g.n2 + x;
  }
  auto at = [&](int64_t z, int64_t c) -> double {
    if (z < 0) return halo_lo ? __ldg(halo_lo + (int64_t)i * plane + c) : 0.0;
    if (z >= g.nz) return halo_hi ? __ldg(halo_hi + (int64_t)i * plane + c) : 0.0;
    return __ldg(ui + z * plane + c);
  };
  double zm[J], c[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    zm[j] = xin[j] ? at(zs - 1, col[j]) : 0.0;
    c[j] = xin[j] ? at(zs, col[j]) : 0.0;
  }
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t z = zs; z < ze; ++z) {
    double zp[J], ym[J], yp[J], v[J], ve[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      zp[j] = xin[j] ? at(z + 1, col[j]) : 0.0;
      ym[j] = (xin[j] && has_ym) ? __ldg(ui + z * plane + col[j] - g.n2) : 0.0;
      yp[j] = (xin[j] && has_yp) ? __ldg(ui + z * plane + col[j] + g.n2) : 0.0;
      v[j] = xin[j] ? __ldg(vloc + z * plane + col[j]) : 0.0;
      if (EXT) ve[j] = xin[j] ? __ldg(vext + z * plane + col[j]) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      double xm = __shfl_up_sync(0xffffffffu, c[j], 1);
      double xp = __shfl_down_sync(0xffffffffu, c[j], 1);
      const double prev31 = __shfl_sync(0xffffffffu, j > 0 ? c[j > 0 ? j - 1 : 0] : 0.0, 31);
      const double next0 = __shfl_sync(0xffffffffu, j + 1 < J ? c[j + 1 < J ? j + 1 : 0] : 0.0, 0);
      if (lane == 0) xm = prev31;        // x - 1 lives in the previous chunk (0 at x = 0)
      if (lane == TX - 1) xp = next0;    // x + 1 lives in the next chunk
      if (!(lane + 32 * j + 1 < g.n2)) xp = 0.0;
      if (xin[j]) {
        const double cc = c[j];
        const double lap = ((zm[j] - 2.0 * cc + zp[j]) * ih0 + (ym[j] - 2.0 * cc + yp[j]) * ih1) +
                           (xm - 2.0 * cc + xp) * ih2;
        const double h = -0.5 * lap + v[j] * cc;
        if (oi) oi[z * plane + col[j]] = h;
        acc[0] += h * cc;
        acc[1] += lap * cc;
        if (EXT) acc[2] += ve[j] * cc * cc;
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      zm[j] = c[j];
      c[j] = zp[j];
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

template <bool EXT>
void launch_h3(const SlabGeom& g, int N, const double* u, const double* lo, const double* hi,
               const double* vloc, const double* vext, double* out, double* partials,
               cudaStream_t s) {
  dim3 grid((unsigned)((g.n1 + TY - 1) / TY), (unsigned)((g.nz + ZCHUNK2 - 1) / ZCHUNK2), N);
  dim3 block(TX, TY);
  switch ((g.n2 + 31) / 32) {
#define PO_H3(JJ)                                                                               \
  case JJ:                                                                                      \
    hamiltonian3_kernel<JJ, EXT><<<grid, block, 0, s>>>(g, N, u, lo, hi, vloc, vext, out, partials); \
    break;
    PO_H3(1) PO_H3(2) PO_H3(3) PO_H3(4) PO_H3(5) PO_H3(6) PO_H3(7) PO_H3(8)
#undef PO_H3
  }
}

#endif  // PO_MEASUREMENT_VARIANTS

// ---------------------------------------------------------------- v4 (TMA)
// Plane ring: a CTA owns TY full x-rows (y0 .. y0+TY-1) of ONE orbital over a
// z-range. A producer warp streams, per plane, the contiguous block of rows
// y0-1 .. y0+TY (one cp.async.bulk of (TY+2) * n2 * 8 bytes: 7.7 KB at 96^3,
// far above the ~2 KB TMA efficiency threshold measured in
// profiles/r1_tma_probe.txt) and the plane's v_local rows into an NST-deep
// shared-memory ring; 8 consumer warps (one row each, x = lane + 32 j) read all
// seven stencil taps from shared memory — no global loads in the compute —
// and release a plane slot once the step that last needs it (z+1) is done.
// Rows outside [0, n1) stay zero in the ring; planes outside the slab come
// from the halo buffers (or are zero at the global boundary).
struct PlaneRing {
  int nst;
  int64_t urow, vrow;  // doubles per u / v slot
  size_t smem;
};

PlaneRing plane_ring(const SlabGeom& g, int tyr, size_t budget) {
  PlaneRing r;
  r.urow = (tyr + 2) * g.n2;
  r.vrow = tyr * g.n2;
  const size_t per = (size_t)(r.urow + r.vrow) * 8;
  int nst = (int)(budget / per);
  if (nst > 8) nst = 8;
  if (nst < 4) nst = 4;
  r.nst = nst;
  r.smem = 256 + (size_t)nst * per;
  return r;
}

__device__ __forceinline__ bool ring_plane_real(int64_t p, int64_t nz, const double* lo,
                                                const double* hi) {
  return (p >= 0 && p < nz) || (p < 0 && lo) || (p >= nz && hi);
}

template <int J, bool EXT, int TYR>
__global__ void __launch_bounds__(32 * (TYR + 1), 1) hamiltonian4_kernel(
    SlabGeom g, int N, int nst, int zc, const double* __restrict__ u, const double* __restrict__ halo_lo,
    const double* __restrict__ halo_hi, const double* __restrict__ vloc,
    const double* __restrict__ vext, double* __restrict__ out, double* __restrict__ partials,
    int64_t lo_ld, int64_t hi_ld, int nbtot, int boff) {
  // lo_ld / hi_ld: orbital stride of the halo planes (g.plane for the exchange
  // buffers; g.ld when a "halo" is a plane of u itself — the interior / boundary
  // split of a slab, Engine::apply_h); partials of block b land at column boff + b
  // of rows of length nbtot (several launches share one reduction)
  PO_PDL_ENTRY();
  extern __shared__ __align__(128) unsigned char hsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(hsm);
  uint64_t* empty = full + 8;
  double* ring = reinterpret_cast<double*>(hsm + 256);
  __shared__ double red[3 * 32];
  const int64_t n1 = g.n1, n2 = g.n2, plane = g.plane;
  const int64_t urow = (TYR + 2) * n2, vrow = TYR * n2;
  // the orbital is the fastest grid index: CTAs resident together share one
  // (y-tile, z-chunk) of v_local (and, when it exceeds L2 — 134 MB at 256^3 —
  // it is read from HBM once per tile instead of once per orbital)
  const int i = blockIdx.x;
  const int64_t y0 = (int64_t)blockIdx.y * TYR;
  const int64_t zs = (int64_t)blockIdx.z * zc;
  const int64_t ze = min(zs + (int64_t)zc, g.nz);
  const int nplanes = (int)(ze - zs) + 2;  // zs-1 .. ze
  const double* ui = u + (int64_t)i * g.ld;
  const int warp = threadIdx.y, lane = threadIdx.x;  // block (32, 9)
  // valid row window [ra, rb) of the u slot (slot row r <-> grid row y0 - 1 + r)
  const int64_t ra = y0 - 1 < 0 ? 1 : 0;
  const int64_t rb = min((int64_t)TYR + 2, n1 - (y0 - 1));
  const int64_t vb = min((int64_t)TYR, n1 - y0);
  for (int64_t e = threadIdx.x + 32 * threadIdx.y; e < (int64_t)nst * (urow + vrow); e += 32 * (TYR + 1))
    ring[e] = 0.0;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TYR);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == TYR) {  // ------------------------------------------------ producer
    if (lane == 0) {
      // order the generic-proxy zero fill before the async-proxy (TMA) writes
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      for (int k = 0; k < nplanes; ++k) {
        const int s = k % nst;
        if (k >= nst) mbar_wait(&empty[s], (uint32_t)((k / nst) - 1) & 1u);
        const int64_t p = zs - 1 + k;
        double* us = ring + (int64_t)s * (urow + vrow);
        const bool real = ring_plane_real(p, g.nz, halo_lo, halo_hi);
        const bool center = p >= zs && p < ze;
        uint32_t bytes = 0;
        if (real) bytes += (uint32_t)((rb - ra) * n2 * 8);
        if (center) bytes += (uint32_t)(vb * n2 * 8);
        mbar_arrive_expect_tx(&full[s], bytes);
        if (real) {
          const double* src;
          if (p < 0) src = halo_lo + (int64_t)i * lo_ld;
          else if (p >= g.nz) src = halo_hi + (int64_t)i * hi_ld;
          else src = ui + p * plane;
          tma_load_1d(us + ra * n2, src + (y0 - 1 + ra) * n2, (uint32_t)((rb - ra) * n2 * 8),
                      &full[s]);
        }
        if (center)
          tma_load_1d(us + urow, vloc + p * plane + y0 * n2, (uint32_t)(vb * n2 * 8), &full[s]);
      }
    }
    return;
  }
  // ------------------------------------------------------------------ consumers
  // (ring slots and phases advance incrementally and all in-slot offsets are
  // 32-bit: the per-plane index arithmetic — runtime modulo by nst — used to
  // outweigh the stencil math; ncu showed the kernel issue-bound at 71%)
  const int64_t y = y0 + warp;
  const bool yin = y < n1;
  const double ih0 = g.ih2[0], ih1 = g.ih2[1], ih2 = g.ih2[2];
  const int n2i = (int)n2;
  const int slot_stride = (int)(urow + vrow);
  const int rrow = (warp + 1) * n2i;           // slot row of y
  const int vrow_off = (int)urow + warp * n2i;  // v_local row of y
  double acc[3] = {0.0, 0.0, 0.0};
  // planes k = 0 (zs-1) and 1 (zs) before the first step
  mbar_wait(&full[0], 0);
  mbar_wait(&full[1 % nst], (uint32_t)(1 / nst) & 1u);
  int sm = 0, sc = 1 % nst, sp = 2 % nst;  // slots of planes k-1, k, k+1
  uint32_t php = (uint32_t)(2 / nst) & 1u;   // phase of plane k+1's slot
  bool rm = ring_plane_real(zs - 1, g.nz, halo_lo, halo_hi), rc = true;
  double* orow = (out && yin) ? out + (int64_t)i * g.ld + zs * plane + y * n2 : nullptr;
  const double* xrow = (EXT && yin) ? vext + zs * plane + y * n2 : nullptr;
  // z-march with register rotation: each lane keeps its points' values of
  // planes k-1 and k in registers, so a step reads only plane k+1 (z+1), the
  // y/x neighbours in plane k and v_local from shared memory (6 instead of 8
  // loads per point: ncu had the kernel bound by shared-memory bandwidth), and
  // plane k-1's slot is released before the step instead of after it
  double zr_m[J], zr_c[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int x = lane + 32 * j;
    const bool ok = yin && x < n2i;
    zr_m[j] = (ok && rm) ? ring[sm * slot_stride + rrow + x] : 0.0;
    zr_c[j] = ok ? ring[sc * slot_stride + rrow + x] : 0.0;
  }
  for (int k = 1; k + 1 < nplanes; ++k) {  // step on plane z = zs - 1 + k
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sm]);  // plane k-1 lives on in registers only
    mbar_wait(&full[sp], php);
    const double* pc = ring + sc * slot_stride;
    const double* pp = ring + sp * slot_stride;
    const bool rp = ring_plane_real(zs + k, g.nz, halo_lo, halo_hi);
    if (yin) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int x = lane + 32 * j;
        if (x < n2i) {
          const int r = rrow + x;
          const double c = zr_c[j];
          const double zm = zr_m[j];
          const double zp = rp ? pp[r] : 0.0;
          const double ym = pc[r - n2i];  // zero rows outside the box
          const double yp = pc[r + n2i];
          const double xm = x > 0 ? pc[r - 1] : 0.0;
          const double xp = x + 1 < n2i ? pc[r + 1] : 0.0;
          const double lap = ((zm - 2.0 * c + zp) * ih0 + (ym - 2.0 * c + yp) * ih1) +
                             (xm - 2.0 * c + xp) * ih2;
          const double h = -0.5 * lap + pc[vrow_off + x] * c;
          if (orow) orow[x] = h;
          acc[0] += h * c;
          acc[1] += lap * c;
          if (EXT) acc[2] += __ldg(xrow + x) * c * c;
          zr_m[j] = c;
          zr_c[j] = zp;
        }
      }
    }
    if (orow) orow += plane;
    if (EXT && xrow) xrow += plane;
    rm = rc;
    rc = rp;
    sm = sc;
    sc = sp;
    if (++sp == nst) {
      sp = 0;
      php ^= 1u;
    }
  }
  // the last two planes' slots are never re-filled: no arrivals needed
  {
    // block reduction over the 8 consumer warps (the producer warp has exited)
#pragma unroll
    for (int q = 0; q < 3; ++q) acc[q] = warp_sum(acc[q]);
    if (lane == 0)
      for (int q = 0; q < 3; ++q) red[q * 32 + warp] = acc[q];
    asm volatile("bar.sync 1, %0;" ::"n"(TX * TYR));
    if (warp == 0) {
      double v[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) v[q] = warp_sum(lane < TYR ? red[q * 32 + lane] : 0.0);
      if (lane == 0) {
        const int b = boff + blockIdx.y + gridDim.y * blockIdx.z;
#pragma unroll
        for (int q = 0; q < 3; ++q) partials[((int64_t)q * N + i) * nbtot + b] = v[q];
      }
    }
  }
}

struct H4Part {  // a launch's place in a shared partials layout + its halo strides
  int64_t lo_ld = -1, hi_ld = -1;  // -1: g.plane (the exchange buffers)
  int nbtot = -1, boff = 0;        // -1: this launch's own block count
};

template <bool EXT, int TYR = 8>
void launch_h4(const SlabGeom& g, int N, const double* u, const double* lo, const double* hi,
               const double* vloc, const double* vext, double* out, double* partials,
               cudaStream_t s, int zc = ZCHUNK2, size_t budget = 100 * 1024, H4Part pt = H4Part()) {
  const PlaneRing r = plane_ring(g, TYR, budget);
  dim3 grid((unsigned)N, (unsigned)((g.n1 + TYR - 1) / TYR), (unsigned)((g.nz + zc - 1) / zc));
  dim3 block(TX, TYR + 1);
  const int64_t lo_ld = pt.lo_ld < 0 ? g.plane : pt.lo_ld, hi_ld = pt.hi_ld < 0 ? g.plane : pt.hi_ld;
  const int nbtot = pt.nbtot < 0 ? (int)(grid.y * grid.z) : pt.nbtot;
  switch ((g.n2 + 31) / 32) {
#define PO_H4(JJ)                                                                          \
  case JJ: {                                                                               \
    auto k = hamiltonian4_kernel<JJ, EXT, TYR>;                                             \
    set_smem(reinterpret_cast<const void*>(k), (int)r.smem);                               \
    launch_pdl(k, dim3(grid), dim3(block), r.smem, s, g, N, r.nst, zc, u, lo, hi, vloc, vext, out, partials, \
               lo_ld, hi_ld, nbtot, pt.boff);                                               \
    break;                                                                                 \
  }
    PO_H4(1) PO_H4(2) PO_H4(3) PO_H4(4) PO_H4(5) PO_H4(6) PO_H4(7) PO_H4(8)
#undef PO_H4
  }
}

// Production shapes (tools/hu_shape_sweep.py on B200, interleaved rounds,
// profiles/r1_hu_shape_sweep.json): rows per CTA / planes per CTA / ring budget
// by row length. Six rows and a 56 KB ring (4 CTAs / SM) at 96^3 (85% of the
// measured HBM peak after the register z-march; 70.6% before it, 43.6% for the
// first kernel); eight rows win at 64-point rows (fewer, fuller CTAs: 0.77-0.87
// vs 0.63-0.71) and at 128-192 (0.86-0.93); 256-point rows keep six rows (eight
// would leave one CTA per SM). Measured and dropped: two or three rows per
// consumer warp (y neighbours from registers, 5 loads per point): 81% / 71% —
// fewer warps per SM hide less latency than the saved loads buy.
struct H4Shape {
  int tyr, zc;
  size_t budget;
};
H4Shape h4_shape(const SlabGeom& g) {
  if (g.n2 <= 64) return {8, 32, 56 * 1024};
  if (g.n2 <= 96) return {6, 64, 56 * 1024};
  if (g.n2 <= 192) return {8, 48, 70 * 1024};
  return {6, 32, 56 * 1024};
}

bool h4_supported(const SlabGeom& g) {
  // bulk copies need 16-byte multiples / alignment: even n2 (plane rows of 8 n2 bytes)
  return g.n2 % 2 == 0 && g.n2 <= 32 * MAXJ && (g.ld % 2 == 0);
}

}  // namespace

int hamiltonian2_nblk(const SlabGeom& g) {
  if (h4_supported(g)) {  // TMA ring: (y-tile, z-chunk) grid
    const H4Shape h = h4_shape(g);
    return (int)((g.n1 + h.tyr - 1) / h.tyr) * (int)((g.nz + h.zc - 1) / h.zc);
  }
  HGrid h = hgrid(g);
  return h.ntx * h.nty * (int)((g.nz + ZCHUNK2 - 1) / ZCHUNK2);
}

void launch_hamiltonian2(const SlabGeom& g, int N, const double* u, const double* halo_lo,
                         const double* halo_hi, const double* v_local, const double* v_ext,
                         double* hu, double* partials, cudaStream_t s) {
  if (h4_supported(g)) {  // production path: TMA plane ring
    ::po::count_launch();
    const H4Shape h = h4_shape(g);
    if (h.tyr == 8) {
      if (v_ext)
        launch_h4<true, 8>(g, N, u, halo_lo, halo_hi, v_local, v_ext, hu, partials, s, h.zc, h.budget);
      else
        launch_h4<false, 8>(g, N, u, halo_lo, halo_hi, v_local, nullptr, hu, partials, s, h.zc,
                            h.budget);
    } else {
      if (v_ext)
        launch_h4<true, 6>(g, N, u, halo_lo, halo_hi, v_local, v_ext, hu, partials, s, h.zc, h.budget);
      else
        launch_h4<false, 6>(g, N, u, halo_lo, halo_hi, v_local, nullptr, hu, partials, s, h.zc,
                            h.budget);
    }
    return;
  }
  HGrid h = hgrid(g);
  dim3 grid(h.ntx * h.nty, (unsigned)((g.nz + ZCHUNK2 - 1) / ZCHUNK2), N), block(TX, TY);
  ::po::count_launch();
  if (v_ext)
    hamiltonian2_kernel<true, 4, 3><<<grid, block, 0, s>>>(g, N, h.ntx, u, halo_lo, halo_hi,
                                                           v_local, v_ext, hu, partials);
  else
    hamiltonian2_kernel<false, 4, 3><<<grid, block, 0, s>>>(g, N, h.ntx, u, halo_lo, halo_hi,
                                                            v_local, nullptr, hu, partials);
}

// H u of a slab with the halo exchange overlapped (Engine::apply_h, size > 1):
// `interior` launches planes 1 .. nz-2, whose z-neighbours are all local (the
// "halos" of that view are planes 0 and nz-1 of u itself, orbital stride ld);
// `boundary` (after the exchange) launches planes 0 and nz-1 with the received
// planes. Both write one partials layout of hamiltonian_split_nblk columns.
// Returns false where the split is unavailable (caller: launch_hamiltonian2).
int hamiltonian_split_nblk(const SlabGeom& g) {
  const H4Shape h = h4_shape(g);
  const int ny = (int)((g.n1 + h.tyr - 1) / h.tyr);
  return ny * (int)((g.nz - 2 + h.zc - 1) / h.zc) + 2 * ny;
}

bool hamiltonian_split_ok(const SlabGeom& g) { return h4_supported(g) && g.nz >= 3; }

namespace {
template <int TYR>
void h4_any(bool ext, const SlabGeom& g, int N, const double* u, const double* lo, const double* hi,
            const double* vloc, const double* vext, double* out, double* partials, cudaStream_t s,
            int zc, size_t budget, H4Part pt) {
  if (ext)
    launch_h4<true, TYR>(g, N, u, lo, hi, vloc, vext, out, partials, s, zc, budget, pt);
  else
    launch_h4<false, TYR>(g, N, u, lo, hi, vloc, nullptr, out, partials, s, zc, budget, pt);
}

void h4_view(const SlabGeom& g, int64_t z0, int64_t nz, int N, const double* u, const double* lo,
             int64_t lo_ld, const double* hi, int64_t hi_ld, const double* vloc, const double* vext,
             double* out, double* partials, int boff, cudaStream_t s) {
  SlabGeom v = g;
  v.nz = nz;
  const int64_t off = z0 * g.plane;
  const H4Shape h = h4_shape(g);
  H4Part pt;
  pt.lo_ld = lo_ld;
  pt.hi_ld = hi_ld;
  pt.nbtot = hamiltonian_split_nblk(g);
  pt.boff = boff;
  ::po::count_launch();
  if (h.tyr == 8)
    h4_any<8>(vext != nullptr, v, N, u + off, lo, hi, vloc + off, vext ? vext + off : nullptr,
              out ? out + off : nullptr, partials, s, h.zc, h.budget, pt);
  else
    h4_any<6>(vext != nullptr, v, N, u + off, lo, hi, vloc + off, vext ? vext + off : nullptr,
              out ? out + off : nullptr, partials, s, h.zc, h.budget, pt);
}
}  // namespace

void launch_hamiltonian_interior(const SlabGeom& g, int N, const double* u, const double* v_local,
                                 const double* v_ext, double* hu, double* partials, cudaStream_t s) {
  h4_view(g, 1, g.nz - 2, N, u, u, g.ld, u + (g.nz - 1) * g.plane, g.ld, v_local, v_ext, hu, partials, 0,
          s);
}

void launch_hamiltonian_boundary(const SlabGeom& g, int N, const double* u, const double* halo_lo,
                                 const double* halo_hi, const double* v_local, const double* v_ext,
                                 double* hu, double* partials, cudaStream_t s) {
  const H4Shape h = h4_shape(g);
  const int ny = (int)((g.n1 + h.tyr - 1) / h.tyr);
  const int nbi = ny * (int)((g.nz - 2 + h.zc - 1) / h.zc);
  // plane 0: below it the received plane (or zero at the global boundary), above it plane 1
  h4_view(g, 0, 1, N, u, halo_lo, g.plane, u + g.plane, g.ld, v_local, v_ext, hu, partials, nbi, s);
  // plane nz-1: below it plane nz-2, above it the received plane
  h4_view(g, g.nz - 1, 1, N, u, u + (g.nz - 2) * g.plane, g.ld, halo_hi, g.plane, v_local, v_ext, hu,
          partials, nbi + ny, s);
}

#ifdef PO_MEASUREMENT_VARIANTS
// Design-space probe (po_enqueue(PO_OP_HAMILTONIAN_VARIANT + v)): same math,
// different register-group depth / occupancy; v = 0 is the first-generation
// kernel (per-point neighbour loads, with V_ext).
int launch_hamiltonian_variant(int v, const SlabGeom& g, int N, const double* u,
                               const double* v_local, const double* v_ext, double* hu,
                               double* partials, cudaStream_t s) {
  HGrid h = hgrid(g);
  dim3 grid(h.ntx * h.nty, (unsigned)((g.nz + ZCHUNK2 - 1) / ZCHUNK2), N), block(TX, TY);
  ::po::count_launch();
  switch (v) {
    case 0:
      launch_hamiltonian(g, N, u, nullptr, nullptr, v_local, v_ext, hu, partials, s);
      return 0;
    case 1:
      hamiltonian2_kernel<false, 4, 3><<<grid, block, 0, s>>>(g, N, h.ntx, u, nullptr, nullptr,
                                                              v_local, nullptr, hu, partials);
      return 0;
    case 2:
      hamiltonian2_kernel<false, 2, 4><<<grid, block, 0, s>>>(g, N, h.ntx, u, nullptr, nullptr,
                                                              v_local, nullptr, hu, partials);
      return 0;
    case 3:
      hamiltonian2_kernel<false, 4, 2><<<grid, block, 0, s>>>(g, N, h.ntx, u, nullptr, nullptr,
                                                              v_local, nullptr, hu, partials);
      return 0;
    case 4:
      hamiltonian2_kernel<false, 8, 2><<<grid, block, 0, s>>>(g, N, h.ntx, u, nullptr, nullptr,
                                                              v_local, nullptr, hu, partials);
      return 0;
    case 5:
      hamiltonian2_kernel<false, 2, 5><<<grid, block, 0, s>>>(g, N, h.ntx, u, nullptr, nullptr,
                                                              v_local, nullptr, hu, partials);
      return 0;
    case 6:
      hamiltonian2_kernel<false, 1, 6><<<grid, block, 0, s>>>(g, N, h.ntx, u, nullptr, nullptr,
                                                              v_local, nullptr, hu, partials);
      return 0;
    case 7:
      if (g.n2 > 32 * MAXJ) return -1;
      launch_h3<false>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s);
      return 0;
    case 8:
      if (!h4_supported(g)) return -1;
      launch_h4<false>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s);
      return 0;
    case 9:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 8>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, 32,
                          56 * 1024);
      return 0;
    case 10:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 4>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, 32,
                          32 * 1024);
      return 0;
    case 11:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 8>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, 16,
                          70 * 1024);
      return 0;
    case 12:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 8>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, 32,
                          70 * 1024);
      return 0;
    case 13:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 4>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, 48,
                          40 * 1024);
      return 0;
    case 14:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 8>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, 48,
                          70 * 1024);
      return 0;
    case 15:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 6>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, 32,
                          56 * 1024);
      return 0;
    case 16:
    case 17:
    case 18:
    case 19:
    case 20:
    case 21: {
      if (!h4_supported(g)) return -1;
      static const int zcs[6] = {16, 48, 64, 32, 32, 96};
      static const int kbs[6] = {56, 56, 56, 40, 84, 56};
      const int q = v - 16;
      launch_h4<false, 6>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, zcs[q],
                          (size_t)kbs[q] * 1024);
      return 0;
    }
    case 22:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 4>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, 32,
                          40 * 1024);
      return 0;
    case 23:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 8>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, 32,
                          72 * 1024);
      return 0;
    case 24:
    case 25:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 3>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s,
                          v == 24 ? 32 : 64, 48 * 1024);
      return 0;
    case 26:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 4>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s, 64,
                          48 * 1024);
      return 0;
    case 27:
    case 28:
      if (!h4_supported(g)) return -1;
      launch_h4<false, 2>(g, N, u, nullptr, nullptr, v_local, nullptr, hu, partials, s,
                          v == 27 ? 32 : 64, 40 * 1024);
      return 0;
  }
  return -1;
}
#endif  // PO_MEASUREMENT_VARIANTS

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
