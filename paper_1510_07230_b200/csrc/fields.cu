// Pointwise / per-orbital streaming kernels (HBM-bound) for the parorb hot path.
// Each replaces a reference CPU loop, cited per kernel. Reductions produce
// per-CTA partials that launch_reduce_rows sums in a fixed order, so every
// result is bitwise reproducible run to run (the reference's determinism
// contract, parallel.hpp:16-19).
#include <math.h>

#include "kernels.h"

namespace po {

namespace {

constexpr int PT = 256;         // threads per CTA for point-parallel kernels
constexpr int PMAXBLK = 148 * 8;

// energy.cpp:67-76 density + 212-226 Dirac exchange + 4 pi rho (energy.cpp:207-209)
__global__ void __launch_bounds__(PT) density_xc_kernel(SlabGeom g, int N,
                                                        const double* __restrict__ u, double occ,
                                                        int xc, double* __restrict__ rho,
                                                        double* __restrict__ vxc,
                                                        double* __restrict__ b,
                                                        const double* __restrict__ vext,
                                                        double* __restrict__ partials,
                                                        const double* __restrict__ guard) {
  PO_PDL_ENTRY();
  if (guard && *guard == 0.0) return;  // device-side branch (CholeskyQR2 repair)
  __shared__ double red[2 * 32];
  double acc[2] = {0.0, 0.0};
  const double cx = dirac_cx();
  const double four_pi = 4.0 * 3.141592653589793238462643383279502884;
  for (int64_t p = (int64_t)blockIdx.x * PT + threadIdx.x; p < g.ngl;
       p += (int64_t)gridDim.x * PT) {
    double s = 0.0;
    int i = 0;
    for (; i + 4 <= N; i += 4) {  // 4 independent loads in flight, ascending-i sum
      const double a0 = __ldg(u + (int64_t)i * g.ld + p);
      const double a1 = __ldg(u + (int64_t)(i + 1) * g.ld + p);
      const double a2 = __ldg(u + (int64_t)(i + 2) * g.ld + p);
      const double a3 = __ldg(u + (int64_t)(i + 3) * g.ld + p);
      s += a0 * a0;
      s += a1 * a1;
      s += a2 * a2;
      s += a3 * a3;
    }
    for (; i < N; ++i) {
      const double a = __ldg(u + (int64_t)i * g.ld + p);
      s += a * a;
    }
    const double r = occ == 1.0 ? s : s * occ;
    rho[p] = r;
    if (xc) {
      const double eps = -cx * cbrt(r);
      vxc[p] = eps * (4.0 / 3.0);
      acc[0] += eps * r;
    } else {
      vxc[p] = 0.0;
    }
    if (b) {
      const double bb = r * four_pi;
      b[p] = bb;
    }
    if (vext) acc[1] += __ldg(vext + p) * r;  // E_ext = w <V_ext, rho> (energy.cpp:286-291 summed)
  }
  block_sum<2>(acc, red);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = acc[0];
    partials[gridDim.x + blockIdx.x] = acc[1];
  }
}

// vh_src: the Poisson solution slab (copied into the state's v_H here) or null
// for "no Hartree" (v_H = 0 written). xc_here >= 0: v_xc is formed here from
// rho (the Dirac term of energy.cpp:212-226 when xc_here = 1, zero when 0) and
// the partials carry [<v_H, rho> | <eps, rho> | <V_ext, rho>] — the trial
// rotation then only writes rho (its cube roots ran on 4 of 32 lanes there);
// xc_here < 0: v_xc was written by the density pass, partials [<v_H, rho>].
// bfull / xfull (non-null, full grid): the Poisson check rides along — sums of
// r^2 and b^2 with r = b - (-lap_h x) at the slab's points, partial rows 3 and 4
// (and the CG status words cg_out = {0, 0}: no CG kernel ran).
__global__ void __launch_bounds__(PT) vlocal_kernel(SlabGeom g, const double* __restrict__ vext,
                                                    const double* __restrict__ vh_src,
                                                    double* __restrict__ vh,
                                                    double* __restrict__ vxc,
                                                    const double* __restrict__ rho,
                                                    double* __restrict__ vloc,
                                                    double* __restrict__ partials, int xc_here,
                                                    const double* __restrict__ bfull,
                                                    const double* __restrict__ xfull,
                                                    int* __restrict__ cg_out) {
  PO_PDL_ENTRY();
  __shared__ double red[5 * 32];
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const double cx = dirac_cx();
  if (cg_out && blockIdx.x == 0 && threadIdx.x < 2) cg_out[threadIdx.x] = 0;
  const int n1 = (int)g.n1, n2 = (int)g.n2, n0 = (int)g.n0;
  const int plane = n1 * n2;
  for (int64_t p = (int64_t)blockIdx.x * PT + threadIdx.x; p < g.ngl;
       p += (int64_t)gridDim.x * PT) {
    const double h = vh_src ? vh_src[p] : 0.0;
    const double r = rho[p];
    vh[p] = h;
    double x;
    if (xc_here < 0) {
      x = vxc[p];
    } else if (xc_here) {
      const double eps = -cx * cbrt(r);
      x = eps * (4.0 / 3.0);
      vxc[p] = x;
      acc[1] += eps * r;
    } else {
      x = 0.0;
      vxc[p] = 0.0;
    }
    const double ve = vext[p];
    vloc[p] = ve + (h + x);
    acc[0] += h * r;
    acc[2] += ve * r;
    if (xfull) {  // -lap_h x at this point (grid.cpp:94-122 stencil, zero outside the box)
      const int q = (int)(g.z0 * plane + p);
      const int z = q / plane, rem = q - z * plane, y = rem / n2, xx = rem - y * n2;
      const double c = xfull[q];
      const double zm = z > 0 ? xfull[q - plane] : 0.0, zp = z + 1 < n0 ? xfull[q + plane] : 0.0;
      const double ym = y > 0 ? xfull[q - n2] : 0.0, yp = y + 1 < n1 ? xfull[q + n2] : 0.0;
      const double xm = xx > 0 ? xfull[q - 1] : 0.0, xp = xx + 1 < n2 ? xfull[q + 1] : 0.0;
      const double lap = ((zm - 2.0 * c + zp) * g.ih2[0] + (ym - 2.0 * c + yp) * g.ih2[1]) +
                         (xm - 2.0 * c + xp) * g.ih2[2];
      const double bq = bfull[q];
      const double res = bq + lap;  // b - A x, A = -lap_h
      acc[3] += res * res;
      acc[4] += bq * bq;
    }
  }
  block_sum<5>(acc, red);
  if (threadIdx.x == 0) {
    if (xc_here >= 0) {  // rows in S_EXC, S_EEXT, S_EH order: one grouped reduction
      partials[blockIdx.x] = acc[1];
      partials[gridDim.x + blockIdx.x] = acc[2];
      partials[2 * gridDim.x + blockIdx.x] = acc[0];
      if (xfull) {
        partials[3 * gridDim.x + blockIdx.x] = acc[3];
        partials[4 * gridDim.x + blockIdx.x] = acc[4];
      }
    } else {
      partials[blockIdx.x] = acc[0];
    }
  }
}

// grid: (nblk, N)
__global__ void __launch_bounds__(PT) residual_diag_kernel(SlabGeom g, int N,
                                                           const double* __restrict__ u,
                                                           const double* __restrict__ hu,
                                                           const double* __restrict__ sig,
                                                           double* __restrict__ z,
                                                           double* __restrict__ partials) {
  __shared__ double red[32];
  const int i = blockIdx.y;
  const double ms = -sig[i];
  const double* ui = u + (int64_t)i * g.ld;
  const double* hi = hu + (int64_t)i * g.ld;
  double* zi = z + (int64_t)i * g.ld;
  double acc[1] = {0.0};
  for (int64_t p = (int64_t)blockIdx.x * PT + threadIdx.x; p < g.ngl;
       p += (int64_t)gridDim.x * PT) {
    const double v = hi[p] + ms * ui[p];
    zi[p] = v;
    acc[0] += v * v;
  }
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) partials[(int64_t)i * gridDim.x + blockIdx.x] = acc[0];
}

__global__ void __launch_bounds__(PT) bb_kernel(SlabGeom g, int N, const double* __restrict__ w,
                                                const double* __restrict__ wp,
                                                const double* __restrict__ z,
                                                const double* __restrict__ zp,
                                                double* __restrict__ partials) {
  __shared__ double red[3 * 32];
  const int i = blockIdx.y;
  const int64_t o = (int64_t)i * g.ld;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t p = (int64_t)blockIdx.x * PT + threadIdx.x; p < g.ngl;
       p += (int64_t)gridDim.x * PT) {
    const double s = wp ? w[o + p] - wp[o + p] : w[o + p];
    const double y = zp ? z[o + p] - zp[o + p] : z[o + p];
    acc[0] += s * s;
    acc[1] += s * y;
    acc[2] += y * y;
  }
  block_sum<3>(acc, red);
  if (threadIdx.x == 0) {
    const int nb = gridDim.x;
#pragma unroll
    for (int q = 0; q < 3; ++q) partials[((int64_t)q * N + i) * nb + blockIdx.x] = acc[q];
  }
}

// residual_diag + BB products in one pass (N > 48 path; the small-N path does
// this inside directions_tma_kernel): z_i = hu_i - sigma_ii u_i written, partial
// rows [zz | ss | sy | yy] with s = u - u_prev, y = z - z_prev
// (manifold.cpp:204-216, optimizer.cpp:386-397).
__global__ void __launch_bounds__(PT) residual_bb_kernel(SlabGeom g, int N,
                                                         const double* __restrict__ u,
                                                         const double* __restrict__ hu,
                                                         const double* __restrict__ sig,
                                                         const double* __restrict__ up,
                                                         const double* __restrict__ zp,
                                                         double* __restrict__ z,
                                                         double* __restrict__ partials) {
  __shared__ double red[4 * 32];
  const int i = blockIdx.y;
  const double ms = -sig[i];
  const int64_t o = (int64_t)i * g.ld;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t p = (int64_t)blockIdx.x * PT + threadIdx.x; p < g.ngl;
       p += (int64_t)gridDim.x * PT) {
    const double w = u[o + p];
    const double v = hu[o + p] + ms * w;
    z[o + p] = v;
    acc[0] += v * v;
    const double sv = w - up[o + p];
    const double yv = v - zp[o + p];
    acc[1] += sv * sv;
    acc[2] += sv * yv;
    acc[3] += yv * yv;
  }
  block_sum<4>(acc, red);
  if (threadIdx.x == 0) {
    const int nb = gridDim.x;
    partials[(int64_t)i * nb + blockIdx.x] = acc[0];
#pragma unroll
    for (int q = 0; q < 3; ++q) partials[((int64_t)(1 + q) * N + i) * nb + blockIdx.x] = acc[1 + q];
  }
}

// The elementwise half of compute_directions for N > 64 when ||D_i||^2 comes
// from the Grams (launch_dnorm_grams): z_i = fma(-sigma_ii, u_i, hu_i) (the
// FMA every z path uses; written only when z is stored), ||z_i||^2 and the BB
// products against (u_prev, z_prev), z_prev = fma(-sigma_prev, u_prev, hu_prev)
// rebuilt (sigp) or read (xp is a stored z_prev). Four streams, 16-byte loads.
// partials [4][N][nblk]: zz, ss, sy, yy (rows 1..3 only with a history).
template <bool HIST, bool ZPI>
__global__ void __launch_bounds__(PT) residual_bb_stream_kernel(
    SlabGeom g, int N, const double* __restrict__ u, const double* __restrict__ hu,
    const double* __restrict__ sig, const double* __restrict__ up, const double* __restrict__ xp,
    const double* __restrict__ sigp, double* __restrict__ z, double* __restrict__ partials) {
  PO_PDL_ENTRY();
  __shared__ double red[4 * 32];
  const int i = blockIdx.y;
  const double ms = -sig[i];
  const double msp = ZPI ? -sigp[i] : 0.0;
  const int64_t o = (int64_t)i * g.ld;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t npair = g.ngl >> 1;
  auto point = [&](double w, double h, double wq, double xq, double& zv) {
    zv = fma(ms, w, h);
    acc[0] += zv * zv;
    if (HIST) {
      const double zq = ZPI ? fma(msp, wq, xq) : xq;
      const double sv = w - wq, yv = zv - zq;
      acc[1] += sv * sv;
      acc[2] += sv * yv;
      acc[3] += yv * yv;
    }
  };
  for (int64_t q = (int64_t)blockIdx.x * PT + threadIdx.x; q < npair; q += (int64_t)gridDim.x * PT) {
    const int64_t p = o + 2 * q;
    const double2 w = __ldg(reinterpret_cast<const double2*>(u + p));
    const double2 h = __ldg(reinterpret_cast<const double2*>(hu + p));
    double2 wq = make_double2(0.0, 0.0), xq = make_double2(0.0, 0.0);
    if (HIST) {
      wq = __ldg(reinterpret_cast<const double2*>(up + p));
      xq = __ldg(reinterpret_cast<const double2*>(xp + p));
    }
    double2 zz;
    point(w.x, h.x, wq.x, xq.x, zz.x);
    point(w.y, h.y, wq.y, xq.y, zz.y);
    if (z) *reinterpret_cast<double2*>(z + p) = zz;
  }
  if ((g.ngl & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd point count: the last point
    const int64_t p = o + g.ngl - 1;
    double zv;
    point(u[p], hu[p], HIST ? up[p] : 0.0, HIST ? xp[p] : 0.0, zv);
    if (z) z[p] = zv;
  }
  block_sum<4>(acc, red);
  if (threadIdx.x == 0) {
    const int nb = gridDim.x;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q == 0 || HIST) partials[((int64_t)q * N + i) * nb + blockIdx.x] = acc[q];
  }
}

__global__ void __launch_bounds__(PT) abs_sum_kernel(SlabGeom g, int N,
                                                     const double* __restrict__ x,
                                                     double* __restrict__ partials) {
  __shared__ double red[32];
  const int i = blockIdx.y;
  double acc[1] = {0.0};
  for (int64_t p = (int64_t)blockIdx.x * PT + threadIdx.x; p < g.ngl;
       p += (int64_t)gridDim.x * PT)
    acc[0] += fabs(x[(int64_t)i * g.ld + p]);
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) partials[(int64_t)i * gridDim.x + blockIdx.x] = acc[0];
}

__global__ void __launch_bounds__(PT) lincomb_kernel(int64_t total, const double* __restrict__ a,
                                                     double sc, const double* __restrict__ b,
                                                     double* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * PT + threadIdx.x; p < total;
       p += (int64_t)gridDim.x * PT)
    out[p] = a[p] + sc * b[p];
}

// z = HW - sigma W written out (a direction the fused path kept implicit),
// with the directions pass's FMA so the block is bitwise what it would have stored
__global__ void __launch_bounds__(PT) z_from_hw_kernel(int64_t total, int64_t ld,
                                                       const double* __restrict__ w,
                                                       const double* __restrict__ hw,
                                                       const double* __restrict__ sig,
                                                       double* __restrict__ z) {
  for (int64_t p = (int64_t)blockIdx.x * PT + threadIdx.x; p < total;
       p += (int64_t)gridDim.x * PT)
    z[p] = fma(-sig[p / ld], w[p], hw[p]);
}

// One warp per row; lanes stride the partials, then a fixed shuffle tree.
// rows in [grp, 2 grp) take scale2, rows from 2 grp on scale3 (grp = 0: one scale)
__global__ void reduce_rows_kernel(const double* __restrict__ partials, int rows, int nblk,
                                   double scale, double* __restrict__ out,
                                   const double* __restrict__ guard, int grp, double scale2,
                                   double scale3) {
  PO_PDL_ENTRY();
  if (guard && *guard == 0.0) return;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const double* p = partials + (int64_t)warp * nblk;
  double s = 0.0;
  for (int b = lane; b < nblk; b += 32) s += p[b];
  s = warp_sum(s);
  const double sc = grp <= 0 || warp < grp ? scale : (warp < 2 * grp ? scale2 : scale3);
  if (lane == 0) out[warp] = sc * s;
}

// energy.cpp:78-99 (softened Coulomb) or BASELINE C5 Gaussian wells.
__global__ void __launch_bounds__(PT) potential_kernel(SlabGeom g, double h0, double h1,
                                                       double h2, const double* __restrict__ at,
                                                       int natoms, int gaussian,
                                                       double* __restrict__ v) {
  for (int64_t p = (int64_t)blockIdx.x * PT + threadIdx.x; p < g.ngl;
       p += (int64_t)gridDim.x * PT) {
    const int64_t k2 = p % g.n2;
    const int64_t k1 = (p / g.n2) % g.n1;
    const int64_t k0 = p / g.plane + g.z0;
    const double xyz[3] = {(double)(k0 + 1) * h0, (double)(k1 + 1) * h1, (double)(k2 + 1) * h2};
    double acc = 0.0;
    for (int a = 0; a < natoms; ++a) {
      const double* q = at + 5 * a;
      if (!gaussian) {
        double r2 = q[4] * q[4];
        for (int d = 0; d < 3; ++d) {
          const double dx = xyz[d] - q[d];
          r2 += dx * dx;
        }
        acc -= q[3] / sqrt(r2);
      } else {
        double r2 = 0.0;
        for (int d = 0; d < 3; ++d) {
          const double dx = xyz[d] - q[d];
          r2 += dx * dx;
        }
        acc += q[3] * exp(-r2 / (2.0 * q[4] * q[4]));
      }
    }
    v[p] = acc;
  }
}

__global__ void __launch_bounds__(PT) pack_plane_kernel(SlabGeom g, int N,
                                                        const double* __restrict__ u,
                                                        int64_t plane_idx,
                                                        double* __restrict__ dst) {
  const int i = blockIdx.y;
  for (int64_t q = (int64_t)blockIdx.x * PT + threadIdx.x; q < g.plane;
       q += (int64_t)gridDim.x * PT)
    dst[(int64_t)i * g.plane + q] = u[(int64_t)i * g.ld + plane_idx * g.plane + q];
}

int nblk_for(int64_t work) {
  int64_t b = (work + PT - 1) / PT;
  if (b > PMAXBLK) b = PMAXBLK;
  if (b < 1) b = 1;
  return (int)b;
}

// u holds the noise on entry; adds the Gaussian in the reference's operation
// order (no contraction: r2 and the exponent argument rounded step by step)
__global__ void __launch_bounds__(PT) init_orbitals_kernel(SlabGeom g, int N, double h0, double h1,
                                                           double h2,
                                                           const double* __restrict__ centers,
                                                           const double* __restrict__ widths,
                                                           double* __restrict__ u) {
  const int i = blockIdx.y;
  const double cx = centers[3 * i], cy = centers[3 * i + 1], cz = centers[3 * i + 2];
  const double w = widths[i];
  const double den = __dmul_rn(__dmul_rn(2.0, w), w);
  double* ui = u + (int64_t)i * g.ld;
  for (int64_t p = (int64_t)blockIdx.x * PT + threadIdx.x; p < g.ngl;
       p += (int64_t)gridDim.x * PT) {
    const int64_t k2 = p % g.n2;
    const int64_t k1 = (p / g.n2) % g.n1;
    const int64_t k0 = p / g.plane + g.z0;
    const double d0 = __dsub_rn(__dmul_rn((double)(k0 + 1), h0), cx);
    const double d1 = __dsub_rn(__dmul_rn((double)(k1 + 1), h1), cy);
    const double d2 = __dsub_rn(__dmul_rn((double)(k2 + 1), h2), cz);
    double r2 = __dmul_rn(d0, d0);
    r2 = __dadd_rn(r2, __dmul_rn(d1, d1));
    r2 = __dadd_rn(r2, __dmul_rn(d2, d2));
    ui[p] = __dadd_rn(exp(__ddiv_rn(-r2, den)), ui[p]);
  }
}

// one coarse line value with the reference's virtual end points (grid.cpp:178-189)
template <class L>
__device__ __forceinline__ double pline(int64_t i, int64_t n, L line) {
  if (i < 0) return n >= 2 ? __dsub_rn(__dmul_rn(2.0, line(0)), line(1)) : line(0);
  if (i >= n)
    return n >= 2 ? __dsub_rn(__dmul_rn(2.0, line(n - 1)), line(n - 2)) : line(n - 1);
  return line(i);
}

// fine index j of a line of n coarse values (grid.cpp:190-194)
template <class L>
__device__ __forceinline__ double pfine(int64_t j, int64_t n, L line) {
  if (j % 2 == 1) return pline((j - 1) / 2, n, line);
  return __dmul_rn(0.5, __dadd_rn(pline(j / 2 - 1, n, line), pline(j / 2, n, line)));
}

// Every fine value is the reference's three passes (axis 0, then 1, then 2)
// evaluated for that point only: the same operations on the same operands, so
// the result is bitwise that of prolongate().
__global__ void __launch_bounds__(PT) prolongate_kernel(int N, int64_t c0, int64_t c1, int64_t c2,
                                                        int64_t ldc, const double* __restrict__ C,
                                                        int64_t f0, int64_t f1, int64_t f2,
                                                        int64_t ldf, double* __restrict__ F) {
  const int i = blockIdx.y;
  const double* ci = C + (int64_t)i * ldc;
  double* fi = F + (int64_t)i * ldf;
  const int64_t nf = f0 * f1 * f2;
  for (int64_t q = (int64_t)blockIdx.x * PT + threadIdx.x; q < nf; q += (int64_t)gridDim.x * PT) {
    const int64_t j2 = q % f2, j1 = (q / f2) % f1, j0 = q / (f1 * f2);
    fi[q] = pfine(j2, c2, [&](int64_t k2) {
      return pfine(j1, c1, [&](int64_t k1) {
        return pfine(j0, c0, [&](int64_t k0) { return ci[(k0 * c1 + k1) * c2 + k2]; });
      });
    });
  }
}

}  // namespace

void launch_init_orbitals(const SlabGeom& g, int N, const double* h3, const double* centers,
                          const double* widths, double* u, cudaStream_t s) {
  dim3 grid(per_orbital_nblk(g, N), N);
  ::po::count_launch();
  init_orbitals_kernel<<<grid, PT, 0, s>>>(g, N, h3[0], h3[1], h3[2], centers, widths, u);
}

void launch_prolongate(int N, const int64_t nc[3], int64_t ldc, const double* C,
                       const int64_t nf[3], int64_t ldf, double* F, cudaStream_t s) {
  const int64_t total = nf[0] * nf[1] * nf[2];
  int64_t b = (total + PT - 1) / PT;
  if (b > 2048) b = 2048;
  dim3 grid((unsigned)b, N);
  ::po::count_launch();
  prolongate_kernel<<<grid, PT, 0, s>>>(N, nc[0], nc[1], nc[2], ldc, C, nf[0], nf[1], nf[2], ldf,
                                        F);
}

int points_nblk(const SlabGeom& g) { return nblk_for(g.ngl); }

// Per-orbital kernels use fewer CTAs per orbital so N * nblk stays ~ a few waves.
int per_orbital_nblk(const SlabGeom& g, int N) {
  int64_t target = (148 * 8 + N - 1) / N;
  if (target < 8) target = 8;
  int64_t b = (g.ngl + PT - 1) / PT;
  return (int)(b < target ? b : target);
}

void launch_density_xc(const SlabGeom& g, int N, const double* u, double occupation, int xc,
                       double* rho, double* v_xc, double* b, const double* v_ext, double* partials,
                       cudaStream_t s, const double* guard) {
  ::po::count_launch();
  launch_pdl(density_xc_kernel, dim3(points_nblk(g)), dim3(PT), 0, s, g, N, u, occupation, xc, rho, v_xc, b, v_ext,
                                                  partials, guard);
}

void launch_vlocal(const SlabGeom& g, const double* v_ext, const double* v_h_src, double* v_h,
                   double* v_xc, const double* rho, double* v_local, double* partials,
                   cudaStream_t s, int xc_here, const double* bfull, const double* xfull,
                   int* cg_out) {
  ::po::count_launch();
  launch_pdl(vlocal_kernel, dim3(points_nblk(g)), dim3(PT), 0, s, g, v_ext, v_h_src, v_h, v_xc, rho,
             v_local, partials, xc_here, bfull, xfull, cg_out);
}

void launch_residual_diag(const SlabGeom& g, int N, const double* u, const double* hu,
                          const double* sigma_diag, double* z, double* partials, cudaStream_t s) {
  dim3 grid(per_orbital_nblk(g, N), N);
  ::po::count_launch();
  residual_diag_kernel<<<grid, PT, 0, s>>>(g, N, u, hu, sigma_diag, z, partials);
}

void launch_residual_bb(const SlabGeom& g, int N, const double* u, const double* hu,
                        const double* sigma_diag, const double* up, const double* zp, double* z,
                        double* partials, cudaStream_t s) {
  dim3 grid(per_orbital_nblk(g, N), N);
  ::po::count_launch();
  residual_bb_kernel<<<grid, PT, 0, s>>>(g, N, u, hu, sigma_diag, up, zp, z, partials);
}

int launch_residual_bb_stream(const SlabGeom& g, int N, const double* u, const double* hu,
                              const double* sigma_diag, const double* up, const double* xp,
                              const double* sig_prev, double* z, double* partials, cudaStream_t s) {
  const int nb = per_orbital_nblk(g, N);
  dim3 grid(nb, N);
  ::po::count_launch();
  if (!up)
    launch_pdl(residual_bb_stream_kernel<false, false>, grid, dim3(PT), 0, s, g, N, u, hu, sigma_diag,
               up, xp, sig_prev, z, partials);
  else if (sig_prev)
    launch_pdl(residual_bb_stream_kernel<true, true>, grid, dim3(PT), 0, s, g, N, u, hu, sigma_diag, up,
               xp, sig_prev, z, partials);
  else
    launch_pdl(residual_bb_stream_kernel<true, false>, grid, dim3(PT), 0, s, g, N, u, hu, sigma_diag, up,
               xp, sig_prev, z, partials);
  return nb;
}

void launch_bb(const SlabGeom& g, int N, const double* w, const double* wp, const double* z,
               const double* zp, double* partials, cudaStream_t s) {
  dim3 grid(per_orbital_nblk(g, N), N);
  ::po::count_launch();
  bb_kernel<<<grid, PT, 0, s>>>(g, N, w, wp, z, zp, partials);
}

void launch_abs_sum(const SlabGeom& g, int N, const double* x, double* partials,
                    cudaStream_t s) {
  dim3 grid(per_orbital_nblk(g, N), N);
  ::po::count_launch();
  abs_sum_kernel<<<grid, PT, 0, s>>>(g, N, x, partials);
}

void launch_z_from_hw(const SlabGeom& g, int N, const double* w, const double* hw,
                      const double* sig, double* z, cudaStream_t s) {
  const int64_t total = (int64_t)N * g.ld;
  ::po::count_launch();
  z_from_hw_kernel<<<nblk_for(total), PT, 0, s>>>(total, g.ld, w, hw, sig, z);
}

void launch_lincomb(const SlabGeom& g, int N, const double* a, double sc, const double* b,
                    double* out, cudaStream_t s) {
  const int64_t total = (int64_t)N * g.ld;
  ::po::count_launch();
  lincomb_kernel<<<nblk_for(total), PT, 0, s>>>(total, a, sc, b, out);
}

void launch_reduce_rows(const double* partials, int rows, int nblk, double scale, double* out,
                        cudaStream_t s, const double* guard) {
  const int threads = 256;
  const int blocks = (rows * 32 + threads - 1) / threads;
  ::po::count_launch();
  launch_pdl(reduce_rows_kernel, dim3(blocks), dim3(threads), 0, s, partials, rows, nblk, scale, out, guard,
             0, 0.0, 0.0);
}

void launch_reduce_rows_grouped(const double* partials, int grp, int ngroups, int nblk,
                                const double* scales, double* out, cudaStream_t s, int rows) {
  if (rows <= 0) rows = grp * ngroups;
  const int threads = 256;
  const int blocks = (rows * 32 + threads - 1) / threads;
  ::po::count_launch();
  launch_pdl(reduce_rows_kernel, dim3(blocks), dim3(threads), 0, s, partials, rows, nblk, scales[0], out,
             (const double*)nullptr, grp, ngroups > 1 ? scales[1] : 0.0, ngroups > 2 ? scales[2] : 0.0);
}

void launch_external_potential(const SlabGeom& g, const double* h3, const double* atoms,
                               int natoms, int gaussian, double* v, cudaStream_t s) {
  ::po::count_launch();
  potential_kernel<<<points_nblk(g), PT, 0, s>>>(g, h3[0], h3[1], h3[2], atoms, natoms, gaussian,
                                                 v);
}

void launch_pack_plane(const SlabGeom& g, int N, const double* u, int64_t plane_idx, double* dst,
                       cudaStream_t s) {
  dim3 grid((unsigned)((g.plane + PT - 1) / PT), N);
  ::po::count_launch();
  pack_plane_kernel<<<grid, PT, 0, s>>>(g, N, u, plane_idx, dst);
}

}  // namespace po
