// Hartree Poisson solve -lap v = 4 pi rho (zero Dirichlet) on B200.
//
// Restates the reference's plain CG (energy.cpp:105-143): x0 = 0 (or a warm
// start), stop when ||r|| <= 1e-10 ||b||, <= 20000 iterations per pass, up to
// 3 restarts from the true residual b - A x, SolverError when p.Ap <= 0 or the
// tolerance is never met. The whole solve is ONE persistent cooperative
// kernel: no host round trip per iteration (the reference needs 158-790
// iterations per solve). Each iteration is two grid-wide phases:
//   phase 1: p <- r + beta p (recomputed at the 6 neighbours from r and the
//            previous p, so no extra barrier), Ap = -lap p, sum p.Ap;
//   phase 2: x += alpha p, r -= alpha Ap, sum r.r.
// Grid reductions: per-CTA partials, one grid barrier, then every CTA sums
// all partials in the same fixed order (identical alpha/beta everywhere,
// bitwise reproducible). The working fields (x, r, p, p', Ap) of a 96^3 grid
// are 35 MB — L2-resident on B200's 126 MB L2.
#include <math.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "kernels.h"

namespace po {

namespace {

constexpr int CT = 512;
int g_cg_blocks = 0;

struct CgArgs {
  int64_t n0, n1, n2, ng, plane;
  double ih0, ih1, ih2;
  const double* b;
  double* x;
  double* r;
  double* p0;
  double* p1;
  double* ap;
  double* red;       // 2 x gridDim.x partial slots
  unsigned* bar;     // [0] arrive counter, [1] generation
  int warm;
  int* out_i;        // {status, iters}
  double* out_d;     // {bnorm, final rel residual}
};

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Deterministic grid-wide sum; every CTA returns the same value.
__device__ double grid_sum(double v, const CgArgs& a, unsigned& slot, double* sh) {
  double vv[1] = {v};
  block_sum<1>(vv, sh);
  double* red = a.red + (slot & 1u) * gridDim.x;
  if (threadIdx.x == 0) red[blockIdx.x] = vv[0];
  ++slot;
  grid_barrier(a.bar, gridDim.x);
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += 32) s += __ldcg(red + k);
    s = warp_sum(s);
    if (threadIdx.x == 0) sh[32] = s;
  }
  __syncthreads();
  const double out = sh[32];
  __syncthreads();
  return out;
}

// Two deterministic grid-wide sums with one barrier.
__device__ void grid_sum2(double& v0, double& v1, const CgArgs& a, unsigned& slot, double* sh) {
  double vv[2] = {v0, v1};
  block_sum<2>(vv, sh);
  double* red = a.red + (slot & 1u) * 2 * gridDim.x;
  if (threadIdx.x == 0) {
    red[2 * blockIdx.x] = vv[0];
    red[2 * blockIdx.x + 1] = vv[1];
  }
  ++slot;
  grid_barrier(a.bar, gridDim.x);
  if (threadIdx.x < 32) {
    double s0 = 0.0, s1 = 0.0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += 32) {
      s0 += __ldcg(red + 2 * k);
      s1 += __ldcg(red + 2 * k + 1);
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (threadIdx.x == 0) {
      sh[64] = s0;
      sh[65] = s1;
    }
  }
  __syncthreads();
  v0 = sh[64];
  v1 = sh[65];
  __syncthreads();
}

// -lap f at point q (Dirichlet zero outside), f given by a functor of the index.
template <class F>
__device__ __forceinline__ double neg_lap(const CgArgs& a, int64_t q, F f) {
  const int64_t k2 = q % a.n2;
  const int64_t k1 = (q / a.n2) % a.n1;
  const int64_t k0 = q / a.plane;
  const double c = f(q);
  const double zm = k0 > 0 ? f(q - a.plane) : 0.0;
  const double zp = k0 + 1 < a.n0 ? f(q + a.plane) : 0.0;
  const double ym = k1 > 0 ? f(q - a.n2) : 0.0;
  const double yp = k1 + 1 < a.n1 ? f(q + a.n2) : 0.0;
  const double xm = k2 > 0 ? f(q - 1) : 0.0;
  const double xp = k2 + 1 < a.n2 ? f(q + 1) : 0.0;
  const double lap = ((zm - 2.0 * c + zp) * a.ih0 + (ym - 2.0 * c + yp) * a.ih1) +
                     (xm - 2.0 * c + xp) * a.ih2;
  return -lap;
}

__global__ void __launch_bounds__(CT) cg_kernel(CgArgs a) {
  __shared__ double sh[66];
  unsigned slot = 0;
  const int64_t stride = (int64_t)gridDim.x * CT;
  const int64_t t0 = (int64_t)blockIdx.x * CT + threadIdx.x;
  const double* __restrict__ b = a.b;
  double* __restrict__ x = a.x;
  double* __restrict__ r = a.r;
  double* __restrict__ ap = a.ap;

  // b norm and initial residual (one pass and one barrier for a warm start:
  // after the DST solve this is usually the whole kernel)
  double acc = 0.0, acc_r = 0.0;
  for (int64_t q = t0; q < a.ng; q += stride) {
    const double bq = b[q];
    if (!a.warm) {
      x[q] = 0.0;
    } else {
      const double rt = bq - neg_lap(a, q, [&](int64_t k) { return __ldcg(x + k); });
      r[q] = rt;
      acc_r += rt * rt;
    }
    acc += bq * bq;
  }
  double bb = acc, rr0 = acc_r;
  grid_sum2(bb, rr0, a, slot, sh);
  const double bnorm = sqrt(bb);
  if (bnorm == 0.0) {
    for (int64_t q = t0; q < a.ng; q += stride) x[q] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.out_i[0] = 0;
      a.out_i[1] = 0;
      a.out_d[0] = 0.0;
      a.out_d[1] = 0.0;
    }
    return;
  }
  const double thr = 1e-10 * bnorm;
  double rr;
  if (!a.warm) {
    for (int64_t q = t0; q < a.ng; q += stride) r[q] = b[q];
    rr = bb;  // r = b: same sum as b.b
  } else {
    rr = rr0;
    if (sqrt(rr) <= thr) {  // converged at iteration 0: the true residual is this one
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.out_i[0] = 0;
        a.out_i[1] = 0;
        a.out_d[0] = bnorm;
        a.out_d[1] = sqrt(rr) / bnorm;
      }
      return;
    }
  }
  int iters = 0, status = 3;
  double final_rr = rr;
  for (int pass = 0; pass <= 3; ++pass) {
    double* pold = a.p0;
    double* pnew = a.p1;
    double beta = 0.0;
    bool first = true;
    for (int it = 0; it < 20000; ++it) {
      if (sqrt(rr) <= thr) break;
      // phase 1
      acc = 0.0;
      for (int64_t q = t0; q < a.ng; q += stride) {
        double pq;
        double aq;
        if (first) {
          aq = neg_lap(a, q, [&](int64_t k) { return __ldcg(r + k); });
          pq = __ldcg(r + q);
        } else {
          aq = neg_lap(a, q, [&](int64_t k) { return __ldcg(r + k) + beta * __ldcg(pold + k); });
          pq = __ldcg(r + q) + beta * __ldcg(pold + q);
        }
        pnew[q] = pq;
        ap[q] = aq;
        acc += pq * aq;
      }
      const double pap = grid_sum(acc, a, slot, sh);
      if (!(pap > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
          a.out_i[0] = 3;
          a.out_i[1] = iters;
          a.out_d[0] = bnorm;
          a.out_d[1] = sqrt(rr) / bnorm;
        }
        return;
      }
      const double alpha = rr / pap;
      const double malpha = -alpha;
      // phase 2
      acc = 0.0;
      for (int64_t q = t0; q < a.ng; q += stride) {
        const double pq = pnew[q];
        x[q] += alpha * pq;
        const double rq = r[q] + malpha * ap[q];
        r[q] = rq;
        acc += rq * rq;
      }
      const double rr_new = grid_sum(acc, a, slot, sh);
      beta = rr_new / rr;
      rr = rr_new;
      double* t = pold;
      pold = pnew;
      pnew = t;
      first = false;
      ++iters;
    }
    // true residual b - A x (energy.cpp:136-141)
    acc = 0.0;
    for (int64_t q = t0; q < a.ng; q += stride) {
      const double rt = b[q] + -1.0 * neg_lap(a, q, [&](int64_t k) { return __ldcg(x + k); });
      r[q] = rt;
      acc += rt * rt;
    }
    rr = grid_sum(acc, a, slot, sh);
    final_rr = rr;
    if (sqrt(rr) <= thr) {
      status = 0;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out_i[0] = status;
    a.out_i[1] = iters;
    a.out_d[0] = bnorm;
    a.out_d[1] = sqrt(final_rr) / bnorm;
  }
}

}  // namespace

int cg_grid_blocks() {
  if (g_cg_blocks == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cg_kernel, CT, 0);
    if (per < 1) per = 1;
    if (per > 2) per = 2;
    g_cg_blocks = sms * per;
  }
  return g_cg_blocks;
}

size_t cg_workspace_doubles(int64_t ng) { return (size_t)4 * ng + 4 * 4096; }

void launch_cg(int64_t n0, int64_t n1, int64_t n2, const double ih2[3], const double* b,
               double* x, int warm, double* ws, unsigned* bar, int* out_i, double* out_d,
               cudaStream_t s) {
  CgArgs a;
  a.n0 = n0;
  a.n1 = n1;
  a.n2 = n2;
  a.plane = n1 * n2;
  a.ng = n0 * n1 * n2;
  a.ih0 = ih2[0];
  a.ih1 = ih2[1];
  a.ih2 = ih2[2];
  a.b = b;
  a.x = x;
  a.r = ws;
  a.p0 = ws + a.ng;
  a.p1 = ws + 2 * a.ng;
  a.ap = ws + 3 * a.ng;
  a.red = ws + 4 * a.ng;
  a.bar = bar;
  a.warm = warm;
  a.out_i = out_i;
  a.out_d = out_d;
  cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), s);
  const int blocks = cg_grid_blocks();
  void* args[] = {&a};
  ::po::count_launch();
  cudaLaunchCooperativeKernel((void*)cg_kernel, dim3(blocks), dim3(CT), args, 0, s);
}

}  // namespace po

// ===================================================================== DST
// Fast diagonalisation of the 7-point Dirichlet Laplacian (the same operator
// as grid.cpp:94-122): -lap_h = (S0 x S1 x S2) diag(lam) (S0 x S1 x S2) * c,
// S_a[j][k] = sin(pi (j+1)(k+1) / (n_a+1)), lam_a[j] = 4 sin^2(pi (j+1) /
// (2 (n_a+1))) / h_a^2, c = prod_a 2 / (n_a + 1). The six axis transforms are
// batched left-multiplies on the FP64 tensor cores (launch_mix_batched); the
// contiguous axis is brought to the middle by an in-plane transpose.
namespace po {

namespace {

constexpr int TT = 32;

// dst[b][c][r] = src[b][r][c] (r < rows, c < cols); dst[b][c][r] = 0 for rows <= r < dstride
__global__ void transpose_planes_kernel(const double* __restrict__ src, int64_t rows,
                                        int64_t cols, int64_t sstride, int64_t splane,
                                        double* __restrict__ dst, int64_t dstride,
                                        int64_t dplane) {
  __shared__ double tile[TT][TT + 1];
  const int64_t b = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.x * TT, c0 = (int64_t)blockIdx.y * TT;
  const double* sp = src + b * splane;
  double* dp = dst + b * dplane;
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (r < rows && c < cols) ? sp[r * sstride + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (c < cols && r < dstride) dp[c * dstride + r] = tile[threadIdx.x][k];
  }
}

// natural (unpadded) <-> natural padded rows
__global__ void pad_rows_kernel(const double* __restrict__ src, int64_t nrows, int64_t w,
                                int64_t sw, double* __restrict__ dst, int64_t dw) {
  const int64_t total = nrows * dw;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / dw, c = e % dw;
    dst[e] = c < w ? src[r * sw + c] : 0.0;
  }
}

__global__ void dst_scale_kernel(double* __restrict__ t, int64_t n0, int64_t n1, int64_t n2,
                                 int64_t n1p, const double* __restrict__ lam, double norm) {
  const int64_t total = n0 * n2 * n1p;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k1 = e % n1p;
    const int64_t k2 = (e / n1p) % n2;
    const int64_t k0 = e / (n1p * n2);
    if (k1 < n1) t[e] *= norm / ((lam[k0] + lam[n0 + k1]) + lam[n0 + n1 + k2]);
  }
}

int64_t rup32(int64_t x) { return (x + 31) / 32 * 32; }

}  // namespace

void DstPoisson::init(int64_t a0, int64_t a1, int64_t a2, const double h[3]) {
  n0 = a0;
  n1 = a1;
  n2 = a2;
  n1p = rup32(n1);
  n2p = rup32(n2);
  len = n0 * std::max(n1 * n2p, n2 * n1p);
  const int64_t ns[3] = {n0, n1, n2};
  std::vector<double> lam_h;
  const double pi = 3.141592653589793238462643383279502884;
  norm = 1.0;
  for (int a = 0; a < 3; ++a) {
    const int64_t n = ns[a];
    std::vector<double> S((size_t)(n * n));
    for (int64_t j = 0; j < n; ++j)
      for (int64_t k = 0; k < n; ++k)
        S[(size_t)(j * n + k)] = std::sin(pi * (double)((j + 1) * (k + 1) % (2 * (n + 1))) /
                                          (double)(n + 1));
    cudaMalloc(&this->S[a], sizeof(double) * n * n);
    cudaMemcpy(this->S[a], S.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    for (int64_t j = 0; j < n; ++j) {
      const double sn = std::sin(pi * (double)(j + 1) / (2.0 * (double)(n + 1)));
      lam_h.push_back(4.0 * sn * sn / (h[a] * h[a]));
    }
    norm *= 2.0 / (double)(n + 1);
  }
  cudaMalloc(&lam, sizeof(double) * lam_h.size());
  cudaMemcpy(lam, lam_h.data(), sizeof(double) * lam_h.size(), cudaMemcpyHostToDevice);
  if (dst_fused_supported(n0, n1, n2)) {  // spectral factors of the plane kernel, same rounding
    std::vector<double> sc((size_t)(n0 * n1 * n2));
    for (int64_t k0 = 0; k0 < n0; ++k0)
      for (int64_t k1 = 0; k1 < n1; ++k1)
        for (int64_t k2 = 0; k2 < n2; ++k2)
          sc[(size_t)((k0 * n1 + k1) * n2 + k2)] =
              norm / ((lam_h[(size_t)k0] + lam_h[(size_t)(n0 + k1)]) + lam_h[(size_t)(n0 + n1 + k2)]);
    cudaMalloc(&scale, sizeof(double) * sc.size());
    cudaMemcpy(scale, sc.data(), sizeof(double) * sc.size(), cudaMemcpyHostToDevice);
  }
  cudaMalloc(&t0, sizeof(double) * len);
  cudaMalloc(&t1, sizeof(double) * len);
  cudaMemset(t0, 0, sizeof(double) * len);
  cudaMemset(t1, 0, sizeof(double) * len);
}

void DstPoisson::release() {
  for (auto& s : S)
    if (s) cudaFree(s), s = nullptr;
  if (lam) cudaFree(lam), lam = nullptr;
  if (scale) cudaFree(scale), scale = nullptr;
  if (t0) cudaFree(t0), t0 = nullptr;
  if (t1) cudaFree(t1), t1 = nullptr;
}

void DstPoisson::solve(const double* b, double* x, cudaStream_t s) {
  if (launch_dst_fused(*this, b, x, s)) return;
  const int64_t pn = n1 * n2p;  // natural padded plane
  const int64_t pt = n2 * n1p;  // transposed padded plane
  const dim3 tb(TT, 8);
  auto blocks = [](int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16); };
  // b -> t0 (natural padded)
  ::po::count_launch();
  pad_rows_kernel<<<blocks(n0 * n1 * n2p), 256, 0, s>>>(b, n0 * n1, n2, n2, t0, n2p);
  // forward: axis 0, axis 1, transpose, axis 2
  launch_mix_batched((int)n0, pn, pn, 1, 0, t0, S[0], t1, s);
  launch_mix_batched((int)n1, n2p, n2p, (int)n0, pn, t1, S[1], t0, s);
  ::po::count_launch();
  transpose_planes_kernel<<<dim3((unsigned)((n1p + TT - 1) / TT), (unsigned)((n2 + TT - 1) / TT),
                                 (unsigned)n0), tb, 0, s>>>(t0, n1, n2, n2p, pn, t1, n1p, pt);
  launch_mix_batched((int)n2, n1p, n1p, (int)n0, pt, t1, S[2], t0, s);
  ::po::count_launch();
  dst_scale_kernel<<<blocks(n0 * pt), 256, 0, s>>>(t0, n0, n1, n2, n1p, lam, norm);
  // inverse: axis 2, transpose back, axis 1, axis 0
  launch_mix_batched((int)n2, n1p, n1p, (int)n0, pt, t0, S[2], t1, s);
  ::po::count_launch();
  transpose_planes_kernel<<<dim3((unsigned)((n2p + TT - 1) / TT), (unsigned)((n1 + TT - 1) / TT),
                                 (unsigned)n0), tb, 0, s>>>(t1, n2, n1, n1p, pt, t0, n2p, pn);
  launch_mix_batched((int)n1, n2p, n2p, (int)n0, pn, t0, S[1], t1, s);
  launch_mix_batched((int)n0, pn, pn, 1, 0, t1, S[0], t0, s);
  ::po::count_launch();
  pad_rows_kernel<<<blocks(n0 * n1 * n2), 256, 0, s>>>(t0, n0 * n1, n2, n2p, x, n2);
}

}  // namespace po
