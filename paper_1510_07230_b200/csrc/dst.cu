// Three-kernel DST-I Poisson solve for grids up to 128 points per axis.
//
// -lap_h = (S0 x S1 x S2) diag(lam) (S0 x S1 x S2) * c (see poisson.cu). The
// axis-1/axis-2 transforms, the spectral scaling and their inverses are all
// local to one axis-0 plane once the axis-0 transform is done, so the solve is
//   axis-0 GEMM (b -> t)  ->  per-plane kernel in shared memory
//   (t_k0 <- S1 [ (S1 t_k0 S2) ./ (lam0[k0] + lam1 + lam2) * c ] S2)
//   ->  axis-0 GEMM (t -> x)
// with no transposes, no padding passes and the working set (the grid, a few
// MB) resident in L2. All products are FP64 mma.sync.m8n8k4 (DMMA); the plane
// lives in shared memory with a row stride of (n8 + 4) doubles, which keeps
// both fragment shapes (8 rows x 4 k, 4 k x 8 cols) bank-conflict free.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"

namespace po {

namespace {

// S[j][k]: from global (zero outside n x n) or from a zero-padded smem copy (stride ss)
template <bool SG>
__device__ __forceinline__ double sld(const double* S, int ss, int n, int j, int k) {
  if constexpr (SG) return (j < n && k < n) ? __ldg(S + j * n + k) : 0.0;
  else return S[j * ss + k];
}

// warp grid WR x WC over the fragment tiles; warp (wr, wc) owns row frags
// wr*RB.. and col frags wc*CB..
template <int WC>
__device__ __forceinline__ void warp_pos(int& wr, int& wc) {
  const int warp = threadIdx.x >> 5;
  wr = warp / WC;
  wc = warp % WC;
}

// acc(r, c) = sum_k X[r][k] S[k][c]  (X in smem, stride ps)
template <int RB, int CB, int WC, bool SG>
__device__ __forceinline__ void mul_right(const double* X, int ps, const double* S, int ss, int n,
                                          int nf, double (&acc)[RB][CB][2]) {
  const int lane = threadIdx.x & 31, gq = lane >> 2, t4 = lane & 3;
  int wr, wc;
  warp_pos<WC>(wr, wc);
#pragma unroll
  for (int a = 0; a < RB; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nks = (n + 3) / 4;
  for (int ks = 0; ks < nks; ++ks) {
    const int k = 4 * ks + t4;
    double af[RB], bf[CB];
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      const int rf = wr * RB + a;
      af[a] = rf < nf ? X[(8 * rf + gq) * ps + k] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int cf = wc * CB + b;
      bf[b] = cf < nf ? sld<SG>(S, ss, n, k, 8 * cf + gq) : 0.0;
    }
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
      for (int b = 0; b < CB; ++b) dmma_8x8x4(acc[a][b], af[a], bf[b]);
  }
}

// acc(j, c) = sum_k S[j][k] X[k][c]
template <int RB, int CB, int WC, bool SG>
__device__ __forceinline__ void mul_left(const double* X, int ps, const double* S, int ss, int n,
                                         int nf, double (&acc)[RB][CB][2]) {
  const int lane = threadIdx.x & 31, gq = lane >> 2, t4 = lane & 3;
  int wr, wc;
  warp_pos<WC>(wr, wc);
#pragma unroll
  for (int a = 0; a < RB; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nks = (n + 3) / 4;
  for (int ks = 0; ks < nks; ++ks) {
    const int k = 4 * ks + t4;
    double af[RB], bf[CB];
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      const int rf = wr * RB + a;
      af[a] = rf < nf ? sld<SG>(S, ss, n, 8 * rf + gq, k) : 0.0;
    }
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int cf = wc * CB + b;
      bf[b] = cf < nf ? X[k * ps + 8 * cf + gq] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
      for (int b = 0; b < CB; ++b) dmma_8x8x4(acc[a][b], af[a], bf[b]);
  }
}

// write the warp's tiles back into the plane (zero outside the nr x nc interior),
// optionally times the spectral scale c / (lam0[k0] + lam1[r] + lam2[c])
template <int RB, int CB, int WC>
__device__ __forceinline__ void store_tiles(double* X, int ps, int nr, int nc, int nf,
                                            const double (&acc)[RB][CB][2],
                                            const double* __restrict__ scale) {
  const int lane = threadIdx.x & 31, gq = lane >> 2, t4 = lane & 3;
  int wr, wc;
  warp_pos<WC>(wr, wc);
#pragma unroll
  for (int a = 0; a < RB; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int rf = wr * RB + a, cf = wc * CB + b;
      if (rf >= nf || cf >= nf) continue;
      const int r = 8 * rf + gq;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = 8 * cf + 2 * t4 + j;
        double v = acc[a][b][j];
        if (scale && r < nr && c < nc) v *= __ldg(scale + r * nc + c);
        X[r * ps + c] = (r < nr && c < nc) ? v : 0.0;
      }
    }
}

// copy an n x n matrix into a zero-padded [n8][n8 + 4] smem array
__device__ __forceinline__ void load_s(double* dst, const double* __restrict__ S, int n, int n8) {
  const int ps = n8 + 4;
  for (int e = threadIdx.x; e < n8 * ps; e += blockDim.x) {
    const int j = e / ps, k = e % ps;
    dst[e] = (j < n && k < n) ? S[j * n + k] : 0.0;
  }
}

// one CTA (16 warps, 4 x 4 warp grid) per axis-0 plane k0 (already transformed
// along axis 0). SG: DST matrices read from global/L1 (planes too large to
// also hold them in shared memory, or n1 != n2).
constexpr int PW = 16;
template <int NF, bool SG>
__global__ void __launch_bounds__(PW * 32) dst_plane_kernel(double* __restrict__ t, int n0, int n1,
                                                            int n2, const double* __restrict__ S1,
                                                            const double* __restrict__ S2,
                                                            const double* __restrict__ scale) {
  PO_PDL_ENTRY();
  constexpr int WC = 4, RB = (NF + 3) / 4, CB = (NF + WC - 1) / WC;
  extern __shared__ double dsm[];
  const int nf = (max(n1, n2) + 7) / 8;
  const int n8 = 8 * nf;
  const int ps = n8 + 4;
  double* X = dsm;  // [n8][ps]
  const double* s1 = S1;
  const double* s2 = S2;
  if constexpr (!SG) {  // n1 == n2: one shared copy serves both axes
    double* Ss = dsm + n8 * ps;
    load_s(Ss, S1, n1, n8);
    s1 = s2 = Ss;
  }
  const int k0 = blockIdx.x;
  double* tp = t + (int64_t)k0 * n1 * n2;
  for (int e = threadIdx.x; e < n8 * ps; e += blockDim.x) {
    const int r = e / ps, c = e % ps;
    X[e] = (r < n1 && c < n2) ? tp[r * n2 + c] : 0.0;
  }
  __syncthreads();
  double acc[RB][CB][2];
  // forward: axis 2 (X S2), axis 1 (S1 X) + spectral scale; inverse: axis 1, axis 2
  mul_right<RB, CB, WC, SG>(X, ps, s2, ps, n2, nf, acc);
  __syncthreads();
  store_tiles<RB, CB, WC>(X, ps, n1, n2, nf, acc, nullptr);
  __syncthreads();
  mul_left<RB, CB, WC, SG>(X, ps, s1, ps, n1, nf, acc);
  __syncthreads();
  store_tiles<RB, CB, WC>(X, ps, n1, n2, nf, acc, scale + (int64_t)k0 * n1 * n2);
  __syncthreads();
  mul_left<RB, CB, WC, SG>(X, ps, s1, ps, n1, nf, acc);
  __syncthreads();
  store_tiles<RB, CB, WC>(X, ps, n1, n2, nf, acc, nullptr);
  __syncthreads();
  mul_right<RB, CB, WC, SG>(X, ps, s2, ps, n2, nf, acc);
  __syncthreads();
  store_tiles<RB, CB, WC>(X, ps, n1, n2, nf, acc, nullptr);
  __syncthreads();
  for (int e = threadIdx.x; e < n1 * n2; e += blockDim.x) tp[e] = X[(e / n2) * ps + e % n2];
}

// y[j][p] = sum_k S0[j][k] x[k][p] over a 32-point column tile of the planes
constexpr int AW = 8;
template <int NF, bool SG, int A0P>
__global__ void __launch_bounds__(AW * 32) dst_axis0_kernel(const double* __restrict__ x,
                                                            double* __restrict__ y, int n0,
                                                            int64_t plane,
                                                            const double* __restrict__ S0) {
  PO_PDL_ENTRY();
  constexpr int WC = 2, RB = (NF + 3) / 4, CB = A0P / 8 / WC;
  extern __shared__ double dsm[];
  constexpr int xs = A0P + 4;
  const int nf = (n0 + 7) / 8;
  const int n8 = 8 * nf;
  double* X = dsm;  // [n8][xs]
  const double* s0 = S0;
  if constexpr (!SG) {
    double* Ss = dsm + n8 * xs;
    load_s(Ss, S0, n0, n8);
    s0 = Ss;
  }
  const int64_t p0 = (int64_t)blockIdx.x * A0P;
  for (int e = threadIdx.x; e < n8 * A0P; e += blockDim.x) {
    const int k = e / A0P, c = e % A0P;
    X[k * xs + c] = (k < n0 && p0 + c < plane) ? x[(int64_t)k * plane + p0 + c] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, gq = lane >> 2, t4 = lane & 3;
  int wr, wc;
  warp_pos<WC>(wr, wc);
  double acc[RB][CB][2];
#pragma unroll
  for (int a = 0; a < RB; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nks = (n0 + 3) / 4;
  // unrolled by 4: the S / X fragment loads of later k-steps issue ahead of the
  // DMMAs (a k-step at a time exposed the L1 / shared-memory latency)
#pragma unroll 4
  for (int ks = 0; ks < nks; ++ks) {
    const int k = 4 * ks + t4;
    double af[RB], bf[CB];
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      const int rf = wr * RB + a;
      af[a] = rf < nf ? sld<SG>(s0, n8 + 4, n0, 8 * rf + gq, k) : 0.0;
    }
#pragma unroll
    for (int b = 0; b < CB; ++b) bf[b] = X[k * xs + 8 * (wc * CB + b) + gq];
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
      for (int b = 0; b < CB; ++b) dmma_8x8x4(acc[a][b], af[a], bf[b]);
  }
#pragma unroll
  for (int a = 0; a < RB; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int j = 8 * (wr * RB + a) + gq;
      const int64_t p = p0 + 8 * (wc * CB + b) + 2 * t4;
      if (j < n0) {
        double* yp = y + (int64_t)j * plane + p;
        if (p + 1 < plane && (plane & 1) == 0) {  // 16-B aligned only for even planes
          *reinterpret_cast<double2*>(yp) = make_double2(acc[a][b][0], acc[a][b][1]);
        } else {
          if (p < plane) yp[0] = acc[a][b][0];
          if (p + 1 < plane) yp[1] = acc[a][b][1];
        }
      }
    }
}

constexpr size_t kSmemMax = 227 * 1024;

template <int NF, int A0P, bool ASG>
void launch_axis0(const DstPoisson& d, const double* x, double* y, cudaStream_t s) {
  const int64_t plane = d.n1 * d.n2;
  const int n80 = 8 * (int)((d.n0 + 7) / 8);
  const size_t sh0 = sizeof(double) * n80 * (A0P + 4) + (ASG ? 0 : sizeof(double) * n80 * (n80 + 4));
  auto ka = dst_axis0_kernel<NF, ASG, A0P>;
  set_smem(reinterpret_cast<const void*>(ka), (int)sh0);
  ::po::count_launch();
  launch_pdl(ka, dim3((unsigned)((plane + A0P - 1) / A0P)), dim3(AW * 32), sh0, s, x, y, (int)d.n0, plane, d.S[0]);
}

template <int NF>
void launch_axis0_pick(const DstPoisson& d, const double* x, double* y, cudaStream_t s) {
  static int cfg = -1;
  if (cfg < 0) {
    const char* e = getenv("PO_DST_A0");  // measurement override: 0..5
    cfg = e ? atoi(e) : 2;  // measured best at 96^3: 32-point tiles, S0 through L1
  }
  switch (cfg) {
    case 0: launch_axis0<NF, 32, false>(d, x, y, s); break;
    case 2: launch_axis0<NF, 32, true>(d, x, y, s); break;
    case 3: launch_axis0<NF, 64, true>(d, x, y, s); break;
    case 4: launch_axis0<NF, 128, false>(d, x, y, s); break;
    case 5: launch_axis0<NF, 128, true>(d, x, y, s); break;
    default: launch_axis0<NF, 64, false>(d, x, y, s); break;
  }
}


// Column-split form of the per-plane transforms for n1 == n2 <= 96: the plane's
// work (four n^3 DMMA GEMMs on one CTA per plane = 96 of 148 SMs at 96^3) runs
// as two launches of (32-column part, plane) CTAs, two per SM (S from L1):
//   out[:, cols] = [scale .] S1 (in S2[:, cols])
// first on the axis-0-transformed plane (t0 -> t1, with the spectral scale),
// then on the scaled plane (t1 -> t0). Each part needs the whole input plane
// but only its own columns of the intermediate, so no CTA waits on another.
constexpr int PP = 32;  // columns per part
template <int NF>
__global__ void __launch_bounds__(256, 2) dst_plane_part_kernel(const double* __restrict__ in,
                                                               double* __restrict__ out, int n,
                                                               const double* __restrict__ S1,
                                                               const double* __restrict__ S2,
                                                               const double* __restrict__ scale) {
  PO_PDL_ENTRY();
  constexpr int RB = NF / 4, CB = 2;  // 8 warps: 4 row groups x 2 column groups
  extern __shared__ double dsm[];
  const int n8 = 8 * NF, ps = n8 + 4, qs = PP + 4;
  double* X = dsm;              // [n8][ps]: the input plane
  double* P = dsm + n8 * ps;    // [n8][qs]: in S2[:, cols]
  const int c0 = blockIdx.x * PP, k0 = blockIdx.y;
  const double* ip = in + (int64_t)k0 * n * n;
  for (int e = threadIdx.x; e < n8 * ps; e += blockDim.x) {
    const int r = e / ps, c = e % ps;
    X[e] = (r < n && c < n) ? ip[r * n + c] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, gq = lane >> 2, t4 = lane & 3;
  const int warp = threadIdx.x >> 5, wr = warp >> 1, wc = warp & 1;
  const int nks = (n + 3) / 4;
  double acc[RB][CB][2];
  // P = X S2[:, c0 + ...]
#pragma unroll
  for (int a = 0; a < RB; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int ks = 0; ks < nks; ++ks) {
    const int k = 4 * ks + t4;
    double af[RB], bf[CB];
#pragma unroll
    for (int a = 0; a < RB; ++a) af[a] = X[(8 * (wr * RB + a) + gq) * ps + k];
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const int col = c0 + 8 * (wc * CB + b) + gq;
      bf[b] = (k < n && col < n) ? __ldg(S2 + k * n + col) : 0.0;
    }
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
      for (int b = 0; b < CB; ++b) dmma_8x8x4(acc[a][b], af[a], bf[b]);
  }
#pragma unroll
  for (int a = 0; a < RB; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        P[(8 * (wr * RB + a) + gq) * qs + 8 * (wc * CB + b) + 2 * t4 + j] = acc[a][b][j];
  __syncthreads();
  // out[:, cols] = S1 P
#pragma unroll
  for (int a = 0; a < RB; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int ks = 0; ks < nks; ++ks) {
    const int k = 4 * ks + t4;
    double af[RB], bf[CB];
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      const int row = 8 * (wr * RB + a) + gq;
      af[a] = (row < n && k < n) ? __ldg(S1 + row * n + k) : 0.0;
    }
#pragma unroll
    for (int b = 0; b < CB; ++b) bf[b] = P[k * qs + 8 * (wc * CB + b) + gq];
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
      for (int b = 0; b < CB; ++b) dmma_8x8x4(acc[a][b], af[a], bf[b]);
  }
  double* op = out + (int64_t)k0 * n * n;
  const double* sp = scale ? scale + (int64_t)k0 * n * n : nullptr;
#pragma unroll
  for (int a = 0; a < RB; ++a)
#pragma unroll
    for (int b = 0; b < CB; ++b)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = 8 * (wr * RB + a) + gq, c = c0 + 8 * (wc * CB + b) + 2 * t4 + j;
        if (r < n && c < n) {
          double v = acc[a][b][j];
          if (sp) v *= __ldg(sp + r * n + c);
          op[r * n + c] = v;
        }
      }
}

template <int NF>
void launch_plane_parts(const DstPoisson& d, cudaStream_t s) {
  const int n = (int)d.n1, n8 = 8 * NF;
  const size_t sh = sizeof(double) * ((size_t)n8 * (n8 + 4) + (size_t)n8 * (PP + 4));
  auto k = dst_plane_part_kernel<NF>;
  set_smem(reinterpret_cast<const void*>(k), (int)sh);
  const dim3 grid((unsigned)((n + PP - 1) / PP), (unsigned)d.n0);
  ::po::count_launch();
  launch_pdl(k, grid, dim3(256), sh, s, (const double*)d.t0, d.t1, n, (const double*)d.S[1],
             (const double*)d.S[2], (const double*)d.scale);
  ::po::count_launch();
  launch_pdl(k, grid, dim3(256), sh, s, (const double*)d.t1, d.t0, n, (const double*)d.S[1],
             (const double*)d.S[2], (const double*)nullptr);
}

template <int NF>
void launch_fused(const DstPoisson& d, const double* b, double* x, cudaStream_t s) {
  const int n8 = 8 * (int)((std::max(d.n1, d.n2) + 7) / 8);
  const size_t pl = sizeof(double) * n8 * (n8 + 4);
  const bool p_sg = d.n1 != d.n2 || 2 * pl > kSmemMax;
  const size_t sh1 = p_sg ? pl : 2 * pl;
  auto kp = p_sg ? dst_plane_kernel<NF, true> : dst_plane_kernel<NF, false>;
  set_smem(reinterpret_cast<const void*>(kp), (int)sh1);
  launch_axis0_pick<NF>(d, b, d.t0, s);
  static const int parts_env = getenv("PO_DST_PARTS") ? atoi(getenv("PO_DST_PARTS")) : 1;  // measurement
  if (parts_env && NF <= 12 && d.n1 == d.n2 && d.n1 > 8 * (NF - 4)) {
    launch_plane_parts<NF>(d, s);
  } else {
    ::po::count_launch();
    launch_pdl(kp, dim3((unsigned)d.n0), dim3(PW * 32), sh1, s, d.t0, (int)d.n0, (int)d.n1, (int)d.n2, d.S[1],
               d.S[2], d.scale);
  }
  launch_axis0_pick<NF>(d, d.t0, x, s);
}

}  // namespace

bool dst_fused_supported(int64_t n0, int64_t n1, int64_t n2) {
  return n0 <= 128 && n1 <= 128 && n2 <= 128;
}

bool launch_dst_fused(const DstPoisson& d, const double* b, double* x, cudaStream_t s) {
  if (!dst_fused_supported(d.n0, d.n1, d.n2)) return false;
  const int64_t m = std::max(d.n0, std::max(d.n1, d.n2));
  if (m <= 64)
    launch_fused<8>(d, b, x, s);
  else if (m <= 96)
    launch_fused<12>(d, b, x, s);
  else
    launch_fused<16>(d, b, x, s);
  return true;
}

}  // namespace po
