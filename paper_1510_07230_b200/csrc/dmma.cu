// FP64 tensor-core contractions for the orbital block (sm_100a).
//
// tcgen05.mma has no f64 kind on sm_100a, so FP64 tensor math is the warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4). Two contractions dominate the
// orthonormalisation step of the reference:
//   gram  (manifold.cpp:41-61): G = w U^T V, a tall-skinny SYRK/GEMM with
//         K = N_g up to 7e6 -> split-K over grid points, deterministic
//         fixed-order reduction of the per-split partials;
//   mix   (manifold.cpp:67-85): out = U M, (N_g x N)(N x N) — the rotation
//         U L^{-T}, the residual HU - U Sigma and the subspace rotation W P.
// Both stage tiles through shared memory with register double-buffering
// (global loads of stage s+1 are in flight while stage s feeds the DMMAs).
// Fusions: the trial point W - tau Z is formed while loading (no trial block
// is ever written), and mix can add beta*C and emit per-orbital squared norms
// of its result instead of storing it (grad-norm of HU - U Sigma).
#include <cstdlib>

#include "kernels.h"

namespace po {

namespace {

// ------------------------------------------------------------------- Gram
constexpr int GB = 64;     // output tile (GB x GB)
constexpr int GK = 32;     // points per stage
constexpr int GKP = GK + 4;  // smem row stride (doubles): conflict-free fragment reads
constexpr int GT = 256;    // 8 warps: 4 along m x 2 along n, warp tile 16 x 32

struct GramPlan {
  int mt;       // tiles per side
  int ntiles;   // tiles computed (upper only if sym)
  int nsplit;   // K splits
  int64_t kchunk;
};

GramPlan gram_plan(const SlabGeom& g, int N, int sym) {
  GramPlan p;
  p.mt = (N + GB - 1) / GB;
  p.ntiles = sym ? p.mt * (p.mt + 1) / 2 : p.mt * p.mt;
  const int target = 148 * 3;
  int ns = (target + p.ntiles - 1) / p.ntiles;
  const int64_t kb = (g.ld + GK - 1) / GK;  // K blocks
  if (ns > kb) ns = (int)kb;
  if (ns < 1) ns = 1;
  p.kchunk = ((kb + ns - 1) / ns) * GK;
  p.nsplit = (int)((g.ld + p.kchunk - 1) / p.kchunk);
  return p;
}

__device__ __forceinline__ void tile_index(int t, int mt, int sym, int& tm, int& tn) {
  if (!sym) {
    tm = t / mt;
    tn = t % mt;
    return;
  }
  // enumerate upper triangle row by row
  int r = 0, rem = t;
  while (rem >= mt - r) {
    rem -= mt - r;
    ++r;
  }
  tm = r;
  tn = r + rem;
}

// Load a GB x GK tile of (X + s Xb) rows [r0, r0+GB), points [k0, k0+GK) into regs.
__device__ __forceinline__ void gram_load(double (&reg)[8], const double* X, const double* Xb,
                                          double s, int N, int64_t ld, int r0, int64_t k0,
                                          int64_t kend) {
  const int t = threadIdx.x;
  const int row = t >> 2;           // 0..63
  const int c0 = (t & 3) * 8;       // 0, 8, 16, 24
  const int r = r0 + row;
  const int64_t k = k0 + c0;
  if (r < N && k < kend) {          // kend is a multiple of 8 (ld padded to 32)
    const double2* src = reinterpret_cast<const double2*>(X + (int64_t)r * ld + k);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double2 v = __ldg(src + j);
      reg[2 * j] = v.x;
      reg[2 * j + 1] = v.y;
    }
    if (Xb) {
      const double2* sb = reinterpret_cast<const double2*>(Xb + (int64_t)r * ld + k);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double2 v = __ldg(sb + j);
        reg[2 * j] += s * v.x;
        reg[2 * j + 1] += s * v.y;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) reg[j] = 0.0;
  }
}

__device__ __forceinline__ void gram_store(const double (&reg)[8], double* S) {
  const int t = threadIdx.x;
  const int row = t >> 2;
  const int c0 = (t & 3) * 8;
#pragma unroll
  for (int j = 0; j < 8; ++j) S[row * GKP + c0 + j] = reg[j];
}

__global__ void __launch_bounds__(GT) gram_kernel(int N, int64_t ld, int64_t kchunk, int mt,
                                                  int sym, const double* __restrict__ A,
                                                  const double* __restrict__ Ab, double sa,
                                                  const double* __restrict__ B,
                                                  const double* __restrict__ Bb, double sb,
                                                  double* __restrict__ ws,
    const double* __restrict__ guard) {
  if (guard && *guard == 0.0) return;  // device-side branch (CholeskyQR2 repair)
  extern __shared__ __align__(16) double gsm[];
  double (*As)[GB * GKP] = reinterpret_cast<double (*)[GB * GKP]>(gsm);
  double (*Bs)[GB * GKP] = reinterpret_cast<double (*)[GB * GKP]>(gsm + 2 * GB * GKP);
  int tm, tn;
  tile_index(blockIdx.x, mt, sym, tm, tn);
  const int m0 = tm * GB, n0 = tn * GB;
  const int64_t kbeg = (int64_t)blockIdx.y * kchunk;
  const int64_t kend = min(kbeg + kchunk, ld);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 1, wn = warp & 1;  // 4 x 2 warps
  const int gq = lane >> 2, t4 = lane & 3;
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  double ra[8], rb[8];
  const bool same = sym && tm == tn;
  gram_load(ra, A, Ab, sa, N, ld, m0, kbeg, kend);
  if (!same) gram_load(rb, B, Bb, sb, N, ld, n0, kbeg, kend);
  int buf = 0;
  for (int64_t k0 = kbeg; k0 < kend; k0 += GK) {
    gram_store(ra, As[buf]);
    gram_store(same ? ra : rb, Bs[buf]);
    __syncthreads();
    if (k0 + GK < kend) {  // prefetch next stage into registers
      gram_load(ra, A, Ab, sa, N, ld, m0, k0 + GK, kend);
      if (!same) gram_load(rb, B, Bb, sb, N, ld, n0, k0 + GK, kend);
    }
    const double* as = As[buf];
    const double* bs = Bs[buf];
#pragma unroll
    for (int kk = 0; kk < GK / 4; ++kk) {
      double af[2], bf[4];
#pragma unroll
      for (int fm = 0; fm < 2; ++fm) af[fm] = as[(wm * 16 + fm * 8 + gq) * GKP + kk * 4 + t4];
#pragma unroll
      for (int fn = 0; fn < 4; ++fn) bf[fn] = bs[(wn * 32 + fn * 8 + gq) * GKP + kk * 4 + t4];
#pragma unroll
      for (int fm = 0; fm < 2; ++fm)
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) dmma_8x8x4(acc[fm][fn], af[fm], bf[fn]);
    }
    buf ^= 1;
  }
  // partial tile -> ws[split][tile][GB][GB]
  double* out = ws + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (GB * GB);
#pragma unroll
  for (int fm = 0; fm < 2; ++fm)
#pragma unroll
    for (int fn = 0; fn < 4; ++fn) {
      const int r = wm * 16 + fm * 8 + gq;
      const int c = wn * 32 + fn * 8 + 2 * t4;
      out[r * GB + c] = acc[fm][fn][0];
      out[r * GB + c + 1] = acc[fm][fn][1];
    }
}

__global__ void gram_reduce_kernel(int N, int mt, int sym, int ntiles, int nsplit, double w,
                                   const double* __restrict__ ws, double* __restrict__ G,
    const double* __restrict__ guard) {
  if (guard && *guard == 0.0) return;  // device-side branch (CholeskyQR2 repair)
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)N * N) return;
  int i = (int)(e / N), j = (int)(e % N);
  if (sym && j < i) {
    const int t = i;
    i = j;
    j = t;
  }
  const int tm = i / GB, tn = j / GB;
  int tile;
  if (!sym) {
    tile = tm * mt + tn;
  } else {
    tile = 0;
    for (int r = 0; r < tm; ++r) tile += mt - r;
    tile += tn - tm;
  }
  const int r = i - tm * GB, c = j - tn * GB;
  double s = 0.0;
  for (int k = 0; k < nsplit; ++k) s += ws[((int64_t)k * ntiles + tile) * (GB * GB) + r * GB + c];
  G[e] = w * s;
}

// ------------------------------------------- small-N streaming kernels (N <= 56)
// Tall-skinny contractions for small N, fed by plain vectorised loads.
// Measured on B200 (profiles/r1_tma_probe.txt): 1D TMA bulk copies are
// request-rate bound (512 B rows -> 2.1 TB/s, 1 KB -> 4.0 TB/s, 2 KB -> 6.2 TB/s
// whatever the ring depth), and a stage of N rows x 2 KB does not fit a
// multi-stage ring, whereas vectorised LDG with several CTAs per SM reaches
// 6.2-6.4 TB/s. So each CTA streams its point range in 64-point stages:
// all 256 threads prefetch the next stage (double2 per row, rows x 64 points,
// the trial combination W - tau Z formed on the fly) into registers while the
// DMMAs run on the current stage in shared memory. Warp w owns points
// [8w, 8w + 8) of a stage; the row stride of 72 doubles (16 words mod 32)
// keeps the fragment reads conflict-free.
constexpr int SK = 64;
constexpr int SKP = SK + 8;
constexpr int ST = 256;

template <int F, bool SYM>
struct SmallPairs {
  static constexpr int NP = SYM ? F * (F + 1) / 2 : F * F;
};

template <int NPAD>
struct Tile {
  static constexpr int NV = (NPAD * (SK / 2) + ST - 1) / ST;  // double2 per thread per tile
};

template <int NPAD>
__device__ __forceinline__ void tile_load(double2 (&v)[Tile<NPAD>::NV], const double* X,
                                          const double* Xb, double s, int N, int64_t ld,
                                          int64_t k0, int64_t kend) {
#pragma unroll
  for (int j = 0; j < Tile<NPAD>::NV; ++j) {
    const int e = threadIdx.x + j * ST;
    const int row = e / (SK / 2), c2 = e % (SK / 2);
    const int64_t k = k0 + 2 * c2;
    if (row < N && k < kend) {
      double2 x = __ldg(reinterpret_cast<const double2*>(X + (int64_t)row * ld + k));
      if (Xb) {
        const double2 y = __ldg(reinterpret_cast<const double2*>(Xb + (int64_t)row * ld + k));
        x.x += s * y.x;
        x.y += s * y.y;
      }
      v[j] = x;
    } else {
      v[j] = make_double2(0.0, 0.0);
    }
  }
}

template <int NPAD>
__device__ __forceinline__ void tile_store(const double2 (&v)[Tile<NPAD>::NV], double* S) {
#pragma unroll
  for (int j = 0; j < Tile<NPAD>::NV; ++j) {
    const int e = threadIdx.x + j * ST;
    const int row = e / (SK / 2), c2 = e % (SK / 2);
    if (row < NPAD) *reinterpret_cast<double2*>(S + row * SKP + 2 * c2) = v[j];
  }
}

// TMA-ring variant of the small-N Gram (faster than LDG staging for the Gram:
// profiles/r1_*): a producer warp streams the stage's row segments with 1D
// bulk copies into an NST-stage ring, eight consumer warps run the DMMAs and
// release stages through "empty" mbarriers.
constexpr int SC = 8;
constexpr int RING_THREADS = (SC + 1) * 32;
constexpr size_t RING_SMEM_BUDGET = 200 * 1024;

struct RingCfg {
  int ks = 64, nst = 2;
  size_t stage_doubles = 0, smem = 0;
};

RingCfg ring_cfg(int nsrc, int npad, size_t min_smem_doubles) {
  RingCfg c;
  auto stage = [&](int ks) { return (size_t)nsrc * npad * (ks + 8); };
  c.ks = (3 * stage(128) * 8 <= RING_SMEM_BUDGET) ? 128 : 64;
  c.stage_doubles = stage(c.ks);
  c.nst = (int)(RING_SMEM_BUDGET / 8 / c.stage_doubles);
  if (c.nst > 6) c.nst = 6;
  if (c.nst < 2) c.nst = 2;
  size_t d = (size_t)c.nst * c.stage_doubles;
  if (d < min_smem_doubles) d = min_smem_doubles;
  c.smem = 128 + d * 8;
  return c;
}

__device__ __forceinline__ void ring_produce(const double* const* srcs, int nsrc, int N, int npad,
                                             int64_t ld, int64_t kbeg, int64_t kend, int ks,
                                             int nst, size_t sdoubles, double* stage0,
                                             uint64_t* full, uint64_t* empty, int lane) {
  const int nstage = kend > kbeg ? (int)((kend - kbeg + ks - 1) / ks) : 0;
  const int rs = ks + 8;
  for (int st = 0; st < nstage; ++st) {
    const int s = st % nst;
    const uint32_t ph = (uint32_t)(st / nst) & 1u;
    if (st >= nst) mbar_wait(&empty[s], ph ^ 1u);
    const int64_t k0 = kbeg + (int64_t)st * ks;
    const int cnt = (int)min((int64_t)ks, kend - k0);
    if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)(nsrc * N * cnt * 8));
    __syncwarp();
    double* sb = stage0 + (size_t)s * sdoubles;
    for (int e = lane; e < nsrc * N; e += 32) {
      const int q = e / N, r = e % N;
      tma_load_1d(sb + ((size_t)q * npad + r) * rs, srcs[q] + (int64_t)r * ld + k0,
                  (uint32_t)cnt * 8u, &full[s]);
    }
  }
}

template <int F, bool SYM>
__global__ void __launch_bounds__(RING_THREADS, 1) gram_ring_kernel(
    int N, int64_t ld, int64_t kchunk, int ks, int nst, const double* __restrict__ A,
    const double* __restrict__ Ab, double sa, const double* __restrict__ B,
    const double* __restrict__ Bb, double sb, double* __restrict__ ws,
    const double* __restrict__ guard) {
  if (guard && *guard == 0.0) return;  // device-side branch (CholeskyQR2 repair)
  constexpr int NP = SmallPairs<F, SYM>::NP;
  constexpr int NPAD = 8 * F;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + 8;
  double* stage0 = reinterpret_cast<double*>(smraw + 128);
  const double* srcs[4];
  int nsrc = 0;
  srcs[nsrc++] = A;
  const int qa_b = Ab ? nsrc : -1;
  if (Ab) srcs[nsrc++] = Ab;
  int qb = 0, qb_b = -1;
  if (!SYM) {
    qb = nsrc;
    srcs[nsrc++] = B;
    if (Bb) {
      qb_b = nsrc;
      srcs[nsrc++] = Bb;
    }
  }
  const int rs = ks + 8;
  const size_t sdoubles = (size_t)nsrc * NPAD * rs;
  for (size_t e = threadIdx.x; e < (size_t)nst * sdoubles; e += RING_THREADS) stage0[e] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SC);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t kbeg = (int64_t)blockIdx.x * kchunk;
  const int64_t kend = min(kbeg + kchunk, ld);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t4 = lane & 3;
  double acc[NP][2];
#pragma unroll
  for (int q = 0; q < NP; ++q) acc[q][0] = acc[q][1] = 0.0;
  if (warp == SC) {
    ring_produce(srcs, nsrc, N, NPAD, ld, kbeg, kend, ks, nst, sdoubles, stage0, full, empty, lane);
  } else {
    const int nstage = kend > kbeg ? (int)((kend - kbeg + ks - 1) / ks) : 0;
    for (int st = 0; st < nstage; ++st) {
      const int s = st % nst;
      mbar_wait(&full[s], (uint32_t)(st / nst) & 1u);
      const double* sbuf = stage0 + (size_t)s * sdoubles;
      const int cnt = (int)min((int64_t)ks, kend - (kbeg + (int64_t)st * ks));
      for (int c = warp * 8; c < cnt; c += SC * 8) {
        double2 a[F], b[SYM ? 1 : F];
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const int off = (8 * f + gq) * rs + c + 2 * t4;
          a[f] = *reinterpret_cast<const double2*>(sbuf + off);
          if (qa_b >= 0) {
            const double2 z = *reinterpret_cast<const double2*>(sbuf + (size_t)qa_b * NPAD * rs + off);
            a[f].x += sa * z.x;
            a[f].y += sa * z.y;
          }
          if constexpr (!SYM) {
            b[f] = *reinterpret_cast<const double2*>(sbuf + (size_t)qb * NPAD * rs + off);
            if (qb_b >= 0) {
              const double2 z = *reinterpret_cast<const double2*>(sbuf + (size_t)qb_b * NPAD * rs + off);
              b[f].x += sb * z.x;
              b[f].y += sb * z.y;
            }
          }
        }
        int q = 0;
#pragma unroll
        for (int fm = 0; fm < F; ++fm)
#pragma unroll
          for (int fn = SYM ? fm : 0; fn < F; ++fn, ++q) {
            const double2 bv = SYM ? a[fn] : b[SYM ? 0 : fn];
            dmma_8x8x4(acc[q], a[fm].x, bv.x);
            dmma_8x8x4(acc[q], a[fm].y, bv.y);
          }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  double* red = stage0;
  if (warp < SC) {
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      red[(warp * NP + q) * 64 + lane * 2] = acc[q][0];
      red[(warp * NP + q) * 64 + lane * 2 + 1] = acc[q][1];
    }
  }
  __syncthreads();
  double* out = ws + (int64_t)blockIdx.x * NPAD * NPAD;
  for (int e = threadIdx.x; e < NP * 64; e += RING_THREADS) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < SC; ++w) sum += red[(w * NP) * 64 + e];
    const int q = e / 64, l = (e % 64) / 2, j = e % 2;
    int fm = 0, fn = 0, c = 0;
    for (int m = 0; m < F; ++m)
      for (int n = SYM ? m : 0; n < F; ++n, ++c)
        if (c == q) {
          fm = m;
          fn = n;
        }
    out[(8 * fm + (l >> 2)) * NPAD + 8 * fn + 2 * (l & 3) + j] = sum;
  }
}

// one warp per output element, lanes stride over the splits (fixed order)
__global__ void gram_small_reduce_kernel(int N, int npad, int sym, int nsplit, double w,
                                         const double* __restrict__ ws, double* __restrict__ G,
    const double* __restrict__ guard) {
  if (guard && *guard == 0.0) return;  // device-side branch (CholeskyQR2 repair)
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= (int64_t)N * N) return;
  int i = (int)(wid / N), j = (int)(wid % N);
  if (sym && j < i) {
    const int t = i;
    i = j;
    j = t;
  }
  double s = 0.0;
  for (int k = lane; k < nsplit; k += 32) s += ws[(int64_t)k * npad * npad + i * npad + j];
  s = warp_sum(s);
  if (lane == 0) G[wid] = w * s;
}

int g_sms = 0;
int num_sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_sms;
}

constexpr int SMALL_SPLITS_PER_SM = 4;

template <int F>
void launch_gram_small_f(int N, int64_t ld, int sym, const double* A, const double* Ab, double sa,
                         const double* B, const double* Bb, double sb, double* ws, double* G,
                         double w, cudaStream_t s, const double* guard) {
  const int nsrc = 1 + (Ab ? 1 : 0) + (sym ? 0 : 1 + (Bb ? 1 : 0));
  const int np = sym ? F * (F + 1) / 2 : F * F;
  const RingCfg cfg = ring_cfg(nsrc, 8 * F, (size_t)SC * np * 64);
  const int64_t kblocks = (ld + cfg.ks - 1) / cfg.ks;
  int nsplit = num_sms();
  if (nsplit > kblocks) nsplit = (int)kblocks;
  const int64_t kchunk = ((kblocks + nsplit - 1) / nsplit) * cfg.ks;
  nsplit = (int)((ld + kchunk - 1) / kchunk);
  ::po::count_launch();
  if (sym) {
    auto k = gram_ring_kernel<F, true>;
    set_smem(reinterpret_cast<const void*>(k), (int)(cfg.smem));
    k<<<nsplit, RING_THREADS, cfg.smem, s>>>(N, ld, kchunk, cfg.ks, cfg.nst, A, Ab, sa, A, Ab, sa, ws, guard);
  } else {
    auto k = gram_ring_kernel<F, false>;
    set_smem(reinterpret_cast<const void*>(k), (int)(cfg.smem));
    k<<<nsplit, RING_THREADS, cfg.smem, s>>>(N, ld, kchunk, cfg.ks, cfg.nst, A, Ab, sa, B, Bb, sb, ws, guard);
  }
  const int64_t threads = (int64_t)N * N * 32;
  ::po::count_launch();
  gram_small_reduce_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(N, 8 * F, sym, nsplit,
                                                                             w, ws, G, guard);
}

// Small-N mix: out_i[p] = alpha sum_k (A + sa Ab)_k[p] M(k, i) + beta C_i[p].
// Warp w owns the 8 points [8w, 8w+8) of a stage (one DMMA row fragment) and
// all N outputs; M sits in shared memory for the whole CTA; C is prefetched
// with the inputs; UPPER skips the k > i fragments of an upper-triangular M.
template <int F, bool UPPER>
__global__ void __launch_bounds__(ST, 2) mix_small_kernel(
    int N, int64_t ld, int64_t ngl, int64_t pchunk, const double* __restrict__ A,
    const double* __restrict__ Ab, double sa, const double* __restrict__ M, double alpha,
    const double* __restrict__ C, double beta, double* __restrict__ out,
    double* __restrict__ norms, const double* __restrict__ guard) {
  if (guard && *guard == 0.0) return;  // device-side branch (CholeskyQR2 repair)
  constexpr int NPAD = 8 * F;
  constexpr int NV = Tile<NPAD>::NV;
  extern __shared__ __align__(16) double msmem[];
  double* Ms = msmem;                     // [NPAD][NPAD]
  double* sA = Ms + NPAD * NPAD;          // [NPAD][SKP]
  double* sC = sA + NPAD * SKP;           // [NPAD][SKP] (only if C)
  double* nred = sC + (C ? NPAD * SKP : 0);  // [8][NPAD]
  for (int e = threadIdx.x; e < NPAD * NPAD; e += ST) {
    const int k = e / NPAD, i = e % NPAD;
    Ms[e] = (k < N && i < N) ? M[(int64_t)k * N + i] : 0.0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t4 = lane & 3;
  const int64_t pbeg = (int64_t)blockIdx.x * pchunk;
  const int64_t pend = min(pbeg + pchunk, ld);
  const int ksteps = (N + 3) / 4;
  double nrm[F][2];
#pragma unroll
  for (int fi = 0; fi < F; ++fi) nrm[fi][0] = nrm[fi][1] = 0.0;
  double2 va[NV], vc[NV];
  tile_load<NPAD>(va, A, Ab, sa, N, ld, pbeg, pend);
  if (C) tile_load<NPAD>(vc, C, nullptr, 0.0, N, ld, pbeg, pend);
  for (int64_t k0 = pbeg; k0 < pend; k0 += SK) {
    __syncthreads();
    tile_store<NPAD>(va, sA);
    if (C) tile_store<NPAD>(vc, sC);
    __syncthreads();
    if (k0 + SK < pend) {
      tile_load<NPAD>(va, A, Ab, sa, N, ld, k0 + SK, pend);
      if (C) tile_load<NPAD>(vc, C, nullptr, 0.0, N, ld, k0 + SK, pend);
    }
    const int c = warp * 8;
    double acc[F][2];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f][0] = acc[f][1] = 0.0;
    for (int ks = 0; ks < ksteps; ++ks) {
      const int krow = 4 * ks + t4;
      const double av = sA[krow * SKP + c + gq];
#pragma unroll
      for (int fi = 0; fi < F; ++fi) {
        if (UPPER && 4 * ks > 8 * fi + 7) continue;
        dmma_8x8x4(acc[fi], av, Ms[krow * NPAD + 8 * fi + gq]);
      }
    }
    const int64_t p = k0 + c + gq;
#pragma unroll
    for (int fi = 0; fi < F; ++fi)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int i = 8 * fi + 2 * t4 + j;
        if (p < ngl && i < N) {
          double v = alpha * acc[fi][j];
          if (C) v += beta * sC[i * SKP + c + gq];
          if (out) out[(int64_t)i * ld + p] = v;
          nrm[fi][j] += v * v;
        }
      }
  }
  if (norms) {
#pragma unroll
    for (int fi = 0; fi < F; ++fi)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double v = nrm[fi][j];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (gq == 0) nred[warp * NPAD + 8 * fi + 2 * t4 + j] = v;
      }
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += ST) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < ST / 32; ++w) sum += nred[w * NPAD + i];
      norms[(int64_t)i * gridDim.x + blockIdx.x] = sum;
    }
  }
}

template <int F>
int launch_mix_small_f(int N, int64_t ld, int64_t ngl, const double* A, const double* Ab,
                       double sa, const double* M, double alpha, const double* C, double beta,
                       int upper, double* out, double* norms, cudaStream_t s,
                       const double* guard) {
  const size_t smem = sizeof(double) * ((size_t)(8 * F) * (8 * F) +
                                        (size_t)(C ? 2 : 1) * 8 * F * SKP + 8 * 8 * F);
  const int64_t kb = (ld + SK - 1) / SK;
  int nblk = num_sms() * SMALL_SPLITS_PER_SM;
  if (nblk > kb) nblk = (int)kb;
  const int64_t pchunk = ((kb + nblk - 1) / nblk) * SK;
  nblk = (int)((ld + pchunk - 1) / pchunk);
  ::po::count_launch();
  if (upper) {
    auto k = mix_small_kernel<F, true>;
    set_smem(reinterpret_cast<const void*>(k), (int)(smem));
    k<<<nblk, ST, smem, s>>>(N, ld, ngl, pchunk, A, Ab, sa, M, alpha, C, beta, out, norms, guard);
  } else {
    auto k = mix_small_kernel<F, false>;
    set_smem(reinterpret_cast<const void*>(k), (int)(smem));
    k<<<nblk, ST, smem, s>>>(N, ld, ngl, pchunk, A, Ab, sa, M, alpha, C, beta, out, norms, guard);
  }
  return nblk;
}

// -------------------------------------------------------------------- mix
constexpr int MP = 128;       // points per CTA tile
constexpr int MI = 64;        // orbitals per CTA tile
constexpr int MK = 16;        // k (input orbitals) per stage
constexpr int MPP = MP + 8;   // smem strides
constexpr int MIP = MI + 8;
constexpr int MT = 256;       // 8 warps: 4 along p x 2 along i; warp tile 32 x 32

__device__ __forceinline__ void mix_load(double (&ra)[8], double (&rm)[4], const double* A,
                                         const double* Ab, double sa, const double* M, int N,
                                         int64_t ld, int64_t ngl, int64_t p0, int i0, int k0) {
  const int t = threadIdx.x;
  {  // A: MK rows (k) x MP points: thread -> row t/16, 8 points
    const int row = t >> 4;
    const int c0 = (t & 15) * 8;
    const int k = k0 + row;
    const int64_t p = p0 + c0;
    if (k < N && p < ld) {
      const double2* src = reinterpret_cast<const double2*>(A + (int64_t)k * ld + p);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double2 v = __ldg(src + j);
        ra[2 * j] = v.x;
        ra[2 * j + 1] = v.y;
      }
      if (Ab) {
        const double2* sb = reinterpret_cast<const double2*>(Ab + (int64_t)k * ld + p);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double2 v = __ldg(sb + j);
          ra[2 * j] += sa * v.x;
          ra[2 * j + 1] += sa * v.y;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) ra[j] = 0.0;
    }
  }
  {  // M: MK rows (k) x MI cols (i): thread -> row t/16, 4 cols
    const int row = t >> 4;
    const int c0 = (t & 15) * 4;
    const int k = k0 + row;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + c0 + j;
      rm[j] = (k < N && i < N) ? __ldg(M + (int64_t)k * N + i) : 0.0;
    }
  }
}

__global__ void __launch_bounds__(MT) mix_kernel(int N, int64_t ld, int64_t ngl, int64_t bstride,
                                                 int upper,
                                                 const double* __restrict__ A,
                                                 const double* __restrict__ Ab, double sa,
                                                 const double* __restrict__ M, double alpha,
                                                 const double* __restrict__ C, double beta,
                                                 double* __restrict__ out,
                                                 double* __restrict__ norms,
                                                 const double* __restrict__ guard) {
  if (guard && *guard == 0.0) return;  // device-side branch (CholeskyQR2 repair)
  extern __shared__ __align__(16) double msm[];
  double (*As)[MK * MPP] = reinterpret_cast<double (*)[MK * MPP]>(msm);
  double (*Ms)[MK * MIP] = reinterpret_cast<double (*)[MK * MIP]>(msm + 2 * MK * MPP);
  double (*nred)[MI] = reinterpret_cast<double (*)[MI]>(msm + 2 * MK * MPP + 2 * MK * MIP);
  const int64_t p0 = (int64_t)blockIdx.x * MP;
  if (blockIdx.z) {  // batched left-multiplies (DST transforms): independent row sets
    A += blockIdx.z * bstride;
    if (Ab) Ab += blockIdx.z * bstride;
    if (C) C += blockIdx.z * bstride;
    if (out) out += blockIdx.z * bstride;
  }
  const int i0 = blockIdx.y * MI;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wp = warp >> 1, wi = warp & 1;
  const int gq = lane >> 2, t4 = lane & 3;
  int kend = N;
  if (upper) kend = min(N, i0 + MI);  // M(k, i) = 0 for k > i
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  double ra[8], rm[4];
  mix_load(ra, rm, A, Ab, sa, M, N, ld, ngl, p0, i0, 0);
  int buf = 0;
  for (int k0 = 0; k0 < kend; k0 += MK) {
    {
      const int t = threadIdx.x;
      const int row = t >> 4;
#pragma unroll
      for (int j = 0; j < 8; ++j) As[buf][row * MPP + (t & 15) * 8 + j] = ra[j];
#pragma unroll
      for (int j = 0; j < 4; ++j) Ms[buf][row * MIP + (t & 15) * 4 + j] = rm[j];
    }
    __syncthreads();
    if (k0 + MK < kend) mix_load(ra, rm, A, Ab, sa, M, N, ld, ngl, p0, i0, k0 + MK);
    const double* as = As[buf];
    const double* ms = Ms[buf];
#pragma unroll
    for (int kk = 0; kk < MK / 4; ++kk) {
      double af[4], bf[4];
#pragma unroll
      for (int fm = 0; fm < 4; ++fm) af[fm] = as[(kk * 4 + t4) * MPP + wp * 32 + fm * 8 + gq];
#pragma unroll
      for (int fn = 0; fn < 4; ++fn) bf[fn] = ms[(kk * 4 + t4) * MIP + wi * 32 + fn * 8 + gq];
#pragma unroll
      for (int fm = 0; fm < 4; ++fm)
#pragma unroll
        for (int fn = 0; fn < 4; ++fn) dmma_8x8x4(acc[fm][fn], af[fm], bf[fn]);
    }
    buf ^= 1;
  }
  // epilogue: acc[fm][fn][j] = Out[p = p0 + wp*32 + fm*8 + gq][i = i0 + wi*32 + fn*8 + 2*t4 + j]
  double nrm[4][2];
#pragma unroll
  for (int fn = 0; fn < 4; ++fn) nrm[fn][0] = nrm[fn][1] = 0.0;
#pragma unroll
  for (int fm = 0; fm < 4; ++fm) {
    const int64_t p = p0 + wp * 32 + fm * 8 + gq;
#pragma unroll
    for (int fn = 0; fn < 4; ++fn)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int i = i0 + wi * 32 + fn * 8 + 2 * t4 + j;
        if (p < ngl && i < N) {
          double v = alpha * acc[fm][fn][j];
          if (C) v += beta * C[(int64_t)i * ld + p];
          if (out) out[(int64_t)i * ld + p] = v;
          nrm[fn][j] += v * v;
        }
      }
  }
  if (norms) {
    // reduce over gq (lane bits 2..4), then over the 4 warps along p
#pragma unroll
    for (int fn = 0; fn < 4; ++fn)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double v = nrm[fn][j];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (gq == 0) nred[wp][wi * 32 + fn * 8 + 2 * t4 + j] = v;
      }
    __syncthreads();
    if (threadIdx.x < MI) {
      const int i = i0 + threadIdx.x;
      if (i < N) {
        const double s = ((nred[0][threadIdx.x] + nred[1][threadIdx.x]) + nred[2][threadIdx.x]) +
                         nred[3][threadIdx.x];
        norms[(int64_t)i * gridDim.x + blockIdx.x] = s;
      }
    }
  }
}

}  // namespace

size_t gram_workspace_doubles(const SlabGeom& g, int N) {
  GramPlan p = gram_plan(g, N, 0);
  const size_t tiled = (size_t)p.nsplit * p.ntiles * GB * GB;
  const size_t small = (size_t)148 * 4 * 64 * 64;
  size_t w = tiled > small ? tiled : small;
  const size_t big = gram_big_workspace_doubles(g.ld, N);
  return big > w ? big : w;
}

static bool gram_small_ok(int N, int sym) { return sym ? N <= 48 : N <= 40; }

void launch_gram(const SlabGeom& g, int N, const double* A, const double* Ab, double sa,
                 const double* B, const double* Bb, double sb, int sym, double* ws, double* G,
                 cudaStream_t s, const double* guard) {
  if (gram_small_ok(N, sym)) {
    static const bool no_tma = getenv("PO_NO_TMA") != nullptr;  // measurement: LDG paths
    if (!no_tma && launch_gram_tma(N, g.ld, sym, A, Ab, sa, B, Bb, sb, ws, G, g.w, s, guard)) return;
    switch ((N + 7) / 8) {
#define PO_GS(F)                                                                  \
  case F:                                                                         \
    launch_gram_small_f<F>(N, g.ld, sym, A, Ab, sa, B, Bb, sb, ws, G, g.w, s, guard);    \
    return;
      PO_GS(1) PO_GS(2) PO_GS(3) PO_GS(4) PO_GS(5) PO_GS(6) PO_GS(7) PO_GS(8)
#undef PO_GS
    }
  }
  if (launch_gram_big(N, g.ld, sym, A, Ab, sa, B, Bb, sb, ws, gram_workspace_doubles(g, N), G,
                      g.w, s, guard))
    return;
  GramPlan p = gram_plan(g, N, sym);
  dim3 grid(p.ntiles, p.nsplit);
  constexpr size_t shm = sizeof(double) * 4 * GB * GKP;
  static bool attr = false;
  if (!attr) {
    set_smem(reinterpret_cast<const void*>(gram_kernel), (int)(shm));
    attr = true;
  }
  ::po::count_launch();
  gram_kernel<<<grid, GT, shm, s>>>(N, g.ld, p.kchunk, p.mt, sym, A, Ab, sa, B, Bb, sb, ws, guard);
  const int64_t total = (int64_t)N * N;
  ::po::count_launch();
  gram_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(N, p.mt, sym, p.ntiles,
                                                                      p.nsplit, g.w, ws, G, guard);
}

int mix_nblk(const SlabGeom& g) { return (int)((g.ngl + MP - 1) / MP); }

// Largest norm-partials row any mix path can write (tiled: one per 128-point
// tile; small-N: up to SMALL_SPLITS_PER_SM CTAs per SM).
int mix_nblk_max(const SlabGeom& g) {
  const int small = num_sms() * SMALL_SPLITS_PER_SM;
  const int tiled = mix_nblk(g);
  return small > tiled ? small : tiled;
}

int launch_mix(const SlabGeom& g, int N, const double* A, const double* Ab, double sa,
               const double* M, double alpha, const double* C, double beta, int upper,
               double* out, double* norms, cudaStream_t s, const double* guard,
               const double* zsig) {
  if (zsig) {  // implicit direction: only the large-N TMA tiles rebuild z = HW - zsig W
    if (N <= 64 || !Ab) return -2;
    const int nb = launch_mix_big(N, g.ld, g.ngl, A, Ab, sa, M, alpha, C, beta, upper, out, norms, s,
                                  guard, zsig);
    return nb >= 0 ? nb : -2;
  }
  // measurement switch (the large-N TMA mix at N = 49..64 measured slower: 0.49 vs 0.53 of HBM)
  static const int big_min = getenv("PO_MIX_BIG_MIN") ? atoi(getenv("PO_MIX_BIG_MIN")) : 65;
  if (N < big_min && N <= 64) {  // small-N paths (return their partials row length)
    static const bool no_tma = getenv("PO_NO_TMA") != nullptr;
    const int nb = no_tma ? -1 : launch_mix_tma(N, g.ld, g.ngl, A, Ab, sa, M, alpha, C, beta, upper, out, norms,
                                  s, guard);
    if (nb >= 0) return nb;
    switch ((N + 7) / 8) {
#define PO_MS(F) \
  case F:        \
    return launch_mix_small_f<F>(N, g.ld, g.ngl, A, Ab, sa, M, alpha, C, beta, upper, out, norms, s, guard);
      PO_MS(1) PO_MS(2) PO_MS(3) PO_MS(4) PO_MS(5) PO_MS(6) PO_MS(7) PO_MS(8)
#undef PO_MS
    }
  }
  {
    const int nb = launch_mix_big(N, g.ld, g.ngl, A, Ab, sa, M, alpha, C, beta, upper, out, norms, s,
                                  guard);
    if (nb >= 0) return nb;
  }
  dim3 grid(mix_nblk(g), (N + MI - 1) / MI);
  constexpr size_t shm = sizeof(double) * (2 * MK * MPP + 2 * MK * MIP + 4 * MI);
  static bool attr = false;
  if (!attr) {
    set_smem(reinterpret_cast<const void*>(mix_kernel), (int)(shm));
    attr = true;
  }
  ::po::count_launch();
  mix_kernel<<<grid, MT, shm, s>>>(N, g.ld, g.ngl, 0, upper, A, Ab, sa, M, alpha, C, beta, out,
                                   norms, guard);
  return mix_nblk(g);
}

void launch_mix_batched(int N, int64_t ld, int64_t ngl, int batch, int64_t bstride,
                        const double* A, const double* M, double* out, cudaStream_t s) {
  dim3 grid((unsigned)((ngl + MP - 1) / MP), (N + MI - 1) / MI, batch);
  constexpr size_t shm = sizeof(double) * (2 * MK * MPP + 2 * MK * MIP + 4 * MI);
  static bool attr = false;
  if (!attr) {
    set_smem(reinterpret_cast<const void*>(mix_kernel), (int)(shm));
    attr = true;
  }
  ::po::count_launch();
  mix_kernel<<<grid, MT, shm, s>>>(N, ld, ngl, bstride, 0, A, nullptr, 0.0, M, 1.0, nullptr, 0.0,
                                   out, nullptr, nullptr);
}

}  // namespace po
