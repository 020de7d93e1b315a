// Tall-skinny FP64 tensor-core contractions fed by 2D tensor-map TMA: small-N (N <= 64)
// streamed stages (first part of this file) and large-N tiles (gram_big / mix_big).
//
// Small-N stages (measured on B200, profiles/r1_tma_probe.txt and
// r1_tma2d_probe.txt): 1D bulk copies are request-rate bound (512 B per request
// caps a ring at ~2.1 TB/s), and so are 2D boxes of 128-B rows (16 points,
// 128-B swizzle: ~4.2 TB/s); rows of >= 64 points reach 6+ TB/s. So a stage of
// 64 points is one cp.async.bulk.tensor box {72 points x N rows} per source
// (rows >= N never read; the 8 extra points pad the shared-memory row stride so
// the DMMA fragment reads are bank-conflict free, see PADW). A producer warp
// keeps an NST-deep ring full; eight consumer warps run mma.sync.m8n8k4.f64
// (DMMA) from shared memory.
//   gram: G = w (A + sa Ab)^T (B + sb Bb)        (manifold.cpp:41-61)
//   mix : out = alpha (A + sa Ab) M + beta C     (manifold.cpp:67-85, 181-202)
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "kernels.h"

namespace po {

namespace {

constexpr int BOX = 16;           // points per box (128 B rows, SWIZZLE_128B)
constexpr int TKS = 64;           // points per stage (4 boxes)
constexpr int TSC = 8;            // consumer warps
// 8 consumer warps (warpgroups 0-1) + a producer warpgroup (one lane issues the
// boxes) that hands its registers to the consumers via setmaxnreg (40 / 232).
constexpr int TTH = (TSC + 4) * 32;
constexpr size_t TBUDGET = 180 * 1024;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Encoded tensor maps are cached by (base, ld, rows, box rows): the solver's
// blocks come from pools and recur every iteration, and encoding is a driver
// call on the launch path.
struct MapKey {
  const double* base;
  int64_t ld;
  int rows, npad, bx;
  bool operator==(const MapKey& o) const {
    return base == o.base && ld == o.ld && rows == o.rows && npad == o.npad && bx == o.bx;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.base) ^ (size_t)(k.ld * 31 + k.rows * 131 + k.npad + k.bx * 7919);
  }
};

bool encode_map(CUtensorMap* m, const double* base, int64_t ld, int rows, int npad, int bx);

// box {bx, npad}: bx = 16 with 128-B swizzle (the large-N tiles), otherwise
// unswizzled rows of bx points (the small-N stages, see PADW)
bool make_map(CUtensorMap* m, const double* base, int64_t ld, int rows, int npad, int bx = 16) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  const MapKey key{base, ld, rows, npad, bx};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *m = it->second;
      return true;
    }
  }
  if (!encode_map(m, base, ld, rows, npad, bx)) return false;
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *m);
  return true;
}

// rows x ld doubles, row stride ld; box {bx, npad}
bool encode_map(CUtensorMap* m, const double* base, int64_t ld, int rows, int npad, int bx) {
  auto fn = encode_fn();
  if (!fn || !base) return false;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)npad};
  cuuint32_t es[2] = {1, 1};
  static const int promo = getenv("PO_TMA_PROMO") ? atoi(getenv("PO_TMA_PROMO")) : 3;
  const CUtensorMapL2promotion pr = promo == 0   ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                    : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                 : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            bx == BOX ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, pr,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Sources of a streamed contraction (one tensor map per source block).
struct Maps {
  CUtensorMap m[4];
};

// Small-N stage layout. Measured (tools/tma2d_probe.cu, profiles/r1_tma2d_probe.txt):
// a 2D-TMA stream of 128-B box rows (16 points, 128-B swizzle) tops out at
// ~4.2 TB/s on B200, boxes of >= 64-point rows (unswizzled) at 6.0-6.6 TB/s.
// So a stage of 64 points is ONE box per source, {PADW points x N rows}: the
// 8 extra points per row (the next stage's first points, L2 hits) pad the
// shared-memory row stride to 72 doubles, which makes both fragment access
// patterns conflict-free: 8 rows x 16-B pairs (Gram operands) and 4 rows x
// 8 consecutive points (rotation / mix operands), because row r starts at
// 16-byte chunk 4 r (mod 8).
constexpr int PADW = 72;

bool make_map2(Maps& M, int i, const double* base, int64_t ld, int rows, int /*npad*/) {
  return make_map(&M.m[i], base, ld, rows, rows, PADW);  // boxes of exactly N rows
}



__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// swizzled address of element (row, point p in the stage) in a source's stage
// area: 4 boxes of nb rows x 16 doubles back to back (the area is padded to a
// multiple of 8 rows, so it starts 1024-B aligned); the hardware XORs the
// 16-byte chunk index with bits [7:9] of the shared address, i.e. with the
// area row (b * nb + row) mod 8.
__device__ __forceinline__ int swz(int row, int p, int nb) {
  const int b = p >> 4, o = p & 15;
  const int r = b * nb + row;
  const int j = (o >> 1) ^ (r & 7);
  return r * BOX + j * 2 + (o & 1);
}

// small-N stage: element (row, point p < 64) of a source's area
__device__ __forceinline__ int pad(int row, int p) { return row * PADW + p; }

// doubles per source per stage (nb padded rows, areas 128-B aligned)
__host__ __device__ constexpr size_t qs_of(int nb) {
  return ((size_t)nb * PADW + 15) & ~(size_t)15;
}

struct TCfg {
  int nst;
  size_t stage_doubles, smem;
};

size_t tbudget() {
  static size_t b = 0;
  if (!b) {
    const char* e = getenv("PO_TMA_BUDGET_KB");  // measurement override
    b = (e ? (size_t)atoi(e) : 0) * 1024;
    if (b < 64 * 1024 || b > 220 * 1024) b = TBUDGET;
  }
  return b;
}

TCfg tcfg(int nsrc, int npad, size_t extra_doubles) {
  TCfg c;
  c.stage_doubles = (size_t)nsrc * qs_of(npad);
  const size_t avail = tbudget() / 8 - extra_doubles;
  c.nst = (int)(avail / c.stage_doubles);
  if (c.nst > 8) c.nst = 8;
  if (c.nst < 2) c.nst = 2;
  // + barriers / alignment slack + tail (fragment rows past N: up to 7 padded rows)
  c.smem = 3072 + 8 * PADW * 8 + ((size_t)c.nst * c.stage_doubles + extra_doubles) * 8;
  return c;
}

// producer warp: lane 0 recycles the stage and arms its barrier, then one lane
// per (source, box) issues that box — the boxes of a stage go out in parallel
// instead of one after another from a single thread
__device__ __forceinline__ void tma_produce(const CUtensorMap* maps, int nsrc, int npad,
                                            int64_t kbeg, int64_t kend, int nst, size_t sdoubles,
                                            double* stage0, uint64_t* full, uint64_t* empty) {
  const int lane = threadIdx.x & 31;
  const int nstage = kend > kbeg ? (int)((kend - kbeg + TKS - 1) / TKS) : 0;
  const uint32_t bytes = (uint32_t)(nsrc * npad * PADW * 8);
  const size_t qs = qs_of(npad);
  for (int st = 0; st < nstage; ++st) {
    const int s = st % nst;
    if (lane == 0) {
      if (st >= nst) mbar_wait(&empty[s], ((uint32_t)(st / nst) & 1u) ^ 1u);
      mbar_arrive_expect_tx(&full[s], bytes);
    }
    __syncwarp();
    const int64_t k0 = kbeg + (int64_t)st * TKS;
    double* sb = stage0 + (size_t)s * sdoubles;
    if (lane < nsrc) tma_load_2d(sb + lane * qs, &maps[lane], (int)k0, 0, &full[s]);
  }
}

// producer of a small-N stage of ks points (one box {pw points x npad rows} per source)
__device__ __forceinline__ void tma_produce_w(const CUtensorMap* maps, int nsrc, int npad,
                                              int64_t kbeg, int64_t kend, int nst, size_t sdoubles,
                                              double* stage0, uint64_t* full, uint64_t* empty, int ks,
                                              int pw) {
  const int lane = threadIdx.x & 31;
  const int nstage = kend > kbeg ? (int)((kend - kbeg + ks - 1) / ks) : 0;
  const uint32_t bytes = (uint32_t)(nsrc * npad * pw * 8);
  const size_t qs = ((size_t)npad * pw + 15) & ~(size_t)15;
  for (int st = 0; st < nstage; ++st) {
    const int s = st % nst;
    if (lane == 0) {
      if (st >= nst) mbar_wait(&empty[s], ((uint32_t)(st / nst) & 1u) ^ 1u);
      mbar_arrive_expect_tx(&full[s], bytes);
    }
    __syncwarp();
    const int64_t k0 = kbeg + (int64_t)st * ks;
    double* sb = stage0 + (size_t)s * sdoubles;
    if (lane < nsrc) tma_load_2d(sb + lane * qs, &maps[lane], (int)k0, 0, &full[s]);
  }
}

// producer side of every small-N streamed kernel (called by the whole producer warpgroup)
// (measured alternatives, not kept: a cp.async producer warpgroup streamed the
// same stages at about half the rate of the TMA boxes on B200; splitting the
// sources between TMA (half) and cp.async from the idle producer warps (half)
// was slower than TMA alone for every kernel: e.g. Sigma 113 -> 142 us,
// directions 234 -> 266 us; an interleaved stage schedule across CTAs — all
// CTAs reading neighbouring segments of each row — made no difference)
__device__ __forceinline__ void produce(const Maps& mp, int nsrc, int npad, int64_t kbeg,
                                        int64_t kend, int nst, size_t sdoubles, double* stage0,
                                        uint64_t* full, uint64_t* empty) {
  if ((threadIdx.x >> 5) == TSC)
    tma_produce(mp.m, nsrc, npad, kbeg, kend, nst, sdoubles, stage0, full, empty);
}

template <int F, bool SYM>
struct TPairs {
  static constexpr int NP = SYM ? F * (F + 1) / 2 : F * F;
};

// G = w (A + sa Ab)^T (B + sb Bb) over the CTA's point range; with DUAL
// (non-symmetric call only) the same pass also accumulates A^T A, so
// Sigma = (HW)^T W and G_HH = (HW)^T (HW) come from one read of HW and W.
// F = ceil(N/8) fragments; NPAD = 8F. With DUAL and R > 0 (N = 8(F-1) + R,
// R <= 2) the last fragment row — R real orbitals and 8 - R padding ones — is
// contracted with FP64 FMAs instead of DMMA: this pass is DMMA-bound (two
// Grams), and for N = 33 the padding row would cost 18 of its 80 DMMAs.
template <int F, bool SYM, bool DUAL, int R = 0>
__global__ void __launch_bounds__(TTH, 1) gram_tma_kernel(const __grid_constant__ Maps maps,
                                                          int N, int nsrc, int qa_b, int qb,
                                                          int qb_b, int64_t ld, int64_t kchunk,
                                                          int nst, double sa, double sb,
                                                          double* __restrict__ ws,
                                                          const double* __restrict__ guard,
                                                          int probe) {
  PO_PDL_ENTRY();
  if (guard && *guard == 0.0) return;
  constexpr bool REM = DUAL && R > 0;
  constexpr int FD = REM ? F - 1 : F;  // DMMA fragments
  constexpr int NP = TPairs<FD, SYM>::NP;
  constexpr int NP2 = DUAL ? FD * (FD + 1) / 2 : 0;
  constexpr int NPAD = 8 * F;
  constexpr int RQ = REM ? 2 * R * 3 : 0;  // remainder partials per lane: [h][r][3]
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  // SWIZZLE_128B boxes need 1024-byte aligned destinations
  unsigned char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* empty = full + 8;
  double* stage0 = reinterpret_cast<double*>(tsm + 1024);
  const int NB = N;  // box rows: no zero-filled padding rows in the stream
  const size_t qstride = qs_of(NB);
  const size_t sdoubles = (size_t)nsrc * qstride;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TSC);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t kbeg = (int64_t)blockIdx.x * kchunk;
  const int64_t kend = min(kbeg + kchunk, ld);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t4 = lane & 3;
  double* red = stage0;  // after the loop: [8 warps][(NP + NP2) * 64] then [8][RQ][32]
  double* rred = red + (size_t)TSC * (NP + NP2) * 64;
  if (warp >= TSC) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    produce(maps, nsrc, NB, kbeg, kend, nst, sdoubles, stage0, full, empty);
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    double acc[NP > 0 ? NP : 1][2], acc2[NP2 > 0 ? NP2 : 1][2];
#pragma unroll
    for (int q = 0; q < NP; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
    for (int q = 0; q < NP2; ++q) acc2[q][0] = acc2[q][1] = 0.0;
    double racc[REM ? 2 : 1][REM ? R : 1][3];
#pragma unroll
    for (int h = 0; h < (REM ? 2 : 1); ++h)
#pragma unroll
      for (int r = 0; r < (REM ? R : 1); ++r) racc[h][r][0] = racc[h][r][1] = racc[h][r][2] = 0.0;
    const int nstage = kend > kbeg ? (int)((kend - kbeg + TKS - 1) / TKS) : 0;
    const int c = warp * 8;  // this warp's 8-point chunk of every stage
    // (measured: prefetching the next stage's fragments before this stage's
    // DMMAs made the kernel slower — it is bound by the TMA stream, not by
    // shared-memory latency — so load, release, then multiply)
    for (int st = 0; st < nstage; ++st) {
      const int s = st % nst;
      mbar_wait(&full[s], (uint32_t)(st / nst) & 1u);
      const double* sbuf = stage0 + (size_t)s * sdoubles;
      if (probe) {  // measurement hook: stream the ring without consuming it
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        continue;
      }
      if constexpr (REM) {
        // 8 points of one row of source q as 4 double2, in a lane-rotated pair
        // order: rows i = lane (stride PADW = 8 mod 16) then fall on distinct
        // banks within each quarter-warp (the plain order was a 4-way conflict)
        const int rot = (lane >> 1) & 3;
        auto row8 = [&](int row, int q, double2 (&v)[4]) {
#pragma unroll
          for (int m = 0; m < 4; ++m)
            v[m] = *reinterpret_cast<const double2*>(sbuf + q * qstride +
                                                     pad(row, c + 2 * ((m + rot) & 3)));
        };
        auto dot8 = [](const double2 (&x)[4], const double2 (&y)[4], double t) {
          // four independent products chains instead of one 8-deep FMA chain
          double p0 = x[0].x * y[0].x, p1 = x[0].y * y[0].y, p2 = x[1].x * y[1].x, p3 = x[1].y * y[1].y;
          p0 = fma(x[2].x, y[2].x, p0);
          p1 = fma(x[2].y, y[2].y, p1);
          p2 = fma(x[3].x, y[3].x, p2);
          p3 = fma(x[3].y, y[3].y, p3);
          return t + ((p0 + p1) + (p2 + p3));
        };
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int rr = 8 * FD + r;
          double2 ar[4], br[4];
          row8(rr, 0, ar);
          row8(rr, qb, br);
          // N = 33 (R = 1, 32 DMMA rows): rows 0 .. 31 take all 32 lanes below; the
          // entries of row rr itself come from lane 0's own ar / br (the same
          // products in the same order as the general form, which ran a whole
          // pass of loads and dots for that one live lane)
          constexpr bool ONE = R == 1 && 8 * FD == 32;
          if (ONE && lane == 0) {
            racc[1][r][0] = dot8(ar, br, racc[1][r][0]);  // Sigma(rr, rr)
            racc[1][r][2] = dot8(ar, ar, racc[1][r][2]);  // G_HH(rr, rr)
          }
#pragma unroll
          for (int h = 0; h < (ONE ? 1 : 2); ++h) {
            const int i = lane + 32 * h;
            if (!ONE && i >= N) continue;
            double2 ai[4];
            row8(i, 0, ai);
            racc[h][r][0] = dot8(ai, br, racc[h][r][0]);  // Sigma(i, rr)
            if (i <= rr) racc[h][r][2] = dot8(ai, ar, racc[h][r][2]);  // G_HH(i, rr)
            if (i < 8 * FD) {
              double2 bi[4];
              row8(i, qb, bi);
              racc[h][r][1] = dot8(ar, bi, racc[h][r][1]);  // Sigma(rr, i)
            }
          }
        }
      }
      double2 a[FD > 0 ? FD : 1], b[SYM ? 1 : (FD > 0 ? FD : 1)];
#pragma unroll
      for (int f = 0; f < FD; ++f) {
        const int off = pad(8 * f + gq, c + 2 * t4);  // 16-B aligned pair of points
        a[f] = *reinterpret_cast<const double2*>(sbuf + off);
        if (qa_b >= 0) {
          const double2 z = *reinterpret_cast<const double2*>(sbuf + qa_b * qstride + off);
          a[f].x += sa * z.x;
          a[f].y += sa * z.y;
        }
        if constexpr (!SYM) {
          b[f] = *reinterpret_cast<const double2*>(sbuf + qb * qstride + off);
          if (qb_b >= 0) {
            const double2 z = *reinterpret_cast<const double2*>(sbuf + qb_b * qstride + off);
            b[f].x += sb * z.x;
            b[f].y += sb * z.y;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // fragments are in registers: release early
      int q = 0;
#pragma unroll
      for (int fm = 0; fm < FD; ++fm)
#pragma unroll
        for (int fn = SYM ? fm : 0; fn < FD; ++fn, ++q) {
          const double2 bv = SYM ? a[fn] : b[SYM ? 0 : fn];
          dmma_8x8x4(acc[q], a[fm].x, bv.x);
          dmma_8x8x4(acc[q], a[fm].y, bv.y);
        }
      if constexpr (DUAL) {
        int q2 = 0;
#pragma unroll
        for (int fm = 0; fm < FD; ++fm)
#pragma unroll
          for (int fn = fm; fn < FD; ++fn, ++q2) {
            dmma_8x8x4(acc2[q2], a[fm].x, a[fn].x);
            dmma_8x8x4(acc2[q2], a[fm].y, a[fn].y);
          }
      }
    }
    // all consumers are past the ring: reuse it for the CTA reduction (named
    // barrier over the consumer warps only; the producer warpgroup runs with
    // 40 registers and must not hold the accumulators)
    asm volatile("bar.sync 1, %0;\n" ::"n"(TSC * 32) : "memory");
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      red[(warp * (NP + NP2) + q) * 64 + lane * 2] = acc[q][0];
      red[(warp * (NP + NP2) + q) * 64 + lane * 2 + 1] = acc[q][1];
    }
#pragma unroll
    for (int q = 0; q < NP2; ++q) {
      red[(warp * (NP + NP2) + NP + q) * 64 + lane * 2] = acc2[q][0];
      red[(warp * (NP + NP2) + NP + q) * 64 + lane * 2 + 1] = acc2[q][1];
    }
    if constexpr (REM) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int k = 0; k < 3; ++k) rred[(warp * RQ + (h * R + r) * 3 + k) * 32 + lane] = racc[h][r][k];
    }
  }
  __syncthreads();
  // zero the tiles first when a remainder row exists (its entries come from racc)
  for (int e = threadIdx.x; e < (NP + NP2) * 64; e += TTH) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < TSC; ++w) sum += red[(w * (NP + NP2)) * 64 + e];
    const int qq = e / 64, l = (e % 64) / 2, j = e % 2;
    const bool second = qq >= NP;
    const int q = second ? qq - NP : qq;
    const bool sym = second || SYM;
    int fm = 0, fn = 0, cq = 0;
    for (int m = 0; m < FD; ++m)
      for (int n = sym ? m : 0; n < FD; ++n, ++cq)
        if (cq == q) {
          fm = m;
          fn = n;
        }
    double* out = ws + ((second ? gridDim.x : 0) + (int64_t)blockIdx.x) * NPAD * NPAD;
    out[(8 * fm + (l >> 2)) * NPAD + 8 * fn + 2 * (l & 3) + j] = sum;
  }
  if constexpr (REM) {
    for (int e = threadIdx.x; e < RQ * 32; e += TTH) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < TSC; ++w) sum += rred[w * RQ * 32 + e];
      const int l = e % 32, k = (e / 32) % 3, r = (e / 32 / 3) % R, h = e / 32 / 3 / R;
      const int i = l + 32 * h, rr = 8 * FD + r;
      if (i >= N) continue;
      double* o1 = ws + (int64_t)blockIdx.x * NPAD * NPAD;
      double* o2 = ws + ((int64_t)gridDim.x + blockIdx.x) * NPAD * NPAD;
      if (k == 0) o1[i * NPAD + rr] = sum;                      // Sigma(i, rr)
      else if (k == 1 && i < 8 * FD) o1[rr * NPAD + i] = sum;   // Sigma(rr, i)
      else if (k == 2 && i <= rr) o2[i * NPAD + rr] = sum;      // G_HH(i, rr)
    }
  }
}

// Verification Gram G = W~^T W~ (symmetric) of a rotated block with the density
// / Dirac xc of W~ in the same pass (energy.cpp:67-76, 212-226): rho = occ sum_i
// W~_i^2, v_xc, 4 pi rho into bvec (when non-null), partial rows
// [<eps, rho> | <V_ext, rho>] x grid in dpart. The split form of the trial
// rotation (launch_rotate_fused): the rotation itself runs as the two-source
// mix at ~90% of HBM, this pass reads W~ once.
template <int F>
__global__ void __launch_bounds__(TTH, 1) gram_density_kernel(
    const __grid_constant__ Maps maps, int N, int64_t ld, int64_t ngl, int64_t kchunk, int nst,
    double* __restrict__ ws, double occ, int xc, double* __restrict__ rho, double* __restrict__ vxc,
    double* __restrict__ bvec, const double* __restrict__ vext, double* __restrict__ dpart) {
  PO_PDL_ENTRY();
  constexpr int NP = F * (F + 1) / 2;
  constexpr int NPAD = 8 * F;
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* empty = full + 8;
  double* stage0 = reinterpret_cast<double*>(tsm + 1024);
  const size_t sdoubles = qs_of(N);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TSC);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t kbeg = (int64_t)blockIdx.x * kchunk;
  const int64_t kend = min(kbeg + kchunk, ld);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t4 = lane & 3;
  const double cx = dirac_cx();
  const double four_pi = 4.0 * 3.141592653589793238462643383279502884;
  double* red = stage0;  // after the loop: [8 warps][NP * 64], then energies
  double* ered = red + (size_t)TSC * NP * 64;
  if (warp >= TSC) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    produce(maps, 1, N, kbeg, kend, nst, sdoubles, stage0, full, empty);
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    double acc[NP][2];
#pragma unroll
    for (int q = 0; q < NP; ++q) acc[q][0] = acc[q][1] = 0.0;
    double eacc[2] = {0.0, 0.0};
    const int nstage = kend > kbeg ? (int)((kend - kbeg + TKS - 1) / TKS) : 0;
    const int c = warp * 8;  // this warp's 8 points of every stage
    for (int st = 0; st < nstage; ++st) {
      const int s = st % nst;
      const int64_t p0 = kbeg + (int64_t)st * TKS + c + 2 * t4;  // this lane's two points
      double vx[2] = {0.0, 0.0};
      if (vext && xc >= 0 && gq == 0) {  // requested before the stage wait (latency under the TMA)
        if (p0 < ngl) vx[0] = __ldg(vext + p0);
        if (p0 + 1 < ngl) vx[1] = __ldg(vext + p0 + 1);
      }
      mbar_wait(&full[s], (uint32_t)(st / nst) & 1u);
      const double* sbuf = stage0 + (size_t)s * sdoubles;
      double2 a[F];
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int f = 0; f < F; ++f) {
        a[f] = *reinterpret_cast<const double2*>(sbuf + pad(8 * f + gq, c + 2 * t4));
        if (8 * f + gq < N) {  // rows past N are another area's data
          d0 = fma(a[f].x, a[f].x, d0);
          d1 = fma(a[f].y, a[f].y, d1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      int q = 0;
#pragma unroll
      for (int fm = 0; fm < F; ++fm)
#pragma unroll
        for (int fn = fm; fn < F; ++fn, ++q) {
          dmma_8x8x4(acc[q], a[fm].x, a[fn].x);
          dmma_8x8x4(acc[q], a[fm].y, a[fn].y);
        }
      // density of the lane's two points: sum over the 8 row groups (gq)
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        d0 += __shfl_xor_sync(0xffffffffu, d0, o);
        d1 += __shfl_xor_sync(0xffffffffu, d1, o);
      }
      if (gq == 0) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t p = p0 + e;
          if (p >= ngl) continue;
          const double dv = e ? d1 : d0;
          const double r = occ == 1.0 ? dv : dv * occ;
          rho[p] = r;
          if (xc > 0) {
            const double eps = -cx * cbrt(r);
            vxc[p] = eps * (4.0 / 3.0);
            eacc[0] += eps * r;
          } else if (xc == 0) {
            vxc[p] = 0.0;
          }  // xc < 0: v_xc and the energies come from the v_local pass
          if (bvec) bvec[p] = r * four_pi;
          if (xc >= 0) eacc[1] += vx[e] * r;
        }
      }
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(TSC * 32) : "memory");
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      red[(warp * NP + q) * 64 + lane * 2] = acc[q][0];
      red[(warp * NP + q) * 64 + lane * 2 + 1] = acc[q][1];
    }
    const double e0 = warp_sum(eacc[0]), e1 = warp_sum(eacc[1]);
    if (lane == 0) {
      ered[warp] = e0;
      ered[TSC + warp] = e1;
    }
  }
  __syncthreads();
  double* o = ws + (int64_t)blockIdx.x * NPAD * NPAD;
  for (int e = threadIdx.x; e < NP * 64; e += TTH) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < TSC; ++w) sum += red[(w * NP) * 64 + e];
    const int q = e / 64, l = (e % 64) / 2, j = e % 2;
    int fm = 0, fn = 0, cq = 0;
    for (int m = 0; m < F; ++m)
      for (int n = m; n < F; ++n, ++cq)
        if (cq == q) {
          fm = m;
          fn = n;
        }
    o[(8 * fm + (l >> 2)) * NPAD + 8 * fn + 2 * (l & 3) + j] = sum;
  }
  if (threadIdx.x < 2) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < TSC; ++w) sum += ered[threadIdx.x * TSC + w];
    dpart[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = sum;
  }
}

// G = w sum over splits (one warp per element); blockIdx.y = 1 reduces a second
// matrix (the dual pass's G_HH: ws2 / G2, symmetric) in the same launch, and
// diag (optional) receives G's diagonal (sigma_ii for the directions pass)
__global__ void gram_tma_reduce_kernel(int N, int npad, int sym, int nsplit, double w,
                                       const double* __restrict__ ws, double* __restrict__ G,
                                       const double* __restrict__ guard,
                                       const double* __restrict__ ws2, double* __restrict__ G2,
                                       double* __restrict__ diag) {
  PO_PDL_ENTRY();
  if (guard && *guard == 0.0) return;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= (int64_t)N * N) return;
  const bool second = blockIdx.y == 1;
  if (second) {
    ws = ws2;
    G = G2;
    sym = 1;
  }
  int i = (int)(wid / N), j = (int)(wid % N);
  if (sym && j < i) {
    const int t = i;
    i = j;
    j = t;
  }
  double s = 0.0;
  for (int k = lane; k < nsplit; k += 32) s += ws[(int64_t)k * npad * npad + i * npad + j];
  s = warp_sum(s);
  if (lane == 0) {
    G[wid] = w * s;
    if (diag && !second && i == j) diag[i] = w * s;
  }
}

int g_nsm = 0;
int nsm() {
  if (!g_nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_nsm;
}

template <int F>
bool launch_gram_tma_f(int N, int64_t ld, int sym, const double* A, const double* Ab, double sa,
                       const double* B, const double* Bb, double sb, double* ws, double* G,
                       double w, cudaStream_t s, const double* guard, double* G2, double* diag) {
  constexpr int NPAD = 8 * F;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  int nsrc = 0, qa_b = -1, qb = 0, qb_b = -1;
  if (!make_map2(maps, nsrc++, A, ld, N, NPAD)) return false;
  if (Ab) {
    qa_b = nsrc;
    if (!make_map2(maps, nsrc++, Ab, ld, N, NPAD)) return false;
  }
  if (!sym) {
    qb = nsrc;
    if (!make_map2(maps, nsrc++, B, ld, N, NPAD)) return false;
    if (Bb) {
      qb_b = nsrc;
      if (!make_map2(maps, nsrc++, Bb, ld, N, NPAD)) return false;
    }
  }
  const bool dual = G2 != nullptr && !sym;
  static const int no_rem = getenv("PO_NO_REM") ? atoi(getenv("PO_NO_REM")) : 0;  // measurement
  const int R = !no_rem && dual && F > 1 && (N % 8 == 1 || N % 8 == 2) ? N % 8 : 0;
  const int fd = R ? F - 1 : F;
  const int np = (sym ? fd * (fd + 1) / 2 : fd * fd) + (dual ? fd * (fd + 1) / 2 : 0);
  const size_t red = (size_t)TSC * np * 64 + (size_t)TSC * 12 * 32;
  if (3072 + red * 8 > 220 * 1024) return false;  // reduction scratch > shared memory
  TCfg cfg = tcfg(nsrc, N, 0);
  if (cfg.smem < 3072 + red * 8) cfg.smem = 3072 + red * 8;
  const int64_t kblocks = (ld + TKS - 1) / TKS;
  int nsplit = nsm();
  if (nsplit > kblocks) nsplit = (int)kblocks;
  const int64_t kchunk = ((kblocks + nsplit - 1) / nsplit) * TKS;
  nsplit = (int)((ld + kchunk - 1) / kchunk);
  ::po::count_launch();
  auto k = sym    ? gram_tma_kernel<F, true, false>
           : !dual ? gram_tma_kernel<F, false, false>
           : R == 1 ? gram_tma_kernel<F, false, true, (F > 1 ? 1 : 0)>
           : R == 2 ? gram_tma_kernel<F, false, true, (F > 1 ? 2 : 0)>
                    : gram_tma_kernel<F, false, true, 0>;
  set_smem(reinterpret_cast<const void*>(k), (int)cfg.smem);
  const char* pe = getenv("PO_GRAM_PROBE");  // measurement hook (TMA ring without math)
  const int probe = pe ? atoi(pe) : 0;
  launch_pdl(k, dim3(nsplit), dim3(TTH), cfg.smem, s, maps, N, nsrc, qa_b, qb, qb_b, ld, kchunk, cfg.nst, sa, sb, ws,
                                   guard, probe);
  const int64_t threads = (int64_t)N * N * 32;
  ::po::count_launch();
  launch_pdl(gram_tma_reduce_kernel, dim3((unsigned)((threads + 255) / 256), dual ? 2 : 1), dim3(256), 0, s,
             N, NPAD, sym, nsplit, w, ws, G, guard,
             dual ? (const double*)(ws + (size_t)nsplit * NPAD * NPAD) : (const double*)nullptr,
             dual ? G2 : (double*)nullptr, diag);
  return true;
}

// ------------------------------------------------------------------- mix
// Warp w owns the 8 points [8w, 8w+8) of each 64-point stage (one DMMA row
// fragment) and all N outputs; M (N x N) is in shared memory for the CTA.
template <int F, bool UPPER>
__global__ void __launch_bounds__(TTH, 1) mix_tma_kernel(
    const __grid_constant__ Maps maps, int nsrc, int qc, int N, int64_t ld, int64_t ngl,
    int64_t pchunk, int nst, double sa, const double* __restrict__ M, double alpha, double beta,
    double* __restrict__ out, double* __restrict__ norms, const double* __restrict__ guard,
    const double* __restrict__ sa_dev) {
  PO_PDL_ENTRY();
  if (guard && *guard == 0.0) return;
  if (sa_dev) sa = *sa_dev;  // trial scale decided on the device (bb_tau_kernel)
  constexpr int NPAD = 8 * F;
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  // SWIZZLE_128B boxes need 1024-byte aligned destinations
  unsigned char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* empty = full + 8;
  double* stage0 = reinterpret_cast<double*>(tsm + 1024);
  const int NB = N;  // box rows: no zero-filled padding rows in the stream
  const size_t qstride = qs_of(NB);
  const size_t sdoubles = (size_t)nsrc * qstride;
  double* Ms = stage0 + (size_t)nst * sdoubles;  // [NPAD][NPAD]
  double* nred = Ms + NPAD * NPAD;               // [8][NPAD]
  for (int e = threadIdx.x; e < NPAD * NPAD; e += TTH) {
    const int k = e / NPAD, i = e % NPAD;
    Ms[e] = (k < N && i < N) ? M[(int64_t)k * N + i] : 0.0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TSC);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t pbeg = (int64_t)blockIdx.x * pchunk;
  const int64_t pend = min(pbeg + pchunk, ld);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t4 = lane & 3;
  const bool has_ab = nsrc - (qc >= 0 ? 1 : 0) == 2;
  if (warp >= TSC) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    produce(maps, nsrc, NB, pbeg, pend, nst, sdoubles, stage0, full, empty);
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    double nrm[F][2];
#pragma unroll
    for (int fi = 0; fi < F; ++fi) nrm[fi][0] = nrm[fi][1] = 0.0;
    const int nstage = pend > pbeg ? (int)((pend - pbeg + TKS - 1) / TKS) : 0;
    const int ksteps = (N + 3) / 4;
    const int c = warp * 8;
    // upper-triangular M: this lane's B fragments for every (k-step, output fragment)
    double mreg[UPPER ? 2 * F : 1][UPPER ? F : 1];
    if constexpr (UPPER) {
#pragma unroll
      for (int ks = 0; ks < 2 * F; ++ks)
#pragma unroll
        for (int fi = 0; fi < F; ++fi)
          mreg[ks][fi] = 4 * ks > 8 * fi + 7 ? 0.0 : Ms[(4 * ks + t4) * NPAD + 8 * fi + gq];
    }
    for (int st = 0; st < nstage; ++st) {
      const int s = st % nst;
      mbar_wait(&full[s], (uint32_t)(st / nst) & 1u);
      const double* sbuf = stage0 + (size_t)s * sdoubles;
      const int64_t k0 = pbeg + (int64_t)st * TKS;
      double acc[F][2];
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f][0] = acc[f][1] = 0.0;
      if constexpr (UPPER) {
        // all A values of the chunk first (one latency), M fragments from registers
        double av[2 * F];
#pragma unroll
        for (int ks = 0; ks < 2 * F; ++ks) {
          const int off = pad(4 * ks + t4, c + gq);
          av[ks] = sbuf[off];
          if (has_ab) av[ks] += sa * sbuf[qstride + off];
          if (4 * ks + t4 >= N) av[ks] = 0.0;  // rows past N alias the next box
        }
#pragma unroll
        for (int ks = 0; ks < 2 * F; ++ks) {
          // no runtime trip count: k rows >= N are zero in both operands, and a
          // data-dependent exit serialised the unrolled k-steps (load, DMMA, branch)
#pragma unroll
          for (int fi = 0; fi < F; ++fi) {
            if (4 * ks > 8 * fi + 7) continue;
            dmma_8x8x4(acc[fi], av[ks], mreg[ks][fi]);
          }
        }
      } else {
        for (int ks = 0; ks < ksteps; ++ks) {
          const int krow = 4 * ks + t4;
          const int off = pad(krow, c + gq);
          double av = sbuf[off];
          if (has_ab) av += sa * sbuf[qstride + off];
          if (krow >= N) av = 0.0;
#pragma unroll
          for (int fi = 0; fi < F; ++fi) dmma_8x8x4(acc[fi], av, Ms[krow * NPAD + 8 * fi + gq]);
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
            if (qc >= 0) v += beta * sbuf[qc * qstride + pad(i, c + gq)];
            if (out) out[(int64_t)i * ld + p] = v;
            nrm[fi][j] += v * v;
          }
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
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
    }
  }
  if (norms) {
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += TTH) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < TSC; ++w) sum += nred[w * NPAD + i];
      norms[(int64_t)i * gridDim.x + blockIdx.x] = sum;
    }
  }
}

// ------------------------------------------------------------- fused rotation
// The orthonormalisation rotation of a line-search trial with its two
// follow-ups folded into the epilogue (manifold.cpp:97-114 + 136-169,
// energy.cpp:67-76 / 212-226):
//   W~ = (W + sa Z) L^{-T}                 (DMMA, upper-triangular skip; written)
//   G2 partial = W~^T W~ over the CTA's points  (verification Gram, DMMA + FMA tail)
//   rho = occ sum_i W~_i^2, v_xc, 4 pi rho, <eps, rho>, <V_ext, rho> partials
// so the trial's verification Gram and density passes over the block vanish.
// The warp's rotated 8-point chunk goes back into its own slot of the stage
// (same swizzled layout as the source), from where the Gram fragments are read.
// CW consumer warps of 8 points each (stage = 8 CW points): CW = 8 keeps L^{-T}
// in registers next to a producer warpgroup (setmaxnreg); CW = 12 reads it from
// shared memory and has one producer warp (13 warps, at most 4 per SM
// sub-partition: 128 registers; 1.5x the warps in flight for this
// latency-bound pass)
template <int F, int R, int CW, bool ZV = false>
__global__ void __launch_bounds__(CW == 8 ? TTH : (CW + 1) * 32, 1) rotate_fused_kernel(
    const __grid_constant__ Maps maps, int nsrc, int N, int64_t ld, int64_t ngl, int64_t pchunk,
    int nst, double sa, const double* __restrict__ M, double* __restrict__ out,
    double* __restrict__ ws, double occ, int xc, double* __restrict__ rho, double* __restrict__ vxc,
    double* __restrict__ bvec, const double* __restrict__ vext, double* __restrict__ dpart,
    const double* __restrict__ sa_dev, const double* __restrict__ zsig) {
  PO_PDL_ENTRY();
  if (sa_dev) sa = *sa_dev;  // trial scale decided on the device (bb_tau_kernel)
  constexpr int NPAD = 8 * F;
  constexpr int FD = R > 0 ? F - 1 : F;
  constexpr int KS = 8 * CW;                 // points per stage
  // padded row, PW = 4 mod 16 doubles: a half-warp's (gq < 4, t4) reads of
  // rows 4 ks + t4 and writes of rows 2 t4 + j' land in 16 distinct 8-byte
  // slots (64-bit shared accesses are served per half-warp)
  constexpr int PW = KS + 4;
  constexpr int NT = CW == 8 ? TTH : (CW + 1) * 32;
  constexpr int NP = FD * (FD + 1) / 2;
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* empty = full + 8;
  double* stage0 = reinterpret_cast<double*>(tsm + 1024);
  const int NB = N;  // box rows: no zero-filled padding rows in the stream
  const size_t qstride = ((size_t)NB * PW + 15) & ~(size_t)15;
  const size_t sdoubles = (size_t)nsrc * qstride;
  // L^{-T} rows padded to MST = 4 mod 16 doubles (conflict-free fragment reads)
  constexpr int MST = NPAD + 4;
  double* Ms = stage0 + (size_t)nst * sdoubles;  // [NPAD][MST]
  for (int e = threadIdx.x; e < NPAD * MST; e += NT) {
    const int k = e / MST, i = e % MST;
    Ms[e] = (k < N && i < N) ? M[(int64_t)k * N + i] : 0.0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t pbeg = (int64_t)blockIdx.x * pchunk;
  const int64_t pend = min(pbeg + pchunk, ld);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t4 = lane & 3;
  const double cx = dirac_cx();
  const double four_pi = 4.0 * 3.141592653589793238462643383279502884;
  double* red = stage0;
  constexpr int RS = 2 * (R > 0 ? R : 1) * 32;
  double* rred = red + (size_t)CW * NP * 64;
  double* ered = rred + (size_t)CW * RS;
  if (warp >= CW) {
    if constexpr (CW == 8) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == CW) tma_produce_w(maps.m, nsrc, NB, pbeg, pend, nst, sdoubles, stage0, full, empty, KS, PW);
  } else {
    if constexpr (CW == 8) asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    double gacc[NP > 0 ? NP : 1][2];
#pragma unroll
    for (int q = 0; q < NP; ++q) gacc[q][0] = gacc[q][1] = 0.0;
    double racc[2][R > 0 ? R : 1];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int r = 0; r < (R > 0 ? R : 1); ++r) racc[h][r] = 0.0;
    double eacc[2] = {0.0, 0.0};
    const int nstage = pend > pbeg ? (int)((pend - pbeg + KS - 1) / KS) : 0;
    const int c = warp * 8;
    // this lane's fragments of the upper-triangular L^{-T}; with R > 0 the last
    // fragment column (R real orbitals) is a per-lane FMA dot instead of DMMA
    constexpr bool MREG = CW <= 8;  // L^{-T} fragments in registers
    double mreg[MREG ? 2 * F : 1][MREG ? F : 1];
    if constexpr (MREG) {
#pragma unroll
      for (int ks = 0; ks < 2 * F; ++ks)
#pragma unroll
        for (int fi = 0; fi < F; ++fi)
          mreg[ks][fi] = 4 * ks > 8 * fi + 7 ? 0.0 : Ms[(4 * ks + t4) * MST + 8 * fi + gq];
    }
    double mrem[R > 0 ? R : 1][2 * F];
#pragma unroll
    for (int r = 0; r < (R > 0 ? R : 1); ++r)
#pragma unroll
      for (int ks = 0; ks < 2 * F; ++ks)
        mrem[r][ks] = (R > 0 && 4 * ks + t4 < N) ? Ms[(4 * ks + t4) * MST + 8 * FD + r] : 0.0;
    // zsig: the second source is HW and the direction z = HW - sigma W is rebuilt
    // here with the directions pass's FMA (bitwise the value it would have stored)
    double mz[ZV ? 2 * F : 1];
    if constexpr (ZV) {
#pragma unroll
      for (int ks = 0; ks < 2 * F; ++ks) mz[ks] = 4 * ks + t4 < N ? -zsig[4 * ks + t4] : 0.0;
    }
    // V_ext of the next chunk is requested one stage ahead (a global load in
    // the epilogue stalled every warp for its full latency)
    double vx_next = (vext && t4 == 0 && pbeg + c + gq < ngl) ? __ldg(vext + pbeg + c + gq) : 0.0;
    int s = 0;         // ring slot and phase parity, stepped without a division
    uint32_t fph = 0;
    for (int st = 0; st < nstage; ++st) {
      const int64_t p = pbeg + (int64_t)st * KS + c + gq;
      const double vx = vx_next;
      const int64_t pn = p + KS;
      if (vext && t4 == 0 && st + 1 < nstage && pn < ngl) vx_next = __ldg(vext + pn);
      mbar_wait(&full[s], fph);
      double* sbuf = stage0 + (size_t)s * sdoubles;
      double acc[F][2];
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f][0] = acc[f][1] = 0.0;
      {
        double av[2 * F];
#pragma unroll
        for (int ks = 0; ks < 2 * F; ++ks) {
          const int off = (4 * ks + t4) * PW + c + gq;
          av[ks] = sbuf[off];
          if (ZV || nsrc == 2) {
            double zb = sbuf[qstride + off];
            if constexpr (ZV) zb = fma(mz[ZV ? ks : 0], av[ks], zb);
            av[ks] += sa * zb;
          }
          // rows past N alias the next box (N > 8 (F - 1): only the last k-steps can hold one)
          if (4 * ks + 3 > 8 * (F - 1))
            if (4 * ks + t4 >= N) av[ks] = 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < 2 * F; ++ks) {
          // no runtime trip count: k rows >= N are zero in both operands, and a
          // data-dependent exit serialised the unrolled k-steps (load, DMMA, branch)
#pragma unroll
          for (int fi = 0; fi < FD; ++fi) {
            if (4 * ks > 8 * fi + 7) continue;
            if constexpr (MREG)
              dmma_8x8x4(acc[fi], av[ks], mreg[ks][fi]);
            else
              dmma_8x8x4(acc[fi], av[ks], Ms[(4 * ks + t4) * MST + 8 * fi + gq]);
          }
        }
        if constexpr (R > 0) {  // out_rr(point c + gq) = sum_k A_k M(k, rr), k split over t4
#pragma unroll
          for (int r = 0; r < R; ++r) {
            // two independent chains (a 2F-deep dependent FMA chain sat on every stage)
            double t = 0.0, t2 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 2 * F; ks += 2) {
              t = fma(av[ks], mrem[r][ks], t);
              if (ks + 1 < 2 * F) t2 = fma(av[ks + 1], mrem[r][ks + 1], t2);
            }
            t += t2;
            t += __shfl_xor_sync(0xffffffffu, t, 1);
            t += __shfl_xor_sync(0xffffffffu, t, 2);
            acc[FD][r] = t;  // read back below for i = 8 FD + r (lanes with t4 == 0)
          }
        }
      }
      __syncwarp();  // every lane is done reading the chunk's source values
      double dsum = 0.0;
      const int jx = t4 >> 1;  // lanes t4 = 2, 3 store their pair swapped (rows mod 4 distinct)
      // The loop is issue-bound (~800 instructions per stage and warp, most of them
      // integer / control): every fragment below the last holds 8 real orbitals, so
      // only the last one checks i < N; the row offsets are lane constants and the
      // stores are predicated on one point test (same values, same summation order).
      const bool pin = p < ngl;
      double* const outp = out + (int64_t)(2 * t4) * ld + p;
      double* const sp = sbuf + (2 * t4) * PW + c + gq;
      const int64_t lda = jx ? ld : 0, ldb = jx ? 0 : ld;  // first / second stored row of the pair
      const int pwa = jx ? PW : 0, pwb = jx ? 0 : PW;
#pragma unroll
      for (int fi = 0; fi < F; ++fi) {
        const double va = jx ? acc[fi][1] : acc[fi][0];  // element j ^ jx for j = 0, 1
        const double vb = jx ? acc[fi][0] : acc[fi][1];
        if (fi < F - 1) {
          if (pin) {
            outp[(int64_t)(8 * fi) * ld + lda] = va;
            outp[(int64_t)(8 * fi) * ld + ldb] = vb;
          }
          sp[8 * fi * PW + pwa] = va;
          sp[8 * fi * PW + pwb] = vb;
          dsum += va * va;
          dsum += vb * vb;
        } else {
          const int ia = 8 * fi + 2 * t4 + jx, ib = 8 * fi + 2 * t4 + (jx ^ 1);
          if (ia < N) {
            if (pin) outp[(int64_t)(8 * fi) * ld + lda] = va;
            sp[8 * fi * PW + pwa] = va;
            dsum += va * va;
          }
          if (ib < N) {
            if (pin) outp[(int64_t)(8 * fi) * ld + ldb] = vb;
            sp[8 * fi * PW + pwb] = vb;
            dsum += vb * vb;
          }
        }
      }
      // density of the rotated chunk: sum over the 4 lanes sharing point c + gq
      dsum += __shfl_xor_sync(0xffffffffu, dsum, 1);
      dsum += __shfl_xor_sync(0xffffffffu, dsum, 2);
      if (t4 == 0 && p < ngl) {
        const double r = occ == 1.0 ? dsum : dsum * occ;
        rho[p] = r;
        if (xc > 0) {
          const double eps = -cx * cbrt(r);
          vxc[p] = eps * (4.0 / 3.0);
          eacc[0] += eps * r;
        } else if (xc == 0) {
          vxc[p] = 0.0;
        }  // xc < 0: v_xc and the energies are formed by the v_local pass
        if (bvec) bvec[p] = r * four_pi;
        if (vext && xc >= 0) eacc[1] += vx * r;
      }
      __syncwarp();  // rotated chunk visible to the whole warp
      if constexpr (R > 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int rr = 8 * FD + r;
          // point pairs visited in a lane-rotated order: rows i = lane (stride
          // PW = 4 mod 16) then hit distinct banks within each quarter-warp
          const int rot = lane >> 2;
          double2 bv[4];
#pragma unroll
          for (int m = 0; m < 4; ++m)
            bv[m] = *reinterpret_cast<const double2*>(sbuf + (rr) * PW + c + 2 * ((m + rot) & 3));
          if (R == 1 && 8 * FD == 32) {
            // rows 0 .. 31 below take all 32 lanes; the one entry left, (rr, rr), is
            // lane 0's own bv (same products, same order as the general form, which
            // ran 4 loads and 8 FP64 instructions for one live lane)
            if (lane == 0) {
              double p0 = bv[0].x * bv[0].x, p1 = bv[0].y * bv[0].y, p2 = bv[1].x * bv[1].x,
                     p3 = bv[1].y * bv[1].y;
              p0 = fma(bv[2].x, bv[2].x, p0);
              p1 = fma(bv[2].y, bv[2].y, p1);
              p2 = fma(bv[3].x, bv[3].x, p2);
              p3 = fma(bv[3].y, bv[3].y, p3);
              racc[1][r] += (p0 + p1) + (p2 + p3);
            }
          }
#pragma unroll
          for (int h = 0; h < ((R == 1 && 8 * FD == 32) ? 1 : 2); ++h) {
            const int i = lane + 32 * h;
            if (!(R == 1 && 8 * FD == 32) && (i >= N || i > rr)) continue;
            double2 av[4];
#pragma unroll
            for (int m = 0; m < 4; ++m)
              av[m] = *reinterpret_cast<const double2*>(sbuf + (i) * PW + c + 2 * ((m + rot) & 3));
            double p0 = av[0].x * bv[0].x, p1 = av[0].y * bv[0].y, p2 = av[1].x * bv[1].x,
                   p3 = av[1].y * bv[1].y;
            p0 = fma(av[2].x, bv[2].x, p0);
            p1 = fma(av[2].y, bv[2].y, p1);
            p2 = fma(av[3].x, bv[3].x, p2);
            p3 = fma(av[3].y, bv[3].y, p3);
            racc[h][r] += (p0 + p1) + (p2 + p3);
          }
        }
      }
      // G2 fragments: k = points t4 and 4 + t4 of the chunk (two 64-bit reads,
      // conflict-free at PW = 4 mod 16)
      double2 a[FD > 0 ? FD : 1];
#pragma unroll
      for (int f = 0; f < FD; ++f) {
        a[f].x = sbuf[(8 * f + gq) * PW + c + t4];
        a[f].y = sbuf[(8 * f + gq) * PW + c + 4 + t4];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      int q = 0;
#pragma unroll
      for (int fm = 0; fm < FD; ++fm)
#pragma unroll
        for (int fn = fm; fn < FD; ++fn, ++q) {
          dmma_8x8x4(gacc[q], a[fm].x, a[fn].x);
          dmma_8x8x4(gacc[q], a[fm].y, a[fn].y);
        }
      if (++s == nst) {
        s = 0;
        fph ^= 1u;
      }
    }
    // CTA reductions (consumers only, ring reused): G2 partial tile -> ws[block];
    // energies -> dpart[2][grid]
    asm volatile("bar.sync 1, %0;\n" ::"n"(CW * 32) : "memory");
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      red[(warp * NP + q) * 64 + lane * 2] = gacc[q][0];
      red[(warp * NP + q) * 64 + lane * 2 + 1] = gacc[q][1];
    }
    if constexpr (R > 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int r = 0; r < R; ++r) rred[warp * RS + (h * R + r) * 32 + lane] = racc[h][r];
    }
    double e0 = warp_sum(eacc[0]), e1 = warp_sum(eacc[1]);
    if (lane == 0) {
      ered[warp] = e0;
      ered[CW + warp] = e1;
    }
  }
  __syncthreads();
  double* o = ws + (int64_t)blockIdx.x * NPAD * NPAD;
  for (int e = threadIdx.x; e < NP * 64; e += NT) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < CW; ++w) sum += red[(w * NP) * 64 + e];
    const int q = e / 64, l = (e % 64) / 2, j = e % 2;
    int fm = 0, fn = 0, cq = 0;
    for (int m = 0; m < FD; ++m)
      for (int n = m; n < FD; ++n, ++cq)
        if (cq == q) {
          fm = m;
          fn = n;
        }
    o[(8 * fm + (l >> 2)) * NPAD + 8 * fn + 2 * (l & 3) + j] = sum;
  }
  if constexpr (R > 0) {
    for (int e = threadIdx.x; e < RS; e += NT) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < CW; ++w) sum += rred[w * RS + e];
      const int l = e % 32, r = (e / 32) % R, h = e / 32 / R;
      const int i = l + 32 * h, rr = 8 * FD + r;
      if (i < N && i <= rr) o[i * NPAD + rr] = sum;
    }
  }
  if (threadIdx.x < 2) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < CW; ++w) sum += ered[threadIdx.x * CW + w];
    dpart[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = sum;
  }
}

template <int F>
int launch_rotate_fused_f(int N, int64_t ld, int64_t ngl, const double* A, const double* Ab,
                          double sa, const double* M, double* out, double* ws, double* G, double w,
                          double occ, int xc, double* rho, double* vxc, double* bvec,
                          const double* vext, double* dpart, cudaStream_t s,
                          const double* sa_dev, const double* zsig) {
  constexpr int NPAD = 8 * F;
  if (xc < 0) vext = nullptr;  // <V_ext, rho> belongs to the v_local pass then: no per-stage V_ext prefetch
  static const int cw_env = getenv("PO_RF_CW") ? atoi(getenv("PO_RF_CW")) : 8;  // measurement (12: slower, 228 vs 215 us at C2)
  const int R = (N % 8 == 1 || N % 8 == 2) && N > 8 ? N % 8 : 0;
  // 12 consumer warps where they fit 128 registers without spilling (N <= 33)
  const int CW = zsig || cw_env == 8 ? 8 : cw_env == 6 ? 6 : (F > 5 || (F == 5 && R == 2) ? 8 : 12);
  const int KS = 8 * CW, PW = KS + 4;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  int nsrc = 0;
  if (!make_map(&maps.m[nsrc++], A, ld, N, N, PW)) return -1;
  if (Ab && !make_map(&maps.m[nsrc++], Ab, ld, N, N, PW)) return -1;
  const int fd = R ? F - 1 : F;
  const size_t red = (size_t)CW * (fd * (fd + 1) / 2) * 64 + (size_t)CW * 2 * 2 * 32 + 2 * CW;
  const size_t extra = (size_t)NPAD * (NPAD + 4);
  // ring: stages of KS points, padded rows; tail for fragment rows past N
  const size_t qs = ((size_t)N * PW + 15) & ~(size_t)15;
  const size_t sd = (size_t)nsrc * qs;
  int nst = (int)((tbudget() / 8 - extra) / sd);
  if (nst > 8) nst = 8;
  if (nst < 2) nst = 2;
  size_t smem = 3072 + (size_t)8 * PW * 8 + ((size_t)nst * sd + extra) * 8;
  if (smem < 2048 + red * 8) smem = 2048 + red * 8;
  const int64_t kb = (ld + KS - 1) / KS;
  int nblk = nsm();
  if (nblk > kb) nblk = (int)kb;
  const int64_t pchunk = ((kb + nblk - 1) / nblk) * KS;
  nblk = (int)((ld + pchunk - 1) / pchunk);
  auto k = zsig ? (F == 1 || R == 0 ? rotate_fused_kernel<F, 0, 8, true>
                             : R == 1 ? rotate_fused_kernel<F, 1, 8, true> : rotate_fused_kernel<F, 2, 8, true>)
         : CW == 6 ? (F == 1 || R == 0 ? rotate_fused_kernel<F, 0, 6>
                                       : R == 1 ? rotate_fused_kernel<F, 1, 6> : rotate_fused_kernel<F, 2, 6>)
         : CW == 8 ? (F == 1 || R == 0 ? rotate_fused_kernel<F, 0, 8>
                                       : R == 1 ? rotate_fused_kernel<F, 1, 8> : rotate_fused_kernel<F, 2, 8>)
                   : (F == 1 || R == 0 ? rotate_fused_kernel<F, 0, 12>
                                       : rotate_fused_kernel<F, 1, (F <= 5 ? 12 : 8)>);
  const int nthreads = CW == 8 ? TTH : (CW + 1) * 32;
  TCfg cfg{nst, sd, smem};
  ::po::count_launch();
  set_smem(reinterpret_cast<const void*>(k), (int)cfg.smem);
  launch_pdl(k, dim3(nblk), dim3(nthreads), cfg.smem, s, maps, nsrc, N, ld, ngl, pchunk, cfg.nst, sa, M, out, ws, occ, xc,
                                 rho, vxc, bvec, vext, dpart, sa_dev, zsig);
  const int64_t threads = (int64_t)N * N * 32;
  ::po::count_launch();
  launch_pdl(gram_tma_reduce_kernel, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, s, N, NPAD, 1,
             nblk, w, ws, G, (const double*)nullptr, (const double*)nullptr, (double*)nullptr,
             (double*)nullptr);
  return nblk;
}

// ---------------------------------------------------------- fused directions
// compute_directions + the BB products in ONE pass over the blocks
// (optimizer.cpp:265-320 and 376-411; manifold.cpp:181-202):
//   z_i  = HW_i - sigma_ii W_i                  (written; ||z_i||^2)
//   D_i  = HW_i - sum_k Sigma_ki W_k  [DD]      (DMMA, not written; ||D_i||^2)
//   s_i  = W_i - WP_i, y_i = z_i - ZP_i [HIST]  (<s,s>, <s,y>, <y,y>)
// Sources in the ring: 0 = W, 1 = HW, 2 = WP, 3 = ZP. Per-orbital partial rows
// [zz | dd | ss | sy | yy] x gridDim.x (dd = 0 without DD).
// LDGH: W_prev / Z_prev are read by the consumers with plain loads issued at the
// top of the stage (they are only needed elementwise, for the BB products), so
// the TMA ring carries two sources and holds twice the stages
// CW consumer warps (stage = 8 CW points): CW = 6 with a 52-point padded row
// gives a three-deep ring for the four streamed sources at N = 33 (CW = 8: two
// stages of 76 KB, i.e. one stage in flight while one is consumed)
// ZM: 0 = z stored, ZP is the previous z; 1 = z not stored (implicit), ZP is
// the previous z; 2 = z not stored, ZP is the previous HW (previous z implicit)
template <int F, bool DD, bool HIST, bool LDGH, int CW, int ZM = 0>
__global__ void __launch_bounds__(CW == 8 ? TTH : (CW + 1) * 32, 1) directions_tma_kernel(
    const __grid_constant__ Maps maps, int N, int64_t ld, int64_t ngl, int64_t pchunk, int nst,
    const double* __restrict__ Sigma, const double* __restrict__ sig, double* __restrict__ Z,
    double* __restrict__ partials, const double* __restrict__ WP, const double* __restrict__ ZP,
    const double* __restrict__ psig, double* __restrict__ sig_out) {
  PO_PDL_ENTRY();
  constexpr int NPAD = 8 * F;
  constexpr int NSRC = HIST && !LDGH ? 4 : 2;
  constexpr int NQ = HIST ? 5 : 2;
  constexpr int KS = 8 * CW;
  constexpr int PW = CW == 8 ? PADW : KS + 4;  // conflict-free padded row (see PADW)
  constexpr int NT = CW == 8 ? TTH : (CW + 1) * 32;
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* empty = full + 8;
  double* stage0 = reinterpret_cast<double*>(tsm + 1024);
  const int NB = N;  // box rows: no zero-filled padding rows in the stream
  const size_t qstride = ((size_t)NB * PW + 15) & ~(size_t)15;
  const size_t sdoubles = NSRC * qstride;
  // Sigma rows padded to MST = 4 mod 16 doubles: the fragment reads of rows
  // 4 ks + t4 are then conflict-free per half-warp
  constexpr int MST = NPAD + 4;
  double* Ms = stage0 + (size_t)nst * sdoubles;  // [NPAD][MST] (DD)
  double* msig = Ms + NPAD * MST;                // [NPAD]: -sigma_ii
  double* mpsig = msig + NPAD;                   // [NPAD]: -sigma_ii of the previous iterate
  double* nred = mpsig + NPAD;                   // [8][NQ][NPAD]
  for (int e = threadIdx.x; e < NPAD * MST; e += NT) {
    const int k = e / MST, i = e % MST;
    Ms[e] = (DD && k < N && i < N) ? Sigma[(int64_t)k * N + i] : 0.0;
  }
  for (int i = threadIdx.x; i < NPAD; i += NT) {
    msig[i] = i < N ? -sig[i] : 0.0;
    mpsig[i] = ZM == 2 && i < N ? -psig[i] : 0.0;
    if (sig_out && blockIdx.x == 0 && i < N) sig_out[i] = sig[i];  // the sigma z is built from
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t pbeg = (int64_t)blockIdx.x * pchunk;
  const int64_t pend = min(pbeg + pchunk, ld);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t4 = lane & 3;
  if (warp >= CW) {
    if constexpr (CW == 8) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == CW) tma_produce_w(maps.m, NSRC, NB, pbeg, pend, nst, sdoubles, stage0, full, empty, KS, PW);
  } else {
    if constexpr (CW == 8) asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    double nrm[NQ][F][2];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int fi = 0; fi < F; ++fi) nrm[q][fi][0] = nrm[q][fi][1] = 0.0;
    const int nstage = pend > pbeg ? (int)((pend - pbeg + KS - 1) / KS) : 0;
    const int c = warp * 8;
    // lanes t4 = 2, 3 visit their pair of orbitals swapped: rows 2 t4 + j'
    // then differ mod 4 across the half-warp (PW = 4 mod 16, conflict-free);
    // slot j of nrm holds orbital 8 fi + 2 t4 + (j ^ jx)
    const int jx = t4 >> 1;
    // this lane's -sigma values in registers (the ring waits clobber memory,
    // so shared-memory copies would be re-read every stage)
    double msr[F][2], mpr[ZM == 2 ? F : 1][2];
#pragma unroll
    for (int fi = 0; fi < F; ++fi)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int i = 8 * fi + 2 * t4 + (j ^ jx);
        msr[fi][j] = msig[i];
        if constexpr (ZM == 2) mpr[fi][j] = mpsig[i];
      }
    int s = 0;         // ring slot and phase parity, stepped without a division
    uint32_t fph = 0;
    for (int st = 0; st < nstage; ++st) {
      mbar_wait(&full[s], fph);
      const double* sbuf = stage0 + (size_t)s * sdoubles;
      const int64_t p = pbeg + (int64_t)st * KS + c + gq;
      double acc[F][2];
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f][0] = acc[f][1] = 0.0;
      double wpv[LDGH ? F : 1][2], zpv[LDGH ? F : 1][2];
      if constexpr (HIST && LDGH) {
#pragma unroll
        for (int fi = 0; fi < F; ++fi)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int i = 8 * fi + 2 * t4 + (j ^ (t4 >> 1));
            const bool ok = p < ngl && i < N;
            wpv[fi][j] = ok ? __ldcs(WP + (int64_t)i * ld + p) : 0.0;
            zpv[fi][j] = ok ? __ldcs(ZP + (int64_t)i * ld + p) : 0.0;
          }
      }
      if constexpr (DD) {
        // even / odd k-steps into separate accumulators: 2F independent DMMA chains
        // instead of F chains of length 2F (the loop is unrolled over the 2F slots)
        double acc2[F][2];
#pragma unroll
        for (int f = 0; f < F; ++f) acc2[f][0] = acc2[f][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 2 * F; ++ks) {
          // no runtime trip count: k rows >= N are zero in both operands, and a
          // data-dependent exit serialised the unrolled k-steps (load, DMMA, branch)
          const int krow = 4 * ks + t4;
          // (N > 8 (F - 1): only the last k-steps can hold a row past N, which aliases the next area)
          const double av = (4 * ks + 3 <= 8 * (F - 1) || krow < N) ? sbuf[(krow) * PW + c + gq] : 0.0;
#pragma unroll
          for (int fi = 0; fi < F; ++fi) {
            if (ks & 1)
              dmma_8x8x4(acc2[fi], av, Ms[krow * MST + 8 * fi + gq]);
            else
              dmma_8x8x4(acc[fi], av, Ms[krow * MST + 8 * fi + gq]);
          }
        }
#pragma unroll
        for (int f = 0; f < F; ++f) {
          acc[f][0] += acc2[f][0];
          acc[f][1] += acc2[f][1];
        }
      }
#pragma unroll
      for (int fi = 0; fi < F; ++fi)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = 8 * fi + 2 * t4 + (j ^ jx);
          // the loop is issue-bound: fragments below the last hold 8 real orbitals
          // (no row test), and points past ngl are zero padding in every block —
          // they add exact zeros to the sums, only a stored z needs the point test
          if (fi < F - 1 || i < N) {
            const int off = (i) * PW + c + gq;
            const double wv = sbuf[off], hv = sbuf[qstride + off];
            if constexpr (DD) {
              double d = -(jx ? acc[fi][j ^ 1] : acc[fi][j]);
              d += hv;
              nrm[1][fi][j] += d * d;
            }
            // z = HW - sigma W (one FMA; rotate_fused and the previous-z term
            // below rebuild exactly this value when z is not stored, Z == null)
            const double z = fma(msr[fi][j], wv, hv);
            if constexpr (ZM == 0) {
              if (p < ngl) Z[(int64_t)i * ld + p] = z;
            }
            nrm[0][fi][j] += z * z;
            if constexpr (HIST) {
              const double wp = LDGH ? wpv[fi][j] : sbuf[2 * qstride + off];
              double zp = LDGH ? zpv[fi][j] : sbuf[3 * qstride + off];
              if constexpr (ZM == 2) zp = fma(mpr[ZM == 2 ? fi : 0][j], wp, zp);  // source 3: previous HW
              const double sv = wv - wp;
              const double yv = z - zp;
              nrm[2][fi][j] += sv * sv;
              nrm[3][fi][j] += sv * yv;
              nrm[4][fi][j] += yv * yv;
            }
          }
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == nst) {
        s = 0;
        fph ^= 1u;
      }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int fi = 0; fi < F; ++fi)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          double v = nrm[q][fi][j];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          if (gq == 0) nred[(warp * NQ + q) * NPAD + 8 * fi + 2 * t4 + (j ^ (t4 >> 1))] = v;
        }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NQ * N; e += NT) {
    const int q = e / N, i = e % N;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < CW; ++w) sum += nred[(w * NQ + q) * NPAD + i];
    partials[((int64_t)q * N + i) * gridDim.x + blockIdx.x] = sum;
  }
}

template <int F, bool DD, bool HIST>
int launch_directions_fdh(const double* W, const double* HW, int N, int64_t ld, int64_t ngl,
                          const double* Sigma, const double* sig, double* Z, double* partials,
                          cudaStream_t s, const double* WP, const double* ZP, const double* psig,
                          double* sig_out) {
  constexpr int NPAD = 8 * F;
  constexpr int NQ = HIST ? 5 : 2;
  // (measured and dropped: W_prev / Z_prev through direct loads instead of the
  // ring, 286 vs 244 us at C2 — the kernel keeps the LDGH template switch)
  const bool ldgh = false;
  // six consumer warps where the 8-warp ring would hold only two stages of the
  // four streamed sources (measurement switch PO_DIR_CW = 6 / 8)
  static const int cw_env = getenv("PO_DIR_CW") ? atoi(getenv("PO_DIR_CW")) : 0;
  const int nsrc = HIST && !ldgh ? 4 : 2;
  const int zm = Z ? 0 : (HIST && psig ? 2 : 1);
  // implicit z (zm = 2, no stores): eight consumer warps with a two-deep ring
  // measured 173 vs 197 us for six warps / three stages at C2 (PO_DIR_CW=6 compares)
  // (F <= 5: two stages of the four sources fit shared memory)
  const int CW = zm == 2 ? (cw_env == 6 || F > 5 ? 6 : 8)
                         : zm == 0 && cw_env >= 4 && cw_env <= 8 && cw_env != 7 ? cw_env
                                                                                 : (nsrc == 4 ? 6 : 8);
  const int KS = 8 * CW, PW = CW == 8 ? PADW : KS + 4;
  const size_t extra = (size_t)NPAD * (NPAD + 4) + 2 * NPAD + (size_t)CW * NQ * NPAD;
  const size_t sd = (size_t)nsrc * (((size_t)N * PW + 15) & ~(size_t)15);
  int nst = (int)((tbudget() / 8 - extra) / sd);
  if (nst > 8) nst = 8;
  if (nst < 2) nst = 2;
  const TCfg cfg{nst, sd, 3072 + (size_t)8 * PW * 8 + ((size_t)nst * sd + extra) * 8};
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  const double* srcs[4] = {W, HW, WP, ZP};
  for (int q = 0; q < nsrc; ++q)
    if (!make_map(&maps.m[q], srcs[q], ld, N, N, PW)) return -1;
  const int64_t kb = (ld + KS - 1) / KS;
  int nblk = nsm();
  if (nblk > kb) nblk = (int)kb;
  const int64_t pchunk = ((kb + nblk - 1) / nblk) * KS;
  nblk = (int)((ld + pchunk - 1) / pchunk);
  ::po::count_launch();
  auto k = zm == 1   ? (HIST ? directions_tma_kernel<F, DD, HIST, false, 6, 1>
                               : directions_tma_kernel<F, DD, HIST, false, 8, 1>)
           : zm == 2 ? (CW == 8 ? directions_tma_kernel<F, DD, HIST, false, 8, 2>
                                : directions_tma_kernel<F, DD, HIST, false, 6, 2>)
           : CW == 8 ? directions_tma_kernel<F, DD, HIST, false, 8>
           : CW == 6 ? directions_tma_kernel<F, DD, HIST, false, 6>
           : CW == 5 ? directions_tma_kernel<F, DD, HIST, false, 5>
                     : directions_tma_kernel<F, DD, HIST, false, 4>;
  set_smem(reinterpret_cast<const void*>(k), (int)cfg.smem);
  launch_pdl(k, dim3(nblk), dim3(CW == 8 ? TTH : (CW + 1) * 32), cfg.smem, s, maps, N, ld, ngl, pchunk, cfg.nst, Sigma, sig, Z,
             partials, WP, ZP, psig, sig_out);
  return nblk;
}

template <int F>
int launch_directions_f(int N, int64_t ld, int64_t ngl, const double* W, const double* HW,
                        const double* WP, const double* ZP, const double* Sigma, const double* sig,
                        double* Z, double* partials, cudaStream_t s, const double* psig,
                        double* sig_out) {
  const bool hist = WP && ZP;
  if (Sigma)
    return hist ? launch_directions_fdh<F, true, true>(W, HW, N, ld, ngl, Sigma, sig, Z, partials, s, WP, ZP, psig, sig_out)
                : launch_directions_fdh<F, true, false>(W, HW, N, ld, ngl, Sigma, sig, Z, partials, s, WP, ZP, psig, sig_out);
  return hist ? launch_directions_fdh<F, false, true>(W, HW, N, ld, ngl, Sigma, sig, Z, partials, s, WP, ZP, psig, sig_out)
              : launch_directions_fdh<F, false, false>(W, HW, N, ld, ngl, Sigma, sig, Z, partials, s, WP, ZP, psig, sig_out);
}

template <int F>
int launch_mix_tma_f(int N, int64_t ld, int64_t ngl, const double* A, const double* Ab, double sa,
                     const double* M, double alpha, const double* C, double beta, int upper,
                     double* out, double* norms, cudaStream_t s, const double* guard,
                     const double* sa_dev = nullptr) {
  constexpr int NPAD = 8 * F;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  int nsrc = 0, qc = -1;
  if (!make_map2(maps, nsrc++, A, ld, N, NPAD)) return -1;
  if (Ab && !make_map2(maps, nsrc++, Ab, ld, N, NPAD)) return -1;
  if (C) {
    qc = nsrc;
    if (!make_map2(maps, nsrc++, C, ld, N, NPAD)) return -1;
  }
  const size_t extra = (size_t)NPAD * NPAD + (size_t)TSC * NPAD;
  const TCfg cfg = tcfg(nsrc, N, extra);
  const int64_t kb = (ld + TKS - 1) / TKS;
  int nblk = nsm();
  if (nblk > kb) nblk = (int)kb;
  const int64_t pchunk = ((kb + nblk - 1) / nblk) * TKS;
  nblk = (int)((ld + pchunk - 1) / pchunk);
  ::po::count_launch();
  if (upper) {
    auto k = mix_tma_kernel<F, true>;
    set_smem(reinterpret_cast<const void*>(k), (int)cfg.smem);
    launch_pdl(k, dim3(nblk), dim3(TTH), cfg.smem, s, maps, nsrc, qc, N, ld, ngl, pchunk, cfg.nst, sa, M, alpha, beta,
                                   out, norms, guard, sa_dev);
  } else {
    auto k = mix_tma_kernel<F, false>;
    set_smem(reinterpret_cast<const void*>(k), (int)cfg.smem);
    launch_pdl(k, dim3(nblk), dim3(TTH), cfg.smem, s, maps, nsrc, qc, N, ld, ngl, pchunk, cfg.nst, sa, M, alpha, beta,
                                   out, norms, guard, sa_dev);
  }
  return nblk;
}

// ------------------------------------------------------- large-N tiled Gram
// G = w (A + sa Ab)^T (B + sb Bb) for N > 48, tiled 128 x 128 over orbital
// pairs and split over points (deterministic fixed-order reduction of the
// per-split partial tiles). Each 16-point stage of a source is ONE box
// {16 points x 128 rows} (16 KB, SWIZZLE_128B, rows >= N zero-filled), so a
// producer warp keeps up to 8 stages in flight with a handful of requests.
// Eight consumer warps own 32 x 64 sub-tiles (4 x 8 DMMA fragments): per 8
// points a warp loads 4 + 8 double2 fragments and issues 64 DMMAs. In the
// symmetric case only tiles on/above the diagonal exist, diagonal tiles skip
// fragment pairs below the diagonal and never load B.

__device__ __forceinline__ void big_tile_index(int t, int mt, int sym, int& tm, int& tn) {
  if (!sym) {
    tm = t / mt;
    tn = t % mt;
    return;
  }
  int r = 0, rem = t;
  while (rem >= mt - r) {
    rem -= mt - r;
    ++r;
  }
  tm = r;
  tn = r + rem;
}

// T = 128: a producer warpgroup (one lane issues the boxes) that hands its
// registers to the two consumer warpgroups (setmaxnreg 40 / 232); T = 64: one
// producer warp. (ptxas still compiles the whole kernel for 168 registers, and
// a 9-warp block cannot have more: the register file is split over the four
// SM sub-partitions and one of them holds 3 of the 9 warps — measured as a
// launch failure at 216 registers x 288 threads.)
template <int GT_T>
struct BigCfg {  // consumer warps WM x WN, warp tile (T/WM) x (T/WN)
  static constexpr int WM = 4, WN = 2;
  static constexpr int NW = WM * WN;
  static constexpr int PW = GT_T == 128 ? 4 : 1;  // producer warps (first)
  static constexpr int THREADS = (NW + PW) * 32;
  static constexpr int FM = GT_T / (8 * WM), FN = GT_T / (8 * WN);
};

// Stage loop of a T = 128 symmetric diagonal tile (gram_big_kernel). The 16
// fragment rows form an 8 x 8 grid of 16 x 16 super-blocks; warp a of each
// half owns super-rows a and a + 4 and the circulant slots (R, (R + k) mod 8),
// k = 0..3, plus the one slot (a, a + 4): 9 super-blocks = 36 DMMA blocks per
// k-step, the same straight-line code for every warp (8 of the 144 issued
// blocks, the lower halves of the diagonal super-blocks, are wasted; every
// unordered super-block pair appears exactly once). Per 8 points a warp loads
// the 16 fragments once (16 LDS.128) for 72 DMMAs. acc0[k] = (a, a + k),
// acc1[k] = (a + 4, (a + 4 + k) mod 8). TWO: the operand is A + sa Ab, formed at
// the fragment load.
struct DensArgs {  // DENS: the tile's density rides on the stage loop (see gram_big_kernel)
  double* rho;
  double* bvec;
  double occ;
  int64_t p0, ngl;  // first point of the CTA's range, points of the slab
  int w8;           // consumer warp 0..7
};

template <bool TWO, bool DENS>
__device__ __forceinline__ void sym_diag_stages(double (&acc0)[5][2][2][2], double (&acc1)[4][2][2][2],
                                                int a, const double* stage0, size_t sdoubles,
                                                int nstage, int nst, uint64_t* full, uint64_t* empty,
                                                int q0, int qb2, double sa, int t4, int gq, int lane,
                                                const DensArgs& da) {
  constexpr int QS = 128 * BOX;
  // doubles offset of fragment (2 sr(j), row gq, points 2 t4 ..) in an area; the
  // second fragment of the super-row is + 8 rows, the second 8 points ^ 8
  int off[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) off[j] = q0 * QS + swz(16 * ((a + j) & 7) + gq, 2 * t4, 128);
  const int dz = TWO ? (qb2 - q0) * QS : 0;
  for (int st = 0; st < nstage; ++st) {
    const int s = st % nst;
    mbar_wait(&full[s], (uint32_t)(st / nst) & 1u);
    const double* sbuf = stage0 + (size_t)s * sdoubles;
    if constexpr (DENS) {
      // rho of 4 of the stage's 32 points per warp, before the fragments are
      // loaded: lane (q, c) sums the squares of orbitals 8 j + c at point
      // 4 (w8 & 3) + q of half w8 >> 2 (a half-warp's 8 rows x 2 points are 16
      // distinct 8-byte slots under the swizzle), then the 8 classes meet by
      // shuffles. 16 DFMAs per lane in the warp's own stream (a separate density
      // warp's DFMAs waited behind the consumers' DMMAs on the FP64 pipe).
      const int o = 4 * (da.w8 & 3) + (lane >> 3), c = lane & 7;
      const double* area = sbuf + (size_t)(da.w8 >> 2) * QS;
      double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;  // four independent chains of four
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const double v0 = area[swz(8 * j + c, o, 128)], v1 = area[swz(8 * j + 8 + c, o, 128)];
        const double v2 = area[swz(8 * j + 16 + c, o, 128)], v3 = area[swz(8 * j + 24 + c, o, 128)];
        d0 = fma(v0, v0, d0);
        d1 = fma(v1, v1, d1);
        d2 = fma(v2, v2, d2);
        d3 = fma(v3, v3, d3);
      }
      double d = (d0 + d1) + (d2 + d3);
      d += __shfl_xor_sync(0xffffffffu, d, 1);
      d += __shfl_xor_sync(0xffffffffu, d, 2);
      d += __shfl_xor_sync(0xffffffffu, d, 4);
      const int64_t p = da.p0 + (int64_t)st * 2 * BOX + 16 * (da.w8 >> 2) + o;
      if (c == 0 && p < da.ngl) {
        const double r = da.occ == 1.0 ? d : d * da.occ;
        da.rho[p] = r;
        if (da.bvec) da.bvec[p] = r * (4.0 * 3.141592653589793238462643383279502884);
      }
    }
#pragma unroll
    for (int kg = 0; kg < 2; ++kg) {
      double2 f[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double* src = sbuf + ((off[j] + e * 8 * BOX) ^ (8 * kg));
          f[j][e] = *reinterpret_cast<const double2*>(src);
          if (TWO) {
            const double2 zb = *reinterpret_cast<const double2*>(src + dz);
            f[j][e].x += sa * zb.x;
            f[j][e].y += sa * zb.y;
          }
        }
      if (kg == 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // all fragments of the stage are in registers
      }
#pragma unroll
      for (int k = 0; k < 5; ++k)
#pragma unroll
        for (int ea = 0; ea < 2; ++ea)
#pragma unroll
          for (int eb = 0; eb < 2; ++eb) dmma_8x8x4(acc0[k][ea][eb], f[0][ea].x, f[k][eb].x);
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int ea = 0; ea < 2; ++ea)
#pragma unroll
          for (int eb = 0; eb < 2; ++eb) dmma_8x8x4(acc1[k][ea][eb], f[4][ea].x, f[4 + k][eb].x);
#pragma unroll
      for (int k = 0; k < 5; ++k)
#pragma unroll
        for (int ea = 0; ea < 2; ++ea)
#pragma unroll
          for (int eb = 0; eb < 2; ++eb) dmma_8x8x4(acc0[k][ea][eb], f[0][ea].y, f[k][eb].y);
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int ea = 0; ea < 2; ++ea)
#pragma unroll
          for (int eb = 0; eb < 2; ++eb) dmma_8x8x4(acc1[k][ea][eb], f[4][ea].y, f[4 + k][eb].y);
    }
  }
}

// BB: the elementwise half of compute_directions rides on the Sigma Gram
// (N > 64, non-symmetric 128-tiles: area 0 holds HW rows of tile tm, area qb W
// rows of tile tn — on the tiles with tm == tn every orbital of both blocks
// passes through shared memory anyway; for N <= 128 that is the only tile). Each lane pair of
// the eight consumer warps owns one orbital and, per stage, reads its 16 points
// of HW, W and — from two extra ring areas — W_prev and HW_prev
// (or a stored Z_prev): z = fma(-sigma_i, W, HW) (the FMA of every z path),
// ||z_i||^2 and the BB products <s,s>, <s,y>, <y,y> against (W_prev, z_prev)
// (manifold.cpp:204-216, optimizer.cpp:386-397) accumulate in registers over
// the CTA's point range; one partial per (sum, orbital, split). sigma_i is the
// H u pass's own <HW_i, W_i> (the Gram's diagonal does not exist yet). The
// separate streaming pass over four blocks (1.24 ms at C3) disappears; the
// FP64-bound Gram hides the two extra streams.
struct GramBBArgs {
  const double* sig;    // sigma_i of the current iterate (device, N)
  const double* sigp;   // previous sigma (z_prev implicit) or null (area holds Z_prev)
  double* part;         // [4][N][nsplit]: zz, ss, sy, yy (raw sums)
  int hist;             // history valid: W_prev / X_prev areas are streamed
  int N;
};

template <int GT_T, bool BB = false>
__global__ void __launch_bounds__(BigCfg<GT_T>::THREADS, 1) gram_big_kernel(const __grid_constant__ Maps maps,
                                                          int nsrc, int qa_b, int qb, int qb_b,
                                                          int mt, int sym, int64_t ld,
                                                          int64_t kchunk, int nst, double sa,
                                                          double sb, double* __restrict__ ws,
                                                          const double* __restrict__ guard,
                                                          double* __restrict__ rho,
                                                          double* __restrict__ bvec, double occ,
                                                          int64_t ngl, const GramBBArgs bb) {
  // rho (T = 128, one symmetric diagonal tile, one source): the verification
  // Gram of a rotated trial also yields its density (energy.cpp:67-76) and
  // 4 pi rho — each consumer warp sums the squares of all N orbitals at 4 of a
  // stage's 32 points (sym_diag_stages<.., DENS>), so the trial needs no
  // separate density pass
  PO_PDL_ENTRY();
  if (guard && *guard == 0.0) return;
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* empty = full + 8;
  double* stage0 = reinterpret_cast<double*>(tsm + 1024);
  constexpr size_t QS = (size_t)GT_T * BOX;  // doubles per source per stage
  const int nbb_areas = BB && bb.hist ? 2 : 0;  // extra ring areas: W_prev, X_prev
  const size_t sdoubles = (size_t)(nsrc + nbb_areas) * QS;
  int tm, tn;
  big_tile_index(blockIdx.x, mt, sym, tm, tn);
  const bool diag = !BB && sym && tm == tn;
  // BB on N > 128: the tiles with tm == tn hold HW_i and W_i of the same 128
  // orbitals — they carry the sums (and the two extra streams); the others are
  // plain Sigma tiles with the same stage layout
  const bool bbt = BB && tm == tn;
  const int nbb = bbt ? nbb_areas : 0;
  // sources fetched per 16-point half: A (+Ab); B (+Bb) unless this is a symmetric diagonal tile
  const int nload = diag ? (qa_b >= 0 ? 2 : 1) : nsrc;
  using Cfg = BigCfg<GT_T>;
  const bool dens = GT_T == 128 && rho && diag && nload == 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t kbeg = (int64_t)blockIdx.y * kchunk;
  const int64_t kend = min(kbeg + kchunk, ld);
  // a diagonal tile consumes 32 points per stage (two 16-point halves, see below)
  const int pps = diag ? 2 * BOX : BOX;
  const int nstage = kend > kbeg ? (int)((kend - kbeg + pps - 1) / pps) : 0;
  const int lane = threadIdx.x & 31;
  int warp = threadIdx.x >> 5;
  if (warp < Cfg::PW) {
    // (40 x 128 + 232 x 256 = the 168 x 384 registers the CTA is launched with:
    // a setmaxnreg.inc asking for more than that waits forever)
    if constexpr (Cfg::PW == 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      for (int q = 0; q < nload + nbb; ++q)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[q])));
      const int nbox = diag ? 2 * nload : nload + nbb;
      const uint32_t bytes = (uint32_t)(nbox * QS * 8);
      for (int st = 0; st < nstage; ++st) {
        const int s = st % nst;
        if (st >= nst) mbar_wait(&empty[s], ((uint32_t)(st / nst) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&full[s], bytes);
        const int x = (int)(kbeg + (int64_t)st * pps);
        double* sbuf = stage0 + (size_t)s * sdoubles;
        if (diag) {  // areas [A(x), Ab(x)?, A(x+16), Ab(x+16)?], all rows of tile tm
          for (int h = 0; h < 2; ++h)
            for (int q = 0; q < nload; ++q)
              tma_load_2d(sbuf + (h * nload + q) * QS, &maps.m[q], x + h * BOX, tm * GT_T, &full[s]);
        } else {
          for (int q = 0; q < nload; ++q) {
            const int row0 = (q == qb || q == qb_b) ? tn * GT_T : tm * GT_T;
            tma_load_2d(sbuf + q * QS, &maps.m[q], x, row0, &full[s]);
          }
          for (int q = nload; q < nload + nbb; ++q)  // BB: W_prev, X_prev of the same points / orbitals
            tma_load_2d(sbuf + q * QS, &maps.m[q], x, tm * GT_T, &full[s]);
        }
      }
    }
  } else {
    if constexpr (Cfg::PW == 4) asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    warp -= Cfg::PW;
    const int gq = lane >> 2, t4 = lane & 3;
    constexpr int FM = Cfg::FM, FN = Cfg::FN, WM = Cfg::WM, WN = Cfg::WN;
    const int wm = warp / WN, wn = warp % WN;
    double acc[FM][FN][2];
#pragma unroll
    for (int a = 0; a < FM; ++a)
#pragma unroll
      for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    // fragment row / column f of this warp: WM f + wm / WN f + wn (interleaved)
    auto load_frag = [&](const double* base, int qa, int qb2, double sc, int frag, int p) {
      const int off = swz(8 * frag + gq, p, GT_T);
      double2 v = *reinterpret_cast<const double2*>(base + qa * QS + off);
      if (qb2 >= 0) {
        const double2 z = *reinterpret_cast<const double2*>(base + qb2 * QS + off);
        v.x += sc * z.x;
        v.y += sc * z.y;
      }
      return v;
    };
    if (!diag) {
      // one-source operands (Sigma, off-diagonal symmetric tiles) get a loop with
      // no predicated combine in their fragment loads (as the diagonal tiles)
      // BB: lane pair (2 l, 2 l + 1) of consumer warp w owns orbital 16 w + l and
      // one 8-point half of its 16 points per stage (4 chunks of 16 bytes; a
      // quarter-warp's 4 rows x 2 halves hit 8 distinct chunks under the swizzle)
      const int bi = BB ? 16 * warp + (lane >> 1) : 0, bh = lane & 1;
      const int gi = tm * GT_T + bi;  // the orbital (bi: its row in the tile)
      double bms = 0.0, bmsp = 0.0, r0 = 0.0, r1 = 0.0, r2 = 0.0, r3 = 0.0;
      if constexpr (BB) {
        bms = (bbt && gi < bb.N) ? -bb.sig[gi] : 0.0;
        bmsp = (bbt && bb.sigp && gi < bb.N) ? -bb.sigp[gi] : 0.0;
      }
      const bool bhist = BB && bb.hist != 0, bzpi = BB && bb.sigp != nullptr;
      auto stages = [&](auto two, auto dobb) {
        constexpr bool TWO = decltype(two)::value;
        constexpr bool DOBB = decltype(dobb)::value;  // this tile carries the sums (compile-time loop variant)
        for (int st = 0; st < nstage; ++st) {
          const int s = st % nst;
          mbar_wait(&full[s], (uint32_t)(st / nst) & 1u);
          const double* sbuf = stage0 + (size_t)s * sdoubles;
          if constexpr (DOBB) {
            // the stage's elementwise work in this warp's own instruction stream,
            // before its fragments are loaded (their registers are free): 64 DFMAs
            // against the stage's 128 DMMAs per warp. (As the job of separate warps
            // the same DFMAs starved behind the consumers' DMMAs on the FP64 pipe and
            // held the ring: 2.66 ms instead of the plain Gram's 1.92 at C3.)
            const double* hA = sbuf + bi * BOX;                       // HW rows (area 0)
            const double* wA = sbuf + (size_t)qb * QS + bi * BOX;     // W rows
            const double* pA = sbuf + (size_t)nsrc * QS + bi * BOX;   // W_prev
            const double* xA = pA + QS;                               // HW_prev or Z_prev
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              const int off = ((4 * bh + cc) ^ (bi & 7)) << 1;
              const double2 h = *reinterpret_cast<const double2*>(hA + off);
              const double2 w = *reinterpret_cast<const double2*>(wA + off);
              const double z0 = fma(bms, w.x, h.x), z1 = fma(bms, w.y, h.y);
              r0 += z0 * z0;
              r0 += z1 * z1;
              if (bhist) {
                const double2 wq = *reinterpret_cast<const double2*>(pA + off);
                const double2 xq = *reinterpret_cast<const double2*>(xA + off);
                const double q0 = bzpi ? fma(bmsp, wq.x, xq.x) : xq.x;
                const double q1 = bzpi ? fma(bmsp, wq.y, xq.y) : xq.y;
                const double s0 = w.x - wq.x, y0 = z0 - q0;
                const double s1 = w.y - wq.y, y1 = z1 - q1;
                r1 += s0 * s0;
                r1 += s1 * s1;
                r2 += s0 * y0;
                r2 += s1 * y1;
                r3 += y0 * y0;
                r3 += y1 * y1;
              }
            }
          }
#pragma unroll
          for (int kg = 0; kg < 2; ++kg) {
            const int p = 8 * kg + 2 * t4;
            double2 a[FM], b[FN];
#pragma unroll
            for (int f = 0; f < FM; ++f) a[f] = load_frag(sbuf, 0, TWO ? qa_b : -1, sa, WM * f + wm, p);
#pragma unroll
            for (int f = 0; f < FN; ++f) b[f] = load_frag(sbuf, qb, TWO ? qb_b : -1, sb, WN * f + wn, p);
            if (kg == 1) {
              __syncwarp();
              if (lane == 0) mbar_arrive(&empty[s]);  // all fragments of the stage are in registers
            }
#pragma unroll
            for (int fm = 0; fm < FM; ++fm)
#pragma unroll
              for (int fn = 0; fn < FN; ++fn) {
                dmma_8x8x4(acc[fm][fn], a[fm].x, b[fn].x);
                dmma_8x8x4(acc[fm][fn], a[fm].y, b[fn].y);
              }
          }
        }
      };
      if (BB && bbt)
        stages(std::false_type{}, std::integral_constant<bool, BB>{});
      else if (qa_b >= 0 || qb_b >= 0)
        stages(std::true_type{}, std::false_type{});
      else
        stages(std::false_type{}, std::false_type{});
      if constexpr (BB) {  // the two halves of an orbital's points meet; one partial per split
        r0 += __shfl_xor_sync(0xffffffffu, r0, 1);
        r1 += __shfl_xor_sync(0xffffffffu, r1, 1);
        r2 += __shfl_xor_sync(0xffffffffu, r2, 1);
        r3 += __shfl_xor_sync(0xffffffffu, r3, 1);
        if (bbt && bh == 0 && gi < bb.N) {
          const int64_t nb = gridDim.y;
          bb.part[((int64_t)0 * bb.N + gi) * nb + blockIdx.y] = r0;
          if (bhist) {
            bb.part[((int64_t)1 * bb.N + gi) * nb + blockIdx.y] = r1;
            bb.part[((int64_t)2 * bb.N + gi) * nb + blockIdx.y] = r2;
            bb.part[((int64_t)3 * bb.N + gi) * nb + blockIdx.y] = r3;
          }
        }
      }
    } else if constexpr (BB) {
      return;  // (never: a BB launch has no symmetric tiles)
    } else if constexpr (GT_T == 128) {
      // Diagonal tile of a symmetric Gram, T = 128 (16 fragment rows): warps 0-3
      // take the first 16-point half of every stage, warps 4-7 the second; warp a
      // of either half owns the circulant super-block slots described at
      // sym_diag_stages. The two halves' partial blocks meet in the epilogue.
      const int hf = warp >> 2, a = warp & 3;
      double acc0[5][2][2][2], acc1[4][2][2][2];
#pragma unroll
      for (int k = 0; k < 5; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc0[k][e >> 1][e & 1][0] = acc0[k][e >> 1][e & 1][1] = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc1[k][e >> 1][e & 1][0] = acc1[k][e >> 1][e & 1][1] = 0.0;
      const int q0 = hf * nload, qb2 = qa_b >= 0 ? hf * nload + qa_b : -1;
      // one-source (G_HH, G2) and two-source (a trial's G0) loops are separate
      // instantiations: the one-source loop carries no combine
      const DensArgs da{rho, bvec, occ, kbeg, ngl, warp};
      if (qb2 >= 0)
        sym_diag_stages<true, false>(acc0, acc1, a, stage0, sdoubles, nstage, nst, full, empty, q0, qb2,
                                     sa, t4, gq, lane, da);
      else if (dens)
        sym_diag_stages<false, true>(acc0, acc1, a, stage0, sdoubles, nstage, nst, full, empty, q0, qb2,
                                     sa, t4, gq, lane, da);
      else
        sym_diag_stages<false, false>(acc0, acc1, a, stage0, sdoubles, nstage, nst, full, empty, q0, qb2,
                                      sa, t4, gq, lane, da);
      constexpr int SP = GT_T + 8;
      double* S = stage0;
      asm volatile("bar.sync 1, %0;\n" ::"n"(Cfg::NW * 32) : "memory");  // ring fully consumed
      // pass 0: half 0 stores its blocks; pass 1: half 1 adds (same block set).
      // Slots whose column wrapped below their row land transposed; the lower
      // block of a diagonal super-block is dropped.
      auto put = [&](int pass, int R, int C, int ea, int eb, const double (&v)[2]) {
        if (R == C && ea > eb) return;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int r = 16 * R + 8 * ea + gq, c = 16 * C + 8 * eb + 2 * t4 + j;
          const int idx = R <= C ? r * SP + c : c * SP + r;
          if (pass == 0)
            S[idx] = v[j];
          else
            S[idx] += v[j];
        }
      };
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        if (hf == pass) {
#pragma unroll
          for (int k = 0; k < 5; ++k)
#pragma unroll
            for (int e = 0; e < 4; ++e) put(pass, a, a + k, e >> 1, e & 1, acc0[k][e >> 1][e & 1]);
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int e = 0; e < 4; ++e)
              put(pass, a + 4, (a + 4 + k) & 7, e >> 1, e & 1, acc1[k][e >> 1][e & 1]);
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(Cfg::NW * 32) : "memory");
      }
      double* outd = ws + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (GT_T * GT_T);
      const int ct = threadIdx.x - Cfg::PW * 32;
      for (int e = ct; e < GT_T * GT_T / 2; e += Cfg::NW * 32) {
        const int r = (2 * e) / GT_T, c = (2 * e) % GT_T;
        *reinterpret_cast<double2*>(outd + r * GT_T + c) =
            make_double2(S[r * SP + c], S[r * SP + c + 1]);
      }
      return;
    } else {
      // Diagonal tile of a symmetric Gram with no wasted DMMA and one code path
      // for all warps. Each stage holds two 16-point halves. With R = T / 8
      // fragment rows, warp w owns rows r = w + 8 m (m < R / 8) and the R
      // circulant offsets k: slot (m, k) accumulates block (r, c = (r + k) mod R).
      // Every unordered pair {x, y} of fragments appears in exactly two slots,
      // (x, y - x) and (y, x - y) (mod R): offsets 1 .. R/2 - 1 take the first
      // half, R/2 + 1 .. R - 1 the second, offset R/2 the first half on rows
      // < R/2 (its partner slot has row >= R/2); offset 0 (the diagonal
      // blocks) takes both. So each slot's half is fixed per (m, k) — the same
      // for every warp — and the two contributions of a pair meet in the
      // epilogue (shared memory, transposed where r > c).
      constexpr int R = GT_T / 8, RW = R / 8;
      const int wq = warp;  // 0..7
      double gacc[RW][R][2];
#pragma unroll
      for (int m = 0; m < RW; ++m)
#pragma unroll
        for (int k = 0; k < R; ++k) gacc[m][k][0] = gacc[m][k][1] = 0.0;
      const int h1 = nload;  // first area of the second half
      for (int st = 0; st < nstage; ++st) {
        const int s = st % nst;
        mbar_wait(&full[s], (uint32_t)(st / nst) & 1u);
        const double* sbuf = stage0 + (size_t)s * sdoubles;
#pragma unroll
        for (int kg = 0; kg < 2; ++kg) {
          const int p = 8 * kg + 2 * t4;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int q0 = h * h1, qb2 = qa_b >= 0 ? h * h1 + qa_b : -1;
            const double* base = sbuf;
            double2 ar[RW];
#pragma unroll
            for (int m = 0; m < RW; ++m) ar[m] = load_frag(base, q0, qb2, sa, wq + 8 * m, p);
#pragma unroll
            for (int m = 0; m < RW; ++m)
#pragma unroll
              for (int k = 0; k < R; ++k) {
                // half of slot (m, k); -1: offset R/2 with a runtime row test (RW == 1)
                constexpr int dummy = 0;
                (void)dummy;
                const int hs = k == 0 ? 2 : (k < R / 2 ? 0 : (k > R / 2 ? 1 : (RW == 2 ? m : -1)));
                if (hs == 2 || hs == h) {
                  const double2 bc = load_frag(base, q0, qb2, sa, (wq + 8 * m + k) % R, p);
                  dmma_8x8x4(gacc[m][k], ar[m].x, bc.x);
                  dmma_8x8x4(gacc[m][k], ar[m].y, bc.y);
                } else if (hs == -1 && h == 0) {
                  // offset R/2 with one row per warp: rows < R/2 use the first
                  // half, the others the second (operands selected, no predicate)
                  const bool first = wq < R / 2;
                  const int qs = first ? 0 : h1, qsb = qa_b >= 0 ? qs + qa_b : -1;
                  const double2 ra = load_frag(base, qs, qsb, sa, wq, p);
                  const double2 bc = load_frag(base, qs, qsb, sa, (wq + R / 2) % R, p);
                  dmma_8x8x4(gacc[m][k], ra.x, bc.x);
                  dmma_8x8x4(gacc[m][k], ra.y, bc.y);
                }
              }
            asm volatile("" ::: "memory");
          }
          if (kg == 1) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
          }
        }
      }
      constexpr int SP = GT_T + 8;
      double* S = stage0;
      asm volatile("bar.sync 1, %0;\n" ::"n"(Cfg::NW * 32) : "memory");  // ring fully consumed
      // pass 0: first-half and diagonal slots store; pass 1: second-half slots add
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
        for (int m = 0; m < RW; ++m)
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const int r = wq + 8 * m, c = (r + k) % R;
            const int hs = k == 0 ? 0 : (k < R / 2 ? 0 : (k > R / 2 ? 1 : (r < R / 2 ? 0 : 1)));
            if (hs != pass) continue;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int idx = r <= c ? (8 * r + gq) * SP + 8 * c + 2 * t4 + j
                                     : (8 * c + 2 * t4 + j) * SP + 8 * r + gq;
              if (pass == 0)
                S[idx] = gacc[m][k][j];
              else
                S[idx] += gacc[m][k][j];
            }
          }
        asm volatile("bar.sync 1, %0;\n" ::"n"(Cfg::NW * 32) : "memory");
      }
      double* outd = ws + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (GT_T * GT_T);
      const int ct = threadIdx.x - Cfg::PW * 32;
      for (int e = ct; e < GT_T * GT_T / 2; e += Cfg::NW * 32) {
        const int r = (2 * e) / GT_T, c = (2 * e) % GT_T;
        *reinterpret_cast<double2*>(outd + r * GT_T + c) =
            make_double2(S[r * SP + c], S[r * SP + c + 1]);
      }
      return;
    }
    double* out = ws + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (GT_T * GT_T);
#pragma unroll
    for (int fm = 0; fm < FM; ++fm)
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) {
        const int r = 8 * (WM * fm + wm) + gq, c = 8 * (WN * fn + wn) + 2 * t4;
        // (lower blocks of a diagonal tile hold the transposed second half: never read)
        *reinterpret_cast<double2*>(out + r * GT_T + c) = make_double2(acc[fm][fn][0], acc[fm][fn][1]);
      }
  }
}

// G(i, j) = w sum_k ws[k](tile of (i, j)); 8 split groups per element summed
// in a fixed order (deterministic), 32 consecutive elements per block
__global__ void __launch_bounds__(256) gram_big_reduce_kernel(int GT_T, int N, int mt, int sym,
                                                              int ntiles, int nsplit, double w,
                                                              const double* __restrict__ ws,
                                                              double* __restrict__ G,
                                                              const double* __restrict__ guard) {
  PO_PDL_ENTRY();
  if (guard && *guard == 0.0) return;
  __shared__ double part[8][33];
  const int64_t e = (int64_t)blockIdx.x * 32 + threadIdx.x;
  double s = 0.0;
  int64_t off = 0;
  if (e < (int64_t)N * N) {
    int i = (int)(e / N), j = (int)(e % N);
    if (sym && j < i) {
      const int t = i;
      i = j;
      j = t;
    }
    const int tm = i / GT_T, tn = j / GT_T;
    int tile;
    if (!sym) {
      tile = tm * mt + tn;
    } else {
      tile = 0;
      for (int r = 0; r < tm; ++r) tile += mt - r;
      tile += tn - tm;
    }
    off = (int64_t)tile * GT_T * GT_T + (i - tm * GT_T) * GT_T + (j - tn * GT_T);
    const int64_t stride = (int64_t)ntiles * GT_T * GT_T;
    for (int k = threadIdx.y; k < nsplit; k += 8) s += ws[k * stride + off];
  }
  part[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && e < (int64_t)N * N) {
    double t = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) t += part[g][threadIdx.x];
    G[e] = w * t;
  }
}

struct BigPlan {
  int mt, ntiles, nsplit;
  int64_t kchunk;
};

// splits so that tiles x splits fills whole waves of one CTA per SM
// Tile side. Measured at N = 128 (C3, 128^3): 128-wide tiles win for every
// Gram once diagonal tiles stopped issuing wasted DMMAs (symmetric 1.45 ms vs
// 1.74 ms with 64-wide tiles; before, 64 won at 2.04 vs 2.26 ms); with two
// streamed sources the 64-tile CTAs are bound by the 2D-TMA row rate.
int big_tile(int N, int sym, bool two_src) {
  static int forced = -1;
  if (forced < 0) {
    const char* e = getenv("PO_GRAM_TILE");  // measurement override: 64 or 128
    forced = e ? atoi(e) : 0;
  }
  if (forced == 64 || forced == 128) return forced;
  (void)sym;
  (void)two_src;
  return N <= 64 ? 64 : 128;
}

BigPlan big_plan(int64_t ld, int N, int sym, int sms, int GT_T) {
  BigPlan p;
  p.mt = (N + GT_T - 1) / GT_T;
  p.ntiles = sym ? p.mt * (p.mt + 1) / 2 : p.mt * p.mt;
  const int64_t kb = (ld + BOX - 1) / BOX;
  int cap = 4096 / p.ntiles;
  if (cap < 1) cap = 1;
  if (cap > kb) cap = (int)kb;
  // the fewest splits that fill whole waves (a 0.97-full wave left 4 of 148 SMs
  // idle for the whole of the C3 Grams), else the best fill
  int best = 1;
  double beste = 0.0;
  for (int ns = 1; ns <= cap; ++ns) {
    const int64_t units = (int64_t)p.ntiles * ns;
    const int64_t waves = (units + sms - 1) / sms;
    const double eff = (double)units / (double)(waves * sms);
    if (eff > beste + 1e-3) {
      beste = eff;
      best = ns;
    }
    if (eff >= 0.999) break;
  }
  // chunks of a multiple of 32 points: diagonal tiles consume 32-point stages
  p.kchunk = (((kb + best - 1) / best + 1) / 2) * 2 * BOX;
  p.nsplit = (int)((ld + p.kchunk - 1) / p.kchunk);
  return p;
}

// ------------------------------------------------------------------ large-N mix
// out_i = alpha sum_k (A + sa Ab)_k M(k, i) + beta C_i for N > 64
// (manifold.cpp:67-85; the orthonormalisation rotation W L^{-T} with M upper
// triangular, manifold.cpp:97-114, and the gradient D = HW - W Sigma,
// manifold.cpp:181-202). Persistent CTAs walk 128-point x 128-orbital output
// tiles; each stage brings 16 input orbitals of the tile's 128 points
// (8 boxes {16 points x 16 rows}, 128-B swizzle) per source plus the matching
// 16 columns of M^T (one box {16 k x 128 i}) — M is transposed into a padded
// scratch by the launcher so that one 16-byte shared load gives a lane the B
// fragments of two k-steps. The A side pairs points instead: a lane's 16-byte
// load holds points 2q, 2q+1, i.e. the same (row, k) element of two DMMA row
// fragments.
// Consumer warp w owns the output fragments F = w and F = 15 - w (8 orbitals
// each) over all 128 points of the tile. With an upper-triangular M the
// 8-input block kb of the tile's diagonal block only meets fragments F >= kb,
// so the pair does kb-blocks 0..w and 0..15-w: 17 per warp, balanced, and
// every skipped block is a warp-uniform branch around whole DMMA groups (a
// predicated-off DMMA still occupies the tensor pipe; per-stage code variants
// thrashed the instruction cache: ncu "no instruction" stalls).
constexpr int XP = 128;  // points per tile
constexpr int XI = 128;  // orbitals per tile
constexpr int XK = 16;   // input orbitals per stage
constexpr int XTH = 384;

// one 8-input block (k8 .. k8 + 7 = stage rows 8h ..) for the warp's active fragments
template <bool A0, bool A1>
__device__ __forceinline__ void mix_big_slice(double (&acc)[2][16][2], const double* sb,
                                              const double* sbb, double sa, double2 b0, double2 b1,
                                              int h, int gq, int t4) {
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    double2 a[2];
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const int off = swz(8 * h + 2 * t4 + s2, 16 * g + 2 * gq, XK);
      a[s2] = *reinterpret_cast<const double2*>(sb + off);
      if (sbb) {
        const double2 z = *reinterpret_cast<const double2*>(sbb + off);
        a[s2].x += sa * z.x;
        a[s2].y += sa * z.y;
      }
    }
    if (A0) {
      dmma_8x8x4(acc[0][2 * g], a[0].x, b0.x);
      dmma_8x8x4(acc[0][2 * g + 1], a[0].y, b0.x);
      dmma_8x8x4(acc[0][2 * g], a[1].x, b0.y);
      dmma_8x8x4(acc[0][2 * g + 1], a[1].y, b0.y);
    }
    if (A1) {
      dmma_8x8x4(acc[1][2 * g], a[0].x, b1.x);
      dmma_8x8x4(acc[1][2 * g + 1], a[0].y, b1.x);
      dmma_8x8x4(acc[1][2 * g], a[1].x, b1.y);
      dmma_8x8x4(acc[1][2 * g + 1], a[1].y, b1.y);
    }
  }
}

__global__ void __launch_bounds__(XTH, 1) mix_big_kernel(
    const __grid_constant__ Maps maps, int has_ab, int N, int64_t ld, int64_t ngl, int n_pt,
    int n_it, int upper, int nst, double sa, double alpha, const double* __restrict__ C,
    double beta, double* __restrict__ out, double* __restrict__ norms,
    const double* __restrict__ guard, const double* __restrict__ zsig) {
  PO_PDL_ENTRY();
  if (guard && *guard == 0.0) return;
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* empty = full + 8;
  uint64_t* ready = full + 16;  // two-source stages: A + sa Ab formed in place
  double* mst = reinterpret_cast<double*>(tsm + 512);  // -sigma of a stage (implicit z)
  double* stage0 = reinterpret_cast<double*>(tsm + 1024);
  constexpr size_t QA = (size_t)XP * XK;  // doubles per source per stage
  const int nsrc = has_ab ? 2 : 1;
  const size_t sdoubles = (size_t)(nsrc + 1) * QA;  // + the M^T box
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
      mbar_init(&ready[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int ntiles = n_pt * n_it;
  // heavy (last) orbital tiles first: with the triangular skip their k range is longest
  auto tile_of = [&](int t, int& pt, int& it) {
    it = n_it - 1 - t / n_pt;
    pt = t % n_pt;
  };
  auto kend_of = [&](int it) { return upper ? min(N, (it + 1) * XI) : N; };
  const int lane = threadIdx.x & 31;
  int warp = threadIdx.x >> 5;
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      for (int q = 0; q <= nsrc; ++q)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[q])));
      const uint32_t bytes = (uint32_t)((nsrc + 1) * QA * 8);
      int g = 0;  // global stage counter (ring position)
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int pt, it;
        tile_of(t, pt, it);
        const int nk = (kend_of(it) + XK - 1) / XK;
        for (int c = 0; c < nk; ++c, ++g) {
          const int s = g % nst;
          if (g >= nst) mbar_wait(&empty[s], ((uint32_t)(g / nst) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], bytes);
          double* sb = stage0 + (size_t)s * sdoubles;
          for (int q = 0; q < nsrc; ++q)
            for (int b = 0; b < XP / BOX; ++b)
              tma_load_2d(sb + q * QA + b * BOX * XK, &maps.m[q], pt * XP + b * BOX, c * XK, &full[s]);
          tma_load_2d(sb + nsrc * QA, &maps.m[nsrc], c * XK, it * XI, &full[s]);
        }
      }
    } else if (warp > 0 && has_ab) {
      // the other three producer warps form A + sa Ab in place for every stage
      // (the trial rotation's W - tau Z), so the consumers read one source
      const int ct = threadIdx.x - 32;  // 0..95
      int g = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int pt, it;
        tile_of(t, pt, it);
        const int nk = (kend_of(it) + XK - 1) / XK;
        for (int c = 0; c < nk; ++c, ++g) {
          const int s = g % nst;
          mbar_wait(&full[s], (uint32_t)(g / nst) & 1u);
          double2* a2 = reinterpret_cast<double2*>(stage0 + (size_t)s * sdoubles);
          const double2* b2 = reinterpret_cast<const double2*>(stage0 + (size_t)s * sdoubles + QA);
          if (zsig) {  // -sigma of the stage's 16 orbitals, once per stage
            if (ct < XK) {
              const int k = c * XK + ct;
              mst[ct] = k < N ? -zsig[k] : 0.0;
            }
            asm volatile("bar.sync 2, 96;\n" ::: "memory");
          }
          for (int e = ct; e < (int)(QA / 2); e += 96) {
            double2 v = a2[e];
            double2 z = b2[e];
            if (zsig) {  // Ab is HW: z = HW - sigma_k W rebuilt with the directions pass's FMA
              const double ms = mst[(e & 127) >> 3];  // the swizzle permutes within a 16-point row
              z.x = fma(ms, v.x, z.x);
              z.y = fma(ms, v.y, z.y);
            }
            v.x += sa * z.x;
            v.y += sa * z.y;
            a2[e] = v;
          }
          // generic writes into a TMA-filled slot: ordered before the slot's refill
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          asm volatile("bar.sync 2, 96;\n" ::: "memory");
          if (ct == 0) mbar_arrive(&ready[s]);
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    warp -= 4;
    const int gq = lane >> 2, t4 = lane & 3;
    const int F0 = warp, F1 = 15 - warp;  // this warp's output fragments
    int g = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int pt, it;
      tile_of(t, pt, it);
      const int i0 = it * XI;
      const int kend = kend_of(it);
      const int nk = (kend + XK - 1) / XK;
      const bool real0 = i0 + 8 * F0 < N, real1 = i0 + 8 * F1 < N;  // padding fragments
      double acc[2][16][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 16; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
      for (int c = 0; c < nk; ++c, ++g) {
        const int s = g % nst;
        mbar_wait(has_ab ? &ready[s] : &full[s], (uint32_t)(g / nst) & 1u);
        const double* sb = stage0 + (size_t)s * sdoubles;
        const double* sbb = nullptr;
        const double* mt = sb + nsrc * QA;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k8 = c * XK + 8 * h;
          if (k8 >= kend) break;
          const int kb = (k8 - i0) >> 3;  // 8-block index relative to the tile's orbitals
          const bool a0 = real0 && (!upper || kb <= F0);
          const bool a1 = real1 && (!upper || kb <= F1);
          const double2 b0 = *reinterpret_cast<const double2*>(mt + swz(8 * F0 + gq, 8 * h + 2 * t4, XI));
          const double2 b1 = *reinterpret_cast<const double2*>(mt + swz(8 * F1 + gq, 8 * h + 2 * t4, XI));
          if (a0 && a1)
            mix_big_slice<true, true>(acc, sb, sbb, sa, b0, b1, h, gq, t4);
          else if (a1)
            mix_big_slice<false, true>(acc, sb, sbb, sa, b0, b1, h, gq, t4);
          else if (a0)
            mix_big_slice<true, false>(acc, sb, sbb, sa, b0, b1, h, gq, t4);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // the stage's fragments were consumed
      }
      // epilogue: acc[q][2 g + e][j] = out(point 16 g + 2 gq + e, orbital i0 + 8 F_q + 2 t4 + j)
      const int64_t pb = (int64_t)pt * XP + 2 * gq;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (!(q ? real1 : real0)) continue;
        const int F = q ? F1 : F0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = i0 + 8 * F + 2 * t4 + j;
          double nrm = 0.0;
          if (i < N) {
#pragma unroll
            for (int gg = 0; gg < 8; ++gg) {
              const int64_t p = pb + 16 * gg;
              if (p >= ngl) continue;
              double v0 = alpha * acc[q][2 * gg][j], v1 = alpha * acc[q][2 * gg + 1][j];
              const bool two = p + 1 < ngl;
              if (C) {
                if (two) {
                  const double2 cv = *reinterpret_cast<const double2*>(C + (int64_t)i * ld + p);
                  v0 += beta * cv.x;
                  v1 += beta * cv.y;
                } else {
                  v0 += beta * C[(int64_t)i * ld + p];
                }
              }
              if (!two) v1 = 0.0;
              if (out) {
                if (two)
                  *reinterpret_cast<double2*>(out + (int64_t)i * ld + p) = make_double2(v0, v1);
                else
                  out[(int64_t)i * ld + p] = v0;
              }
              nrm += v0 * v0 + v1 * v1;
            }
          }
          if (norms) {
            nrm += __shfl_xor_sync(0xffffffffu, nrm, 4);
            nrm += __shfl_xor_sync(0xffffffffu, nrm, 8);
            nrm += __shfl_xor_sync(0xffffffffu, nrm, 16);
            if (gq == 0 && i < N) norms[(int64_t)i * n_pt + pt] = nrm;
          }
        }
      }
    }
  }
}


// ------------------------------------------------------- large-N directions pass
// compute_directions for N > 64 (manifold.cpp:181-216, optimizer.cpp:265-320,
// 386-397) with every operand streamed by TMA and no epilogue loads.
// Tiles of 128 points x 128 orbitals as in mix_big_kernel; ring A carries, per
// stage, 16 input orbitals of W (the DMMA A operand) and 16 columns of Sigma^T.
// The stages whose 16 orbitals are the tile's own (the "diagonal" stages, all
// of them for N <= 128) additionally get ring E: HW, W_prev and HW_prev (or a
// stored Z_prev) of the same 16 orbitals x 128 points. The consumer warp that
// owns an orbital fragment, at the diagonal stage holding it,
//   * forms z = HW - sigma_ii W with the same FMA the stored-z passes use
//     (fma(-sigma_i, W, HW)) and, only if a caller needs it stored, writes it;
//   * reduces ||z||^2 and the BB products ss, sy, yy against
//     (W_prev, z_prev = HW_prev - sigma_prev W_prev) — the previous iteration's
//     direction rebuilt, never stored (or read from Z_prev);
//   * subtracts HW from its DMMA accumulators, so the tile's accumulators end
//     as W Sigma - HW = -D and ||D_i||^2 needs no memory at all.
// Every block is read once through TMA (W, HW, W_prev, HW_prev: 4 blocks) and
// nothing is written on the implicit path; the old form (mix_big_kernel<DIR>)
// wrote z and re-read HW / W / W_prev / Z_prev with plain loads after the DMMA
// loop while the tensor pipe idled (5.2 ms at C3).
struct Maps5 {
  CUtensorMap m[5];
};
constexpr int DNA = 4;  // ring A stages (16 input orbitals of W: 16 KB each)
constexpr int DNE = 3;  // ring E stages (HW, W_prev, HW_prev: 3 x 16.25 KB each)
// Sigma^T is not staged: its B fragments come from the padded transpose in
// global memory (128 KB at N = 128, L2-resident), one stage ahead in
// registers, so the shared memory goes to ring depth (ncu: the consumers'
// dominant stall was the wait for ring E with 3 A + 2 E stages of 32 / 48 KB)
// Ring E boxes are unswizzled rows of EW = 130 points (one box per block per
// stage): 1-KB+ TMA rows stream at full rate where the 128-B rows of the
// swizzled DMMA boxes cap near 4.2 TB/s (profiles/r1_tma2d_probe.txt), and the
// 1040-B row pitch puts the rows 2 t4 + j a lane quarter reads at 16-B chunks
// 2 t4 (mod 8) apart: the elementwise reads are bank-conflict free. The 2
// extra points per row are the next tile's first two (L2 hits).
constexpr int EW = 130;
constexpr size_t QE = (size_t)XK * EW;  // doubles per block per E stage (a multiple of 128 B)

template <int Q>
__device__ __forceinline__ void dir_big_elementwise(
    double (&acc)[2][16][2], const double* sa_, const double* se, int hist, int hh, int gq, int t4,
    int i0, int F, int N, int64_t ld, int64_t ngl, int64_t p0, const double* __restrict__ sig,
    const double* __restrict__ sigp, double* __restrict__ zout, double* __restrict__ dpart, int n_pt,
    int pt) {
  const double* sh = se;               // HW
  const double* swp = se + QE;         // W_prev
  const double* sx = se + 2 * QE;      // HW_prev (implicit z_prev) or Z_prev
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int i = i0 + 8 * F + 2 * t4 + j;
    const bool live = i < N;
    const double ms = live ? -sig[i] : 0.0;
    const double msp = (live && sigp) ? -sigp[i] : 0.0;
    const int row = 8 * hh + 2 * t4 + j;
    double r4[4] = {0.0, 0.0, 0.0, 0.0};  // zz, ss, sy, yy
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const int off = swz(row, 16 * g + 2 * gq, XK);  // the swizzled A (W) stage
      const int oe = row * EW + 16 * g + 2 * gq;       // the ring E rows
      const double2 wv = *reinterpret_cast<const double2*>(sa_ + off);
      const double2 hv = *reinterpret_cast<const double2*>(sh + oe);
      // accumulators: W Sigma - HW (points past ngl hold zeros on both sides)
      acc[Q][2 * g][j] -= hv.x;
      acc[Q][2 * g + 1][j] -= hv.y;
      // z = HW - sigma_ii W (residual_bb_kernel / launch_z_from_hw: the same FMA)
      const double v0 = fma(ms, wv.x, hv.x), v1 = fma(ms, wv.y, hv.y);
      r4[0] += v0 * v0 + v1 * v1;
      const int64_t p = p0 + 16 * g + 2 * gq;
      if (zout && live && p < ngl) {
        if (p + 1 < ngl)
          *reinterpret_cast<double2*>(zout + (int64_t)i * ld + p) = make_double2(v0, v1);
        else
          zout[(int64_t)i * ld + p] = v0;
      }
      if (hist) {
        const double2 wq = *reinterpret_cast<const double2*>(swp + oe);
        const double2 xq = *reinterpret_cast<const double2*>(sx + oe);
        const double zq0 = sigp ? fma(msp, wq.x, xq.x) : xq.x;
        const double zq1 = sigp ? fma(msp, wq.y, xq.y) : xq.y;
        const double s0 = wv.x - wq.x, y0 = v0 - zq0;
        const double s1 = wv.y - wq.y, y1 = v1 - zq1;
        r4[1] += s0 * s0 + s1 * s1;
        r4[2] += s0 * y0 + s1 * y1;
        r4[3] += y0 * y0 + y1 * y1;
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double v = r4[r];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      const int row_out = r == 0 ? 0 : r + 1;  // [zz | dd | ss | sy | yy]
      if (gq == 0 && live && (hist || r == 0)) dpart[((int64_t)row_out * N + i) * n_pt + pt] = v;
    }
  }
}

__global__ void __launch_bounds__(XTH, 1) dir_big_kernel(
    const __grid_constant__ Maps5 maps, int N, int64_t ld, int64_t ngl, int n_pt, int n_it, int hist,
    const double* __restrict__ sig, const double* __restrict__ sigp, double* __restrict__ zout,
    double* __restrict__ sig_save, double* __restrict__ dpart, const double* __restrict__ mtg, int np) {
  PO_PDL_ENTRY();
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
  uint64_t* fullA = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* emptyA = fullA + 8;
  uint64_t* fullE = fullA + 16;
  uint64_t* emptyE = fullA + 24;
  constexpr size_t QA = (size_t)XP * XK;  // doubles per block per stage
  constexpr size_t SA = QA;               // ring A stage: W
  constexpr size_t SE = 3 * QE;           // ring E stage: HW, W_prev, HW_prev / Z_prev
  double* ringA = reinterpret_cast<double*>(tsm + 1024);
  double* ringE = ringA + DNA * SA;
  if (threadIdx.x == 0) {
    for (int s = 0; s < DNA; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 8);
    }
    for (int s = 0; s < DNE; ++s) {
      mbar_init(&fullE[s], 1);
      // every consumer warp waits on and releases every E stage (only the two
      // owning the stage's fragments read it): with parity waits a warp must
      // never skip a phase of a slot, or a stale phase could satisfy its wait
      mbar_init(&emptyE[s], 8);
    }
    fence_mbar_init();
  }
  if (sig_save && blockIdx.x == 0)
    for (int i = threadIdx.x; i < N; i += blockDim.x) sig_save[i] = sig[i];
  __syncthreads();
  const int ntiles = n_pt * n_it;
  const int nk = (N + XK - 1) / XK;
  auto tile_of = [&](int t, int& pt, int& it) {
    it = n_it - 1 - t / n_pt;
    pt = t % n_pt;
  };
  const int lane = threadIdx.x & 31;
  int warp = threadIdx.x >> 5;
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 0 && lane == 0) {  // ring A: W for every stage
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[0])));
      int g = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int pt, it;
        tile_of(t, pt, it);
        for (int c = 0; c < nk; ++c, ++g) {
          const int s = g % DNA;
          if (g >= DNA) mbar_wait(&emptyA[s], ((uint32_t)(g / DNA) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&fullA[s], (uint32_t)(SA * 8));
          double* sb = ringA + (size_t)s * SA;
          for (int b = 0; b < XP / BOX; ++b)
            tma_load_2d(sb + b * BOX * XK, &maps.m[0], pt * XP + b * BOX, c * XK, &fullA[s]);
        }
      }
    } else if (warp == 1 && lane == 0) {  // ring E: the tile's own orbitals only
      const int ne = hist ? 3 : 1;
      for (int q = 0; q < ne; ++q)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[2 + q])));
      int ge = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int pt, it;
        tile_of(t, pt, it);
        const int c1 = min(nk, (it + 1) * (XI / XK));
        for (int c = it * (XI / XK); c < c1; ++c, ++ge) {
          const int s = ge % DNE;
          if (ge >= DNE) mbar_wait(&emptyE[s], ((uint32_t)(ge / DNE) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&fullE[s], (uint32_t)(ne * QE * 8));
          double* sb = ringE + (size_t)s * SE;
          for (int q = 0; q < ne; ++q)
            tma_load_2d(sb + q * QE, &maps.m[2 + q], pt * XP, c * XK, &fullE[s]);
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
    warp -= 4;
    const int gq = lane >> 2, t4 = lane & 3;
    const int F0 = warp, F1 = 15 - warp;  // this warp's output fragments
    // B fragments (Sigma^T rows i, the stage's k pairs) of stage (c, it), from global
    auto load_b = [&](int c, int it, double2 (&b)[2][2]) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int i = it * XI + 8 * (q ? F1 : F0) + gq;
          const int k = c * XK + 8 * h + 2 * t4;
          b[h][q] = i < np ? __ldg(reinterpret_cast<const double2*>(mtg + (int64_t)i * np + k))
                           : make_double2(0.0, 0.0);
        }
    };
    double2 bnext[2][2];
    if (blockIdx.x < ntiles) {
      int pt, it;
      tile_of(blockIdx.x, pt, it);
      load_b(0, it, bnext);
    }
    int g = 0, ge = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int pt, it;
      tile_of(t, pt, it);
      const int i0 = it * XI;
      const bool real0 = i0 + 8 * F0 < N, real1 = i0 + 8 * F1 < N;  // padding fragments
      const int64_t p0 = (int64_t)pt * XP;
      int ptn = 0, itn = 0;  // the next tile (B prefetch across the tile boundary)
      if (t + (int)gridDim.x < ntiles) tile_of(t + gridDim.x, ptn, itn);
      double acc[2][16][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 16; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
      for (int c = 0; c < nk; ++c, ++g) {
        double2 bcur[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          bcur[h][0] = bnext[h][0];
          bcur[h][1] = bnext[h][1];
        }
        if (c + 1 < nk)
          load_b(c + 1, it, bnext);
        else if (t + (int)gridDim.x < ntiles)
          load_b(0, itn, bnext);
        const int s = g % DNA;
        mbar_wait(&fullA[s], (uint32_t)(g / DNA) & 1u);
        const double* sb = ringA + (size_t)s * SA;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k8 = c * XK + 8 * h;
          if (k8 >= N) break;
          if (real0 && real1)
            mix_big_slice<true, true>(acc, sb, nullptr, 0.0, bcur[h][0], bcur[h][1], h, gq, t4);
          else if (real0)
            mix_big_slice<true, false>(acc, sb, nullptr, 0.0, bcur[h][0], bcur[h][1], h, gq, t4);
        }
        const int crel = c - it * (XI / XK);  // diagonal stage index within the tile
        if (crel >= 0 && crel < XI / XK) {
          const bool upper_half = crel >= 4;  // fragments 2 crel, 2 crel + 1 are >= 8: the F1 side
          const int F = upper_half ? F1 : F0;
          const int se = ge % DNE;
          mbar_wait(&fullE[se], (uint32_t)(ge / DNE) & 1u);
          if ((F >> 1) == crel && (upper_half ? real1 : real0)) {
            const double* sbe = ringE + (size_t)se * SE;
            if (upper_half)
              dir_big_elementwise<1>(acc, sb, sbe, hist, F & 1, gq, t4, i0, F, N, ld, ngl, p0, sig,
                                     sigp, zout, dpart, n_pt, pt);
            else
              dir_big_elementwise<0>(acc, sb, sbe, hist, F & 1, gq, t4, i0, F, N, ld, ngl, p0, sig,
                                     sigp, zout, dpart, n_pt, pt);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&emptyE[se]);
          ++ge;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyA[s]);
      }
      // ||D_i||^2 from the registers: acc = W Sigma - HW = -D
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (!(q ? real1 : real0)) continue;
        const int F = q ? F1 : F0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = i0 + 8 * F + 2 * t4 + j;
          double v = 0.0;
#pragma unroll
          for (int gg = 0; gg < 8; ++gg) {
            const double d0 = acc[q][2 * gg][j], d1 = acc[q][2 * gg + 1][j];
            v += d0 * d0 + d1 * d1;
          }
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          if (gq == 0 && i < N) dpart[((int64_t)N + i) * n_pt + pt] = v;
        }
      }
    }
  }
}


// Upper-triangular mix (the orthonormalisation rotation W L^{-T}) with the
// triangle balanced per SM sub-partition. A 128-point tile is split into two
// 64-point halves: consumer warps 0-3 (one per sub-partition) walk the k
// chunks of the first half forwards, warps 4-7 those of the second half
// backwards, and warp a of either half owns output fragments
// {a, 7-a, 8+a, 15-a}. In the diagonal block an 8-input slice kb meets the
// fragments >= kb, so a sub-partition (warp a forwards at slice kb, warp 4+a
// backwards at 15-kb) always has 4 or 5 active fragment groups — constant
// DMMA pressure instead of 4 -> 1 over the block (mix_big_kernel: 60% of FP64
// on the triangle vs 82% dense). A stage carries both halves' chunks and both
// M^T boxes. N a multiple of 128 (every fragment real).
template <int CNT>
__device__ __forceinline__ void mix_tri_slice(double (&acc)[4][8][2], const double* sa_,
                                              const double* mt, int h, int a, int gq, int t4) {
  // the CNT highest of the warp's sorted fragments {a, 7-a, 8+a, 15-a} take part
  const int fr[4] = {a, 7 - a, 8 + a, 15 - a};
  double2 b[4];
#pragma unroll
  for (int f = 4 - CNT; f < 4; ++f)
    b[f] = *reinterpret_cast<const double2*>(mt + swz(8 * fr[f] + gq, 8 * h + 2 * t4, XI));
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    double2 av[2];
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2)
      av[s2] = *reinterpret_cast<const double2*>(sa_ + swz(8 * h + 2 * t4 + s2, 16 * g + 2 * gq, XK));
#pragma unroll
    for (int f = 4 - CNT; f < 4; ++f) {
      dmma_8x8x4(acc[f][2 * g], av[0].x, b[f].x);
      dmma_8x8x4(acc[f][2 * g + 1], av[0].y, b[f].x);
      dmma_8x8x4(acc[f][2 * g], av[1].x, b[f].y);
      dmma_8x8x4(acc[f][2 * g + 1], av[1].y, b[f].y);
    }
  }
}

__global__ void __launch_bounds__(XTH, 1) mix_tri_kernel(
    const __grid_constant__ Maps maps, int has_ab, int N, int64_t ld, int64_t ngl, int n_pt,
    int n_it, int nst, double sa, double alpha, double* __restrict__ out,
    const double* __restrict__ guard, const double* __restrict__ zsig, int mres, int qform) {
  // qform: zsig holds q_k and M^T is already scaled by sa (transpose_pad_kernel):
  // the trial point is sa (HW_k + q_k W_k), one FMA per element
  // mres (one orbital tile, N = 128): M^T stays resident in shared memory for
  // the whole kernel (8 boxes = 128 KB, loaded once) instead of two 16 KB boxes
  // per stage — per tile that was as much TMA traffic (L2) as the operands, all
  // in 128-B rows, the request-rate-bound kind (profiles/r1_tma2d_probe.txt)
  PO_PDL_ENTRY();
  if (guard && *guard == 0.0) return;
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm);
  uint64_t* empty = full + 8;
  uint64_t* ready = full + 16;
  double* mst = reinterpret_cast<double*>(tsm + 512);  // -sigma of a stage (implicit z)
  double* stage0 = reinterpret_cast<double*>(tsm + 1024);
  constexpr size_t QH = (size_t)64 * XK;  // doubles per half per source per stage
  constexpr size_t QM = (size_t)XI * XK;  // one M^T box
  const int nsrc = has_ab ? 2 : 1;
  // stage: [A half 0][A half 1]([Ab half 0][Ab half 1])[M^T chunk of half 0][M^T chunk of half 1]
  // (mres: no M^T chunks; the resident M^T follows the ring)
  const size_t mofs = (size_t)2 * nsrc * QH;
  const size_t sdoubles = mofs + (mres ? 0 : 2 * QM);
  double* mtres = stage0 + (size_t)nst * sdoubles;  // [XI / XK boxes][QM]
  uint64_t* mbar_res = full + 24;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
      mbar_init(&ready[s], 3);  // one arrival per combining warp
    }
    mbar_init(mbar_res, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int ntiles = n_pt * n_it;
  auto tile_of = [&](int t, int& pt, int& it) {
    it = n_it - 1 - t / n_pt;
    pt = t % n_pt;
  };
  const int lane = threadIdx.x & 31;
  int warp = threadIdx.x >> 5;
  if (warp < 4) {
    // 88 registers (not 40): the three combining warps form W - tau z for every
    // stage and were the consumers' dominant wait (ncu: `ready` barrier); the
    // headroom keeps four independent element chains in flight (C3 implicit
    // rotation 1.81 -> 1.75 ms; forming the trial values in the consumers
    // instead, at their fragment loads, measured 2.5 ms: the per-load branch and
    // the 4x redundant forms broke the DMMA schedule even on one source)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      for (int q = 0; q <= nsrc; ++q)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[q])));
      const uint32_t bytes = (uint32_t)(sdoubles * 8);
      if (mres) {  // the whole (padded) M^T once: box ck holds k = 16 ck .. 16 ck + 15
        mbar_arrive_expect_tx(mbar_res, (uint32_t)((XI / XK) * QM * 8));
        for (int ck = 0; ck < XI / XK; ++ck)
          tma_load_2d(mtres + (size_t)ck * QM, &maps.m[nsrc], ck * XK, 0, mbar_res);
      }
      int g = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int pt, it;
        tile_of(t, pt, it);
        const int nk = (it + 1) * XI / XK;  // upper: k < i0 + 128
        for (int c = 0; c < nk; ++c, ++g) {
          const int s = g % nst;
          if (g >= nst) mbar_wait(&empty[s], ((uint32_t)(g / nst) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], bytes);
          double* sb = stage0 + (size_t)s * sdoubles;
          for (int hf = 0; hf < 2; ++hf) {
            const int ck = hf ? nk - 1 - c : c;  // the second half walks k backwards
            for (int q = 0; q < nsrc; ++q)
              for (int b = 0; b < 4; ++b)
                tma_load_2d(sb + (q * 2 + hf) * QH + b * BOX * XK, &maps.m[q],
                            pt * XP + hf * 64 + b * BOX, ck * XK, &full[s]);
            if (!mres) tma_load_2d(sb + mofs + hf * QM, &maps.m[nsrc], ck * XK, it * XI, &full[s]);
          }
        }
      }
    } else if (warp > 0 && has_ab) {  // A + sa Ab in place (both halves)
      const int ct = threadIdx.x - 32;
      int g = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int pt, it;
        tile_of(t, pt, it);
        const int nk = (it + 1) * XI / XK;
        for (int c = 0; c < nk; ++c, ++g) {
          const int s = g % nst;
          mbar_wait(&full[s], (uint32_t)(g / nst) & 1u);
          double2* a2 = reinterpret_cast<double2*>(stage0 + (size_t)s * sdoubles);
          const double2* b2 = reinterpret_cast<const double2*>(stage0 + (size_t)s * sdoubles + 2 * QH);
          if (zsig && !qform) {  // -sigma of the stage's 2 x 16 orbitals (half 1 walks k backwards)
            if (ct < 2 * XK) {
              const int k = ((ct >= XK) ? nk - 1 - c : c) * XK + (ct & (XK - 1));
              mst[ct] = k < N ? (qform ? zsig[k] : -zsig[k]) : 0.0;
            }
            asm volatile("bar.sync 2, 96;\n" ::: "memory");
          }
          if (qform) {
#pragma unroll 4
            for (int e = ct; e < (int)QH; e += 96) {
              double2 v = a2[e];
              const double2 z = b2[e];
              // q_k straight from the 1-KB vector (L1): no staging, no CTA-level barrier
              const int k = (((2 * e) / (int)QH) ? nk - 1 - c : c) * XK + ((e & 127) >> 3);
              const double q = __ldg(zsig + k);
              v.x = fma(q, v.x, z.x);
              v.y = fma(q, v.y, z.y);
              a2[e] = v;
            }
          } else {
#pragma unroll 4
            for (int e = ct; e < (int)QH; e += 96) {  // 2 * QH doubles = QH double2
              double2 v = a2[e];
              double2 z = b2[e];
              if (zsig) {  // Ab is HW: z = HW - sigma_k W (the directions pass's FMA)
                const double ms = mst[((2 * e) / (int)QH) * XK + ((e & 127) >> 3)];
                z.x = fma(ms, v.x, z.x);
                z.y = fma(ms, v.y, z.y);
              }
              v.x += sa * z.x;
              v.y += sa * z.y;
              a2[e] = v;
            }
          }
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&ready[s]);
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    warp -= 4;
    const int gq = lane >> 2, t4 = lane & 3;
    const int hf = warp >> 2, a = warp & 3;  // half (0 forwards, 1 backwards), fragment set
    const int fr[4] = {a, 7 - a, 8 + a, 15 - a};
    if (mres) mbar_wait(mbar_res, 0);
    int g = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int pt, it;
      tile_of(t, pt, it);
      const int i0 = it * XI;
      const int nk = (it + 1) * XI / XK;
      double acc[4][8][2];
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int m = 0; m < 8; ++m) acc[f][m][0] = acc[f][m][1] = 0.0;
      for (int c = 0; c < nk; ++c, ++g) {
        const int s = g % nst;
        mbar_wait(has_ab ? &ready[s] : &full[s], (uint32_t)(g / nst) & 1u);
        const double* sb = stage0 + (size_t)s * sdoubles;
        const double* sa_ = sb + hf * QH;
        const int ck = hf ? nk - 1 - c : c;
        const double* mt = mres ? mtres + (size_t)ck * QM : sb + mofs + hf * QM;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int h = hf ? 1 - hh : hh;
          const int kb = (ck * XK + 8 * h - i0) >> 3;  // slice index relative to the tile
          const int cnt = (kb <= fr[0]) + (kb <= fr[1]) + (kb <= fr[2]) + (kb <= fr[3]);
          if (cnt == 4)
            mix_tri_slice<4>(acc, sa_, mt, h, a, gq, t4);
          else if (cnt == 3)
            mix_tri_slice<3>(acc, sa_, mt, h, a, gq, t4);
          else if (cnt == 2)
            mix_tri_slice<2>(acc, sa_, mt, h, a, gq, t4);
          else if (cnt == 1)
            mix_tri_slice<1>(acc, sa_, mt, h, a, gq, t4);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      // epilogue: acc[f][2 g + e][j] = out(point 64 hf + 16 g + 2 gq + e, orbital i0 + 8 fr[f] + 2 t4 + j)
      const int64_t pb = (int64_t)pt * XP + 64 * hf + 2 * gq;
      if (alpha == 1.0 && (int64_t)(pt + 1) * XP <= ngl) {
        // interior tile of the rotation (every tile but the last): plain stores, no
        // per-store point tests or scaling (the general form below issues ~12
        // instructions per store, 32 stores per lane and tile)
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            double* o = out + (int64_t)(i0 + 8 * fr[f] + 2 * t4 + j) * ld + pb;
#pragma unroll
            for (int gg = 0; gg < 4; ++gg)
              *reinterpret_cast<double2*>(o + 16 * gg) = make_double2(acc[f][2 * gg][j], acc[f][2 * gg + 1][j]);
          }
        continue;
      }
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = i0 + 8 * fr[f] + 2 * t4 + j;
#pragma unroll
          for (int gg = 0; gg < 4; ++gg) {
            const int64_t p = pb + 16 * gg;
            if (p >= ngl) continue;
            const double v0 = alpha * acc[f][2 * gg][j], v1 = alpha * acc[f][2 * gg + 1][j];
            if (p + 1 < ngl)
              *reinterpret_cast<double2*>(out + (int64_t)i * ld + p) = make_double2(v0, v1);
            else
              out[(int64_t)i * ld + p] = v0;
          }
        }
    }
  }
}

// Mt = (padded) M^T. With zq != null (the implicit-z trial rotation of
// mix_tri_kernel): W - tau z = sa (HW_k + q_k W_k) with sa = -tau and
// q_k = (1 - sa sigma_k) / sa, so M^T is scaled by sa here and q_k goes to zq —
// the combine is then ONE FMA per element, fma(q_k, W, HW) (it was z = fma(-sigma, W,
// HW), then W + sa z: the combining warps' DFMAs queue behind the consumers'
// DMMAs on the FP64 pipe, so their count is what the consumers wait for).
__global__ void transpose_pad_kernel(int N, int np, const double* __restrict__ M,
                                     double* __restrict__ Mt, double sa = 1.0,
                                     const double* __restrict__ zsig = nullptr,
                                     double* __restrict__ zq = nullptr) {
  PO_PDL_ENTRY();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)np * np) return;
  const int i = (int)(e / np), k = (int)(e % np);
  const double v = (i < N && k < N) ? M[(int64_t)k * N + i] : 0.0;
  Mt[e] = zq ? sa * v : v;
  if (zq && i == 0) zq[k] = k < N ? (1.0 - sa * zsig[k]) / sa : 0.0;
}

}  // namespace

// per-stream padded M^T scratch of the large-N mix (engines on different
// streams / host threads never share one)
static double* mix_big_scratch(cudaStream_t s, size_t doubles) {
  static std::mutex mu;
  static std::unordered_map<cudaStream_t, std::pair<double*, size_t>> bufs;
  std::lock_guard<std::mutex> g(mu);
  auto& b = bufs[s];
  if (b.second < doubles) {
    if (b.first) {
      cudaStreamSynchronize(s);
      cudaFree(b.first);
    }
    b.first = nullptr;
    b.second = 0;
    if (cudaMalloc(&b.first, doubles * 8) != cudaSuccess) return nullptr;
    b.second = doubles;
  }
  return b.first;
}

int mix_big_nblk(int64_t ngl) { return (int)((ngl + XP - 1) / XP); }

int launch_mix_big(int N, int64_t ld, int64_t ngl, const double* A, const double* Ab, double sa,
                   const double* M, double alpha, const double* C, double beta, int upper,
                   double* out, double* norms, cudaStream_t s, const double* guard,
                   const double* zsig) {
  static const bool off = getenv("PO_NO_MIX_BIG") != nullptr;  // measurement: tiled LDG mix
  static const bool dbg = getenv("PO_MIX_DEBUG") != nullptr;
#define PO_MB_FAIL(why)                                                 \
  do {                                                                  \
    if (dbg) fprintf(stderr, "launch_mix_big(N=%d): %s\n", N, why);     \
    return -1;                                                          \
  } while (0)
  if (off || !tma2d_available()) PO_MB_FAIL("disabled / no TMA");
  const int np = (N + 15) & ~15;
  double* mt = mix_big_scratch(s, (size_t)np * np + np);
  if (!mt) PO_MB_FAIL("scratch");
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  int q = 0;
  if (!make_map(&maps.m[q++], A, ld, N, XK)) PO_MB_FAIL("map A");
  if (Ab && !make_map(&maps.m[q++], Ab, ld, N, XK)) PO_MB_FAIL("map Ab");
  if (!make_map(&maps.m[q++], mt, np, np, XI)) PO_MB_FAIL("map Mt");
  const int nsrc = Ab ? 2 : 1;
  static const int tri_env = getenv("PO_MIX_TRI") ? atoi(getenv("PO_MIX_TRI")) : 1;  // measurement
  const bool tri = tri_env && upper && !C && !norms && N % XI == 0;
  static const int mres_env = getenv("PO_MT_RESIDENT") ? atoi(getenv("PO_MT_RESIDENT")) : 1;
  const bool mres = tri && N == XI && mres_env;  // resident M^T (128 KB) + a 3..6-stage ring
  const size_t sdoubles = tri ? (size_t)2 * nsrc * 64 * XK + (mres ? 0 : 2 * XI * XK)
                              : (size_t)(nsrc + 1) * XP * XK;
  const size_t fixed = 1024 + 1024;  // barriers, alignment slack
  const size_t resd = mres ? (size_t)XI * XI : 0;
  int nst = (int)(((mres ? 227 : 200) * 1024 - fixed - resd * 8) / (sdoubles * 8));
  if (nst > 8) nst = 8;
  if (nst < 2) PO_MB_FAIL("shared memory");
#undef PO_MB_FAIL
  const size_t smem = fixed + ((size_t)nst * sdoubles + resd) * 8;
  ::po::count_launch();
  // implicit-z triangular rotation: one-FMA combine against a scaled M^T (q_k after the matrix)
  const bool qform = tri && Ab && zsig && sa != 0.0;
  double* zq = mt + (size_t)np * np;
  launch_pdl(transpose_pad_kernel, dim3((unsigned)(((int64_t)np * np + 255) / 256)), dim3(256), 0, s, N, np, M, mt,
             qform ? sa : 1.0, qform ? zsig : (const double*)nullptr, qform ? zq : (double*)nullptr);
  const int n_pt = mix_big_nblk(ngl);
  const int n_it = (N + XI - 1) / XI;
  const int ntiles = n_pt * n_it;
  const int grid = ntiles < nsm() ? ntiles : nsm();
  if (tri) {
    set_smem(reinterpret_cast<const void*>(mix_tri_kernel), (int)smem);
    ::po::count_launch();
    launch_pdl(mix_tri_kernel, dim3(grid), dim3(XTH), smem, s, maps, Ab ? 1 : 0, N, ld, ngl, n_pt, n_it,
               nst, sa, alpha, out, guard, qform ? (const double*)zq : (Ab ? zsig : (const double*)nullptr),
               mres ? 1 : 0, qform ? 1 : 0);
    return n_pt;
  }
  set_smem(reinterpret_cast<const void*>(mix_big_kernel), (int)smem);
  ::po::count_launch();
  launch_pdl(mix_big_kernel, dim3(grid), dim3(XTH), smem, s, maps, Ab ? 1 : 0, N, ld, ngl, n_pt,
             n_it, upper, nst, sa, alpha, C, beta, out, norms, guard, Ab ? zsig : (const double*)nullptr);
  return n_pt;
}

int launch_directions_big(int N, int64_t ld, int64_t ngl, const double* W, const double* HW,
                          const double* WP, const double* XP_, const double* sig_prev,
                          const double* Sigma, const double* sig, double* Z, double* sig_save,
                          double* partials, cudaStream_t s) {
  static const int off = getenv("PO_NO_DIR_BIG") ? atoi(getenv("PO_NO_DIR_BIG")) : 0;  // measurement
  if (off || N <= 64 || !tma2d_available()) return -1;
  const int hist = WP != nullptr;
  const int np = (N + 15) & ~15;
  double* mt = mix_big_scratch(s, (size_t)np * np);
  if (!mt) return -1;
  Maps5 maps;
  std::memset(&maps, 0, sizeof maps);
  if (!make_map(&maps.m[0], W, ld, N, XK)) return -1;
  if (!make_map(&maps.m[2], HW, ld, N, XK, EW)) return -1;  // m[1] unused (Sigma^T from global)
  if (hist && (!make_map(&maps.m[3], WP, ld, N, XK, EW) || !make_map(&maps.m[4], XP_, ld, N, XK, EW)))
    return -1;
  const size_t smem = 2048 + ((size_t)DNA * XP * XK + (size_t)DNE * 3 * QE) * 8;
  ::po::count_launch();
  launch_pdl(transpose_pad_kernel, dim3((unsigned)(((int64_t)np * np + 255) / 256)), dim3(256), 0, s, N,
             np, Sigma, mt, 1.0, (const double*)nullptr, (double*)nullptr);
  const int n_pt = mix_big_nblk(ngl);
  const int n_it = (N + XI - 1) / XI;
  const int ntiles = n_pt * n_it;
  const int grid = ntiles < nsm() ? ntiles : nsm();
  set_smem(reinterpret_cast<const void*>(dir_big_kernel), (int)smem);
  ::po::count_launch();
  launch_pdl(dir_big_kernel, dim3(grid), dim3(XTH), smem, s, maps, N, ld, ngl, n_pt, n_it, hist, sig,
             hist ? sig_prev : (const double*)nullptr, Z, sig_save, partials, (const double*)mt, np);
  return n_pt;
}

size_t gram_big_workspace_doubles(int64_t ld, int N) {
  if (N <= 48) return 0;
  size_t w = 0;
  for (int t : {64, 128})
    for (int sym : {0, 1}) {
      const BigPlan p = big_plan(ld, N, sym, nsm(), t);
      const size_t a = (size_t)p.nsplit * p.ntiles * t * t;
      if (a > w) w = a;
    }
  return w;
}

bool launch_gram_big(int N, int64_t ld, int sym, const double* A, const double* Ab, double sa,
                     const double* B, const double* Bb, double sb, double* ws, size_t ws_doubles,
                     double* G, double w, cudaStream_t s, const double* guard, double* rho,
                     double* bvec, double occ, int64_t ngl, GramBB* bbl) {
  const int GT_T = big_tile(N, sym, Ab != nullptr || !sym);
  // the fused elementwise pass: Sigma = <(HW)^T W> as one non-symmetric 128-tile
  static const bool bb_off = getenv("PO_NO_GRAM_BB") != nullptr;  // measurement switch
  if (bbl && (bb_off || sym || Ab || Bb || GT_T != 128 || N <= 64 || rho)) return false;
  // the fused density needs the whole orbital set in one diagonal tile
  if (rho && !(sym && !Ab && GT_T == 128 && N <= 128 && N > 64)) return false;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  int nsrc = 0, qa_b = -1, qb = 0, qb_b = -1;
  if (!make_map(&maps.m[nsrc++], A, ld, N, GT_T)) return false;
  if (Ab) {
    qa_b = nsrc;
    if (!make_map(&maps.m[nsrc++], Ab, ld, N, GT_T)) return false;
  }
  if (sym) {
    qb = 0;
  } else {
    qb = nsrc;
    if (!make_map(&maps.m[nsrc++], B, ld, N, GT_T)) return false;
    if (Bb) {
      qb_b = nsrc;
      if (!make_map(&maps.m[nsrc++], Bb, ld, N, GT_T)) return false;
    }
  }
  if (sym) {  // off-diagonal symmetric tiles read the B side from the same block
    qb = nsrc;
    maps.m[nsrc++] = maps.m[0];
    if (Ab) {
      qb_b = nsrc;
      maps.m[nsrc++] = maps.m[qa_b];
    }
    sb = sa;
  }
  const BigPlan p = big_plan(ld, N, sym, nsm(), GT_T);
  if ((size_t)p.nsplit * p.ntiles * GT_T * GT_T > ws_doubles) return false;
  GramBBArgs bba{nullptr, nullptr, nullptr, 0, N};
  int nbb = 0;
  if (bbl) {
    if (bbl->wp) {  // history: W_prev and HW_prev / Z_prev ride in two more ring areas
      if (!make_map(&maps.m[nsrc], bbl->wp, ld, N, GT_T) || !make_map(&maps.m[nsrc + 1], bbl->xp, ld, N, GT_T))
        return false;
      nbb = 2;
    }
    bba = GramBBArgs{bbl->sig, bbl->wp ? bbl->sigp : nullptr, bbl->partials, bbl->wp ? 1 : 0, N};
    bbl->nsplit = p.nsplit;
  }
  const size_t sdoubles = (size_t)(nsrc + nbb) * GT_T * BOX;
  int nst = (int)(((bbl ? 224 : 200) * 1024 / 8) / sdoubles);
  if (nst > 8) nst = 8;
  if (nst < 2) return false;
  const size_t smem = 2048 + (size_t)nst * sdoubles * 8;
  ::po::count_launch();
  auto k = bbl ? gram_big_kernel<128, true> : GT_T == 64 ? gram_big_kernel<64> : gram_big_kernel<128>;
  const int threads = GT_T == 64 ? BigCfg<64>::THREADS : BigCfg<128>::THREADS;
  set_smem(reinterpret_cast<const void*>(k), (int)smem);
  launch_pdl(k, dim3(dim3(p.ntiles, p.nsplit)), dim3(threads), smem, s, maps, nsrc, qa_b, qb, qb_b, p.mt, sym, ld, p.kchunk,
                                                 nst, sa, sb, ws, guard, rho, bvec, occ, ngl, bba);
  const int64_t total = (int64_t)N * N;
  ::po::count_launch();
  launch_pdl(gram_big_reduce_kernel, dim3((unsigned)((total + 31) / 32)), dim3(dim3(32, 8)), 0, s, GT_T, N, p.mt, sym, p.ntiles,
                                                                               p.nsplit, w, ws, G, guard);
  return true;
}

bool tma2d_available() { return encode_fn() != nullptr; }

// Dynamic shared-memory limit, set once per kernel and size (a driver call kept
// off the launch path), plus the max-shared carveout for the big-ring kernels.
void set_smem(const void* k, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> done;
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find(k);
  if (it != done.end() && it->second >= bytes) return;
  // (kernels staging through registers / L1 keep the default carveout: the
  // tiled LDG mix lost 20% at C3 with the max-shared carveout)
  if (it == done.end() && bytes >= 64 * 1024)
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
  if (bytes > 0) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done[k] = bytes;
}

// split trial rotation: two-source mix (W + sa Z) L^{-T} (device-side scale
// possible), then the verification Gram + density / xc of W~ in one pass
template <int F>
int launch_rotation_split_f(int N, int64_t ld, int64_t ngl, const double* A, const double* Ab,
                            double sa, const double* M, double* out, double* ws, double* G, double w,
                            double occ, int xc, double* rho, double* vxc, double* bvec,
                            const double* vext, double* dpart, cudaStream_t s, const double* sa_dev) {
  constexpr int NPAD = 8 * F;
  if (launch_mix_tma_f<F>(N, ld, ngl, A, Ab, sa, M, 1.0, nullptr, 0.0, 1, out, nullptr, s, nullptr,
                          sa_dev) < 0)
    return -1;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  if (!make_map2(maps, 0, out, ld, N, NPAD)) return -1;
  const size_t red = (size_t)TSC * (F * (F + 1) / 2) * 64 + 2 * TSC;
  TCfg cfg = tcfg(1, N, 0);
  if (cfg.smem < 3072 + red * 8) cfg.smem = 3072 + red * 8;
  const int64_t kblocks = (ld + TKS - 1) / TKS;
  int nsplit = nsm();
  if (nsplit > kblocks) nsplit = (int)kblocks;
  const int64_t kchunk = ((kblocks + nsplit - 1) / nsplit) * TKS;
  nsplit = (int)((ld + kchunk - 1) / kchunk);
  ::po::count_launch();
  auto k = gram_density_kernel<F>;
  set_smem(reinterpret_cast<const void*>(k), (int)cfg.smem);
  launch_pdl(k, dim3(nsplit), dim3(TTH), cfg.smem, s, maps, N, ld, ngl, kchunk, cfg.nst, ws, occ, xc,
             rho, vxc, bvec, vext, dpart);
  const int64_t threads = (int64_t)N * N * 32;
  ::po::count_launch();
  launch_pdl(gram_tma_reduce_kernel, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, s, N, NPAD,
             1, nsplit, w, ws, G, (const double*)nullptr, (const double*)nullptr, (double*)nullptr,
             (double*)nullptr);
  return nsplit;
}

int launch_rotate_fused(int N, int64_t ld, int64_t ngl, const double* A, const double* Ab,
                        double sa, const double* M, double* out, double* ws, double* G, double w,
                        double occ, int xc, double* rho, double* vxc, double* bvec,
                        const double* vext, double* dpart, cudaStream_t s, const double* sa_dev,
                        const double* zsig) {
  // measurement switch: rotation as the two-source mix + a Gram/density pass (slower: 250 vs 218 us at C2)
  static const int split = getenv("PO_ROT_SPLIT") ? atoi(getenv("PO_ROT_SPLIT")) : 0;
  if (split && !zsig) {
    switch ((N + 7) / 8) {
#define PO_RS(F) \
  case F:        \
    return launch_rotation_split_f<F>(N, ld, ngl, A, Ab, sa, M, out, ws, G, w, occ, xc, rho, vxc, bvec, vext, dpart, s, sa_dev);
      PO_RS(1) PO_RS(2) PO_RS(3) PO_RS(4) PO_RS(5) PO_RS(6)
#undef PO_RS
    }
    return -1;
  }
  switch ((N + 7) / 8) {
#define PO_RF(F) \
  case F:        \
    return launch_rotate_fused_f<F>(N, ld, ngl, A, Ab, sa, M, out, ws, G, w, occ, xc, rho, vxc, bvec, vext, dpart, s, sa_dev, zsig);
    PO_RF(1) PO_RF(2) PO_RF(3) PO_RF(4) PO_RF(5) PO_RF(6)
#undef PO_RF
  }
  return -1;
}

int launch_directions(int N, int64_t ld, int64_t ngl, const double* W, const double* HW,
                      const double* WP, const double* ZP, const double* Sigma, const double* sig,
                      double* Z, double* partials, cudaStream_t s, const double* psig,
                      double* sig_out) {
  switch ((N + 7) / 8) {
#define PO_DR(F) \
  case F:        \
    return launch_directions_f<F>(N, ld, ngl, W, HW, WP, ZP, Sigma, sig, Z, partials, s, psig, sig_out);
    PO_DR(1) PO_DR(2) PO_DR(3) PO_DR(4) PO_DR(5) PO_DR(6)
#undef PO_DR
  }
  return -1;
}

bool launch_gram_tma(int N, int64_t ld, int sym, const double* A, const double* Ab, double sa,
                     const double* B, const double* Bb, double sb, double* ws, double* G, double w,
                     cudaStream_t s, const double* guard, double* G2, double* diag) {
  switch ((N + 7) / 8) {
#define PO_GT(F) \
  case F:        \
    return launch_gram_tma_f<F>(N, ld, sym, A, Ab, sa, B, Bb, sb, ws, G, w, s, guard, G2, diag);
    PO_GT(1) PO_GT(2) PO_GT(3) PO_GT(4) PO_GT(5) PO_GT(6)
#undef PO_GT
  }
  return false;
}

int launch_mix_tma(int N, int64_t ld, int64_t ngl, const double* A, const double* Ab, double sa,
                   const double* M, double alpha, const double* C, double beta, int upper,
                   double* out, double* norms, cudaStream_t s, const double* guard) {
  switch ((N + 7) / 8) {
#define PO_MT(F) \
  case F:        \
    return launch_mix_tma_f<F>(N, ld, ngl, A, Ab, sa, M, alpha, C, beta, upper, out, norms, s, guard);
    PO_MT(1) PO_MT(2) PO_MT(3) PO_MT(4) PO_MT(5) PO_MT(6) PO_MT(7) PO_MT(8)
#undef PO_MT
  }
  return -1;
}

}  // namespace po
