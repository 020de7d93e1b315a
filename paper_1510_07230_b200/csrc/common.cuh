// Shared device helpers for the parorb B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace po {

constexpr int kWarp = 32;

// Grid geometry of one rank's slab. Points are lexicographic, axis 2 fastest
// (include/parorb/grid.hpp:11-14); a block stores N orbitals with stride ld.
struct SlabGeom {
  int64_t n0, n1, n2;     // global interior points per axis
  int64_t z0, nz;         // local planes [z0, z0 + nz) of axis 0
  int64_t plane;          // n1 * n2
  int64_t ngl;            // nz * plane (local points)
  int64_t ld;             // orbital stride in a block (>= ngl, padded)
  double ih2[3];          // 1 / h_a^2
  double w;               // quadrature weight h0 h1 h2
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction of NQ values; result valid in thread 0.
template <int NQ>
__device__ __forceinline__ void block_sum(double (&v)[NQ], double* smem /* >= 32*NQ */) {
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int warp = tid >> 5;
  const int nwarps = (blockDim.x * blockDim.y + 31) >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) smem[q * 32 + warp] = v[q];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double x = lane < nwarps ? smem[q * 32 + lane] : 0.0;
      v[q] = warp_sum(x);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double dirac_cx() {
  // kDiracCx = 0.75 * cbrt(3 / pi), energy.cpp:18
  return 0.75 * cbrt(3.0 / 3.141592653589793238462643383279502884);
}

// One warp mma.sync m8n8k4 fp64 (SASS DMMA.8x8x4): D = A(8x4, row) B(4x8, col) + C.
// Fragments: a = A[lane/4][lane%4], b = B[lane%4][lane/4],
//            c[j] = C[lane/4][2*(lane%4) + j].
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  // not volatile: no side effects beyond its outputs, so the scheduler may
  // interleave independent DMMAs with the fragment loads around them
  asm(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- TMA / mbarrier
// 1D bulk tensor-memory-accelerator copies (cp.async.bulk, SASS UBLKCP) with
// mbarrier transaction counting: the producer arms a stage's "full" barrier
// with the byte count, the copies complete it; consumers release the stage
// through its "empty" barrier.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy of `bytes` (multiple of 16, 16-B aligned), completing on bar
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gsrc, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------ programmatic dependent launch
// Kernels on the iteration path are launched with programmatic stream
// serialization (launch_pdl): the next kernel may be scheduled while the
// previous one drains, so its launch latency overlaps the tail. Each such
// kernel starts with PO_PDL_ENTRY(): wait for the preceding grid (its memory
// is then visible), then let the following grid start launching (it too waits
// before touching memory). A grid's dependents launch only once every one of
// its CTAs has started, so no waiting CTA can starve the kernel it waits on.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
#define PO_PDL_ENTRY() \
  do {                 \
    pdl_wait();        \
    pdl_trigger();     \
  } while (0)

bool pdl_on();  // PO_PDL=0 disables the attribute (measurement)

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace po
