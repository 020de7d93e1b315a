// Probe: HBM delivery rate of a 2D tensor-map TMA ring vs box shape, for the
// small-N orbital-block stream (C2: 33 rows x 884736 doubles). Each CTA
// streams a contiguous point range of all rows; a stage is KS points of every
// row, fetched as KS/BX boxes {BX points x rows}. BX = 16 uses SWIZZLE_128B
// (the layout the small-N kernels read); BX >= 32 must use SWIZZLE_NONE.
// The consumers only touch one word per stage (no math): this is the ceiling
// the TMA path can deliver for a given box shape.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma2d_probe.cu -o tma2d_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1510_07230_b200/csrc/common.cuh"

using namespace po;

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

struct Maps2 {
  CUtensorMap m[2];
};

__global__ void __launch_bounds__(288, 1) ring2d(const __grid_constant__ Maps2 maps, int nsrc, int rows,
                                                 long ld, long chunk, int ks, int bx, int nst,
                                                 double* sink) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 8;
  double* st0 = (double*)(sm + 1024);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t sd = (size_t)nsrc * rows * ks;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long kbeg = blockIdx.x * chunk, kend = min(kbeg + chunk, ld);
  const int nstage = (int)((kend - kbeg + ks - 1) / ks);
  double acc = 0.0;
  if (warp == 8) {
    if (lane == 0) {
      for (int t = 0; t < nstage; ++t) {
        const int s = t % nst;
        if (t >= nst) mbar_wait(&empty[s], ((t / nst) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], (uint32_t)(sd * 8));
        const long k0 = kbeg + (long)t * ks;
        for (int q = 0; q < nsrc; ++q)
          for (int b = 0; b < ks / bx; ++b)
            tma2d(st0 + s * sd + ((size_t)q * (ks / bx) + b) * rows * bx, &maps.m[q], (int)(k0 + b * bx), 0,
                  &full[s]);
      }
    }
  } else {
    for (int t = 0; t < nstage; ++t) {
      const int s = t % nst;
      mbar_wait(&full[s], (t / nst) & 1);
      acc += st0[s * sd + threadIdx.x];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  const int rows = 33;
  const long ld = 884736;
  double *src, *sink;
  cudaMalloc(&src, sizeof(double) * rows * ld * 2);
  cudaMalloc(&sink, 64);
  cudaMemset(src, 0, sizeof(double) * rows * ld * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ring2d, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  printf("2D TMA ring, %d rows x %ld doubles per source, %d CTAs (one per SM), no math\n", rows, ld, sms);
  for (int nsrc = 1; nsrc <= 2; ++nsrc)
    for (int ks : {64, 128, 256})
      for (int bx : {16, 32, 64, 128, 256}) {
        if (bx > ks) continue;
        Maps2 maps;
        bool ok = true;
        for (int s = 0; s < nsrc; ++s) {
          cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
          cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
          cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)rows};
          cuuint32_t es[2] = {1, 1};
          ok &= enc(&maps.m[s], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src + (size_t)s * rows * ld, dims,
                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    bx == 16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        if (!ok) {
          printf("encode failed ks=%d bx=%d\n", ks, bx);
          continue;
        }
        const size_t sdb = (size_t)nsrc * rows * ks * 8;
        int nst = (int)((200 * 1024) / sdb);
        if (nst > 8) nst = 8;
        if (nst < 2) {
          printf("nsrc=%d ks=%3d bx=%3d: stage %zu KB does not double-buffer\n", nsrc, ks, bx, sdb / 1024);
          continue;
        }
        const long chunk = ((ld + sms - 1) / sms + ks - 1) / ks * ks;
        const size_t smem = 2048 + nst * sdb;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int it = 0; it < 3; ++it)
          ring2d<<<sms, 288, smem>>>(maps, nsrc, rows, ld, chunk, ks, bx, nst, sink);
        cudaEventRecord(a);
        const int reps = 20;
        for (int it = 0; it < reps; ++it)
          ring2d<<<sms, 288, smem>>>(maps, nsrc, rows, ld, chunk, ks, bx, nst, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double us = ms * 1e3 / reps;
        printf("nsrc=%d ks=%3d bx=%3d nst=%d: %7.1f us  %6.0f GB/s  (%s)\n", nsrc, ks, bx, nst, us,
               nsrc * rows * ld * 8.0 / us / 1e3, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
