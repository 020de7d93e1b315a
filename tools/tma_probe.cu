// Probe: HBM delivery rate of a TMA bulk-copy ring vs request size / depth,
// against a plain vectorised-LDG streaming reduction. Shape: R rows of the
// C2 orbital block (N=33 x 884736 doubles), each CTA streams a contiguous
// point range of every row (the Gram / mix access pattern).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_probe.cu -o tma_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1510_07230_b200/csrc/common.cuh"

using namespace po;

__global__ void __launch_bounds__(288, 1) ring_kernel(const double* src, int rows, long ld,
                                                      long chunk, int ks, int nst, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 8;
  double* st0 = (double*)(sm + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t sd = (size_t)rows * ks;
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
    for (int t = 0; t < nstage; ++t) {
      const int s = t % nst;
      if (t >= nst) mbar_wait(&empty[s], ((t / nst) & 1) ^ 1);
      const long k0 = kbeg + (long)t * ks;
      const int cnt = (int)min((long)ks, kend - k0);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], rows * cnt * 8);
      __syncwarp();
      for (int r = lane; r < rows; r += 32)
        tma_load_1d(st0 + s * sd + (size_t)r * ks, src + (long)r * ld + k0, cnt * 8, &full[s]);
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

__global__ void ldg_kernel(const double* src, int rows, long ld, double* sink) {
  double acc = 0.0;
  for (long p = (long)blockIdx.x * blockDim.x + threadIdx.x; p < ld / 2;
       p += (long)gridDim.x * blockDim.x) {
    for (int r = 0; r < rows; r += 4) {
      double2 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        v[j] = r + j < rows ? __ldg((const double2*)(src + (long)(r + j) * ld) + p) : make_double2(0, 0);
#pragma unroll
      for (int j = 0; j < 4; ++j) acc += v[j].x * v[j].y;
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  const int rows = 33;
  const long ld = 884736;
  double *src, *sink;
  cudaMalloc(&src, sizeof(double) * rows * ld);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 0, sizeof(double) * rows * ld);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = 8.0 * rows * ld;
  for (int ks : {64, 128, 256, 512}) {
    for (int nst : {2, 3, 4, 6}) {
      const size_t smem = 128 + (size_t)nst * rows * ks * 8;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const long kb = (ld + ks - 1) / ks;
      const long chunk = ((kb + 147) / 148) * ks;
      const int grid = (int)((ld + chunk - 1) / chunk);
      ring_kernel<<<grid, 288, smem>>>(src, rows, ld, chunk, ks, nst, sink);
      cudaEventRecord(a);
      for (int i = 0; i < 5; ++i) ring_kernel<<<grid, 288, smem>>>(src, rows, ld, chunk, ks, nst, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("ring ks=%4d (%5d B/copy) nst=%d smem=%6zu: %7.1f us  %6.0f GB/s\n", ks, ks * 8, nst, smem,
             1e3 * ms / 5, bytes / (ms / 5 * 1e-3) / 1e9);
    }
  }
  for (int per : {4, 8, 16}) {
    const int grid = 148 * per;
    ldg_kernel<<<grid, 256>>>(src, rows, ld, sink);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) ldg_kernel<<<grid, 256>>>(src, rows, ld, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("ldg  grid=%d: %7.1f us  %6.0f GB/s\n", grid, 1e3 * ms / 5, bytes / (ms / 5 * 1e-3) / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
