// DMMA (mma.sync.m8n8k4.f64) and DFMA issue-rate probe: warps per SM x
// independent accumulator chains. Prints TFLOP/s for each configuration.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_loop(double* out, int iters) {
  double acc[CH][2];
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
          : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[0] = s;
}

template <int CH>
__global__ void dfma_loop(double* out, int iters) {
  double acc[CH];
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x;
  const double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.0) out[0] = s;
}

template <int CH>
void run(const char* name, void (*k)(double*, int), double flops_per_inst_warp, int sms) {
  double* d;
  cudaMalloc(&d, 8);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 20000;
    k<<<sms, warps * 32>>>(d, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    if (cudaGetLastError() != cudaSuccess) {  // e.g. too many registers for the block size
      printf("%s chains=%d warps/SM=%2d : launch failed\n", name, CH, warps);
      continue;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)sms * warps * iters * CH * flops_per_inst_warp;
    printf("%s chains=%d warps/SM=%2d : %6.2f TFLOP/s\n", name, CH, warps, fl / ms / 1e9);
  }
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1>("DMMA", dmma_loop<1>, 512.0, sms);
  run<4>("DMMA", dmma_loop<4>, 512.0, sms);
  run<16>("DMMA", dmma_loop<16>, 512.0, sms);
  run<1>("DFMA", dfma_loop<1>, 64.0, sms);
  run<8>("DFMA", dfma_loop<8>, 64.0, sms);
  return 0;
}
