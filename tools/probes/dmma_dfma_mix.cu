// Probe: do DMMA (FP64 tensor) and DFMA (FP64 CUDA-core) share one pipe?
// One CTA per SM.  Warps [0, nd) run register-fed DMMA.8x8x4 loops (64x32
// accumulators, as the update kernel), warps [nd, nd + nf) run independent
// DFMA chains.  Reported: each kind's TFLOP/s alone and mixed.  If the mix
// exceeds the DMMA-only rate, the two pipes add up.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_dfma_mix dmma_dfma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(512, 1) mix(double* out, int nd, int nf, int iters_d, int iters_f) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double sink = 0.0;
  if (warp < nd) {
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (lane + i);
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = 1e-3 * (lane - j);
    for (int s = 0; s < iters_d; ++s) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) sink += acc[i][j][0] + acc[i][j][1];
  } else if (warp < nd + nf) {
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = 1e-3 * (lane + k);
    const double m = 0.999999, c = 1e-9;
    for (int s = 0; s < iters_f; ++s) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = fma(x[k], m, c);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) sink += x[k];
  }
  if (sink == 12345.678) out[blockIdx.x] = sink;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sms * sizeof(double));
  const int iters_d = 20000, iters_f = 20000;
  // flops: DMMA warp: iters * 32 DMMA * 512; DFMA warp: iters * 8 * 16 * 32 lanes * 2
  struct Cfg { int nd, nf; };
  Cfg cfgs[] = {{8, 0}, {0, 8}, {0, 16}, {8, 4}, {8, 8}, {4, 8}, {12, 4}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<<<sms, 512>>>(out, 8, 8, 100, 100);  // warm-up
  cudaDeviceSynchronize();
  for (const Cfg& c : cfgs) {
    cudaEventRecord(e0);
    mix<<<sms, 512>>>(out, c.nd, c.nf, iters_d, iters_f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fd = (double)sms * c.nd * iters_d * 32.0 * 512.0;
    const double ff = (double)sms * c.nf * iters_f * 8.0 * 16.0 * 32.0 * 2.0;
    printf("{\"dmma_warps\": %d, \"dfma_warps\": %d, \"ms\": %.3f, \"dmma_tflops_if_alone\": %.2f, "
           "\"dfma_tflops_if_alone\": %.2f, \"combined_tflops\": %.2f}\n",
           c.nd, c.nf, ms, fd / (ms * 1e-3) / 1e12, ff / (ms * 1e-3) / 1e12, (fd + ff) / (ms * 1e-3) / 1e12);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
