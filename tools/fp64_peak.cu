// FP64 peak probes for the roofline denominators (DMMA.8x8x4, DFMA, copy).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_tput(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_tput(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <typename K>
float timeit(K k, int reps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k(); cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out; CK(cudaMalloc(&out, 1 << 20));
  const int iters = 20000;
  for (int wps : {4, 8, 16, 32}) {
    int threads = wps * 32;
    float ms = timeit([&] { dmma_tput<8><<<sms, threads>>>(out, iters); }, 3);
    double flop = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)wps * sms;
    printf("{\"probe\":\"dmma_m8n8k4\",\"warps_per_sm\":%d,\"tflops\":%.2f,\"ms\":%.3f}\n", wps, flop / ms / 1e9, ms);
  }
  for (int wps : {8, 16, 32}) {
    int threads = wps * 32;
    float ms = timeit([&] { dfma_tput<8><<<sms, threads>>>(out, iters); }, 3);
    double flop = 2.0 * 8 * (double)iters * threads * sms;
    printf("{\"probe\":\"dfma\",\"warps_per_sm\":%d,\"tflops\":%.2f,\"ms\":%.3f}\n", wps, flop / ms / 1e9, ms);
  }
  // dependent-chain latency: one warp, one accumulator
  {
    float ms = timeit([&] { dmma_tput<1><<<1, 32>>>(out, iters); }, 3);
    printf("{\"probe\":\"dmma_latency\",\"ns_per_dmma\":%.2f,\"clk_mhz_attr\":%d}\n", ms * 1e6 / iters, clk / 1000);
  }
  size_t n = (size_t)1 << 28;  // 2 GiB per buffer
  double4 *a, *b; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
  cudaMemset(a, 0, n * 8);
  float ms = timeit([&] { copy_k<<<sms * 8, 512>>>(a, b, n / 4); }, 5);
  printf("{\"probe\":\"copy\",\"gbs\":%.1f}\n", 2.0 * n * 8 / ms / 1e6);
  return 0;
}
