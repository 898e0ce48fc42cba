// Probe: single-warp issue rates on sm_100a for the latency-bound tile
// POTRF: DFMA (independent chains), dependent DFMA latency, LDS.64 broadcast,
// SHFL of a double, MUFU-based rsqrt(double).  Cycles per instruction of one
// warp (clock64), one CTA of 32 or 256 threads (all warps doing the same).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/warp_rates tools/probes/warp_rates.cu
#include <cstdio>

constexpr int N = 4096;

__global__ void k_dfma_ilp(double* out, long long* cyc) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  const double m = out[0], c = out[1];
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 8; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[2 + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_dfma_dep(double* out, long long* cyc) {
  double a = threadIdx.x;
  const double m = out[0], c = out[1];
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = fma(a, m, c);
  long long t1 = clock64();
  out[2 + threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_lds_bcast(double* out, long long* cyc) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i;
  __syncthreads();
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 8; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] += s[(i * 8 + k) & 1023];  // same address in all lanes
  long long t1 = clock64();
  double t = 0;
  for (int k = 0; k < 8; ++k) t += acc[k];
  out[2 + threadIdx.x] = t;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_shfl(double* out, long long* cyc) {
  double v[8];
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 8; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] += __shfl_sync(0xffffffffu, v[k], (i + k) & 31);
  long long t1 = clock64();
  double t = 0;
  for (int k = 0; k < 8; ++k) t += acc[k];
  out[2 + threadIdx.x] = t;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_rsqrt_dep(double* out, long long* cyc) {
  double a = 2.0 + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 16; ++i) a = rsqrt(a) + 1.5;
  long long t1 = clock64();
  out[2 + threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 4096 * 8);
  cudaMalloc(&c, 8);
  double init[2] = {0.999, 1e-3};
  cudaMemcpy(d, init, 16, cudaMemcpyHostToDevice);
  struct K {
    const char* name;
    void (*f)(double*, long long*);
    int per;
  } ks[] = {{"dfma_ilp8", k_dfma_ilp, N},   {"dfma_dependent", k_dfma_dep, N}, {"lds64_broadcast", k_lds_bcast, N},
            {"shfl_f64", k_shfl, N},        {"rsqrt_f64_dependent", k_rsqrt_dep, N / 16}};
  for (auto& k : ks)
    for (int threads : {32, 128, 256}) {
      long long best = 1ll << 60;
      for (int r = 0; r < 3; ++r) {
        k.f<<<1, threads>>>(d, c);
        long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (h < best) best = h;
      }
      printf("{\"op\": \"%s\", \"threads\": %d, \"cycles_per_op_per_warp\": %.2f}\n", k.name, threads,
             (double)best / k.per);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
