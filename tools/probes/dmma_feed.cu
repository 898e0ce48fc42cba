// Probe: how fast can LDS-fed DMMA.8x8x4 run on one SM?  Each warp owns a
// 64x32 accumulator (8x4 DMMA tiles) and per "stage" issues 64 DMMAs fed by
// MODE-dependent fragment traffic.  Prints TFLOP/s for each variant.
//   MODE 0: fragments in registers (no LDS)
//   MODE 1: 24 LDS.64 per stage, all issued before the stage's DMMAs
//   MODE 2: MODE 1 + split halves (12 LDS before each 32 DMMAs, pipelined)
//   MODE 3: MODE 1 with LDS.128 (12 LDS.128 per stage)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_feed dmma_feed.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int OFF>
__device__ __forceinline__ double lds(unsigned base) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(base), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ void lds2(unsigned base, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2+%3];" : "=d"(x), "=d"(y) : "r"(base), "n"(OFF));
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) feed(double* out, int stages) {
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 24576; i += blockDim.x) sm[i] = 1e-3 * (i & 7);
  __syncthreads();
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double a[2][8], b[2][4];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[t][i] = 1e-3 * (lane + i + t);
#pragma unroll
    for (int j = 0; j < 4; ++j) b[t][j] = 1e-3 * (lane - j + t);
  }
  unsigned base = (unsigned)__cvta_generic_to_shared(sm) + warp * 24576 + lane * 16;
  for (int s = 0; s < stages; ++s) {
    const unsigned sb = base + (s & 3) * 2048;
    if (MODE == 1) {
      a[0][0] = lds<0>(sb); a[0][1] = lds<256>(sb); a[0][2] = lds<512>(sb); a[0][3] = lds<768>(sb);
      a[0][4] = lds<1024>(sb); a[0][5] = lds<1280>(sb); a[0][6] = lds<1536>(sb); a[0][7] = lds<1792>(sb);
      b[0][0] = lds<4096>(sb); b[0][1] = lds<4352>(sb); b[0][2] = lds<4608>(sb); b[0][3] = lds<4864>(sb);
      a[1][0] = lds<8192>(sb); a[1][1] = lds<8448>(sb); a[1][2] = lds<8704>(sb); a[1][3] = lds<8960>(sb);
      a[1][4] = lds<9216>(sb); a[1][5] = lds<9472>(sb); a[1][6] = lds<9728>(sb); a[1][7] = lds<9984>(sb);
      b[1][0] = lds<12288>(sb); b[1][1] = lds<12544>(sb); b[1][2] = lds<12800>(sb); b[1][3] = lds<13056>(sb);
    }
    if (MODE == 3) {
      lds2<0>(sb, a[0][0], a[0][1]); lds2<512>(sb, a[0][2], a[0][3]); lds2<1024>(sb, a[0][4], a[0][5]);
      lds2<1536>(sb, a[0][6], a[0][7]); lds2<4096>(sb, b[0][0], b[0][1]); lds2<4608>(sb, b[0][2], b[0][3]);
      lds2<8192>(sb, a[1][0], a[1][1]); lds2<8704>(sb, a[1][2], a[1][3]); lds2<9216>(sb, a[1][4], a[1][5]);
      lds2<9728>(sb, a[1][6], a[1][7]); lds2<12288>(sb, b[1][0], b[1][1]); lds2<12800>(sb, b[1][2], b[1][3]);
    }
    if (MODE == 2) {
      a[0][0] = lds<0>(sb); a[0][1] = lds<256>(sb); a[0][2] = lds<512>(sb); a[0][3] = lds<768>(sb);
      a[0][4] = lds<1024>(sb); a[0][5] = lds<1280>(sb); a[0][6] = lds<1536>(sb); a[0][7] = lds<1792>(sb);
      b[0][0] = lds<4096>(sb); b[0][1] = lds<4352>(sb); b[0][2] = lds<4608>(sb); b[0][3] = lds<4864>(sb);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[0][i], b[0][j]);
    if (MODE == 2) {
      a[1][0] = lds<8192>(sb); a[1][1] = lds<8448>(sb); a[1][2] = lds<8704>(sb); a[1][3] = lds<8960>(sb);
      a[1][4] = lds<9216>(sb); a[1][5] = lds<9472>(sb); a[1][6] = lds<9728>(sb); a[1][7] = lds<9984>(sb);
      b[1][0] = lds<12288>(sb); b[1][1] = lds<12544>(sb); b[1][2] = lds<12800>(sb); b[1][3] = lds<13056>(sb);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[1][i], b[1][j]);
  }
  double sum = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) sum += acc[i][j][0] + acc[i][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
}

template <int MODE>
void run(double* out, int sms, int warps, int stages) {
  cudaFuncSetAttribute(feed<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  feed<MODE><<<sms, warps * 32, 196608>>>(out, stages);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) feed<MODE><<<sms, warps * 32, 196608>>>(out, stages);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 3;
  double flop = 2.0 * 8 * 8 * 4 * 64.0 * stages * warps * sms;
  printf("{\"probe\":\"dmma_feed\",\"mode\":%d,\"warps_per_sm\":%d,\"tflops\":%.2f}\n", MODE, warps,
         flop / ms / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sms * 1024 * 8);
  for (int w : {4, 8}) {
    run<0>(out, sms, w, 4000);
    run<1>(out, sms, w, 4000);
    run<2>(out, sms, w, 4000);
    run<3>(out, sms, w, 4000);
  }
  return 0;
}
