// Probe: where does the single-CTA tile POTRF spend its time?  Phase stamps
// (clock64) of warp 0 (the diagonal-block chain) and warp 1 (trailing
// blocks) per 32-column step, for tiles 128 / 256 / 512, shared-memory
// (128) and L2 paths, with and without the fused inverse.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DBGP_POTRF_TRACE \
//        -I paper_1305_4886_b200/csrc -o tools/probes/potrf_trace tools/probes/potrf_trace.cu -lcuda
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bgp_common.cuh"
#include "bgp_internal.h"
#include "panel_device.cuh"

using namespace bgp;

static size_t smem_bytes(int b, bool in_smem) {
  return (in_smem ? (size_t)b * b * 8 : 0) + (size_t)(2 * NB * 33 + (b - NB) * PLD + 2 * NB + 2) * 8;
}

__global__ void __launch_bounds__(POTRF_THREADS, 1)
    probe(double* A, int b, double* dinv, unsigned long long* info, double* Linv, int* progress, int mode) {
  extern __shared__ double sm[];
  if (mode == 0) tile_potrf_inv_device(A, b, 0, dinv, info, Linv, sm, threadIdx.x, 0, progress);
  else tile_potrf_device(A, b, 0, dinv, info, sm, threadIdx.x, 0, Linv, false, progress);
}

int main() {
  const int tiles[] = {128, 256, 512};
  for (int b : tiles) {
    std::vector<double> h((size_t)b * b);
    srand(1);
    // diagonally dominant SPD tile, column-major lower
    for (int c = 0; c < b; ++c)
      for (int r = 0; r < b; ++r) h[(size_t)c * b + r] = (r == c) ? b : (r > c ? 1.0 / (1 + r - c) : 0.0);
    double *dA, *dD, *dL;
    unsigned long long* dI;
    int* dP;
    cudaMalloc(&dA, h.size() * 8);
    cudaMalloc(&dD, (size_t)b * 32 * 8);
    cudaMalloc(&dL, h.size() * 8);
    cudaMalloc(&dI, 8);
    cudaMalloc(&dP, 4);
    for (int variant = 0; variant < 4; ++variant) {
      // 0: default path (smem at 128), no inverse; 1: + inverse; 2: L2 path
      // with progress (substitution look-ahead); 3: L2 path, no progress
      const bool inv = variant == 1;
      int* prog = variant == 2 ? dP : nullptr;
      const int mode = variant == 3 ? 1 : 0;
      const bool in_smem = (b <= SMEM_TILE) && variant < 2;
      const size_t smem = smem_bytes(b, in_smem);
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      float best = 1e30f;
      std::vector<long long> tr(2 * 1024);
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemcpy(dA, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        cudaMemset(dI, 0, 8);
        cudaMemset(dP, 0, 4);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<1, POTRF_THREADS, smem>>>(dA, b, dD, dI, inv ? dL : nullptr, prog, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) {
          best = ms;
          cudaMemcpyFromSymbol(tr.data(), g_ptrace, tr.size() * 8);
        }
      }
      unsigned long long info;
      cudaMemcpy(&info, dI, 8, cudaMemcpyDeviceToHost);
      // residual of the factor (lower part, column-major) and of Dinv_k L_kk = I
      std::vector<double> L((size_t)b * b), Dv((size_t)b * 32);
      cudaMemcpy(L.data(), dA, L.size() * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(Dv.data(), dD, Dv.size() * 8, cudaMemcpyDeviceToHost);
      double res = 0.0, dres = 0.0;
      for (int c = 0; c < b; ++c)
        for (int r = c; r < b; ++r) {
          double s = 0.0;
          for (int k = 0; k <= c; ++k) s += L[(size_t)k * b + r] * L[(size_t)k * b + c];
          res = fmax(res, fabs(s - h[(size_t)c * b + r]) / b);
        }
      for (int k = 0; k < b / 32; ++k)
        for (int i = 0; i < 32; ++i)
          for (int j = 0; j < 32; ++j) {
            double s = 0.0;  // (Dinv_k L_kk)(i, j), Dinv column-major 32x32
            for (int m = 0; m < 32; ++m) s += Dv[(size_t)k * 1024 + m * 32 + i] * L[(size_t)(k * 32 + j) * b + k * 32 + m];
            dres = fmax(dres, fabs(s - (i == j ? 1.0 : 0.0)));
          }
      cudaError_t e = cudaGetLastError();
      printf("{\"tile\": %d, \"variant\": %d, \"inverse\": %d, \"smem_tile\": %d, \"progress\": %d, \"us\": %.2f, "
             "\"info\": %llu, \"err\": \"%s\", \"resid\": %.3e, \"dinv_resid\": %.3e",
             b, variant, inv, in_smem, prog != nullptr, best * 1e3, info, cudaGetErrorString(e), res, dres);
      // per step: [A phase, barrier A, diag update, potrf32, trinv32 / trailing, barrier B] in cycles
      const long long* w0 = tr.data();
      const long long* w1 = tr.data() + 1024;
      printf(", \"prologue_cyc\": %lld, \"steps\": [", w0[1] - w0[0]);
      const int nbk = b / 32;
      for (int kb = 0; kb + 1 < nbk; ++kb) {
        const int i = 2 + 6 * kb;
        const long long next0 = (kb + 2 < nbk) ? w0[i + 6] : -1;
        printf("%s{\"A\": %lld, \"barA\": %lld, \"diag_upd\": %lld, \"potrf32\": %lld, \"trinv32\": %lld, "
               "\"w1_inv\": %lld, \"barB\": %lld}",
               kb ? ", " : "", w0[i + 1] - w0[i], w0[i + 2] - w0[i + 1], w0[i + 3] - w0[i + 2], w0[i + 4] - w0[i + 3],
               w0[i + 5] - w0[i + 4], w1[i + 3] - w1[i + 2], next0 > 0 ? next0 - w0[i + 5] : -1);
      }
      printf("]}\n");
    }
    cudaFree(dA);
    cudaFree(dD);
    cudaFree(dL);
    cudaFree(dI);
    cudaFree(dP);
  }
  return 0;
}
