// Probe: does cp.reduce.async.bulk.tensor .add work on a FLOAT64 tensor map?
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const __grid_constant__ CUtensorMap map) {
  __shared__ __align__(1024) double buf[16 * 8];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) buf[i] = 1.5 + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned s = (unsigned)__cvta_generic_to_shared(buf);
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
                 :: "l"(&map), "r"(0), "r"(0), "r"(0), "r"(s) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  double* d; cudaMalloc(&d, 64 * 64 * 8);
  double h[64 * 64]; for (int i = 0; i < 64 * 64; ++i) h[i] = 100.0;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[3] = {64, 64, 1}; cuuint64_t str[2] = {64 * 8, 64 * 64 * 8};
  cuuint32_t box[3] = {16, 8, 1}, es[3] = {1, 1, 1};
  CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k<<<1, 128>>>(map);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  // element (row i, col c) of box = buf[c*16 + swz(i)]... just print a few
  double sum = 0; int changed = 0;
  for (int i = 0; i < 64 * 64; ++i) { sum += h[i]; changed += (h[i] != 100.0); }
  printf("changed %d sum_delta %.3f (expect 128 changed, delta %.3f)\n", changed, sum - 100.0 * 4096, 128 * 1.5 + 127 * 128 / 2.0);
  return 0;
}
