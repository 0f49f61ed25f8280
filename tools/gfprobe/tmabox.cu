// TMA box-shape probe: one CTA loads one box of a 3D fp32 tensor.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_2510_01190_b200/csrc/tma.cuh"
using namespace divuq;
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap map, int x, int y, unsigned bytes, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
    mbar_expect_tx(bar, bytes);
    tma_load_3d(sm, &map, bar, x, y, 1);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  if (threadIdx.x == 0) out[0] = reinterpret_cast<float*>(sm)[0];
}

int main() {
  float* d; float* o;
  cudaMalloc(&d, 64 * 16 * 4 * 4); cudaMalloc(&o, 4);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  const int shapes[][4] = {{72, 20, -4, -2}, {68, 20, -4, -2}, {64, 16, 0, -2}, {64, 16, -4, 0},
                           {64, 16, -2, 0}};
  for (auto& s : shapes) {
    for (int promo = 0; promo < 2; ++promo) {
      CUtensorMap map{};
      const cuuint64_t dims[3] = {64, 16, 4};
      const cuuint64_t strides[2] = {64 * 4, 64 * 16 * 4};
      const cuuint32_t box[3] = {cuuint32_t(s[0]), cuuint32_t(s[1]), 1}, es[3] = {1, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      k<<<1, 32, 65536 + 64>>>(map, s[2], s[3], unsigned(s[0] * s[1] * 4), o);
      cudaError_t e = cudaDeviceSynchronize();
      printf("box %dx%d at (%d,%d) promo %d: encode %d, %s\n", s[0], s[1], s[2], s[3], promo, int(r),
             cudaGetErrorString(e));
      if (e != cudaSuccess) { cudaDeviceReset(); cudaMalloc(&d, 64 * 16 * 4 * 4); cudaMalloc(&o, 4);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64); }
    }
  }
  return 0;
}
