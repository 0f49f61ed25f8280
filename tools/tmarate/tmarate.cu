// TMA request-rate probe: one elected thread per CTA issues R 1D tensor loads
// of B bytes per round into shared memory (mbarrier expect_tx / wait), 2 rounds
// in flight; reports requests/clk/SM and bytes/clk/SM for several box sizes.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tmarate/tmarate tools/tmarate/tmarate.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(32) tma_rate(const __grid_constant__ CUtensorMap map, int box, int reqs,
                                               int rounds, long long n_elems) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  if (threadIdx.x != 0) return;
  for (int b = 0; b < 2; ++b)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[b])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const uint32_t bytes = uint32_t(box) * 4u * uint32_t(reqs);
  int pos = int((blockIdx.x * 977LL * box) % (n_elems / 2)) & ~3;
  const int lim = int(n_elems - 2 * box - 8192);
  for (int r = 0; r < rounds; ++r) {
    const int b = r & 1;
    if (r >= 2) {   // wait for round r-2 on this barrier
      const uint32_t par = ((r - 2) >> 1) & 1;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su32(&bar[b])), "r"(par));
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(bytes));
    for (int q = 0; q < reqs; ++q) {
      const int c = pos;
      pos += 4100;
      if (pos > lim) pos -= lim;
      pos &= ~3;
      unsigned char* dst = sm + (size_t(b) * reqs + q) * ((box * 4 + 127) / 128 * 128);
      asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                   ::"r"(su32(dst)), "l"(&map), "r"(c), "r"(su32(&bar[b])) : "memory");
    }
  }
  for (int r = rounds - 2; r < rounds; ++r) {
    const int b = r & 1;
    const uint32_t par = (r >> 1) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(&bar[b])), "r"(par));
  }
}

int main() {
  const long long n = 1LL << 28;   // 1 GB of floats
  float* d;
  cudaMalloc(&d, n * 4);
  cudaMemset(d, 0, n * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  for (int box : {32, 140, 256}) {
    for (int ctas : {1, 2, 4, 8}) {
      CUtensorMap m;
      cuuint64_t dims[1] = {cuuint64_t(n)}, str[1] = {0};
      cuuint32_t bx[1] = {cuuint32_t(box)}, es[1] = {1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, d, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int reqs = box > 140 ? 20 : 40, rounds = 400;
      const size_t smem = size_t(2) * reqs * ((box * 4 + 127) / 128 * 128);
      cudaFuncSetAttribute(tma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      tma_rate<<<sms * ctas, 32, smem>>>(m, box, reqs, 20, n);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      tma_rate<<<sms * ctas, 32, smem>>>(m, box, reqs, rounds, n);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double cyc = ms * 1e-3 * 1.965e9;
      const double req = double(sms) * ctas * reqs * rounds;
      printf("box %3d floats (%4d B), %d CTA/SM: %.3f ms  %.4f req/clk/SM  %.1f B/clk/SM  %.0f GB/s  err=%s\n", box,
             box * 4, ctas, ms, req / cyc / sms, req * box * 4 / cyc / sms, req * box * 4 / (ms * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
