// Streaming-bandwidth calibration on one B200: what a plain, perfectly
// coalesced kernel reaches for the read/write mixes of the hot kernels.
//   copy   1 read : 1 write   (the MEASURED_PEAKS.json figure's pattern)
//   k2mix  6 reads : 4 writes (config 3: u v w su sv sw -> mu sigma p_src p_snk)
//   k3mix 48 reads : 4 writes (config 4: 16 members x 3 components -> 4 outputs)
//   read   1 read : 0 writes
//   c1mix 40 reads : 3 writes at config 1's size (1024^2 points, 172 MB),
//          each launch timed alone after an L2-evicting memset (as bench.py)
// Each thread moves float4s, grid = 148 x 8 CTAs of 256 threads, grid-stride.
#include <cstdio>
#include <cuda_runtime.h>

template <int R, int W>
__global__ void __launch_bounds__(256) mix(const float4* __restrict__ in, float4* __restrict__ out,
                                           long long n4) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n4; i += (long long)gridDim.x * 256) {
    float4 v[R > 0 ? R : 1];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = __ldcs(in + r * n4 + i);
#pragma unroll
    for (int r = 0; r < R; ++r) { acc.x += v[r].x; acc.y += v[r].y; acc.z += v[r].z; acc.w += v[r].w; }
#pragma unroll
    for (int w = 0; w < W; ++w) __stcs(out + w * n4 + i, make_float4(acc.x + w, acc.y, acc.z, acc.w));
  }
  if (W == 0 && acc.x == 12345.f) out[0] = acc;
}

template <int R, int W>
void run(const char* name, float4* in, float4* out, long long n4) {
  const int grid = 148 * 8;
  for (int i = 0; i < 3; ++i) mix<R, W><<<grid, 256>>>(in, out, n4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int K = 20;
  cudaEventRecord(a);
  for (int i = 0; i < K; ++i) mix<R, W><<<grid, 256>>>(in, out, n4);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bytes = double(R + W) * n4 * 16;
  printf("%-6s %2d:%d  %.3f ms  %.0f GB/s\n", name, R, W, ms / K, bytes / (ms / K * 1e-3) / 1e9);
}

int main() {
  const long long n4 = (134217728ll / 4);   // 512^3 floats per array
  float4 *in, *out;
  cudaMalloc(&in, 48ll * n4 * 16 / 8 + 6 * n4 * 16);  // enough for 6 full arrays
  cudaMalloc(&out, 4 * n4 * 16);
  cudaMemset(in, 0, 6 * n4 * 16); cudaMemset(out, 0, 4 * n4 * 16);
  run<1, 1>("copy", in, out, n4);
  run<1, 0>("read", in, out, n4);
  run<6, 4>("k2mix", in, out, n4);
  run<6, 0>("k2rd", in, out, n4);
  run<0, 4>("k2wr", in, out, n4);
  // k3 mix on a 1/8 slab so 48 arrays fit: n4/8 elements per array
  run<48, 4>("k3mix", in, out, n4 / 8);
  // config-1 sized: the small-problem floor (launch ramp + tail) for 172 MB
  {
    const long long c4 = 1024ll * 1024 / 4;
    void* flush = nullptr;
    cudaMalloc(&flush, size_t(256) << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int grid_mul : {1, 2, 4, 8}) {
      float best = 1e9f, sum = 0.f;
      const int K = 20;
      for (int i = 0; i < K + 3; ++i) {
        cudaMemsetAsync(flush, i, size_t(256) << 20);
        cudaEventRecord(a);
        mix<40, 3><<<148 * grid_mul, 256>>>(in, out, c4);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (i >= 3) { sum += ms; best = best < ms ? best : ms; }
      }
      const double bytes = 43.0 * c4 * 16;
      printf("c1mix 40:3 grid 148x%d  avg %.1f us (%.0f GB/s)  best %.1f us\n", grid_mul, sum / K * 1e3,
             bytes / (sum / K * 1e-3) / 1e9, best * 1e3);
    }
  }
  return 0;
}
