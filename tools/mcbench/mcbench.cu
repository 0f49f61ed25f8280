// Stand-alone timing harness for the MC kernel variants (config 2 shape):
// nvcc -DVARIANT... includes the library TU and calls the C ABI directly.
#include "../../paper_2510_01190_b200/csrc/capi.cu"
#include <cstdio>
#include <vector>
#include <random>

int main(int argc, char** argv) {
  const int64_t nx = 256, ny = 256, n = nx * ny, ns = argc > 1 ? atoll(argv[1]) : 2000;
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<double> h(4 * n);
  for (int64_t i = 0; i < 2 * n; ++i) h[i] = 2.0 * U(g) - 1.0;
  for (int64_t i = 2 * n; i < 4 * n; ++i) h[i] = 0.05 + 0.25 * U(g);
  double *d, *out, *scratch; int* err;
  cudaMalloc(&d, 4 * n * 8); cudaMalloc(&out, 2 * n * 8); cudaMalloc(&err, 4);
  cudaMemcpy(d, h.data(), 4 * n * 8, cudaMemcpyHostToDevice); cudaMemset(err, 0, 4);
  cudaMalloc(&scratch, divuq_mc_scratch_bytes(nx, 0, ny, ns));
  auto run = [&]() {
    int r = divuq_mc_divergence2d_f64(d, d + n, d + 2 * n, d + 3 * n, nx, ny, 1.0, 1.0, ns, 12345,
                                      0, ny, out, out + n, scratch, err, nullptr);
    if (r) { printf("err %d\n", r); exit(1); }
  };
  for (int i = 0; i < 3; ++i) run();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int K = 20;
  cudaEventRecord(a);
  for (int i = 0; i < K; ++i) run();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  std::vector<double> o(2 * n);
  cudaMemcpy(o.data(), out, 2 * n * 8, cudaMemcpyDeviceToHost);
  double cs = 0; for (auto x : o) cs += x;
  printf("%s ms/step %.4f  Gvs/s %.2f  checksum %.17g\n", argc > 2 ? argv[2] : "", ms / K,
         double(n) * ns / (ms / K * 1e-3) / 1e9, cs);
  return 0;
}
