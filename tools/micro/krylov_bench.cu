// Micro-benchmark of the CGS2 kernels (krylov.cu) at the cfg3 vector length:
// k_multidot / k_update with the vector count passed by value or read on the
// device (the graph-captured path).  Build and run on a B200:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2509_19777_b200/csrc \
//        tools/micro/krylov_bench.cu paper_2509_19777_b200/csrc/krylov.cu -o /tmp/kb && /tmp/kb
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "kernels.cuh"

using namespace hplmm;

int main() {
  const int64_t n = 2162601, ldv = (n + 31) / 32 * 32;
  const int m = 50;
  double *V, *w, *partial, *hb;
  int* cnt;
  cudaMalloc(&V, (size_t)(m + 1) * ldv * 8);
  cudaMalloc(&w, (size_t)ldv * 8);
  cudaMalloc(&partial, (size_t)krylov_partial_doubles(n) * 8);
  cudaMemset(partial, 0, (size_t)krylov_partial_doubles(n) * 8);
  cudaMalloc(&hb, (size_t)(2 * (m + 1) + 8) * 8);
  cudaMalloc(&cnt, 4);
  cudaMemset(V, 0, (size_t)(m + 1) * ldv * 8);
  cudaMemset(w, 0, (size_t)ldv * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int j : {1, 10, 20, 40}) {
    const int jm1 = j - 1;
    cudaMemcpy(cnt, &jm1, 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
      const int* c = mode ? cnt : nullptr;
      for (int rep = 0; rep < 3; ++rep) launch_multidot(n, mode ? m : j, V, ldv, w, partial, hb, 0, c);
      cudaEventRecord(a);
      for (int rep = 0; rep < 20; ++rep) launch_multidot(n, mode ? m : j, V, ldv, w, partial, hb, 0, c);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double t = ms / 20, bytes = 8.0 * (j + 1) * n;
      cudaEventRecord(a);
      for (int rep = 0; rep < 20; ++rep) launch_update(n, mode ? m : j, V, ldv, hb, w, partial, hb + 2 * (m + 1), 0, c);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms2;
      cudaEventElapsedTime(&ms2, a, b);
      const double t2 = ms2 / 20, bytes2 = 8.0 * (j + 2) * n;
      printf("j=%2d %s multidot %.4f ms %.0f GB/s | update %.4f ms %.0f GB/s\n", j,
             mode ? "device-count" : "host-count  ", t, bytes / t / 1e6, t2, bytes2 / t2 / 1e6);
    }
  }
  return 0;
}
