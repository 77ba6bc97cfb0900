// Variants of the CGS2 multi-dot (krylov.cu k_multidot) at the cfg3 length,
// timed back to back (tools/micro; not part of the library).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int KT = 256;
__device__ __forceinline__ void pair_range(int64_t n, int64_t& i0, int64_t& i1) {
  const int64_t chunk = (((n + gridDim.x - 1) / gridDim.x) + 1) & ~(int64_t)1;
  i0 = min(n, blockIdx.x * chunk);
  i1 = min(n, i0 + chunk);
}
template <int MJ, int UN>
__global__ void __launch_bounds__(KT) k_md(int64_t n, int m, const double* __restrict__ V, int64_t ldv,
                                           const double* __restrict__ w, double* __restrict__ partial) {
  __shared__ double red[MJ][KT / 32];
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t i0, i1;
  pair_range(n, i0, i1);
  const int64_t p1 = i0 + ((i1 - i0) & ~(int64_t)1);
  for (int j0 = 0; j0 < m; j0 += MJ) {
    const int nj = min(MJ, m - j0);
    double s[MJ];
#pragma unroll
    for (int jj = 0; jj < MJ; ++jj) s[jj] = 0.0;
    int64_t i = i0 + 2 * threadIdx.x;
    for (; i + 2 * KT * (UN - 1) < p1; i += 2 * KT * UN) {
      double2 wi[UN], v[UN][MJ];
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        wi[u] = *reinterpret_cast<const double2*>(w + i + 2 * KT * u);
#pragma unroll
        for (int jj = 0; jj < MJ; ++jj)
          v[u][jj] = jj < nj ? __ldcs(reinterpret_cast<const double2*>(V + (j0 + jj) * ldv + i + 2 * KT * u))
                             : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < UN; ++u)
#pragma unroll
        for (int jj = 0; jj < MJ; ++jj) s[jj] = fma(v[u][jj].y, wi[u].y, fma(v[u][jj].x, wi[u].x, s[jj]));
    }
    for (; i < p1; i += 2 * KT) {
      const double2 wi = *reinterpret_cast<const double2*>(w + i);
#pragma unroll
      for (int jj = 0; jj < MJ; ++jj)
        if (jj < nj) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(V + (j0 + jj) * ldv + i));
          s[jj] = fma(v.y, wi.y, fma(v.x, wi.x, s[jj]));
        }
    }
#pragma unroll
    for (int jj = 0; jj < MJ; ++jj)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s[jj] += __shfl_xor_sync(0xffffffffu, s[jj], o);
    __syncthreads();
    if (lane == 0)
#pragma unroll
      for (int jj = 0; jj < MJ; ++jj) red[jj][wp] = s[jj];
    __syncthreads();
    if (threadIdx.x < nj) {
      double t = 0.0;
      for (int q = 0; q < KT / 32; ++q) t += red[threadIdx.x][q];
      partial[(int64_t)blockIdx.x * m + j0 + threadIdx.x] = t;
    }
  }
}
template <int MJ, int UN>
void run(const char* name, int nb, int64_t n, int j, const double* V, int64_t ldv, const double* w, double* part) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) k_md<MJ, UN><<<nb, KT>>>(n, j + 1, V, ldv, w, part);
  cudaEventRecord(a);
  for (int r = 0; r < 20; ++r) k_md<MJ, UN><<<nb, KT>>>(n, j + 1, V, ldv, w, part);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double t = ms / 20;
  printf("j=%2d %-14s nb=%5d %.4f ms %.0f GB/s\n", j, name, nb, t, 8.0 * (j + 2) * n / t / 1e6);
}
int main() {
  const int64_t n = 2162601, ldv = (n + 31) / 32 * 32;
  double *V, *w, *part;
  cudaMalloc(&V, 51 * ldv * 8); cudaMalloc(&w, ldv * 8); cudaMalloc(&part, 8192 * 51 * 8);
  cudaMemset(V, 0, 51 * ldv * 8); cudaMemset(w, 0, ldv * 8);
  for (int j : {10, 20, 40}) {
    for (int nb : {592, 1184, 2368}) {
      run<8, 1>("MJ8 UN1", nb, n, j, V, ldv, w, part);
      run<8, 2>("MJ8 UN2", nb, n, j, V, ldv, w, part);
      run<4, 2>("MJ4 UN2", nb, n, j, V, ldv, w, part);
      run<16, 1>("MJ16 UN1", nb, n, j, V, ldv, w, part);
    }
  }
  return 0;
}
