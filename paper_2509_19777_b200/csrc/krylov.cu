// Arnoldi / GMRES vector kernels (sm_100a, fp64): fused multi-dot, multi-axpy
// with an optional fused norm, all with deterministic two-stage reductions
// (fixed block->range mapping, fixed-order final sums).  CGS2 (R22) uses
// multidot + update twice per Arnoldi step.  Measured and dropped: fusing the
// first update with the second multidot (one DRAM pass over V fewer; the
// element's V values re-read from L1/L2 for the dots) was 0.04 ms per
// iteration SLOWER at cfg3 -- the 2 x 50 per-thread accumulators / operands
// take 255 registers, one CTA per SM, and the per-element FMA chain then
// stalls the stream.
#include "kernels.cuh"

namespace hplmm {

constexpr int KT = 256;

int krylov_blocks(int64_t n) {
  int64_t b = (n + 4 * KT - 1) / (4 * KT);
  if (b > 148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  return (int)b;
}

// multi-dot blocks: half as many, each over twice the range (fewer per-group
// block reductions per byte; cfg3 j = 20: 5.6 vs 5.5 TB/s, tools/micro)
static int md_blocks(int64_t n) {
  int64_t b = (n + 8 * KT - 1) / (8 * KT);
  if (b > 148 * 4) b = 148 * 4;
  if (b < 1) b = 1;
  return (int)b;
}

// The partial-sum buffer of a handle: up to 513 (= max restart + 1) partial
// vectors of krylov_blocks(n) entries, then a completion counter (zeroed once
// at allocation, reset by the last block of every launch).
int64_t krylov_partial_doubles(int64_t n) { return (int64_t)krylov_blocks(n) * 513 + 8; }
static unsigned* krylov_counter(double* partial, int64_t n) {
  return reinterpret_cast<unsigned*>(partial + (int64_t)krylov_blocks(n) * 513);
}

// Last-block completion: every block publishes its partials, then takes a
// ticket; the block drawing the last ticket sums the partials in a fixed
// order (so the result is bitwise the separate k_final_sum's) and resets the
// counter.  Saves one launch per reduction (and its ~10-30 us of latency).
__device__ __forceinline__ bool last_block(unsigned* counter) {
  __shared__ unsigned ticket;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(counter, 1u);
  __syncthreads();
  const bool last = ticket == gridDim.x - 1;
  if (last) __threadfence();
  return last;
}

// out[j] = sum_b partial[j nb + b], j < m: warp per j, lane-strided partial
// sums in b order, then a fixed butterfly
__device__ __forceinline__ void final_sums(int nb, int m, const double* partial, double* out) {
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = wp; j < m; j += blockDim.x >> 5) {
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += __ldcg(partial + (int64_t)j * nb + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[j] = s;
  }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < KT / 32; ++i) s += red[i];
  return s;  // valid in thread 0
}

// partial[b*m + j] = sum_{i in block b's range} V[j][i] w[i].  MD_J basis
// vectors per pass share one read of w; per vector the summation order is
// fixed (per-thread strided fma, warp butterfly, warps in order).
constexpr int MD_J = 8;
// block ranges: even-sized (element pairs), so that every block's first
// element is 16-byte aligned (ldv is a multiple of 32)
__device__ __forceinline__ void pair_range(int64_t n, int64_t& i0, int64_t& i1) {
  const int64_t chunk = (((n + gridDim.x - 1) / gridDim.x) + 1) & ~(int64_t)1;
  i0 = min(n, blockIdx.x * chunk);
  i1 = min(n, i0 + chunk);
}

// cnt: if non-null, the vector count is *cnt + 1 (the Arnoldi step index j
// read on the device, for the graph-captured GMRES cycle) instead of m
__device__ __forceinline__ int vec_count(int m, const int* cnt) { return cnt ? *cnt + 1 : m; }

__global__ void __launch_bounds__(KT) k_multidot(int64_t n, int m, const double* __restrict__ V,
                                                 int64_t ldv, const double* __restrict__ w,
                                                 double* __restrict__ partial,
                                                 const int* __restrict__ cnt,
                                                 double* __restrict__ out,
                                                 unsigned* __restrict__ counter) {
  __shared__ double red[MD_J][KT / 32];
  m = vec_count(m, cnt);
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t i0, i1;
  pair_range(n, i0, i1);
  const int64_t p1 = i0 + ((i1 - i0) & ~(int64_t)1);   // end of the paired part
  for (int j0 = 0; j0 < m; j0 += MD_J) {
    const int nj = min(MD_J, m - j0);
    double s[MD_J];
#pragma unroll
    for (int jj = 0; jj < MD_J; ++jj) s[jj] = 0.0;
    // two elements per thread per step (128-bit loads)
    for (int64_t i = i0 + 2 * threadIdx.x; i < p1; i += 2 * KT) {
      const double2 wi = *reinterpret_cast<const double2*>(w + i);
#pragma unroll
      for (int jj = 0; jj < MD_J; ++jj)
        if (jj < nj) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(V + (j0 + jj) * ldv + i));
          s[jj] = fma(v.y, wi.y, fma(v.x, wi.x, s[jj]));
        }
    }
    if (p1 < i1 && threadIdx.x == 0) {
      const double wi = w[p1];
#pragma unroll
      for (int jj = 0; jj < MD_J; ++jj)
        if (jj < nj) s[jj] = fma(V[(j0 + jj) * ldv + p1], wi, s[jj]);
    }
#pragma unroll
    for (int jj = 0; jj < MD_J; ++jj) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s[jj] += __shfl_xor_sync(0xffffffffu, s[jj], o);
    }
    __syncthreads();
    if (lane == 0)
#pragma unroll
      for (int jj = 0; jj < MD_J; ++jj) red[jj][wp] = s[jj];
    __syncthreads();
    if (threadIdx.x < nj) {
      double t = 0.0;
      for (int q = 0; q < KT / 32; ++q) t += red[threadIdx.x][q];
      partial[(int64_t)(j0 + threadIdx.x) * gridDim.x + blockIdx.x] = t;
    }
  }
  if (last_block(counter)) {
    final_sums(gridDim.x, m, partial, out);
    if (threadIdx.x == 0) *counter = 0u;
  }
}

void launch_multidot(int64_t n, int m, const double* V, int64_t ldv, const double* w,
                     double* partial, double* out, cudaStream_t st, const int* cnt) {
  // with a device count, m is the largest count; partial holds (count) x nb
  // entries, summed by the last block
  const int nb = md_blocks(n);
  k_multidot<<<nb, KT, 0, st>>>(n, m, V, ldv, w, partial, cnt, out, krylov_counter(partial, n));
}

// w -= sum_j V[j] h[j]   (+ partial ||w||^2 per block); per element the
// j-order of the update is fixed; two elements per thread (128-bit loads)
__global__ void __launch_bounds__(KT) k_update(int64_t n, int m, const double* __restrict__ V,
                                               int64_t ldv, const double* __restrict__ h,
                                               double* __restrict__ w, double* __restrict__ partial,
                                               const int* __restrict__ cnt,
                                               double* __restrict__ out_norm2,
                                               unsigned* __restrict__ counter) {
  __shared__ double hs[513];
  __shared__ double red[KT / 32];
  m = vec_count(m, cnt);
  for (int j = threadIdx.x; j < m; j += KT) hs[j] = h[j];
  __syncthreads();
  int64_t i0, i1;
  pair_range(n, i0, i1);
  const int64_t p1 = i0 + ((i1 - i0) & ~(int64_t)1);
  double s = 0.0;
  for (int64_t i = i0 + 2 * threadIdx.x; i < p1; i += 2 * KT) {
    double2 acc = *reinterpret_cast<const double2*>(w + i);
    int j = 0;
    for (; j + 3 < m; j += 4) {
      const double2 v0 = __ldcs(reinterpret_cast<const double2*>(V + j * ldv + i));
      const double2 v1 = __ldcs(reinterpret_cast<const double2*>(V + (j + 1) * ldv + i));
      const double2 v2 = __ldcs(reinterpret_cast<const double2*>(V + (j + 2) * ldv + i));
      const double2 v3 = __ldcs(reinterpret_cast<const double2*>(V + (j + 3) * ldv + i));
      acc.x = fma(-v0.x, hs[j], acc.x);
      acc.y = fma(-v0.y, hs[j], acc.y);
      acc.x = fma(-v1.x, hs[j + 1], acc.x);
      acc.y = fma(-v1.y, hs[j + 1], acc.y);
      acc.x = fma(-v2.x, hs[j + 2], acc.x);
      acc.y = fma(-v2.y, hs[j + 2], acc.y);
      acc.x = fma(-v3.x, hs[j + 3], acc.x);
      acc.y = fma(-v3.y, hs[j + 3], acc.y);
    }
    for (; j < m; ++j) {
      const double2 v = __ldcs(reinterpret_cast<const double2*>(V + j * ldv + i));
      acc.x = fma(-v.x, hs[j], acc.x);
      acc.y = fma(-v.y, hs[j], acc.y);
    }
    *reinterpret_cast<double2*>(w + i) = acc;
    s = fma(acc.x, acc.x, s);
    s = fma(acc.y, acc.y, s);
  }
  if (p1 < i1 && threadIdx.x == 0) {
    double acc = w[p1];
    for (int j = 0; j < m; ++j) acc = fma(-V[j * ldv + p1], hs[j], acc);
    w[p1] = acc;
    s = fma(acc, acc, s);
  }
  if (partial) {
    double t = block_sum(s, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
    if (last_block(counter)) {
      final_sums(gridDim.x, 1, partial, out_norm2);
      if (threadIdx.x == 0) *counter = 0u;
    }
  }
}

void launch_update(int64_t n, int m, const double* V, int64_t ldv, const double* h, double* w,
                   double* partial, double* out_norm2, cudaStream_t st, const int* cnt) {
  int nb = krylov_blocks(n);
  k_update<<<nb, KT, 0, st>>>(n, m, V, ldv, h, w, out_norm2 ? partial : nullptr, cnt, out_norm2,
                              out_norm2 ? krylov_counter(partial, n) : nullptr);
}

__global__ void __launch_bounds__(KT) k_norm2(int64_t n, const double* __restrict__ x,
                                              double* __restrict__ partial,
                                              double* __restrict__ out,
                                              unsigned* __restrict__ counter) {
  __shared__ double red[KT / 32];
  int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  int64_t i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  double s = 0.0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += KT) s = fma(x[i], x[i], s);
  double t = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    final_sums(gridDim.x, 1, partial, out);
    if (threadIdx.x == 0) *counter = 0u;
  }
}

void launch_norm2(int64_t n, const double* x, double* partial, double* out, cudaStream_t st) {
  int nb = krylov_blocks(n);
  k_norm2<<<nb, KT, 0, st>>>(n, x, partial, out, krylov_counter(partial, n));
}

// y = x * s  (invert: y = x / sqrt(s))
__global__ void k_scale(int64_t n, const double* __restrict__ x, const double* __restrict__ s,
                        int invert, double* __restrict__ y) {
  double f = invert ? 1.0 / sqrt(s[0]) : s[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * f;
}

void launch_scale(int64_t n, const double* x, const double* s_dev, int invert, double* y,
                  cudaStream_t st) {
  k_scale<<<krylov_blocks(n), KT, 0, st>>>(n, x, s_dev, invert, y);
}

__global__ void k_combine_basis(int64_t n, int m, const double* __restrict__ V, int64_t ldv,
                                const double* __restrict__ y, double* __restrict__ x) {
  __shared__ double ys[513];
  for (int j = threadIdx.x; j < m; j += blockDim.x) ys[j] = y[j];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = x[i];
    for (int j = 0; j < m; ++j) acc = fma(V[j * ldv + i], ys[j], acc);
    x[i] = acc;
  }
}

void launch_combine_basis(int64_t n, int m, const double* V, int64_t ldv, const double* y,
                          double* x, cudaStream_t st) {
  k_combine_basis<<<krylov_blocks(n), KT, 0, st>>>(n, m, V, ldv, y, x);
}

__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

void launch_axpy(int64_t n, double a, const double* x, double* y, cudaStream_t st) {
  k_axpy<<<krylov_blocks(n), KT, 0, st>>>(n, a, x, y);
}

}  // namespace hplmm
