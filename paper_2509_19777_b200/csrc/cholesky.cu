// Coarse solve by a dense Cholesky factor S = L L^T (coarse_solver = 1): the
// literal reading of SURVEY §8(a) a3 / north_star (4) -- factor once, apply by
// a forward and a backward triangular solve per GMRES iteration.
//
// Storage: the coarse batch's packed lower 64-tiles (one SPD block S), factored
// in place (right-looking tiled Cholesky; the tile products run on the FP64
// tensor cores); the inverse of every 64x64 diagonal factor block L_kk (and its
// transpose) is kept so that each diagonal step of the solves is a product.
//
// Solves: one persistent kernel per sweep.  Block rows are owned round-robin
// by the CTAs (all co-resident); a CTA walks its rows in dependency order and
// consumes the off-diagonal tiles as soon as the block it needs is published
// (per-row flags stamped with the apply's epoch, release/acquire at gpu scope),
// so only the chain of diagonal steps is sequential.  The default coarse
// solver applies the explicit S^-1 instead (half the bytes, no chain): see
// DESIGN.md §6.
#include <algorithm>
#include <climits>

#include "dmma.cuh"
#include "kernels.cuh"

namespace hplmm {

__device__ __forceinline__ int64_t ctid(int64_t I, int64_t J) { return I * (I + 1) / 2 + J; }

// ---- factorisation ---------------------------------------------------------
// T_kk = L_kk L_kk^T in shared memory; L_kk back into the tile (upper part
// zeroed), L_kk^-1 and its transpose into linv / linvT.
__global__ void __launch_bounds__(256) k_chol_diag(int k, double* tiles, double* linv,
                                                   double* linvT, int32_t* err) {
  extern __shared__ double ch_sm[];
  double* a = ch_sm;
  double* x = ch_sm + TILE;
  __shared__ int bad;
  double* T = tiles + ctid(k, k) * TILE;
  for (int e = threadIdx.x; e < TILE; e += blockDim.x) a[e] = T[e];
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < TB; ++j) {
    const double d = a[j * TB + j];
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) bad = 1;
      break;
    }
    const double ljj = sqrt(d);
    __syncthreads();
    if (threadIdx.x == 0) a[j * TB + j] = ljj;
    for (int i = j + 1 + threadIdx.x; i < TB; i += blockDim.x) a[j * TB + i] /= ljj;
    __syncthreads();
    // trailing lower update: a(i, c) -= l(i, j) l(c, j), j < c <= i
    const int m = TB - 1 - j;
    for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
      const int i = j + 1 + t % m, c = j + 1 + t / m;
      if (c <= i) a[c * TB + i] -= a[j * TB + i] * a[j * TB + c];
    }
    __syncthreads();
  }
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) atomicMin(err, k);
    return;
  }
  // column c of L^-1 by forward substitution (thread per column)
  if (threadIdx.x < TB) {
    const int c = threadIdx.x;
    for (int r = 0; r < TB; ++r) x[c * TB + r] = 0.0;
    x[c * TB + c] = 1.0 / a[c * TB + c];
    for (int r = c + 1; r < TB; ++r) {
      double s = 0.0;
      for (int m2 = c; m2 < r; ++m2) s += a[m2 * TB + r] * x[c * TB + m2];
      x[c * TB + r] = -s / a[r * TB + r];
    }
  }
  __syncthreads();
  double* Li = linv + (int64_t)k * TILE;
  double* LiT = linvT + (int64_t)k * TILE;
  for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
    const int c = e >> 6, r = e & 63;
    T[e] = r >= c ? a[e] : 0.0;
    Li[e] = x[e];                 // (r, c) at c*64 + r
    LiT[e] = x[r * TB + c];       // transpose
  }
}

// T_ik <- T_ik L_kk^-T  (i > k)
__global__ void __launch_bounds__(256) k_chol_panel(int k, int nb, double* tiles,
                                                    const double* linv) {
  const int i = k + 1 + blockIdx.x;
  if (i >= nb) return;
  extern __shared__ double ch_sm[];
  double* As = ch_sm;
  double* Bs = ch_sm + TILE;
  double* T = tiles + ctid(i, k) * TILE;
  const double* Li = linv + (int64_t)k * TILE;
  for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
    As[e] = T[e];     // A(r, m) = T(r, m) at m*64 + r
    Bs[e] = Li[e];    // B(m, c) = Li(c, m) at m*64 + c
  }
  __syncthreads();
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  tile_dmma(As, TB, Bs, TB, TB, acc);
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    int r, c;
    dmma_rc(q, r, c);
    T[c * TB + r] = acc[q];
  }
}

// trailing update T_ij -= T_ik T_jk^T for k < j <= i (blockIdx -> (i, j))
__global__ void __launch_bounds__(256) k_chol_update(int k, int nb, double* tiles) {
  const int64_t t = blockIdx.x;
  const int a = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  int aa = a;
  while ((int64_t)(aa + 1) * (aa + 2) / 2 <= t) ++aa;
  while ((int64_t)aa * (aa + 1) / 2 > t) --aa;
  const int b = (int)(t - (int64_t)aa * (aa + 1) / 2);
  const int i = k + 1 + aa, j = k + 1 + b;
  if (i >= nb) return;
  extern __shared__ double ch_sm[];
  double* As = ch_sm;
  double* Bs = ch_sm + TILE;
  const double* Ti = tiles + ctid(i, k) * TILE;
  const double* Tj = tiles + ctid(j, k) * TILE;
  for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
    As[e] = Ti[e];    // A(r, m) = L_ik(r, m)
    Bs[e] = Tj[e];    // B(m, c) = L_jk(c, m) at m*64 + c
  }
  __syncthreads();
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  tile_dmma(As, TB, Bs, TB, TB, acc);
  double* T = tiles + ctid(i, j) * TILE;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    int r, c;
    dmma_rc(q, r, c);
    T[c * TB + r] -= acc[q];
  }
}

void launch_chol_factor(const DevBatch& b, double* linv, double* linvT, cudaStream_t st) {
  const int nb = b.max_nb;
  const size_t sm = 2 * TILE * sizeof(double);
  set_max_dynamic_smem((const void*)k_chol_diag, sm);
  set_max_dynamic_smem((const void*)k_chol_panel, sm);
  set_max_dynamic_smem((const void*)k_chol_update, sm);
  for (int k = 0; k < nb; ++k) {
    k_chol_diag<<<1, 256, sm, st>>>(k, b.tiles, linv, linvT, b.err);
    if (k + 1 < nb) {
      k_chol_panel<<<nb - k - 1, 256, sm, st>>>(k, nb, b.tiles, linv);
      const int64_t m = nb - k - 1;
      k_chol_update<<<(unsigned)(m * (m + 1) / 2), 256, sm, st>>>(k, nb, b.tiles);
    }
  }
}

// ---- triangular solves -----------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// columns 2l, 2l+1 of the per-lane partial column sums cp[c] (recursive halving)
__device__ __forceinline__ double2 transpose_reduce(double (&cp)[64], int lane) {
#pragma unroll
  for (int h = 32, o = 16; h >= 2; h >>= 1, o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int k2 = 0; k2 < h; ++k2) {
      double send = up ? cp[k2] : cp[h + k2];
      double keep = up ? cp[h + k2] : cp[k2];
      cp[k2] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return make_double2(cp[0], cp[1]);
}

// y(2l, 2l+1) += M v with M a col-major 64x64 tile, v held as lane pairs
__device__ __forceinline__ void tile_mv(const double* __restrict__ M, double2 v, int lane,
                                        double& y0, double& y1) {
  const double2* A = reinterpret_cast<const double2*>(M) + lane;
#pragma unroll 16
  for (int c = 0; c < TB; ++c) {
    const double2 a = __ldcs(A + c * (TB / 2));
    const double x = __shfl_sync(0xffffffffu, (c & 1) ? v.y : v.x, c >> 1);
    y0 = fma(a.x, x, y0);
    y1 = fma(a.y, x, y1);
  }
}

constexpr int TR_WARPS = 8;

__device__ __forceinline__ void tr_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
// whole 64x64 tile -> shared memory (same col-major layout)
__device__ __forceinline__ void tr_prefetch(double* dst, const double* src) {
  for (int e = threadIdx.x; e < TILE / 2; e += blockDim.x) tr_cp16(dst + 2 * e, src + 2 * e);
}
// y(2l, 2l+1) += M v, M a col-major 64x64 tile in shared memory
__device__ __forceinline__ void tile_mv_s(const double* M, double2 v, int lane, double& y0,
                                          double& y1) {
  const double2* A = reinterpret_cast<const double2*>(M) + lane;
#pragma unroll 16
  for (int c = 0; c < TB; ++c) {
    const double2 a = A[c * (TB / 2)];
    const double x = __shfl_sync(0xffffffffu, (c & 1) ? v.y : v.x, c >> 1);
    y0 = fma(a.x, x, y0);
    y1 = fma(a.y, x, y1);
  }
}

// The chain of the triangular sweeps runs through the diagonal: row I waits
// for block I-1 (forward) / I+1 (backward) last.  The two tiles that step
// needs -- the adjacent off-diagonal tile and the inverted diagonal block --
// do not depend on the sweep, so they are copied into shared memory (cp.async)
// before the row starts, and the wait-to-publish path reads only shared
// memory.  The other blocks of the row are consumed by all warps as they are
// published (farthest first).

// forward: z_I = L_II^-1 (r_I - sum_{J<I} L_IJ z_J), rows ascending
__global__ void __launch_bounds__(32 * TR_WARPS, 1)
    k_trsv_fwd(int nb, const double* __restrict__ tiles, const double* __restrict__ linv,
               const double* __restrict__ r, double* z, int* flag, int epoch) {
  extern __shared__ __align__(16) double trs[];   // [tile (I, I-1) | L_II^-1]
  __shared__ double red[TR_WARPS][TB];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int I = blockIdx.x; I < nb; I += gridDim.x) {
    if (I > 0) tr_prefetch(trs, tiles + ctid(I, I - 1) * TILE);
    tr_prefetch(trs + TILE, linv + (int64_t)I * TILE);
    asm volatile("cp.async.commit_group;" ::: "memory");
    double y0 = 0.0, y1 = 0.0;
    for (int J = w; J < I - 1; J += TR_WARPS) {
      if (lane == 0)
        while (ld_acquire(flag + J) < epoch) {
        }
      __syncwarp();
      const double2 zj = __ldcg(reinterpret_cast<const double2*>(z + (int64_t)J * TB) + lane);
      tile_mv(tiles + ctid(I, J) * TILE, zj, lane, y0, y1);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (w == 0 && I > 0) {   // the chain step
      if (lane == 0)
        while (ld_acquire(flag + I - 1) < epoch) {
        }
      __syncwarp();
      const double2 zj = __ldcg(reinterpret_cast<const double2*>(z + (int64_t)(I - 1) * TB) + lane);
      tile_mv_s(trs, zj, lane, y0, y1);
    }
    red[w][2 * lane] = y0;
    red[w][2 * lane + 1] = y1;
    __syncthreads();
    if (w == 0) {
      double2 v = reinterpret_cast<const double2*>(r + (int64_t)I * TB)[lane];
#pragma unroll
      for (int q = 0; q < TR_WARPS; ++q) {
        v.x -= red[q][2 * lane];
        v.y -= red[q][2 * lane + 1];
      }
      double o0 = 0.0, o1 = 0.0;
      tile_mv_s(trs + TILE, v, lane, o0, o1);
      __stcg(reinterpret_cast<double2*>(z + (int64_t)I * TB) + lane, make_double2(o0, o1));
      // bar.warp.sync orders the lanes' stores before lane 0's (cumulative) release
      __syncwarp();
      if (lane == 0) st_release(flag + I, epoch);
    }
    __syncthreads();
  }
}

// backward: y_I = L_II^-T (z_I - sum_{J>I} L_JI^T y_J), rows descending
__global__ void __launch_bounds__(32 * TR_WARPS, 1)
    k_trsv_bwd(int nb, const double* __restrict__ tiles, const double* __restrict__ linvT,
               const double* __restrict__ z, double* y, int* flag, int epoch) {
  extern __shared__ __align__(16) double trs[];   // [tile (I+1, I) | L_II^-T]
  __shared__ double red[TR_WARPS][TB];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this CTA's rows, descending
  const int first = blockIdx.x;
  if (first >= nb) return;
  const int last = first + ((nb - 1 - first) / gridDim.x) * gridDim.x;
  for (int I = last; I >= first; I -= gridDim.x) {
    if (I + 1 < nb) tr_prefetch(trs, tiles + ctid(I + 1, I) * TILE);
    tr_prefetch(trs + TILE, linvT + (int64_t)I * TILE);
    asm volatile("cp.async.commit_group;" ::: "memory");
    double cp[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) cp[c] = 0.0;
    // farthest blocks first; the chain block J = I + 1 comes last (below)
    for (int J = nb - 1 - w; J > I + 1; J -= TR_WARPS) {
      if (lane == 0)
        while (ld_acquire(flag + J) < epoch) {
        }
      __syncwarp();
      const double2 yj = __ldcg(reinterpret_cast<const double2*>(y + (int64_t)J * TB) + lane);
      const double2* A = reinterpret_cast<const double2*>(tiles + ctid(J, I) * TILE) + lane;
#pragma unroll
      for (int c = 0; c < TB; ++c) {
        const double2 a = __ldcs(A + c * (TB / 2));   // rows 2l, 2l+1 of column c
        cp[c] = fma(a.x, yj.x, fma(a.y, yj.y, cp[c]));
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (w == 0 && I + 1 < nb) {   // the chain step
      if (lane == 0)
        while (ld_acquire(flag + I + 1) < epoch) {
        }
      __syncwarp();
      const double2 yj = __ldcg(reinterpret_cast<const double2*>(y + (int64_t)(I + 1) * TB) + lane);
      const double2* A = reinterpret_cast<const double2*>(trs) + lane;
#pragma unroll
      for (int c = 0; c < TB; ++c) {
        const double2 a = A[c * (TB / 2)];
        cp[c] = fma(a.x, yj.x, fma(a.y, yj.y, cp[c]));
      }
    }
    const double2 s = transpose_reduce(cp, lane);   // columns 2l, 2l+1
    red[w][2 * lane] = s.x;
    red[w][2 * lane + 1] = s.y;
    __syncthreads();
    if (w == 0) {
      double2 v = reinterpret_cast<const double2*>(z + (int64_t)I * TB)[lane];
#pragma unroll
      for (int q = 0; q < TR_WARPS; ++q) {
        v.x -= red[q][2 * lane];
        v.y -= red[q][2 * lane + 1];
      }
      double o0 = 0.0, o1 = 0.0;
      tile_mv_s(trs + TILE, v, lane, o0, o1);
      __stcg(reinterpret_cast<double2*>(y + (int64_t)I * TB) + lane, make_double2(o0, o1));
      // bar.warp.sync orders the lanes' stores before lane 0's (cumulative) release
      __syncwarp();
      if (lane == 0) st_release(flag + I, epoch);
    }
    __syncthreads();
  }
}

void launch_chol_solve(const DevBatch& b, const double* linv, const double* linvT,
                       const double* r, double* zbuf, double* y, int* flags_fwd, int* flags_bwd,
                       int epoch, cudaStream_t st) {
  const int nb = b.max_nb;
  if (nb <= 0) return;
  // one CTA per SM at most, and a COOPERATIVE launch: the CTAs wait on each
  // other's rows, so they must all be resident -- the launch fails (loudly,
  // checked by the caller) instead of hanging when co-residency is impossible
  // (MPS SM limits, concurrent kernels holding SMs)
  int grid = std::min(nb, device_sm_count());
  set_max_dynamic_smem((const void*)k_trsv_fwd, 2 * TILE * 8);
  set_max_dynamic_smem((const void*)k_trsv_bwd, 2 * TILE * 8);
  const double* tiles = b.tiles;
  void* af[] = {(void*)&nb, (void*)&tiles, (void*)&linv, (void*)&r, (void*)&zbuf, (void*)&flags_fwd,
                (void*)&epoch};
  cudaLaunchCooperativeKernel((const void*)k_trsv_fwd, dim3(grid), dim3(32 * TR_WARPS), af,
                              2 * TILE * 8, st);
  void* ab[] = {(void*)&nb, (void*)&tiles, (void*)&linvT, (void*)&zbuf, (void*)&y, (void*)&flags_bwd,
                (void*)&epoch};
  cudaLaunchCooperativeKernel((const void*)k_trsv_bwd, dim3(grid), dim3(32 * TR_WARPS), ab,
                              2 * TILE * 8, st);
}

}  // namespace hplmm
