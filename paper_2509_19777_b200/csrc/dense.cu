// Batched dense subdomain operators on packed lower 64x64 tiles (sm_100a, fp64).
//
// Exact local solves of the additive-Schwarz smoothers M_zeta and M_g
// (eq:Mg_Mz; local LU "precomputed" per P:739) and of the coarse
// block S (eq:mg_struct with R16/R17).  Each SPD block is inverted once at
// setup with the block sweep operator (symmetric Gauss-Jordan, no pivoting:
// SPD) and stored as packed lower tiles; every apply is then a symmetric
// matrix-vector product that streams the lower triangle ONCE (n^2/2 doubles),
// i.e. half the bytes of a forward+backward triangular-solve pair over a
// Cholesky factor, with no sequential dependency.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "kernels.cuh"
#include "dmma.cuh"
#include "tma.cuh"

#include <map>
#include <mutex>
#include <utility>

namespace hplmm {

void set_max_dynamic_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, func}];
  if (bytes > have) {
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    have = bytes;
  }
}

int device_sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int& n = cache[dev];
  if (n == 0) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// ---------------------------------------------------------------------------
// 64x64x64 fp64 tile product core (256 threads, 4x4 outputs each):
//   acc[i][j] += sum_k As[k*64 + r0+i] * Bs[k*64 + c0+j]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tile_mma(const double* __restrict__ As,
                                         const double* __restrict__ Bs, double acc[4][4],
                                         int r0, int c0) {
#pragma unroll 8
  for (int k = 0; k < TB; ++k) {
    double2 a01 = *reinterpret_cast<const double2*>(As + k * TB + r0);
    double2 a23 = *reinterpret_cast<const double2*>(As + k * TB + r0 + 2);
    double2 b01 = *reinterpret_cast<const double2*>(Bs + k * TB + c0);
    double2 b23 = *reinterpret_cast<const double2*>(Bs + k * TB + c0 + 2);
    double a[4] = {a01.x, a01.y, a23.x, a23.y};
    double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
  }
}

__device__ __forceinline__ void load_tile(double* dst, const double* __restrict__ src) {
  for (int t = threadIdx.x; t < TILE / 2; t += blockDim.x)
    reinterpret_cast<double2*>(dst)[t] = reinterpret_cast<const double2*>(src)[t];
}
// dst[k*64 + r] = src[r*64 + k]
__device__ __forceinline__ void load_tile_T(double* dst, const double* __restrict__ src) {
  for (int t = threadIdx.x; t < TILE; t += blockDim.x) {
    int k = t >> 6, r = t & 63;
    dst[k * TB + r] = src[r * TB + k];
  }
}

__device__ __forceinline__ int64_t tidx(const int64_t* tile_base, int s, int I, int J) {
  return tile_base[s] + (int64_t)I * (I + 1) / 2 + J;
}

// ---------------------------------------------------------------------------
// extraction: tiles <- A^[sub, sub]  (one warp per subdomain node)
// ---------------------------------------------------------------------------
__global__ void k_extract(int total_nodes, int nsub, const int32_t* __restrict__ sub_node_ptr,
                          const int32_t* __restrict__ sub_nodes, const int64_t* tile_base,
                          const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                          const double* __restrict__ val, double* tiles) {
  int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  int lane = threadIdx.x & 31;
  if (w >= total_nodes) return;
  // subdomain of entry w (binary search in sub_node_ptr)
  int lo = 0, hi = nsub;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (sub_node_ptr[mid] <= w) lo = mid; else hi = mid;
  }
  int s = lo;
  const int32_t* nodes = sub_nodes + sub_node_ptr[s];
  int nn = sub_node_ptr[s + 1] - sub_node_ptr[s];
  int lp = w - sub_node_ptr[s];
  int p = nodes[lp];
  for (int e = rp[p] + lane; e < rp[p + 1]; e += 32) {
    int q = col[e];
    int a = 0, b = nn;                       // lower_bound(q)
    while (a < b) {
      int m = (a + b) >> 1;
      if (nodes[m] < q) a = m + 1; else b = m;
    }
    if (a >= nn || nodes[a] != q) continue;
    int lq = a;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        int R = 3 * lp + r, C = 3 * lq + c;
        int I = R >> 6, J = C >> 6;
        if (I < J) continue;
        tiles[tidx(tile_base, s, I, J) * TILE + (C & 63) * TB + (R & 63)] = val[9 * (int64_t)e + 3 * r + c];
      }
  }
}

void launch_extract_local(const DevBatch& b, int total_nodes, const int32_t* sub_node_ptr,
                          const int32_t* sub_nodes, const int32_t* row_ptr, const int32_t* col,
                          const double* val, cudaStream_t st) {
  if (total_nodes <= 0) return;
  int64_t th = 32 * (int64_t)total_nodes;
  k_extract<<<(int)((th + 255) / 256), 256, 0, st>>>(total_nodes, b.nsub, sub_node_ptr, sub_nodes,
                                                     b.tile_base, row_ptr, col, val, b.tiles);
}

__global__ void k_pad_identity(int nsub, const int32_t* nb, const int32_t* ndof,
                               const int64_t* tile_base, double* tiles) {
  int s = blockIdx.x;
  if (s >= nsub) return;
  int np = TB * nb[s];
  for (int R = ndof[s] + threadIdx.x; R < np; R += blockDim.x) {
    int K = R >> 6;
    tiles[tidx(tile_base, s, K, K) * TILE + (R & 63) * TB + (R & 63)] = 1.0;
  }
}

void launch_pad_identity(const DevBatch& b, cudaStream_t st) {
  if (b.nsub <= 0) return;
  k_pad_identity<<<b.nsub, 64, 0, st>>>(b.nsub, b.nb, b.ndof, b.tile_base, b.tiles);
}

// ---------------------------------------------------------------------------
// Block sweep operator (symmetric Gauss-Jordan) on packed lower tiles.
// Sweeping pivot block p of a symmetric A with D = A_pp:
//   A_pp <- -D^-1,  A_ip <- A_ip D^-1,  A_ij <- A_ij - A_ip D^-1 A_pj
// keeps A symmetric; sweeping every block yields -A^-1 (negated at the end).
// ---------------------------------------------------------------------------
// C_i = A_ip (old), W_i = C_i D^-1 for every row block i != p
template <bool DMMA>
__global__ void __launch_bounds__(256) k_sweep_panel(int p, int64_t nrows, const int32_t* row_s,
                                                     const int32_t* row_k, const int32_t* nb,
                                                     const int64_t* tile_base,
                                                     const int64_t* row_base,
                                                     const double* tiles, const double* dinv,
                                                     double* cbuf, double* wbuf) {
  int64_t rb = blockIdx.x;
  if (rb >= nrows) return;
  int s = row_s[rb], i = row_k[rb];
  if (nb[s] <= p || i == p) return;
  extern __shared__ double sm[];
  double* As = sm;
  double* Bs = sm + TILE;
  if (i > p) load_tile(As, tiles + tidx(tile_base, s, i, p) * TILE);
  else load_tile_T(As, tiles + tidx(tile_base, s, p, i) * TILE);
  load_tile(Bs, dinv + (int64_t)s * TILE);   // (k,c) at c*64+k; D^-1 symmetric
  __syncthreads();
  double* W = wbuf + rb * TILE;
  double* C = cbuf + rb * TILE;
  for (int t = threadIdx.x; t < TILE / 2; t += blockDim.x)
    reinterpret_cast<double2*>(C)[t] = reinterpret_cast<const double2*>(As)[t];
  // Bs is used as Bs[k*64 + c] = D^-1[c][k] = D^-1[k][c]
  if (DMMA) {
    double acc[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = 0.0;
    tile_dmma(As, TB, Bs, TB, TB, acc);
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      int r, c;
      dmma_rc(t, r, c);
      W[c * TB + r] = acc[t];
    }
    return;
  }
  int r0 = (threadIdx.x & 15) * 4, c0 = (threadIdx.x >> 4) * 4;
  double acc[4][4] = {};
  tile_mma(As, Bs, acc, r0, c0);
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i2 = 0; i2 < 4; ++i2) W[(c0 + j) * TB + r0 + i2] = acc[i2][j];
}

template <bool DMMA>
__global__ void __launch_bounds__(256) k_sweep_update(int p, int64_t ntiles, const int32_t* tile_s,
                                                      const int32_t* tile_ij, const int32_t* nb,
                                                      const int64_t* row_base, double* tiles,
                                                      const double* dinv, const double* cbuf,
                                                      const double* wbuf) {
  int64_t t = blockIdx.x;
  if (t >= ntiles) return;
  int s = tile_s[t];
  if (nb[s] <= p) return;
  int I = tile_ij[t] >> 16, J = tile_ij[t] & 0xffff;
  double* T = tiles + t * TILE;
  if (I == p && J == p) {
    const double* D = dinv + (int64_t)s * TILE;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) T[e] = -D[e];
    return;
  }
  if (J == p) {            // I > p:  A_ip <- W_i
    const double* W = wbuf + (row_base[s] + I) * TILE;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) T[e] = W[e];
    return;
  }
  if (I == p) {            // J < p:  A_pj <- (W_j)^T
    const double* W = wbuf + (row_base[s] + J) * TILE;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
      int c = e >> 6, r = e & 63;
      T[e] = W[r * TB + c];
    }
    return;
  }
  extern __shared__ double sm[];
  if (DMMA) {
    // padded rows (72 doubles) spread the DMMA fragment loads over the banks
    constexpr int LDP = 72;
    double* As = sm;
    double* Bs = sm + TB * LDP;
    const double* Wg = wbuf + (row_base[s] + I) * TILE;
    const double* Cg = cbuf + (row_base[s] + J) * TILE;
    for (int e = threadIdx.x; e < TILE / 2; e += blockDim.x) {
      const int k = e >> 5, r2 = (e & 31) * 2;
      *reinterpret_cast<double2*>(As + k * LDP + r2) = reinterpret_cast<const double2*>(Wg)[e];
      *reinterpret_cast<double2*>(Bs + k * LDP + r2) = reinterpret_cast<const double2*>(Cg)[e];
    }
    // target values first: their DRAM latency overlaps the tile product
    double tv[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      int r, c;
      dmma_rc(q, r, c);
      tv[q] = T[c * TB + r];
    }
    __syncthreads();
    double acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = 0.0;
    tile_dmma(As, LDP, Bs, LDP, TB, acc);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      int r, c;
      dmma_rc(q, r, c);
      T[c * TB + r] = tv[q] - acc[q];
    }
    return;
  }
  double* As = sm;
  double* Bs = sm + TILE;
  load_tile(As, wbuf + (row_base[s] + I) * TILE);   // W_I (r,k) at k*64+r
  load_tile(Bs, cbuf + (row_base[s] + J) * TILE);   // C_J (c,k) at k*64+c  == (C_J^T)(k,c)
  __syncthreads();
  int r0 = (threadIdx.x & 15) * 4, c0 = (threadIdx.x >> 4) * 4;
  double acc[4][4] = {};
  tile_mma(As, Bs, acc, r0, c0);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double2* col = reinterpret_cast<double2*>(T + (c0 + j) * TB + r0);
    double2 v0 = col[0], v1 = col[1];
    v0.x -= acc[0][j]; v0.y -= acc[1][j]; v1.x -= acc[2][j]; v1.y -= acc[3][j];
    col[0] = v0; col[1] = v1;
  }
}

__global__ void k_negate(int64_t n, double* x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = -x[i];
}

static int g_dmma = -1;   // FP64 tensor cores (DMMA) in the setup tile products; HPLMM_DMMA=0 off

bool use_dmma() {
  if (g_dmma < 0) {
    const char* e = getenv("HPLMM_DMMA");
    g_dmma = (e && e[0] == '0') ? 0 : 1;
  }
  return g_dmma == 1;
}

// ---------------------------------------------------------------------------
// Blocked sweeps (r02): M consecutive pivot tiles P = {p .. p+mg-1} (mg =
// min(M, nb - p) per subdomain) are swept in one pass -- sweeping the pivots
// of P one after the other equals sweeping the (64 mg)^2 block D = A_PP:
//   A_PP <- -D^-1,  A_iP <- A_iP D^-1,  A_ij <- A_ij - A_iP D^-1 A_Pj.
// The update is then a 64 x 64 x 64M DMMA product per tile and every target
// tile is read and written once per M pivots instead of once per pivot: at
// M = 1 the update moves 64 KB of HBM per 0.5 MFLOP, about the B200's FP64
// tensor-core balance, so it cannot be compute-bound (r01: 36.8% DMMA pipe,
// 16 TFLOP/s on the cfg3 coarse block).  D (padded with the identity when
// mg < M) is inverted in registers by one 1024-thread CTA; C_i = A_iP and
// W_i = C_i D^-1 are kept k-major (k * 64 + r, k < 64M) per row block.
// ---------------------------------------------------------------------------

__device__ __forceinline__ double tile_elem_sym(const double* tiles, const int64_t* tile_base,
                                                int s, int I, int J, int r, int c) {
  // element (r, c) of the symmetric block (I, J) from the packed lower tiles
  if (I >= J) return tiles[tidx(tile_base, s, I, J) * TILE + c * TB + r];
  return tiles[tidx(tile_base, s, J, I) * TILE + r * TB + c];
}

// D^-1 by the sweep in registers: one CTA of 1024 threads per subdomain,
// thread i owns row r = i % 64M of the columns c = i / 64M + (1024 / 64M) j.
// Step k updates every element by the same rank-1 formula
//   a_rc <- a_rc - (a_rk / a_kk) a_kc
// and then fixes row k (a_kc / a_kk), column k (a_rk / a_kk) and the pivot
// (-1 / a_kk).  The owners of column k + 1 publish it (and 1 / a_k+1,k+1)
// into a double-buffered shared column as they update it, so a step costs one
// barrier and two instructions per element (r01: 256 threads, the tile in
// shared memory, two barriers and a branchy update per element -- 0.23 ms
// per 64-wide pivot, 12% of the cfg3 setup).  The k loop is unrolled by the
// column stride so that the register holding column k is static.
template <int M>
__global__ void __launch_bounds__(1024) k_sweep_pivot_m(int p, int nsub, const int32_t* nb,
                                                        const int64_t* tile_base,
                                                        const double* tiles, double* dinv,
                                                        int32_t* err) {
  constexpr int N = TB * M, PER = N * N / 1024, CSTEP = 1024 / N;
  const int s = blockIdx.x;
  if (s >= nsub || nb[s] <= p) return;
  const int mg = min(M, nb[s] - p);
  __shared__ double colbuf[2][N];
  __shared__ double invbuf[2];
  const int r = threadIdx.x % N, c0 = threadIdx.x / N;
  double v[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int c = c0 + CSTEP * j;
    const int R = r >> 6, C = c >> 6;
    v[j] = (R < mg && C < mg) ? tile_elem_sym(tiles, tile_base, s, p + R, p + C, r & 63, c & 63)
                              : (r == c ? 1.0 : 0.0);
  }
  bool bad = false;
  if (c0 == 0) {
    colbuf[0][r] = v[0];
    if (r == 0) {
      bad = !(v[0] > 0.0);
      invbuf[0] = 1.0 / v[0];
    }
  }
  __syncthreads();
  const int K = TB * mg;
#pragma unroll
  for (int jj = 0; jj < PER; ++jj) {
#pragma unroll 1
    for (int kk = 0; kk < CSTEP; ++kk) {
      const int k = jj * CSTEP + kk;
      if (k >= K) break;
      const double* colk = colbuf[k & 1];
      const double inv = invbuf[k & 1];
      const double ck_r = colk[r];
      const double f = ck_r * inv;
      double vk = 0.0;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const double ckc = colk[c0 + CSTEP * j];
        v[j] = r == k ? ckc * inv : fma(-f, ckc, v[j]);   // row k, else the rank-1 update
        if (j == jj) vk = v[j];
      }
      if (c0 == kk) vk = r == k ? -inv : f;                // column k and the pivot
#pragma unroll
      for (int j = 0; j < PER; ++j)
        if (j == jj && c0 == kk) v[j] = vk;
      // publish column k + 1 and its pivot's reciprocal
      const int k1 = k + 1, j1 = k1 / CSTEP;
      if (k1 < K && c0 == k1 % CSTEP) {
        double w = 0.0;
#pragma unroll
        for (int j = 0; j < PER; ++j)
          if (j == j1) w = v[j];
        colbuf[k1 & 1][r] = w;
        if (r == k1) {
          if (!(w > 0.0)) bad = true;
          invbuf[k1 & 1] = 1.0 / w;
        }
      }
      __syncthreads();
    }
  }
  if (bad) atomicMin(err, s);
  double* out = dinv + (int64_t)s * N * N;
#pragma unroll
  for (int j = 0; j < PER; ++j) out[(int64_t)(c0 + CSTEP * j) * N + r] = -v[j];
}

// C_i = A_iP (k-major, zero beyond 64 mg), W_i = C_i D^-1 for every row block i
// outside P; one CTA per row block
template <int M>
__global__ void __launch_bounds__(256) k_sweep_panel_m(int p, int64_t nrows, const int32_t* row_s,
                                                       const int32_t* row_k, const int32_t* nb,
                                                       const int64_t* tile_base,
                                                       const double* tiles, const double* dinv,
                                                       double* cbuf, double* wbuf) {
  constexpr int N = TB * M;
  const int64_t rb = blockIdx.x;
  if (rb >= nrows) return;
  const int s = row_s[rb], i = row_k[rb];
  if (nb[s] <= p) return;
  const int mg = min(M, nb[s] - p);
  if (i >= p && i < p + mg) return;
  extern __shared__ double sm[];
  double* As = sm;            // (r, k) at k*64 + r, k < N
  double* Bs = sm + TB * N;   // D^-1, (k, c) at k*N + c (symmetric)
  for (int e = threadIdx.x; e < TB * N; e += blockDim.x) {
    const int k = e >> 6, r = e & 63, b = k >> 6;
    As[e] = b < mg ? tile_elem_sym(tiles, tile_base, s, i, p + b, r, k & 63) : 0.0;
  }
  const double* D = dinv + (int64_t)s * N * N;
  for (int e = threadIdx.x; e < N * N / 2; e += blockDim.x)
    reinterpret_cast<double2*>(Bs)[e] = reinterpret_cast<const double2*>(D)[e];
  __syncthreads();
  double* C = cbuf + rb * (int64_t)(M * TILE);
  double* W = wbuf + rb * (int64_t)(M * TILE);
  for (int e = threadIdx.x; e < TB * N / 2; e += blockDim.x)
    reinterpret_cast<double2*>(C)[e] = reinterpret_cast<const double2*>(As)[e];
#pragma unroll 1
  for (int cb = 0; cb < M; ++cb) {
    double acc[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = 0.0;
    tile_dmma(As, TB, Bs + cb * TB, N, N, acc);
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      int r, c;
      dmma_rc(t, r, c);
      W[(cb * TB + c) * TB + r] = acc[t];
    }
  }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// A_IJ -= W_I C_J^T over K = 64 M for every tile outside P; the tiles of
// row / column P are overwritten with W (and -D^-1).  The K loop streams
// 32-deep chunks of W_I and C_J (L2-resident) through a two-stage cp.async
// ring (rows padded to 72 doubles against bank conflicts) while the target
// tile's values are already in registers.
constexpr int SWU_KC = 32, SWU_LDP = 72;
constexpr size_t SWU_SMEM = 2 * 2 * SWU_KC * SWU_LDP * sizeof(double);

template <int M>
__global__ void __launch_bounds__(256) k_sweep_update_m(int p, int64_t ntiles, const int32_t* tile_s,
                                                        const int32_t* tile_ij, const int32_t* nb,
                                                        const int64_t* row_base, double* tiles,
                                                        const double* dinv, const double* cbuf,
                                                        const double* wbuf) {
  constexpr int N = TB * M;
  const int64_t t = blockIdx.x;
  if (t >= ntiles) return;
  const int s = tile_s[t];
  if (nb[s] <= p) return;
  const int mg = min(M, nb[s] - p);
  const int I = tile_ij[t] >> 16, J = tile_ij[t] & 0xffff;
  const bool inI = I >= p && I < p + mg, inJ = J >= p && J < p + mg;
  double* T = tiles + t * TILE;
  if (inI && inJ) {          // -D^-1 block (I - p, J - p)
    const double* D = dinv + (int64_t)s * N * N;
    const int a = I - p, b = J - p;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
      const int c = e >> 6, r = e & 63;
      T[e] = -D[(int64_t)(b * TB + c) * N + a * TB + r];
    }
    return;
  }
  if (inJ) {                 // I > P:  A_I,p+b <- W_I[:, b]
    const double* W = wbuf + (row_base[s] + I) * (int64_t)(M * TILE) + (J - p) * TILE;
    for (int e = threadIdx.x; e < TILE / 2; e += blockDim.x)
      reinterpret_cast<double2*>(T)[e] = reinterpret_cast<const double2*>(W)[e];
    return;
  }
  if (inI) {                 // J < P:  A_p+a,J <- (W_J[:, a])^T
    const double* W = wbuf + (row_base[s] + J) * (int64_t)(M * TILE) + (I - p) * TILE;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
      const int c = e >> 6, r = e & 63;
      T[e] = W[r * TB + c];
    }
    return;
  }
  extern __shared__ double sm[];
  const double* Wg = wbuf + (row_base[s] + I) * (int64_t)(M * TILE);
  const double* Cg = cbuf + (row_base[s] + J) * (int64_t)(M * TILE);
  const int KC = TB * mg / SWU_KC;   // K chunks (the padding k beyond 64 mg are 0)
  auto issue = [&](int kc) {
    double* As = sm + (kc & 1) * (2 * SWU_KC * SWU_LDP);
    double* Bs = As + SWU_KC * SWU_LDP;
    const double* wsrc = Wg + (int64_t)kc * SWU_KC * TB;
    const double* csrc = Cg + (int64_t)kc * SWU_KC * TB;
    for (int e = threadIdx.x; e < SWU_KC * TB / 2; e += blockDim.x) {
      const int k = e >> 5, r2 = (e & 31) * 2;
      cp_async16(As + k * SWU_LDP + r2, wsrc + 2 * e);
      cp_async16(Bs + k * SWU_LDP + r2, csrc + 2 * e);
    }
    cp_async_commit();
  };
  issue(0);
  if (KC > 1) issue(1);
  double tv[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    int r, c;
    dmma_rc(q, r, c);
    tv[q] = T[c * TB + r];
  }
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (int kc = 0; kc < KC; ++kc) {
    if (kc + 1 < KC) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const double* As = sm + (kc & 1) * (2 * SWU_KC * SWU_LDP);
    tile_dmma(As, SWU_LDP, As + SWU_KC * SWU_LDP, SWU_LDP, SWU_KC, acc);
    __syncthreads();
    if (kc + 2 < KC) issue(kc + 2);
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    int r, c;
    dmma_rc(q, r, c);
    T[c * TB + r] = tv[q] - acc[q];
  }
}

template <int M>
static void sweep_steps_m(const DevBatch& b, cudaStream_t st) {
  constexpr int N = TB * M;
  const size_t sm_panel = (size_t)(TB * N + N * N) * sizeof(double);
  set_max_dynamic_smem((const void*)k_sweep_panel_m<M>, sm_panel);
  set_max_dynamic_smem((const void*)k_sweep_update_m<M>, SWU_SMEM);
  for (int p = 0; p < b.max_nb; p += M) {
    k_sweep_pivot_m<M><<<b.nsub, 1024, 0, st>>>(p, b.nsub, b.nb, b.tile_base, b.tiles, b.dinv, b.err);
    k_sweep_panel_m<M><<<(unsigned)b.nrows, 256, sm_panel, st>>>(p, b.nrows, b.row_s, b.row_k, b.nb,
                                                                 b.tile_base, b.tiles, b.dinv,
                                                                 b.cbuf, b.wbuf);
    k_sweep_update_m<M><<<(unsigned)b.ntiles, 256, SWU_SMEM, st>>>(p, b.ntiles, b.tile_s, b.tile_ij,
                                                                   b.nb, b.row_base, b.tiles,
                                                                   b.dinv, b.cbuf, b.wbuf);
  }
}

template <bool DMMA>
static void sweep_steps(const DevBatch& b, cudaStream_t st) {
  size_t sm2 = 2 * TILE * sizeof(double);
  for (int p = 0; p < b.max_nb; ++p) {
    k_sweep_pivot_m<1><<<b.nsub, 1024, 0, st>>>(p, b.nsub, b.nb, b.tile_base, b.tiles, b.dinv, b.err);
    k_sweep_panel<DMMA><<<(unsigned)b.nrows, 256, sm2, st>>>(p, b.nrows, b.row_s, b.row_k, b.nb,
                                                             b.tile_base, b.row_base, b.tiles,
                                                             b.dinv, b.cbuf, b.wbuf);
    k_sweep_update<DMMA><<<(unsigned)b.ntiles, 256, DMMA ? 2 * TB * 72 * 8 : sm2, st>>>(p, b.ntiles, b.tile_s, b.tile_ij,
                                                               b.nb, b.row_base, b.tiles, b.dinv,
                                                               b.cbuf, b.wbuf);
  }
}

void launch_sweep_invert(const DevBatch& b, cudaStream_t st) {
  if (b.nsub <= 0) return;
  set_max_dynamic_smem((const void*)k_sweep_panel<true>, 2 * TILE * 8);
  set_max_dynamic_smem((const void*)k_sweep_update<true>, 2 * TB * 72 * 8);
  set_max_dynamic_smem((const void*)k_sweep_panel<false>, 2 * TILE * 8);
  set_max_dynamic_smem((const void*)k_sweep_update<false>, 2 * TILE * 8);
  // M = 2 for batches of few large blocks (the coarse S: cfg3 coarse inversion
  // 0.392 -> 0.346 s); M = 1 for the batches of many supernode fronts, whose
  // 1024-thread pivot CTAs (one per front) then keep two CTAs per SM (M = 2:
  // cfg3 grain + contact front inversions 0.21 -> 0.27 s)
  static const int sweep_env = getenv("HPLMM_SWEEP_M") ? atoi(getenv("HPLMM_SWEEP_M")) : -1;
  const int sweep_m = sweep_env >= 0 ? sweep_env : (b.nsub <= 16 && b.max_nb >= 4 ? SWEEP_M : 1);
  if (use_dmma() && sweep_m == 2) sweep_steps_m<2>(b, st);
  else if (use_dmma() && sweep_m == 1) sweep_steps_m<1>(b, st);
  else if (use_dmma()) sweep_steps<true>(b, st);   // HPLMM_SWEEP_M=0: r01 rank-64 kernels
  else sweep_steps<false>(b, st);
  k_negate<<<148 * 8, 256, 0, st>>>(b.ntiles * TILE, b.tiles);
}


// ---------------------------------------------------------------------------
// Packed symmetric matrix-vector product, one warp per lower tile (I,J):
//   part_row[t] = A_IJ x_J        part_col[t] = A_IJ^T x_I   (I != J)
// Lane l owns tile rows 2l, 2l+1: each column is one coalesced 512-byte load.
// The 64 per-lane column partials are reduced by a 5-step recursive-halving
// shuffle transpose (62 shuffles / tile), after which lane l holds columns
// 2l, 2l+1.  No atomics: partials are summed in a fixed order by k_symv_reduce.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_symv_tiles(int64_t ntiles, const int32_t* __restrict__ tile_s,
                                                    const int32_t* __restrict__ tile_ij,
                                                    const int64_t* __restrict__ row_base,
                                                    const double* __restrict__ tiles,
                                                    const double* __restrict__ xloc,
                                                    double* __restrict__ part_row,
                                                    double* __restrict__ part_col) {
  int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  int s = __ldg(tile_s + t);
  int ij = __ldg(tile_ij + t);
  int I = ij >> 16, J = ij & 0xffff;
  int64_t rb = __ldg(row_base + s);
  const double* xJ = xloc + (rb + J) * TB;
  double2 xI = *reinterpret_cast<const double2*>(xloc + (rb + I) * TB + 2 * lane);
  const double2* A = reinterpret_cast<const double2*>(tiles + t * TILE) + lane;
  double y0 = 0.0, y1 = 0.0;
  double cp[64];
#pragma unroll
  for (int c0 = 0; c0 < TB; c0 += 16) {
    double2 a[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) a[u] = __ldcs(A + (c0 + u) * (TB / 2));
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      double xj = __ldg(xJ + c0 + u);
      y0 = fma(a[u].x, xj, y0);
      y1 = fma(a[u].y, xj, y1);
      cp[c0 + u] = fma(a[u].x, xI.x, a[u].y * xI.y);
    }
  }
  reinterpret_cast<double2*>(part_row + t * TB)[lane] = make_double2(y0, y1);
  if (I == J) return;
  // recursive-halving transpose-reduce of cp[0..63] across the warp
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    bool up = lane & 16;
    double send = up ? cp[k] : cp[32 + k];
    double keep = up ? cp[32 + k] : cp[k];
    cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    bool up = lane & 8;
    double send = up ? cp[k] : cp[16 + k];
    double keep = up ? cp[16 + k] : cp[k];
    cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    bool up = lane & 4;
    double send = up ? cp[k] : cp[8 + k];
    double keep = up ? cp[8 + k] : cp[k];
    cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    bool up = lane & 2;
    double send = up ? cp[k] : cp[4 + k];
    double keep = up ? cp[4 + k] : cp[k];
    cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    bool up = lane & 1;
    double send = up ? cp[k] : cp[2 + k];
    double keep = up ? cp[2 + k] : cp[k];
    cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  }
  reinterpret_cast<double2*>(part_col + t * TB)[lane] = make_double2(cp[0], cp[1]);
}

// ---------------------------------------------------------------------------
// TMA-pipelined persistent variant (the production kernel on sm_100a).
// One CTA per SM streams a contiguous range of tiles through a ring of
// SY_STAGES 32-KiB shared-memory stages with 1-D bulk async copies
// (cp.async.bulk, completion via mbarrier transaction counts).  One producer
// lane keeps up to SY_STAGES tiles in flight independently of register
// pressure; SY_CONS consumer warps each take every SY_CONS-th tile and
// compute the same two partial products as k_symv_tiles from shared memory.
// ---------------------------------------------------------------------------
constexpr int SY_STAGES = 6;
constexpr int SY_CONS = 3;
// Stage s is always consumed by warp s % SY_CONS (tile k -> stage k % STAGES,
// warp k % CONS).  That keeps every consumer within one mbarrier phase of the
// stage it waits on, which the parity wait requires.
static_assert(SY_STAGES % SY_CONS == 0, "each stage must belong to one consumer warp");
// multi-column blocks do P times the arithmetic per streamed tile: twice the
// consumer warps (still one stage per warp residue class)
template <int P>
constexpr int sy_cons() { return P == 1 ? SY_CONS : 6; }
static_assert(SY_STAGES % sy_cons<4>() == 0, "each stage must belong to one consumer warp");

// P columns (multi-RHS blocks): each streamed tile is applied to P vectors
// (column c at xloc + c xstr, partials at part_row / part_col + c pstr) while
// it sits in shared memory -- S^-1 is read from HBM once per block
template <int P>
__global__ void __launch_bounds__(32 * (sy_cons<P>() + 1), 1)
    k_symv_tma(int64_t ntiles, const int32_t* __restrict__ tile_s,
               const int32_t* __restrict__ tile_ij, const int64_t* __restrict__ row_base,
               const double* __restrict__ tiles, const double* __restrict__ xloc,
               double* __restrict__ part_row, double* __restrict__ part_col, int64_t xstr,
               int64_t pstr) {
  extern __shared__ __align__(1024) double sm_tiles[];
  __shared__ __align__(8) uint64_t full[SY_STAGES], empty[SY_STAGES];
  constexpr int CONS = sy_cons<P>();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per;
  const int64_t nt = max((int64_t)0, min(ntiles, t0 + per) - t0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < SY_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == CONS) {                       // producer
    if (lane == 0) {
      for (int64_t k = 0; k < nt; ++k) {
        int s = (int)(k % SY_STAGES);
        if (k >= SY_STAGES) mbar_wait(&empty[s], (uint32_t)((k / SY_STAGES - 1) & 1));
        mbar_expect_tx(&full[s], TILE * 8);
        bulk_g2s(sm_tiles + (size_t)s * TILE, tiles + (t0 + k) * TILE, TILE * 8, &full[s]);
      }
    }
    return;
  }
  for (int64_t k = warp; k < nt; k += CONS) {
    const int64_t t = t0 + k;
    const int s = (int)(k % SY_STAGES);
    const int ts = __ldg(tile_s + t);
    const int ij = __ldg(tile_ij + t);
    const int I = ij >> 16, J = ij & 0xffff;
    const int64_t rb = __ldg(row_base + ts);
    // x_I and x_J of every column loaded before the tile wait (lane l holds
    // entries 2l, 2l + 1): their L2 latency overlaps the tile's arrival
    double2 xIc[P], xJc[P];
#pragma unroll
    for (int cc = 0; cc < P; ++cc) {
      const double* xl = xloc + cc * xstr;
      xIc[cc] = *reinterpret_cast<const double2*>(xl + (rb + I) * TB + 2 * lane);
      xJc[cc] = *reinterpret_cast<const double2*>(xl + (rb + J) * TB + 2 * lane);
    }
    mbar_wait(&full[s], (uint32_t)((k / SY_STAGES) & 1));
#pragma unroll 1
    for (int cc = 0; cc < P; ++cc) {
      double2 xI = xIc[0];
      double xj[TB / 32 * 2] = {xJc[0].x, xJc[0].y};
#pragma unroll
      for (int c2 = 1; c2 < P; ++c2)
        if (cc == c2) {
          xI = xIc[c2];
          xj[0] = xJc[c2].x;
          xj[1] = xJc[c2].y;
        }
      const double2* A = reinterpret_cast<const double2*>(sm_tiles + (size_t)s * TILE) + lane;
      double y0 = 0.0, y1 = 0.0;
      double cp[64];
#pragma unroll
      for (int c = 0; c < TB; ++c) {
        double2 a = A[c * (TB / 2)];
        double x = __shfl_sync(0xffffffffu, (c & 1) ? xj[1] : xj[0], c >> 1);
        y0 = fma(a.x, x, y0);
        y1 = fma(a.y, x, y1);
        cp[c] = fma(a.x, xI.x, a.y * xI.y);
      }
      if (cc == P - 1) {   // last read of the stage
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      reinterpret_cast<double2*>(part_row + cc * pstr + t * TB)[lane] = make_double2(y0, y1);
      if (I == J) continue;
#pragma unroll
      for (int k2 = 0; k2 < 32; ++k2) {
        bool up = lane & 16;
        double send = up ? cp[k2] : cp[32 + k2];
        double keep = up ? cp[32 + k2] : cp[k2];
        cp[k2] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) {
        bool up = lane & 8;
        double send = up ? cp[k2] : cp[16 + k2];
        double keep = up ? cp[16 + k2] : cp[k2];
        cp[k2] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
      }
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) {
        bool up = lane & 4;
        double send = up ? cp[k2] : cp[8 + k2];
        double keep = up ? cp[8 + k2] : cp[k2];
        cp[k2] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      }
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) {
        bool up = lane & 2;
        double send = up ? cp[k2] : cp[4 + k2];
        double keep = up ? cp[4 + k2] : cp[k2];
        cp[k2] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2) {
        bool up = lane & 1;
        double send = up ? cp[k2] : cp[2 + k2];
        double keep = up ? cp[2 + k2] : cp[k2];
        cp[k2] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
      reinterpret_cast<double2*>(part_col + cc * pstr + t * TB)[lane] = make_double2(cp[0], cp[1]);
    }
  }
}

// y_K = sum_{J<=K} part_row(K,J) + sum_{I>K} part_col(I,K), fixed order
// y_K = sum_{J<=K} part_row(K,J) + sum_{I>K} part_col(I,K): one CTA of SR_WARPS
// warps per row block; warp w sums the partials of index = w (mod SR_WARPS) in
// ascending order (four loads in flight), then warp 0 adds the warp sums in
// order w = 0..SR_WARPS-1 (fixed order, no atomics)
constexpr int SR_WARPS = 16;
__global__ void __launch_bounds__(32 * SR_WARPS)
    k_symv_reduce(int64_t nrows, const int32_t* __restrict__ row_s,
                  const int32_t* __restrict__ row_k, const int32_t* __restrict__ nb,
                  const int64_t* __restrict__ tile_base, const int64_t* __restrict__ row_base,
                  const double* __restrict__ part_row, const double* __restrict__ part_col,
                  double* __restrict__ yloc, int64_t ystr, int64_t pstr) {
  __shared__ double2 red[SR_WARPS][32];
  // column blockIdx.y of a multi-RHS block (strides ystr / pstr)
  part_row += blockIdx.y * pstr;
  part_col += blockIdx.y * pstr;
  yloc += blockIdx.y * ystr;
  const int64_t rbi = blockIdx.x;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = row_s[rbi], K = row_k[rbi], n = nb[s];
  // index t < n: t <= K -> part_row(K, t), t > K -> part_col(t, K)
  auto part = [&](int t) {
    const double* p = t <= K ? part_row + tidx(tile_base, s, K, t) * TB
                             : part_col + tidx(tile_base, s, t, K) * TB;
    return __ldcs(reinterpret_cast<const double2*>(p) + lane);
  };
  double2 a0 = make_double2(0.0, 0.0), a1 = a0;
  int t = w;
  for (; t + SR_WARPS < n; t += 2 * SR_WARPS) {
    const double2 u = part(t), v = part(t + SR_WARPS);
    a0.x += u.x; a0.y += u.y;
    a1.x += v.x; a1.y += v.y;
  }
  if (t < n) {
    const double2 u = part(t);
    a0.x += u.x; a0.y += u.y;
  }
  red[w][lane] = make_double2(a0.x + a1.x, a0.y + a1.y);
  __syncthreads();
  if (w == 0) {
    double2 acc = red[0][lane];
#pragma unroll
    for (int q = 1; q < SR_WARPS; ++q) {
      acc.x += red[q][lane].x;
      acc.y += red[q][lane].y;
    }
    reinterpret_cast<double2*>(yloc + (row_base[s] + K) * TB)[lane] = acc;
  }
}

__global__ void k_gather(int64_t n, const int32_t* __restrict__ lmap, const double* __restrict__ x,
                         double* __restrict__ xloc, int64_t xld = 0) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  x += blockIdx.y * xld;     // column blockIdx.y of a block (xloc stride n)
  xloc += blockIdx.y * n;
  int g = lmap[i];
  xloc[i] = g >= 0 ? x[g] : 0.0;
}

void launch_gather(const DevBatch& b, const double* x, cudaStream_t st) {
  if (b.nloc <= 0) return;
  k_gather<<<(unsigned)((b.nloc + 255) / 256), 256, 0, st>>>(b.nloc, b.lmap, x, b.xloc);
}

static int g_symv_mode = -1;   // 0 = register kernel, 1 = TMA pipeline (default)

void launch_symv_tiles(const DevBatch& b, cudaStream_t st) {
  if (b.ntiles <= 0) return;
  if (g_symv_mode < 0) {
    const char* e = getenv("HPLMM_SYMV");
    g_symv_mode = (e && e[0] == '0') ? 0 : 1;
  }
  if (g_symv_mode == 1) {
    set_max_dynamic_smem((const void*)k_symv_tma<1>, SY_STAGES * TILE * 8);
    int64_t grid = std::min<int64_t>(device_sm_count(), b.ntiles);
    k_symv_tma<1><<<(unsigned)grid, 32 * (SY_CONS + 1), SY_STAGES * TILE * 8, st>>>(
        b.ntiles, b.tile_s, b.tile_ij, b.row_base, b.tiles, b.xloc, b.part_row, b.part_col, 0, 0);
    return;
  }
  int64_t th = 32 * b.ntiles;
  k_symv_tiles<<<(unsigned)((th + 255) / 256), 256, 0, st>>>(b.ntiles, b.tile_s, b.tile_ij,
                                                             b.row_base, b.tiles, b.xloc,
                                                             b.part_row, b.part_col);
}

void launch_symv_reduce(const DevBatch& b, cudaStream_t st) {
  if (b.nrows <= 0) return;
  k_symv_reduce<<<(unsigned)b.nrows, 32 * SR_WARPS, 0, st>>>(b.nrows, b.row_s, b.row_k, b.nb,
                                                               b.tile_base, b.row_base,
                                                               b.part_row, b.part_col, b.yloc, 0, 0);
}

// P-column block (multi-RHS): y_c = A x_c for c < ncols, with column c of the
// block at xk / yk + c nloc and its partials at prk / pck + c ntiles TB; the
// packed tiles stream once (k_symv_tma<P>)
template <int P>
static void symv_k(const DevBatch& b, int ncols, const double* xk, double* yk, double* prk,
                   double* pck, cudaStream_t st) {
  const int64_t pstr = b.ntiles * TB;
  set_max_dynamic_smem((const void*)k_symv_tma<P>, SY_STAGES * TILE * 8);
  const int64_t grid = std::min<int64_t>(device_sm_count(), b.ntiles);
  k_symv_tma<P><<<(unsigned)grid, 32 * (sy_cons<P>() + 1), SY_STAGES * TILE * 8, st>>>(
      b.ntiles, b.tile_s, b.tile_ij, b.row_base, b.tiles, xk, prk, pck, b.nloc, pstr);
  k_symv_reduce<<<dim3((unsigned)b.nrows, (unsigned)ncols), 32 * SR_WARPS, 0, st>>>(
      b.nrows, b.row_s, b.row_k, b.nb, b.tile_base, b.row_base, prk, pck, yk, b.nloc, pstr);
}

void launch_symv_k(const DevBatch& b, int P, int ncols, const double* xk, double* yk, double* prk,
                   double* pck, cudaStream_t st) {
  if (b.ntiles <= 0 || ncols <= 0) return;
  if (P == 4) symv_k<4>(b, ncols, xk, yk, prk, pck, st);
  else if (P == 2) symv_k<2>(b, ncols, xk, yk, prk, pck, st);
  else symv_k<1>(b, ncols, xk, yk, prk, pck, st);
}

void launch_gather_k(const DevBatch& b, int ncols, const double* x, int64_t xld, double* xk,
                     cudaStream_t st) {
  if (b.nloc <= 0 || ncols <= 0) return;
  k_gather<<<dim3((unsigned)((b.nloc + 255) / 256), (unsigned)ncols), 256, 0, st>>>(b.nloc, b.lmap,
                                                                                    x, xk, xld);
}

void launch_symv(const DevBatch& b, cudaStream_t st) {
  launch_symv_tiles(b, st);
  launch_symv_reduce(b, st);
}

// ---------------------------------------------------------------------------
// B = -(A^-1 X) on the grain batch (shape vectors, eq:col_pk).  One CTA per
// (row block I, 64-column chunk); loops over all tile columns J of the full
// symmetric matrix (tile (J,I)^T above the diagonal).  X, B row-major [.. x ld].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_symm_neg(int64_t nrows, const int32_t* row_s,
                                                  const int32_t* row_k, const int32_t* nb,
                                                  const int64_t* tile_base,
                                                  const double* tiles, const int64_t* x_off,
                                                  const int32_t* ld, const int32_t* kcols,
                                                  const double* X, double* B) {
  int64_t rb = blockIdx.x;
  int q = blockIdx.y;
  int s = row_s[rb], I = row_k[rb], n = nb[s];
  int kc = kcols[s], L = ld[s];
  if (q * TB >= kc) return;
  extern __shared__ double sm[];
  double* As = sm;
  double* Bs = sm + TILE;
  const double* Xs = X + x_off[s];
  int r0 = (threadIdx.x & 15) * 4, c0 = (threadIdx.x >> 4) * 4;
  double acc[4][4] = {};
  for (int J = 0; J < n; ++J) {
    __syncthreads();
    if (J <= I) load_tile(As, tiles + tidx(tile_base, s, I, J) * TILE);
    else load_tile_T(As, tiles + tidx(tile_base, s, J, I) * TILE);
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
      int k = e >> 6, c = e & 63;
      int col = q * TB + c;
      Bs[e] = col < kc ? Xs[(int64_t)(J * TB + k) * L + col] : 0.0;
    }
    __syncthreads();
    tile_mma(As, Bs, acc, r0, c0);
  }
  double* Bo = B + x_off[s];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int col = q * TB + c0 + j;
      if (col < kc) Bo[(int64_t)(I * TB + r0 + i) * L + col] = -acc[i][j];
    }
}

void launch_symm_neg(const DevBatch& b, const int64_t* x_off, const int32_t* ld,
                     const int32_t* kcols, int max_kchunks, const double* X, double* B,
                     cudaStream_t st) {
  if (b.nrows <= 0) return;
  set_max_dynamic_smem((const void*)k_symm_neg, 2 * TILE * 8);
  // grid.y = max column chunks; CTAs beyond a grain's k exit immediately
  if (max_kchunks <= 0) return;
  dim3 grid((unsigned)b.nrows, (unsigned)max_kchunks);
  k_symm_neg<<<grid, 256, 2 * TILE * sizeof(double), st>>>(b.nrows, b.row_s, b.row_k, b.nb,
                                                           b.tile_base, b.tiles, x_off, ld, kcols,
                                                           X, B);
}

// S (dense row-major, leading dim lds) -> packed lower tiles, symmetrised
// from its lower triangle (R16).
__global__ void k_pack_dense(int64_t ntiles, const int32_t* tile_ij, const double* S, int64_t lds,
                             double* tiles) {
  int64_t t = blockIdx.x;
  if (t >= ntiles) return;
  int I = tile_ij[t] >> 16, J = tile_ij[t] & 0xffff;
  for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
    int c = e >> 6, r = e & 63;
    int64_t R = I * TB + r, C = J * TB + c;
    tiles[t * TILE + e] = (R >= C) ? S[R * lds + C] : S[C * lds + R];
  }
}

void launch_pack_dense(const DevBatch& b, const double* S, int64_t lds, cudaStream_t st) {
  if (b.ntiles <= 0) return;
  k_pack_dense<<<(unsigned)b.ntiles, 256, 0, st>>>(b.ntiles, b.tile_ij, S, lds, b.tiles);
}

// ---------------------------------------------------------------------------
__global__ void k_combine_grain(int n, const int32_t* __restrict__ gpos,
                                const double* __restrict__ yloc, const double* __restrict__ a,
                                const double* __restrict__ b, double* __restrict__ out) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  double v = 0.0;
  if (a) v += a[d];
  if (b) v += b[d];
  int g = gpos[d];
  if (g >= 0) v += yloc[g];
  out[d] = v;
}

void launch_combine_grain(int n_dof, const int32_t* gpos, const double* yloc, const double* a,
                          const double* b, double* out, cudaStream_t st) {
  k_combine_grain<<<(n_dof + 255) / 256, 256, 0, st>>>(n_dof, gpos, yloc, a, b, out);
}

__global__ void k_sum_contact(int n, const int32_t* __restrict__ cptr,
                              const int32_t* __restrict__ cidx, const double* __restrict__ yloc,
                              double* __restrict__ out) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  double v = 0.0;
  for (int e = cptr[d]; e < cptr[d + 1]; ++e) v += yloc[cidx[e]];
  out[d] = v;
}

void launch_sum_contact(int n_dof, const int32_t* cptr, const int32_t* cidx, const double* yloc,
                        double* out, cudaStream_t st) {
  k_sum_contact<<<(n_dof + 255) / 256, 256, 0, st>>>(n_dof, cptr, cidx, yloc, out);
}

}  // namespace hplmm
