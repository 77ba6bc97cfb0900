// Multi-RHS applications of the two-level preconditioner (
// the paper's reuse argument): K <= 4 right-hand sides of one
// batch share every streamed operator -- the shape-vector blocks P^_B of the
// restriction / prolongation (eq:mg_struct) are read once for all K vectors;
// the supernodal local solves stream their factors once per launch
// (sn_apply_multi, NRHS = 2 / 4).  Each right-hand side keeps its own
// correction columns c^g = A_g^-1 b^g and D_c (eq:col_cg, R15, R16), held
// apart from P^_B: Ck[c][row] in the grain batch's local row layout.
//
// Vector blocks are K columns of length n_dof with stride ld (column c at
// v + c ld).  Every reduction keeps the single-RHS kernels' fixed order.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace hplmm {

// ---------------------------------------------------------------------------
// per-RHS correction columns (the multi-RHS counterpart of k_set_correction):
// Ck[c] = c_g (grain-batch local rows), Dck[c][g] = b_g . c_g, 0 => no column
// ---------------------------------------------------------------------------
__global__ void k_set_correction_k(const int32_t* nb, const int64_t* row_base, int G,
                                   const double* xloc, const double* yloc, double* Ck,
                                   double* Dck) {
  const int g = blockIdx.x;
  const int n = 64 * nb[g];
  const double* b = xloc + 64 * row_base[g];
  const double* y = yloc + 64 * row_base[g];
  __shared__ double red[256];
  __shared__ int anynz;
  if (threadIdx.x == 0) anynz = 0;
  __syncthreads();
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (b[i] != 0.0) anynz = 1;
    acc += b[i] * y[i];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const int keep = anynz;
  double* out = Ck + 64 * row_base[g];
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = keep ? y[i] : 0.0;
  if (threadIdx.x == 0) Dck[g] = keep ? red[0] : 0.0;
}

void launch_set_correction_k(const DevBatch& gb, int G, double* Ck, double* Dck, cudaStream_t st) {
  if (G <= 0) return;
  k_set_correction_k<<<G, 256, 0, st>>>(gb.nb, gb.row_base, G, gb.xloc, gb.yloc, Ck, Dck);
}

// ---------------------------------------------------------------------------
// Restriction, pass 1: per (grain, 64-row chunk) partials of B_g^T r_c over the
// k_g shape columns, and of c_g^T r_c (column L-1), for every RHS c.
// tk[(chunk_t + j) NRHS + c].  Warp w: rows 8w .. 8w+7; lane: columns.
// ---------------------------------------------------------------------------
template <int NRHS>
__global__ void __launch_bounds__(256, NRHS == 4 ? 3 : 4) k_restrict_chunks_k(DevCoarse c, const int32_t* lmap,
                                                              const int64_t* row_base,
                                                              const double* __restrict__ r,
                                                              int64_t ldr, int ncols,
                                                              const double* __restrict__ Ck,
                                                              int64_t ldc, double* __restrict__ tk) {
  constexpr int MAXL = 640 / NRHS;
  const int64_t ch = blockIdx.x;
  if (ch >= c.n_chunks) return;
  const int g = c.chunk_g[ch];
  const int r0 = c.chunk_r0[ch];
  const int L = c.ld[g];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* Bg = c.B + c.b_off[g] + (int64_t)(r0 + 8 * w) * L;
  const int64_t lrow0 = 64 * row_base[g] + r0;       // grain-batch local row of the chunk
  const int32_t* lm = lmap + lrow0;
  __shared__ __align__(16) double rv[64][NRHS];
  __shared__ double part[8][MAXL + 1][NRHS];
  if (threadIdx.x < 64) {
    const int d = lm[threadIdx.x];
#pragma unroll
    for (int q = 0; q < NRHS; ++q) rv[threadIdx.x][q] = (d >= 0 && q < ncols) ? r[q * ldr + d] : 0.0;
  }
  __syncthreads();
  // the warp's 8 rows of r stay in shared memory (broadcast reads in the FMA
  // loop): an 8 x NRHS register block cost the occupancy that keeps enough
  // B_g loads in flight (NRHS = 4: 2.3 TB/s with it)
  const double* rw = &rv[8 * w][0];
  double* out = tk + c.chunk_t[ch] * NRHS;
  for (int j0 = 0; j0 < L; j0 += MAXL) {
    const int jn = min(MAXL, L - j0);
    for (int jj = lane; jj < jn; jj += 32) {
      const int j = j0 + jj;
      double a[NRHS];
#pragma unroll
      for (int k = 0; k < NRHS; ++k) a[k] = 0.0;
      if (j < L - 1) {
        const double* col = Bg + j;
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = __ldcs(col + (int64_t)q * L);
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int k = 0; k < NRHS; ++k) a[k] = fma(v[q], rw[q * NRHS + k], a[k]);
      } else {   // correction column: each RHS its own c_g
#pragma unroll
        for (int k = 0; k < NRHS; ++k) {
          const double* cc = Ck + k * ldc + lrow0 + 8 * w;
#pragma unroll
          for (int q = 0; q < 8; ++q) a[k] = fma(k < ncols ? cc[q] : 0.0, rw[q * NRHS + k], a[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < NRHS; ++k) part[w][jj][k] = a[k];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < jn * NRHS; t += blockDim.x) {
      const int jj = t / NRHS, k = t - jj * NRHS;
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) a += part[q][jj][k];
      out[(int64_t)(j0 + jj) * NRHS + k] = a;
    }
    __syncthreads();
  }
}

// pass 2: per grain, sum of its chunks' partials (chunk order), gk[(off + j) NRHS + c]
template <int NRHS>
__global__ void k_restrict_grain_k(DevCoarse c, const double* __restrict__ tk,
                                   double* __restrict__ gk) {
  const int g = blockIdx.x;
  const int L = c.ld[g];
  const int c0 = c.chunk_ptr[g], c1 = c.chunk_ptr[g + 1];
  if (c1 <= c0) return;
  const double* t = tk + c.chunk_t[c0] * NRHS;
  double* out = gk + c.yext_off[g] * NRHS;
  const int nch = c1 - c0;
  const int64_t LK = (int64_t)L * NRHS;
  for (int64_t j = threadIdx.x; j < LK; j += blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int ch = 0;
    for (; ch + 3 < nch; ch += 4) {
      a0 += t[ch * LK + j];
      a1 += t[(ch + 1) * LK + j];
      a2 += t[(ch + 2) * LK + j];
      a3 += t[(ch + 3) * LK + j];
    }
    for (; ch < nch; ++ch) a0 += t[ch * LK + j];
    out[j] = (a0 + a1) + (a2 + a3);
  }
}

// pass 3: rm[c Nm + k] = sum over grains + the interface term Q^o[:, k]^T r_c;
// rc[c G + g] = the correction part (0 where D_c[c][g] = 0)
template <int NRHS>
__global__ void k_restrict_final_k(DevCoarse c, const int32_t* mortar_iface,
                                   const double* __restrict__ r, int64_t ldr, int ncols,
                                   const double* __restrict__ gk, const double* __restrict__ Dck,
                                   double* __restrict__ rm, double* __restrict__ rc) {
  constexpr int LPC = 8;
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int k = (int)(gt / LPC), sl = (int)(gt % LPC);
  double acc[NRHS];
#pragma unroll
  for (int q = 0; q < NRHS; ++q) acc[q] = 0.0;
  if (k < c.Nm) {
    const int m = k / 3;
    const int cf = mortar_iface[m];
    const int nu3 = 3 * (c.mortar_ptr[cf + 1] - c.mortar_ptr[cf]);
    const int qq = k - 3 * c.mortar_ptr[cf];
    const double* w = c.W + c.wt_off[cf] + qq;
    const int e0 = c.iface_ptr[cf], e1 = c.iface_ptr[cf + 1];
    for (int e = e0 + sl; e < e1; e += LPC) {
      const int64_t row = 3 * (int64_t)(e - e0);
      const double w0 = w[row * nu3], w1 = w[(row + 1) * nu3], w2 = w[(row + 2) * nu3];
      const int64_t d0 = 3 * (int64_t)c.iface_nodes[e];
#pragma unroll
      for (int q = 0; q < NRHS; ++q)
        if (q < ncols) {
          const double* ry = r + q * ldr + d0;
          acc[q] += w0 * ry[0] + w1 * ry[1] + w2 * ry[2];
        }
    }
  }
#pragma unroll
  for (int q = 0; q < NRHS; ++q)
#pragma unroll
    for (int o = LPC / 2; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o, LPC);
  if (sl != 0) return;
  if (k < c.Nm) {
    for (int e = c.mcol_ptr[k]; e < c.mcol_ptr[k + 1]; ++e) {
      const int g = c.mcol_g[e], j = c.mcol_j[e];
#pragma unroll
      for (int q = 0; q < NRHS; ++q) acc[q] += gk[(c.yext_off[g] + j) * NRHS + q];
    }
#pragma unroll
    for (int q = 0; q < NRHS; ++q)
      if (q < ncols) rm[(int64_t)q * c.Nm + k] = acc[q];
  } else if (k < c.Nm + c.n_grains) {
    const int g = k - c.Nm;
#pragma unroll
    for (int q = 0; q < NRHS; ++q)
      if (q < ncols)
        rc[(int64_t)q * c.n_grains + g] =
            Dck[(int64_t)q * c.n_grains + g] != 0.0 ? gk[(c.yext_off[g] + c.ld[g] - 1) * NRHS + q]
                                                     : 0.0;
  }
}

template <int NRHS>
static void restrict_k(const DevCoarse& c, const double* r, int64_t ldr, int ncols,
                       const double* Ck, int64_t ldc, const double* Dck, double* tk, double* gk,
                       double* rm, double* rc, cudaStream_t st) {
  if (c.n_chunks > 0)
    k_restrict_chunks_k<NRHS><<<(unsigned)c.n_chunks, 256, 0, st>>>(c, c.g_lmap, c.g_row_base, r,
                                                                    ldr, ncols, Ck, ldc, tk);
  const int n = c.Nm + c.n_grains;
  if (c.n_grains > 0) k_restrict_grain_k<NRHS><<<c.n_grains, 256, 0, st>>>(c, tk, gk);
  if (n > 0)
    k_restrict_final_k<NRHS><<<(unsigned)(((int64_t)n * 8 + 255) / 256), 256, 0, st>>>(
        c, c.mortar_iface, r, ldr, ncols, gk, Dck, rm, rc);
}

void launch_restrict_k(const DevCoarse& c, int P, const double* r, int64_t ldr, int ncols,
                       const double* Ck, int64_t ldc, const double* Dck, double* tk, double* gk,
                       double* rm, double* rc, cudaStream_t st) {
  if (P == 4) restrict_k<4>(c, r, ldr, ncols, Ck, ldc, Dck, tk, gk, rm, rc, st);
  else if (P == 2) restrict_k<2>(c, r, ldr, ncols, Ck, ldc, Dck, tk, gk, rm, rc, st);
  else restrict_k<1>(c, r, ldr, ncols, Ck, ldc, Dck, tk, gk, rm, rc, st);
}

// ---------------------------------------------------------------------------
// Prolongation x_c = P^_B y_m,c + sum_g c_g,c y_c,c[g]
// ---------------------------------------------------------------------------
// yk[(off_g + j) NRHS + c]: the grain's coarse values (shape columns from y_m,c,
// column L-1 = the correction coefficient y_c,c[g])
template <int NRHS>
__global__ void k_yext_k(DevCoarse c, const double* __restrict__ ym, const double* __restrict__ yc,
                         const double* __restrict__ Dck, int ncols, double* __restrict__ yk) {
  const int g = blockIdx.x;
  const int L = c.ld[g];
  const int32_t* cols = c.gcols + c.gcols_ptr[g];
  double* out = yk + c.yext_off[g] * NRHS;
  for (int t = threadIdx.x; t < L * NRHS; t += blockDim.x) {
    const int j = t / NRHS, q = t - j * NRHS;
    double v = 0.0;
    if (q < ncols) {
      if (j < L - 1) v = ym[(int64_t)q * c.Nm + cols[j]];
      else if (Dck[(int64_t)q * c.n_grains + g] != 0.0) v = yc[(int64_t)q * c.n_grains + g];
    }
    out[t] = v;
  }
}

// Sum of NV values (a power of two <= 32) of every lane over the warp, one
// value per lane group: each halving step keeps half of the values and
// exchanges the other half (NV - 1 + log2(32 / NV) shuffles instead of
// 5 NV); afterwards lanes with (lane & (32 / NV - 1)) == 0 hold the sum of
// value index idx (bits of the lane at offsets 16, 8, ...).
template <int NV>
__device__ __forceinline__ double warp_transpose_sum(double (&v)[NV], int lane, int& idx) {
  idx = 0;
  int o = 16;
#pragma unroll
  for (int h = NV / 2; h >= 1; h >>= 1, o >>= 1) {
    const bool up = lane & o;
    if (up) idx += h;
#pragma unroll
    for (int t = 0; t < h; ++t) {
      const double send = up ? v[t] : v[h + t];
      const double keep = up ? v[h + t] : v[t];
      v[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  return v[0];
}

// grain rows: one CTA per 64-row block, warp =
// ROWS rows, lanes stride the shape columns (coalesced row reads of B_g, read
// ONCE for the NRHS vectors), transposing warp reduction of ROWS x NRHS sums
template <int NRHS>
__global__ void __launch_bounds__(256) k_prolong_rows_k(DevCoarse c, const int32_t* __restrict__ lmap,
                                                        const int32_t* __restrict__ row_s,
                                                        const int64_t* __restrict__ row_base,
                                                        const double* __restrict__ yk,
                                                        const double* __restrict__ Ck, int64_t ldc,
                                                        int ncols, double* __restrict__ x,
                                                        int64_t ldx) {
  // 8 rows per warp for every NRHS (8 NRHS <= 32 accumulators): each y load
  // serves 8 rows (4 rows per warp with NRHS = 4: 23.9 vs 19.5 ms per cfg3 block)
  constexpr int ROWS = 8;
  constexpr int SPLIT = 8 / ROWS;                    // CTAs per 64-row block
  const int64_t ch = blockIdx.x / SPLIT;
  const int half = (int)(blockIdx.x % SPLIT);
  const int g = row_s[ch];
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = c.ld[g];
  const int roff = half * 8 * ROWS + wp * ROWS;      // row of the warp in the 64-row block
  const int64_t lr0 = (ch - row_base[g]) * 64 + roff;
  const double* Bg = c.B + c.b_off[g] + lr0 * L;
  const double* y = yk + c.yext_off[g] * NRHS;
  const int64_t row0 = 64 * ch + roff;               // grain-batch local row
  double a[ROWS * NRHS];
#pragma unroll
  for (int q = 0; q < ROWS * NRHS; ++q) a[q] = 0.0;
  // two column steps per pass: 2 ROWS streaming loads in flight per lane
  int j = lane;
  for (; j + 32 < L - 1; j += 64) {
    double yj[2][NRHS], b[2][ROWS];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
#pragma unroll
      for (int q = 0; q < ROWS; ++q) b[u][q] = __ldcs(Bg + (int64_t)q * L + j + 32 * u);
#pragma unroll
      for (int k = 0; k < NRHS; ++k) yj[u][k] = __ldg(y + (int64_t)(j + 32 * u) * NRHS + k);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < ROWS; ++q)
#pragma unroll
        for (int k = 0; k < NRHS; ++k) a[q * NRHS + k] = fma(b[u][q], yj[u][k], a[q * NRHS + k]);
  }
  for (; j < L - 1; j += 32) {
    double yj[NRHS];
#pragma unroll
    for (int k = 0; k < NRHS; ++k) yj[k] = __ldg(y + (int64_t)j * NRHS + k);
    double b[ROWS];
#pragma unroll
    for (int q = 0; q < ROWS; ++q) b[q] = __ldcs(Bg + (int64_t)q * L + j);
#pragma unroll
    for (int q = 0; q < ROWS; ++q)
#pragma unroll
      for (int k = 0; k < NRHS; ++k) a[q * NRHS + k] = fma(b[q], yj[k], a[q * NRHS + k]);
  }
  int idx;
  const double v = warp_transpose_sum<ROWS * NRHS>(a, lane, idx);
  if ((lane & (32 / (ROWS * NRHS) - 1)) == 0) {
    const int q = idx / NRHS, k = idx - q * NRHS;
    const int d = lmap[row0 + q];
    if (d >= 0 && k < ncols)
      x[k * ldx + d] = v + Ck[k * ldc + row0 + q] * y[(int64_t)(L - 1) * NRHS + k];
  }
}

template <int NRHS>
__global__ void k_prolong_iface_k(DevCoarse c, const double* __restrict__ ym, int ncols,
                                  double* __restrict__ x, int64_t ldx) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int n3 = 3 * c.n_iface_nodes;
  if (e >= n3) return;
  const int en = e / 3, gam = e - 3 * en;
  const int cf = c.iface_of[en];
  const int nu3 = 3 * (c.mortar_ptr[cf + 1] - c.mortar_ptr[cf]);
  const double* w = c.W + c.wt_off[cf] + (int64_t)(3 * (en - c.iface_ptr[cf]) + gam) * nu3;
  const int kb = 3 * c.mortar_ptr[cf];
  double acc[NRHS];
#pragma unroll
  for (int k = 0; k < NRHS; ++k) acc[k] = 0.0;
  for (int q = 0; q < nu3; ++q) {
    const double wq = w[q];
#pragma unroll
    for (int k = 0; k < NRHS; ++k) acc[k] += wq * ym[(int64_t)k * c.Nm + kb + q];
  }
  const int64_t d = 3 * (int64_t)c.iface_nodes[en] + gam;
#pragma unroll
  for (int k = 0; k < NRHS; ++k)
    if (k < ncols) x[k * ldx + d] = acc[k];
}

template <int NRHS>
static void prolong_k(const DevCoarse& c, const double* ym, const double* yc, const double* Dck,
                      const double* Ck, int64_t ldc, int ncols, double* yk, double* x, int64_t ldx,
                      cudaStream_t st) {
  if (c.n_grains > 0) k_yext_k<NRHS><<<c.n_grains, 128, 0, st>>>(c, ym, yc, Dck, ncols, yk);
  if (c.n_chunks > 0)
    k_prolong_rows_k<NRHS><<<(unsigned)c.n_chunks, 256, 0, st>>>(c, c.g_lmap, c.g_row_s,
                                                                 c.g_row_base, yk, Ck, ldc, ncols,
                                                                 x, ldx);
  if (c.n_iface_nodes > 0)
    k_prolong_iface_k<NRHS><<<(3 * c.n_iface_nodes + 255) / 256, 256, 0, st>>>(c, ym, ncols, x, ldx);
}

void launch_prolong_k(const DevCoarse& c, int P, const double* ym, const double* yc,
                      const double* Dck, const double* Ck, int64_t ldc, int ncols, double* yk,
                      double* x, int64_t ldx, cudaStream_t st) {
  if (P == 4) prolong_k<4>(c, ym, yc, Dck, Ck, ldc, ncols, yk, x, ldx, st);
  else if (P == 2) prolong_k<2>(c, ym, yc, Dck, Ck, ldc, ncols, yk, x, ldx, st);
  else prolong_k<1>(c, ym, yc, Dck, Ck, ldc, ncols, yk, x, ldx, st);
}

// yc[c][g] = rc[c][g] / Dc[c][g] (0 where there is no correction column)
__global__ void k_coarse_diag_k(int n, const double* rc, const double* Dck, double* yc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  yc[t] = Dck[t] != 0.0 ? rc[t] / Dck[t] : 0.0;
}

void launch_coarse_diag_k(int n, const double* rc, const double* Dck, double* yc, cudaStream_t st) {
  if (n <= 0) return;
  k_coarse_diag_k<<<(n + 255) / 256, 256, 0, st>>>(n, rc, Dck, yc);
}

// ---------------------------------------------------------------------------
// local-solve scatter / combine for P interleaved right-hand sides
// ---------------------------------------------------------------------------
// out_c[d] = sum over the contact grids containing DOF d of yloc[pos P + c]
__global__ void k_sum_contact_k(int n, int P, int ncols, const int32_t* __restrict__ cptr,
                                const int32_t* __restrict__ cidx, const double* __restrict__ yloc,
                                double* __restrict__ out, int64_t ldo) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int d = (int)(t / P), c = (int)(t - (int64_t)d * P);
  if (d >= n || c >= ncols) return;
  double v = 0.0;
  for (int e = cptr[d]; e < cptr[d + 1]; ++e) v += yloc[(int64_t)cidx[e] * P + c];
  out[c * ldo + d] = v;
}

void launch_sum_contact_k(int n, int P, int ncols, const int32_t* cptr, const int32_t* cidx,
                          const double* yloc, double* out, int64_t ldo, cudaStream_t st) {
  const int64_t th = (int64_t)n * P;
  k_sum_contact_k<<<(unsigned)((th + 255) / 256), 256, 0, st>>>(n, P, ncols, cptr, cidx, yloc, out,
                                                                ldo);
}

// out_c[d] = a_c[d] + b_c[d] + yloc[gpos[d] P + c]   (a, b optional)
__global__ void k_combine_grain_k(int n, int P, int ncols, const int32_t* __restrict__ gpos,
                                  const double* __restrict__ yloc, const double* __restrict__ a,
                                  const double* __restrict__ b, int64_t ld,
                                  double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int d = (int)(t / P), c = (int)(t - (int64_t)d * P);
  if (d >= n || c >= ncols) return;
  double v = 0.0;
  if (a) v += a[c * ld + d];
  if (b) v += b[c * ld + d];
  const int g = gpos[d];
  if (g >= 0) v += yloc[(int64_t)g * P + c];
  out[c * ld + d] = v;
}

void launch_combine_grain_k(int n, int P, int ncols, const int32_t* gpos, const double* yloc,
                            const double* a, const double* b, int64_t ld, double* out,
                            cudaStream_t st) {
  const int64_t th = (int64_t)n * P;
  k_combine_grain_k<<<(unsigned)((th + 255) / 256), 256, 0, st>>>(n, P, ncols, gpos, yloc, a, b, ld,
                                                                  out);
}

}  // namespace hplmm
