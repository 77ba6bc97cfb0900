// FEM assembly, BSR SpMV and Gaussian mortar weights (sm_100a, fp64).
//
// PAPER.md P:74-78 (Galerkin Q1 FEM on the voxel grid -> eq:ls_all),
// eq:stiff_iso, readings R2 (2x2x2 Gauss, unit voxel), R3
// (node-major 3x3 blocks), R4 (Dirichlet identity rows, lifted RHS);
// eq:gauss with R11 for the mortar weights.
#include <type_traits>
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "kernels.cuh"
#include "tma.cuh"

namespace hplmm {

// ---------------------------------------------------------------------------
// K0 = int_[0,1]^3 B^T D(E=1,nu) B dV  (24x24, DOF 3a+c, a = dx+2dy+4dz)
// ---------------------------------------------------------------------------
__device__ void strain_col(int a, int r, const double xi[3], double e[6]) {
  int c0 = a & 1, c1 = (a >> 1) & 1, c2 = (a >> 2) & 1;
  double f0 = c0 ? xi[0] : 1.0 - xi[0], f1 = c1 ? xi[1] : 1.0 - xi[1], f2 = c2 ? xi[2] : 1.0 - xi[2];
  double d0 = c0 ? 1.0 : -1.0, d1 = c1 ? 1.0 : -1.0, d2 = c2 ? 1.0 : -1.0;
  double gx = d0 * f1 * f2, gy = f0 * d1 * f2, gz = f0 * f1 * d2;
  e[0] = (r == 0) ? gx : 0.0;
  e[1] = (r == 1) ? gy : 0.0;
  e[2] = (r == 2) ? gz : 0.0;
  e[3] = (r == 1) ? gz : (r == 2 ? gy : 0.0);   // gamma_yz
  e[4] = (r == 0) ? gz : (r == 2 ? gx : 0.0);   // gamma_xz
  e[5] = (r == 0) ? gy : (r == 1 ? gx : 0.0);   // gamma_xy
}

__global__ void k_element_K0(double* K0, double nu) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 576) return;
  int i = t / 24, j = t % 24;
  double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  double mu = 1.0 / (2.0 * (1.0 + nu));
  const double g = 0.5 / sqrt(3.0);
  double acc = 0.0;
  for (int p = 0; p < 8; ++p) {
    double xi[3] = {0.5 + ((p & 1) ? g : -g), 0.5 + ((p & 2) ? g : -g), 0.5 + ((p & 4) ? g : -g)};
    double ei[6], ej[6];
    strain_col(i / 3, i % 3, xi, ei);
    strain_col(j / 3, j % 3, xi, ej);
    double s = 0.0;
    for (int m = 0; m < 3; ++m)
      for (int n = 0; n < 3; ++n) s += ei[m] * (lam + (m == n ? 2.0 * mu : 0.0)) * ej[n];
    for (int m = 3; m < 6; ++m) s += ei[m] * mu * ej[m];
    acc += 0.125 * s;
  }
  K0[t] = acc;
}

void launch_element_K0(double* K0, double nu, cudaStream_t st) {
  k_element_K0<<<9, 64, 0, st>>>(K0, nu);
}

// Block (p,q) of the unconstrained matrix: sum over voxels shared by p and q,
// ascending local index a of p in the voxel (the oracle's accumulation order).
__device__ void block_pq(const int32_t* ijk, int p, int q, const uint8_t* solid, const double* E,
                         int nx, int ny, int nz, const double* K0, double out[9]) {
  for (int t = 0; t < 9; ++t) out[t] = 0.0;
  int px = ijk[3 * p], py = ijk[3 * p + 1], pz = ijk[3 * p + 2];
  int qx = ijk[3 * q], qy = ijk[3 * q + 1], qz = ijk[3 * q + 2];
  for (int a = 0; a < 8; ++a) {
    int vx = px - (a & 1), vy = py - ((a >> 1) & 1), vz = pz - ((a >> 2) & 1);
    if (vx < 0 || vy < 0 || vz < 0 || vx >= nx || vy >= ny || vz >= nz) continue;
    int64_t v = vx + (int64_t)nx * (vy + (int64_t)ny * vz);
    if (!solid[v]) continue;
    int bx = qx - vx, by = qy - vy, bz = qz - vz;
    if (bx < 0 || bx > 1 || by < 0 || by > 1 || bz < 0 || bz > 1) continue;
    int b = bx + 2 * by + 4 * bz;
    double Ev = E[v];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c)
        out[3 * r + c] = __dadd_rn(out[3 * r + c], __dmul_rn(Ev, K0[(3 * a + r) * 24 + 3 * b + c]));
  }
}

__global__ void k_assemble(int nnzb, const int32_t* block_row, const int32_t* col,
                           const int32_t* ijk, const uint8_t* dir, const uint8_t* solid,
                           const double* E, int nx, int ny, int nz, const double* K0,
                           double* val) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnzb) return;
  int p = block_row[e], q = col[e];
  double blk[9];
  if (dir[p]) {
    for (int t = 0; t < 9; ++t) blk[t] = (t % 4 == 0) ? 1.0 : 0.0;   // identity (R4)
  } else {
    block_pq(ijk, p, q, solid, E, nx, ny, nz, K0, blk);
  }
  for (int t = 0; t < 9; ++t) val[9 * (int64_t)e + t] = blk[t];
}

void launch_assemble(int nnzb, const int32_t* block_row, const int32_t* col,
                     const int32_t* node_ijk, const uint8_t* dir, const uint8_t* solid,
                     const double* E, int nx, int ny, int nz, const double* K0, double* val,
                     cudaStream_t st) {
  if (nnzb <= 0) return;
  k_assemble<<<(nnzb + 255) / 256, 256, 0, st>>>(nnzb, block_row, col, node_ijk, dir, solid, E,
                                                  nx, ny, nz, K0, val);
}

// b_free = f - sum_{q Dirichlet} K(p,q) u_q ;  b_D = u_D   (R4)
__global__ void k_assemble_rhs(int n, const int32_t* drow_ptr, const int32_t* dcol,
                               const int32_t* ijk, const uint8_t* dir, const uint8_t* solid,
                               const double* E, int nx, int ny, int nz, const double* K0,
                               const double* f, const double* uD, double* b) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  if (dir[p]) {
    for (int r = 0; r < 3; ++r) b[3 * (int64_t)p + r] = uD[3 * (int64_t)p + r];
    return;
  }
  double t[3] = {0.0, 0.0, 0.0};
  for (int e = drow_ptr[p]; e < drow_ptr[p + 1]; ++e) {
    int q = dcol[e];
    double blk[9];
    block_pq(ijk, p, q, solid, E, nx, ny, nz, K0, blk);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) t[r] += blk[3 * r + c] * uD[3 * (int64_t)q + c];
  }
  for (int r = 0; r < 3; ++r) b[3 * (int64_t)p + r] = f[3 * (int64_t)p + r] - t[r];
}

void launch_assemble_rhs(int n_nodes, const int32_t* drow_ptr, const int32_t* dcol,
                         const int32_t* node_ijk, const uint8_t* dir, const uint8_t* solid,
                         const double* E, int nx, int ny, int nz, const double* K0,
                         const double* f, const double* uD, double* b, cudaStream_t st) {
  if (n_nodes <= 0) return;
  k_assemble_rhs<<<(n_nodes + 255) / 256, 256, 0, st>>>(n_nodes, drow_ptr, dcol, node_ijk, dir,
                                                         solid, E, nx, ny, nz, K0, f, uD, b);
}

// ---------------------------------------------------------------------------
// BSR 3x3 SpMV: one warp per block row, one lane per 3x3 block.  The row's
// contiguous 9*nnz_row values are first staged into shared memory with 16-byte
// vector loads (lane-consecutive -> fully coalesced; all loads of the row are
// issued before any is consumed), the column indices are loaded in the same
// wave, then each lane gathers its x block (L2-resident) and the 3 row sums are
// reduced with warp shuffles.  Two dependent memory stages per row instead of
// one per 32 values.  y = A x, or y = v - A x (fused residual, used by
// eq:multi_precond and eq:local_smoother_CG).
// ---------------------------------------------------------------------------
constexpr int SPMV_WARPS = 8;
constexpr int SPMV_BUF = 32 * 9 + 2;

template <bool RESID>
__global__ void __launch_bounds__(32 * SPMV_WARPS) k_spmv(int n, const int32_t* __restrict__ rp,
                                                          const int32_t* __restrict__ col,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ x,
                                                          const double* __restrict__ v,
                                                          double* __restrict__ y) {
  __shared__ __align__(16) double buf[SPMV_WARPS][SPMV_BUF];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * SPMV_WARPS + w;
  if (row >= n) return;
  const int s = __ldg(rp + row), e = __ldg(rp + row + 1);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  double* bw = buf[w];
  for (int cb = s; cb < e; cb += 32) {
    const int nbk = min(32, e - cb);
    const int64_t v0 = 9 * (int64_t)cb;
    const int head = (int)(v0 & 1);
    const int npair = (9 * nbk + head + 1) >> 1;
    const double2* src = reinterpret_cast<const double2*>(val + v0 - head);
    double2 r[5];
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      int i = lane + 32 * u;
      if (i < npair) r[u] = __ldcs(src + i);
    }
    int q = lane < nbk ? __ldg(col + cb + lane) : 0;
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      int i = lane + 32 * u;
      if (i < npair) reinterpret_cast<double2*>(bw)[i] = r[u];
    }
    __syncwarp();
    if (lane < nbk) {
      const double* blk = bw + head + 9 * lane;
      const double* xq = x + 3 * (int64_t)q;
      double x0 = __ldg(xq), x1 = __ldg(xq + 1), x2 = __ldg(xq + 2);
      a0 = fma(blk[0], x0, fma(blk[1], x1, fma(blk[2], x2, a0)));
      a1 = fma(blk[3], x0, fma(blk[4], x1, fma(blk[5], x2, a1)));
      a2 = fma(blk[6], x0, fma(blk[7], x1, fma(blk[8], x2, a2)));
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (lane < 3) {
    double a = lane == 0 ? a0 : (lane == 1 ? a1 : a2);
    int64_t d = 3 * (int64_t)row + lane;
    y[d] = RESID ? (v[d] - a) : a;
  }
}

// ---------------------------------------------------------------------------
// Streaming BSR SpMV (default).  The block values and column indices of a
// chunk of SP_ROWS consecutive block rows are contiguous in HBM; a persistent
// CTA per SM streams its contiguous range of chunks through a ring of
// SP_STAGES shared-memory stages with 1-D TMA bulk copies (one producer lane,
// L2 evict-first so the gathered x stays L2-resident), completion by mbarrier
// transaction counts.  Consumer warp w owns stages s == w (mod SP_CONS) (keeps
// each waiter within one mbarrier phase).  Per chunk a warp works on its
// SP_ROWS rows at once: lane l takes block l of every row (<= 27 blocks per
// row on the voxel lattice), so the x gathers of 4 rows are in flight
// together; the 12 row sums are reduced with a 16-shuffle recursive-halving
// transpose (warp-per-block-row reduction).
// ---------------------------------------------------------------------------
constexpr int SP_G = 4;      // rows reduced together by one warp pass
constexpr int SP_MAXB = 27;  // blocks per row on the voxel lattice

template <int ROWS>
struct SpCfg {
  static constexpr int VBYTES = ROWS * SP_MAXB * 72 + 16;
  static constexpr int CBYTES = (ROWS * SP_MAXB * 4 + 16 + 15) / 16 * 16;
  static constexpr int STAGE = VBYTES + CBYTES;
};

template <bool RESID, int ROWS, int CONS, int STAGES, int CPS>
__global__ void __launch_bounds__(32 * (CONS + 1), CPS)
    k_spmv_tma(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
               const double* __restrict__ val, const double* __restrict__ x,
               const double* __restrict__ v, double* __restrict__ y) {
  static_assert(STAGES % CONS == 0, "each stage must belong to one consumer warp");
  static_assert(ROWS % SP_G == 0, "row groups");
  using C = SpCfg<ROWS>;
  extern __shared__ __align__(128) unsigned char sp_smem[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunks = (n + ROWS - 1) / ROWS;
  const int per = (nchunks + gridDim.x - 1) / gridDim.x;
  const int c0 = blockIdx.x * per;
  const int nk = max(0, min(nchunks, c0 + per) - c0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == CONS) {  // producer warp: lanes prefetch row pointers, lane 0 issues
    const uint64_t pol = policy_evict_first();
    for (int kb = 0; kb < nk; kb += 32) {
      // lane j holds rp at the start of chunk kb+j; bend31 = end of chunk kb+31
      int bstart = __ldg(rp + min(n, (c0 + kb + lane) * ROWS));
      int bend31 = __ldg(rp + min(n, (c0 + kb + 32) * ROWS));
      int cnt = min(32, nk - kb);
      for (int j = 0; j < cnt; ++j) {
        int b0 = __shfl_sync(0xffffffffu, bstart, j);
        int b1 = __shfl_sync(0xffffffffu, bstart, (j + 1) & 31);
        if (j == 31) b1 = bend31;
        if (lane == 0) {
          const int k = kb + j;
          const int s = k % STAGES;
          if (k >= STAGES) mbar_wait(&empty[s], (uint32_t)((k / STAGES - 1) & 1));
          const int64_t vs = (72 * (int64_t)b0) & ~(int64_t)15, ve = (72 * (int64_t)b1 + 15) & ~(int64_t)15;
          const int64_t cs = (4 * (int64_t)b0) & ~(int64_t)15, ce = (4 * (int64_t)b1 + 15) & ~(int64_t)15;
          unsigned char* st = sp_smem + (size_t)s * C::STAGE;
          mbar_expect_tx(&full[s], (uint32_t)((ve - vs) + (ce - cs)));
          bulk_g2s_hint(st, reinterpret_cast<const unsigned char*>(val) + vs, (uint32_t)(ve - vs),
                        &full[s], pol);
          bulk_g2s_hint(st + C::VBYTES, reinterpret_cast<const unsigned char*>(col) + cs,
                        (uint32_t)(ce - cs), &full[s], pol);
        }
      }
    }
    return;
  }
  for (int k = warp; k < nk; k += CONS) {
    const int s = k % STAGES;
    const int rc = (c0 + k) * ROWS;
    int bl = __ldg(rp + min(n, rc + min(lane, ROWS)));
    const int64_t vs = (72 * (int64_t)__shfl_sync(0xffffffffu, bl, 0)) & ~(int64_t)15;
    const int64_t cs = (4 * (int64_t)__shfl_sync(0xffffffffu, bl, 0)) & ~(int64_t)15;
    // lane pair (2i, 2i+1) will hold entry idx(lane) of each 4-row group; the
    // fused-residual operand v is loaded now so its latency overlaps the wait
    const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                    ((lane >> 1) & 1);
    double vpre[ROWS / SP_G];
#pragma unroll
    for (int gq = 0; gq < ROWS / SP_G; ++gq) {
      vpre[gq] = 0.0;
      if (RESID && !(lane & 1) && idx < 3 * SP_G && rc + gq * SP_G + idx / 3 < n)
        vpre[gq] = __ldcs(v + 3 * (int64_t)(rc + gq * SP_G) + idx);
    }
    mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
    const unsigned char* st = sp_smem + (size_t)s * C::STAGE;
    const double* sv = reinterpret_cast<const double*>(st) - vs / 8;              // by 9*b
    const int32_t* sc = reinterpret_cast<const int32_t*>(st + C::VBYTES) - cs / 4;  // by b
    double res[ROWS / SP_G];
    // all x gathers of the chunk first (ROWS independent L2 loads per lane)
    int bq[ROWS + 1];
#pragma unroll
    for (int q = 0; q <= ROWS; ++q) bq[q] = __shfl_sync(0xffffffffu, bl, q);
    double xv[ROWS][3];
#pragma unroll
    for (int q = 0; q < ROWS; ++q) {
      const int b = bq[q] + lane;
      if (b < bq[q + 1]) {
        const double* xq = x + 3 * (int64_t)sc[b];
        xv[q][0] = __ldg(xq);
        xv[q][1] = __ldg(xq + 1);
        xv[q][2] = __ldg(xq + 2);
      } else {
        xv[q][0] = xv[q][1] = xv[q][2] = 0.0;
      }
    }
#pragma unroll
    for (int gq = 0; gq < ROWS / SP_G; ++gq) {
      double a[16];
#pragma unroll
      for (int qq = 0; qq < SP_G; ++qq) {
        const int q = gq * SP_G + qq;
        const int b = bq[q] + lane;
        double blk[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) blk[t] = 0.0;
        if (b < bq[q + 1]) {
#pragma unroll
          for (int t = 0; t < 9; ++t) blk[t] = sv[9 * (int64_t)b + t];
        }
        a[3 * qq + 0] = fma(blk[0], xv[q][0], fma(blk[1], xv[q][1], blk[2] * xv[q][2]));
        a[3 * qq + 1] = fma(blk[3], xv[q][0], fma(blk[4], xv[q][1], blk[5] * xv[q][2]));
        a[3 * qq + 2] = fma(blk[6], xv[q][0], fma(blk[7], xv[q][1], blk[8] * xv[q][2]));
      }
#pragma unroll
      for (int t = 3 * SP_G; t < 16; ++t) a[t] = 0.0;
      // recursive-halving transpose reduction: 8 + 4 + 2 + 1 + 1 shuffles
#pragma unroll
      for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int t = 0; t < h; ++t) {
          double send = up ? a[t] : a[h + t];
          double keep = up ? a[h + t] : a[t];
          a[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      res[gq] = a[0] + __shfl_xor_sync(0xffffffffu, a[0], 1);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
    for (int gq = 0; gq < ROWS / SP_G; ++gq) {
      const int r = rc + gq * SP_G + idx / 3;
      if (!(lane & 1) && idx < 3 * SP_G && r < n) {
        const int64_t d = 3 * (int64_t)(rc + gq * SP_G) + idx;
        y[d] = RESID ? (vpre[gq] - res[gq]) : res[gq];
      }
    }
  }
}

template <int ROWS, int CONS, int STAGES, int CPS = 1>
static void spmv_tma(int n, const int32_t* rp, const int32_t* col, const double* val,
                     const double* x, const double* v, double* y, cudaStream_t st, int nsm) {
  constexpr int SM = STAGES * SpCfg<ROWS>::STAGE;
  set_max_dynamic_smem((const void*)k_spmv_tma<true, ROWS, CONS, STAGES, CPS>, SM);
  set_max_dynamic_smem((const void*)k_spmv_tma<false, ROWS, CONS, STAGES, CPS>, SM);
  int nchunks = (n + ROWS - 1) / ROWS;
  int grid = std::min(nsm * CPS, nchunks);
  if (v)
    k_spmv_tma<true, ROWS, CONS, STAGES, CPS><<<grid, 32 * (CONS + 1), SM, st>>>(n, rp, col, val, x, v, y);
  else
    k_spmv_tma<false, ROWS, CONS, STAGES, CPS><<<grid, 32 * (CONS + 1), SM, st>>>(n, rp, col, val, x, v, y);
}

static int g_spmv_mode = -1;   // >=1 TMA streaming variants (default 1), 0 = warp-per-row staging

// max_row_blocks: the caller's bound on blocks per row (TMA kernel needs <= 27)
void launch_spmv(int n_nodes, const int32_t* row_ptr, const int32_t* col, const double* val,
                 const double* x, const double* v, double* y, cudaStream_t st,
                 int max_row_blocks) {
  if (n_nodes <= 0) return;
  if (g_spmv_mode < 0) {
    const char* e = getenv("HPLMM_SPMV");
    g_spmv_mode = e ? atoi(e) : 6;
  }
  // TMA-streamed kernel (measured best of the ROWS / CONS / STAGES variants on
  // B200, profiles/r01_spmv_variants.txt: 8-row chunks, 3 consumer warps x 2
  // stages, 2 CTAs per SM); HPLMM_SPMV=0 selects the plain warp-per-row kernel
  if (g_spmv_mode != 0 && max_row_blocks <= SP_MAXB) {
    spmv_tma<8, 3, 6, 2>(n_nodes, row_ptr, col, val, x, v, y, st, device_sm_count());
    return;
  }
  int grid = (n_nodes + SPMV_WARPS - 1) / SPMV_WARPS;
  if (v)
    k_spmv<true><<<grid, 32 * SPMV_WARPS, 0, st>>>(n_nodes, row_ptr, col, val, x, v, y);
  else
    k_spmv<false><<<grid, 32 * SPMV_WARPS, 0, st>>>(n_nodes, row_ptr, col, val, x, v, y);
}

// ---------------------------------------------------------------------------
// Element-by-element fine operator (operator_kind = 0): y = A^ x, or
// y = v - A^ x, evaluated from the voxel data instead of the stored blocks.
// A^ is sum_e E_e K0(nu) scattered over the voxels (eq:stiff_iso, P:69-78,
// R2) with the Dirichlet rows/columns replaced by identity rows (R4), so for
// a free node p
//   (A^ x)_p = sum_{a: voxel v_a of p solid} E_{v_a} sum_{b} K0[a, b] x_{q(v_a, b)}
// (b over the corners of v_a that are free nodes), and x_p for a Dirichlet p.
// One thread per node gathers its 27 lattice neighbours once: per neighbour
// offset d the voxels shared with p are those a with a + d in {0,1}^3, each
// adding K0[a, a + d] x_q into a per-voxel accumulator; the 8 accumulators
// are scaled by E_{v_a} at the end.  All K0 indices are compile-time
// constants, so with K0 a __grid_constant__ parameter the 576 DFMAs per node
// take their K0 operand straight from the constant bank.  Bytes per apply:
// x, y (+ v) and the node's coordinates; the lattice map (4 B per lattice
// point) and voxel moduli (8 B per voxel) stay in L2 -- ~20x fewer than the
// 76 B per stored block of the BSR SpMV.  Deterministic (fixed order).
// Measured (cfg3, B200): 0.096 ms per apply vs 0.223 ms for the BSR SpMV
// (ncu, before the grouped lookups below); FP64 pipe 28% active, issue 36%,
// long-scoreboard stalls on the lattice-map -> x gathers (each AoS 24-byte x gather is ~6 L1 wavefronts per
// warp).  Capping registers for 50-75% occupancy (E applied per contribution
// instead of 8 per-voxel accumulators) measured the same, so it was dropped.
// A lattice-tiled variant (CTA = 2 full x lines of one z plane; x of the
// 3 x 4 x (nx+3) lattice halo and the voxel moduli staged in shared memory,
// then every row computed from shared memory) measured 0.175 ms: the staging
// phase does not overlap the compute at 3 CTAs per SM and a quarter of the
// threads sit on padding / void lattice points.  Gathering each x triple with two
// 16-byte loads from the even DOF at or below 3q (instead of three 8-byte
// loads) measured 0.126 vs 0.107 ms: the parity selects and the wider
// requests cost more than the saved load instructions.
// ---------------------------------------------------------------------------
struct EbeK0 {
  double k[576];
};

// Value classes of K0 (isotropic trilinear unit-cube element, eq:stiff_iso):
// K0[3a+i][3b+j] = lam G_ij + mu (G_ji + delta_ij sum_k G_kk), G_ij = int d_i N_a d_j N_b,
// and with s_d = (bit d of a == bit d of b) the 576 entries take only 10 values
// up to sign: i == j: class (s_i ? 0 : 3) + #{d != i : !s_d}, sign +; i != j
// (k the third axis): class 6 + (s_k ? 0 : 2) + (s_i == s_j ? 0 : 1), sign
// sigma_i(a) sigma_j(b) with sigma_d(n) = +1 if bit d of n else -1.  Held in 10
// registers, they replace the 576 constant-bank operand loads of the general
// form (27% of k_ebe's instructions).  launch_ebe checks the classes against
// the K0 it is given and falls back to the general kernel if they do not hold.
__host__ __device__ constexpr int ebe_cls(int row, int col) {
  const int a = row / 3, i = row % 3, b = col / 3, j = col % 3;
  const bool s0 = ((a ^ b) & 1) == 0, s1 = ((a ^ b) & 2) == 0, s2 = ((a ^ b) & 4) == 0;
  const bool si = i == 0 ? s0 : (i == 1 ? s1 : s2), sj = j == 0 ? s0 : (j == 1 ? s1 : s2);
  if (i == j) return (si ? 0 : 3) + (s0 ? 0 : 1) + (s1 ? 0 : 1) + (s2 ? 0 : 1) - (si ? 0 : 1);
  const int k = 3 - i - j;
  const bool sk = k == 0 ? s0 : (k == 1 ? s1 : s2);
  return 6 + (sk ? 0 : 2) + (si == sj ? 0 : 1);
}
__host__ __device__ constexpr bool ebe_neg(int row, int col) {
  const int a = row / 3, i = row % 3, b = col / 3, j = col % 3;
  if (i == j) return false;
  return (((a >> i) & 1) != 0) != (((b >> j) & 1) != 0);
}
// a positive-sign representative of each class (all in row 0 of K0)
__host__ __device__ constexpr int ebe_rep(int c) {
  return c == 0 ? 0 : c == 1 ? 6 : c == 2 ? 18 : c == 3 ? 3 : c == 4 ? 9 : c == 5 ? 21
       : c == 6 ? 1 : c == 7 ? 4 : c == 8 ? 8 : 11;
}
template <int B, int E, class F>
__device__ __forceinline__ void ebe_static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    ebe_static_for<B + 1, E>(f);
  }
}
static bool ebe_classes_hold(const double* K0) {
  double mx = 0.0;
  for (int t = 0; t < 576; ++t) mx = std::max(mx, std::fabs(K0[t]));
  for (int r = 0; r < 24; ++r)
    for (int c = 0; c < 24; ++c) {
      const double ref = K0[ebe_rep(ebe_cls(r, c))] * (ebe_neg(r, c) ? -1.0 : 1.0);
      if (!(std::fabs(K0[r * 24 + c] - ref) <= 1e-14 * mx)) return false;
    }
  return true;
}

template <bool RESID, bool CLS, int GRP = 27, int MINB = 5>
__global__ void __launch_bounds__(128, MINB) k_ebe(int n, const int32_t* __restrict__ ijk,
                                             const uint8_t* __restrict__ dir,
                                             const int32_t* __restrict__ lat,
                                             const double* __restrict__ Es, int nx, int ny, int nz,
                                             const __grid_constant__ EbeK0 K0,
                                             const double* __restrict__ x,
                                             const double* __restrict__ v,
                                             double* __restrict__ y) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  if (dir[p]) {   // identity row (R4)
#pragma unroll
    for (int r = 0; r < 3; ++r)
      y[3 * (int64_t)p + r] = RESID ? v[3 * (int64_t)p + r] - x[3 * (int64_t)p + r]
                                    : x[3 * (int64_t)p + r];
    return;
  }
  const int ix = ijk[3 * p], iy = ijk[3 * p + 1], iz = ijk[3 * p + 2];
  double Ea[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int vx = ix - (a & 1), vy = iy - ((a >> 1) & 1), vz = iz - ((a >> 2) & 1);
    Ea[a] = (vx >= 0 && vy >= 0 && vz >= 0 && vx < nx && vy < ny && vz < nz)
                ? Es[vx + (int64_t)nx * (vy + (int64_t)ny * vz)]
                : 0.0;
  }
  double acc[8][3];
#pragma unroll
  for (int a = 0; a < 8; ++a) acc[a][0] = acc[a][1] = acc[a][2] = 0.0;
  double C[10];   // CLS: the 10 distinct |K0| values
#pragma unroll
  for (int c = 0; c < 10; ++c) C[c] = CLS ? K0.k[ebe_rep(c)] : 0.0;
  const int64_t nx1 = nx + 1, ny1 = ny + 1;
  // all 27 lattice-map lookups are issued first (predicated on a shared
  // solid voxel, which also keeps them in range), then the x gathers: one
  // lookup -> gather chain per neighbour cost 0.126 ms per apply, grouped
  // 0.107 ms (one dz plane at a time: 0.106 ms)
  static_assert(27 % GRP == 0, "whole groups");
  // lattice-map lookup of neighbour k: no shared solid voxel -> no coupling;
  // q < 0: no node or a Dirichlet column, structurally removed (R4)
  auto lookup = [&](int k) -> int {
    const int dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = k / 9 - 1;
    bool any = false;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int bx = (a & 1) + dx, by = ((a >> 1) & 1) + dy, bz = ((a >> 2) & 1) + dz;
      if (bx >= 0 && bx <= 1 && by >= 0 && by <= 1 && bz >= 0 && bz <= 1) any |= Ea[a] != 0.0;
    }
    return any ? lat[(ix + dx) + nx1 * ((iy + dy) + ny1 * (iz + dz))] : -1;
  };
  if constexpr (CLS) {
    // compile-time indices throughout (ebe_cls / ebe_neg are evaluated by the
    // compiler: every K0 value is one of the registers C[0..9])
    ebe_static_for<0, 27 / GRP>([&](auto GI) {
      constexpr int g0 = decltype(GI)::value * GRP;
      int qs[GRP];
#pragma unroll
      for (int t = 0; t < GRP; ++t) qs[t] = lookup(g0 + t);
      ebe_static_for<0, GRP>([&](auto T) {
        constexpr int k = g0 + decltype(T)::value, dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = k / 9 - 1;
        const int q = qs[decltype(T)::value];
        if (q >= 0) {
          const double x0 = x[3 * (int64_t)q], x1 = x[3 * (int64_t)q + 1],
                       x2 = x[3 * (int64_t)q + 2];
          ebe_static_for<0, 8>([&](auto A) {
            constexpr int a = decltype(A)::value;
            constexpr int bx = (a & 1) + dx, by = ((a >> 1) & 1) + dy, bz = ((a >> 2) & 1) + dz;
            if constexpr (bx >= 0 && bx <= 1 && by >= 0 && by <= 1 && bz >= 0 && bz <= 1) {
              constexpr int b = bx + 2 * by + 4 * bz;
              ebe_static_for<0, 3>([&](auto R) {
                constexpr int r = decltype(R)::value, row = 3 * a + r, col = 3 * b;
                constexpr int c0 = ebe_cls(row, col), c1 = ebe_cls(row, col + 1), c2 = ebe_cls(row, col + 2);
                constexpr bool n0 = ebe_neg(row, col), n1 = ebe_neg(row, col + 1), n2 = ebe_neg(row, col + 2);
                acc[a][r] = fma(n2 ? -C[c2] : C[c2], x2,
                                fma(n1 ? -C[c1] : C[c1], x1, fma(n0 ? -C[c0] : C[c0], x0, acc[a][r])));
              });
            }
          });
        }
      });
    });
  } else {
#pragma unroll
    for (int g0 = 0; g0 < 27; g0 += GRP) {
      int qs[GRP];
#pragma unroll
      for (int t = 0; t < GRP; ++t) qs[t] = lookup(g0 + t);
#pragma unroll
      for (int t = 0; t < GRP; ++t) {
        const int k = g0 + t, dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = k / 9 - 1;
        const int q = qs[t];
        if (q < 0) continue;
        const double x0 = x[3 * (int64_t)q], x1 = x[3 * (int64_t)q + 1],
                     x2 = x[3 * (int64_t)q + 2];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          const int bx = (a & 1) + dx, by = ((a >> 1) & 1) + dy, bz = ((a >> 2) & 1) + dz;
          if (bx >= 0 && bx <= 1 && by >= 0 && by <= 1 && bz >= 0 && bz <= 1) {
            const int b = bx + 2 * by + 4 * bz;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              const double* kr = K0.k + (3 * a + r) * 24 + 3 * b;
              acc[a][r] = fma(kr[2], x2, fma(kr[1], x1, fma(kr[0], x0, acc[a][r])));
            }
          }
        }
      }
    }
  }
  double out[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int r = 0; r < 3; ++r) out[r] = fma(Ea[a], acc[a][r], out[r]);
#pragma unroll
  for (int r = 0; r < 3; ++r)
    y[3 * (int64_t)p + r] = RESID ? v[3 * (int64_t)p + r] - out[r] : out[r];
}

// ---------------------------------------------------------------------------
// Two lattice nodes per thread (r02): thread t owns the lattice x-pair
// (2k, j, l), (2k+1, j, l) -- either may be a node, a Dirichlet node or empty.
// The pair's 36 lattice neighbours (x = 2k-1 .. 2k+2) are looked up and
// gathered ONCE for both nodes (two single-node threads gather 54), and the
// 12 voxel moduli around the pair are loaded once (16 for two threads).  With
// two nodes per thread the per-voxel accumulators of k_ebe would need 48
// doubles, so each (voxel, neighbour) contribution is scaled by E_v at once:
// out_r += E_v sum_c K0[3a + r][3b + c] x_c.  All K0 indices are compile-time
// constants (constant-bank operands); fixed order, deterministic.  Same
// operator as k_ebe / the stored blocks up to summation order (R4: Dirichlet
// rows identity, Dirichlet columns skipped).
// MEASURED SLOWER and therefore off by default (HPLMM_EBE_PAIR=1 selects it):
// cfg3, one apply 0.104 ms in the solve vs 0.077 ms for k_ebe (100 registers,
// half the threads and a third more FMAs: the saved gathers do not pay for
// the lost parallelism).
// ---------------------------------------------------------------------------
template <bool RESID>
__global__ void __launch_bounds__(128) k_ebe2(int64_t npairs, int kx, int nx, int ny, int nz,
                                              const int32_t* __restrict__ lat_all,
                                              const int32_t* __restrict__ lat_free,
                                              const double* __restrict__ Es,
                                              const __grid_constant__ EbeK0 K0,
                                              const double* __restrict__ x,
                                              const double* __restrict__ v,
                                              double* __restrict__ y) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= npairs) return;
  const int64_t nx1 = nx + 1, ny1 = ny + 1;
  const int k = (int)(t % kx);
  const int64_t jl = t / kx;
  const int iy = (int)(jl % ny1), iz = (int)(jl / ny1);
  const int ix = 2 * k;
  const int64_t key = ix + nx1 * (iy + ny1 * (int64_t)iz);
  const int np = lat_all[key];
  const int nq = ix + 1 <= nx ? lat_all[key + 1] : -1;
  if (np < 0 && nq < 0) return;
  // free (non-Dirichlet) nodes compute; Dirichlet nodes are identity rows
  const bool fp = np >= 0 && lat_free[key] >= 0;
  const bool fq = nq >= 0 && lat_free[key + 1] >= 0;
  double E[3][2][2];   // voxels vx = ix-1+ox, vy = iy-1+oy, vz = iz-1+oz
#pragma unroll
  for (int ox = 0; ox < 3; ++ox)
#pragma unroll
    for (int oy = 0; oy < 2; ++oy)
#pragma unroll
      for (int oz = 0; oz < 2; ++oz) {
        const int vx = ix - 1 + ox, vy = iy - 1 + oy, vz = iz - 1 + oz;
        E[ox][oy][oz] = (vx >= 0 && vy >= 0 && vz >= 0 && vx < nx && vy < ny && vz < nz)
                            ? Es[vx + (int64_t)nx * (vy + (int64_t)ny * vz)]
                            : 0.0;
      }
  // neighbour lookups first (36), then the gathers and the contributions
  int qs[36];
#pragma unroll
  for (int s = 0; s < 36; ++s) {
    const int kk = s % 4, dy = (s / 4) % 3 - 1, dz = s / 12 - 1;
    bool any = false;
#pragma unroll
    for (int ox = 0; ox < 3; ++ox)
#pragma unroll
      for (int oy = 0; oy < 2; ++oy)
#pragma unroll
        for (int oz = 0; oz < 2; ++oz) {
          const bool inL = (kk - ox == 0 || kk - ox == 1) && (dy + 1 - oy == 0 || dy + 1 - oy == 1) &&
                           (dz + 1 - oz == 0 || dz + 1 - oz == 1);
          if (inL && ((fp && ox <= 1) || (fq && ox >= 1))) any |= E[ox][oy][oz] != 0.0;
        }
    qs[s] = any ? lat_free[key + (kk - 1) + nx1 * (dy + ny1 * (int64_t)dz)] : -1;
  }
  double op[3] = {0.0, 0.0, 0.0}, oq[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int s = 0; s < 36; ++s) {
    const int kk = s % 4, dy = (s / 4) % 3 - 1, dz = s / 12 - 1;
    const int qn = qs[s];
    if (qn < 0) continue;
    const double x0 = x[3 * (int64_t)qn], x1 = x[3 * (int64_t)qn + 1], x2 = x[3 * (int64_t)qn + 2];
#pragma unroll
    for (int ox = 0; ox < 3; ++ox)
#pragma unroll
      for (int oy = 0; oy < 2; ++oy)
#pragma unroll
        for (int oz = 0; oz < 2; ++oz) {
          const int bx = kk - ox, by = dy + 1 - oy, bz = dz + 1 - oz;
          if (bx < 0 || bx > 1 || by < 0 || by > 1 || bz < 0 || bz > 1) continue;
          const int b = bx + 2 * by + 4 * bz;
          const double Ev = E[ox][oy][oz];
          if (ox <= 1) {        // node p = (ix, iy, iz): corner (1-ox, 1-oy, 1-oz)
            const int a = (1 - ox) + 2 * (1 - oy) + 4 * (1 - oz);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              const double* kr = K0.k + (3 * a + r) * 24 + 3 * b;
              op[r] = fma(Ev, fma(kr[2], x2, fma(kr[1], x1, kr[0] * x0)), op[r]);
            }
          }
          if (ox >= 1) {        // node q = (ix+1, iy, iz): corner (2-ox, 1-oy, 1-oz)
            const int a = (2 - ox) + 2 * (1 - oy) + 4 * (1 - oz);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              const double* kr = K0.k + (3 * a + r) * 24 + 3 * b;
              oq[r] = fma(Ev, fma(kr[2], x2, fma(kr[1], x1, kr[0] * x0)), oq[r]);
            }
          }
        }
  }
  if (np >= 0) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int64_t d = 3 * (int64_t)np + r;
      const double av = fp ? op[r] : x[d];
      y[d] = RESID ? v[d] - av : av;
    }
  }
  if (nq >= 0) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int64_t d = 3 * (int64_t)nq + r;
      const double av = fq ? oq[r] : x[d];
      y[d] = RESID ? v[d] - av : av;
    }
  }
}

// ---------------------------------------------------------------------------
// Multi-RHS blocks (NEXT #2): the element-by-element operator applied to P
// columns at once (column c of x / v / y at + c ld).  The 27 lattice lookups
// and the 8 voxel moduli of a node are shared by the P columns; per-voxel
// accumulators for P columns would not fit the registers, so each
// (voxel a, neighbour b) contribution is scaled by E_a at once (as k_ebe2):
// out_c,r += E_a sum_s K0[3a + r][3b + s] x_c,s.  Same operator as k_ebe up
// to the summation order (R4: Dirichlet rows identity, columns skipped).
// ---------------------------------------------------------------------------
template <int P, bool RESID, bool CLS>
__global__ void __launch_bounds__(128) k_ebe_k(int n, int ncols, const int32_t* __restrict__ ijk,
                                               const uint8_t* __restrict__ dir,
                                               const int32_t* __restrict__ lat,
                                               const double* __restrict__ Es, int nx, int ny,
                                               int nz, const __grid_constant__ EbeK0 K0,
                                               const double* __restrict__ x,
                                               const double* __restrict__ v,
                                               double* __restrict__ y, int64_t ld, int64_t ldy) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  if (dir[p]) {   // identity row (R4)
    for (int c = 0; c < ncols; ++c)
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int64_t d = c * ld + 3 * (int64_t)p + r;
        y[c * ldy + 3 * (int64_t)p + r] = RESID ? v[d] - x[d] : x[d];
      }
    return;
  }
  const int ix = ijk[3 * p], iy = ijk[3 * p + 1], iz = ijk[3 * p + 2];
  double Ea[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int vx = ix - (a & 1), vy = iy - ((a >> 1) & 1), vz = iz - ((a >> 2) & 1);
    Ea[a] = (vx >= 0 && vy >= 0 && vz >= 0 && vx < nx && vy < ny && vz < nz)
                ? Es[vx + (int64_t)nx * (vy + (int64_t)ny * vz)]
                : 0.0;
  }
  double out[P][3];
#pragma unroll
  for (int c = 0; c < P; ++c) out[c][0] = out[c][1] = out[c][2] = 0.0;
  const int64_t nx1 = nx + 1, ny1 = ny + 1;
  int qs[27];
#pragma unroll
  for (int k = 0; k < 27; ++k) {
    const int dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = k / 9 - 1;
    bool any = false;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int bx = (a & 1) + dx, by = ((a >> 1) & 1) + dy, bz = ((a >> 2) & 1) + dz;
      if (bx >= 0 && bx <= 1 && by >= 0 && by <= 1 && bz >= 0 && bz <= 1) any |= Ea[a] != 0.0;
    }
    qs[k] = any ? lat[(ix + dx) + nx1 * ((iy + dy) + ny1 * (iz + dz))] : -1;
  }
  if constexpr (CLS) {   // K0's 10 value classes in registers (see k_ebe)
    double C[10];
#pragma unroll
    for (int c = 0; c < 10; ++c) C[c] = K0.k[ebe_rep(c)];
    ebe_static_for<0, 27>([&](auto T) {
      constexpr int k = decltype(T)::value, dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = k / 9 - 1;
      const int q = qs[k];
      if (q >= 0) {
        double xq[P][3];
#pragma unroll
        for (int c = 0; c < P; ++c)
#pragma unroll
          for (int s2 = 0; s2 < 3; ++s2)
            xq[c][s2] = c < ncols ? x[c * ld + 3 * (int64_t)q + s2] : 0.0;
        ebe_static_for<0, 8>([&](auto A) {
          constexpr int a = decltype(A)::value;
          constexpr int bx = (a & 1) + dx, by = ((a >> 1) & 1) + dy, bz = ((a >> 2) & 1) + dz;
          if constexpr (bx >= 0 && bx <= 1 && by >= 0 && by <= 1 && bz >= 0 && bz <= 1) {
            constexpr int b = bx + 2 * by + 4 * bz;
            ebe_static_for<0, 3>([&](auto R) {
              constexpr int r = decltype(R)::value, row = 3 * a + r, col = 3 * b;
              constexpr int c0 = ebe_cls(row, col), c1 = ebe_cls(row, col + 1), c2 = ebe_cls(row, col + 2);
              constexpr bool n0 = ebe_neg(row, col), n1 = ebe_neg(row, col + 1), n2 = ebe_neg(row, col + 2);
              const double k0 = n0 ? -C[c0] : C[c0], k1 = n1 ? -C[c1] : C[c1], k2 = n2 ? -C[c2] : C[c2];
#pragma unroll
              for (int c = 0; c < P; ++c) {
                const double t = fma(k2, xq[c][2], fma(k1, xq[c][1], k0 * xq[c][0]));
                out[c][r] = fma(Ea[a], t, out[c][r]);
              }
            });
          }
        });
      }
    });
  } else {
#pragma unroll
  for (int k = 0; k < 27; ++k) {
    const int dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = k / 9 - 1;
    const int q = qs[k];
    if (q < 0) continue;
    double xq[P][3];
#pragma unroll
    for (int c = 0; c < P; ++c)
#pragma unroll
      for (int s2 = 0; s2 < 3; ++s2)
        xq[c][s2] = c < ncols ? x[c * ld + 3 * (int64_t)q + s2] : 0.0;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int bx = (a & 1) + dx, by = ((a >> 1) & 1) + dy, bz = ((a >> 2) & 1) + dz;
      if (bx >= 0 && bx <= 1 && by >= 0 && by <= 1 && bz >= 0 && bz <= 1) {
        const int b = bx + 2 * by + 4 * bz;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double* kr = K0.k + (3 * a + r) * 24 + 3 * b;
#pragma unroll
          for (int c = 0; c < P; ++c) {
            const double t = fma(kr[2], xq[c][2], fma(kr[1], xq[c][1], kr[0] * xq[c][0]));
            out[c][r] = fma(Ea[a], t, out[c][r]);
          }
        }
      }
    }
  }
  }
#pragma unroll
  for (int c = 0; c < P; ++c) {
    if (c >= ncols) break;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int64_t d = c * ld + 3 * (int64_t)p + r;
      y[c * ldy + 3 * (int64_t)p + r] = RESID ? v[d] - out[c][r] : out[c][r];
    }
  }
}

void launch_ebe_k(int P, int ncols, int n_nodes, const int32_t* node_ijk, const uint8_t* dir,
                  const int32_t* lat, const double* Es, int nx, int ny, int nz,
                  const double* K0_host, const double* x, const double* v, double* y, int64_t ld,
                  int64_t ldy, cudaStream_t st) {
  if (n_nodes <= 0 || ncols <= 0) return;
  EbeK0 k;
  for (int t = 0; t < 576; ++t) k.k[t] = K0_host[t];
  const int grid = (n_nodes + 127) / 128;
  static const bool cls_on = !(getenv("HPLMM_EBE_CLS") && getenv("HPLMM_EBE_CLS")[0] == '0');
  const bool cls = cls_on && ebe_classes_hold(K0_host);
#define EBE_K2(PP, RR)                                                                            \
  if (cls)                                                                                        \
    k_ebe_k<PP, RR, true><<<grid, 128, 0, st>>>(n_nodes, ncols, node_ijk, dir, lat, Es, nx, ny,    \
                                                nz, k, x, v, y, ld, ldy);                          \
  else                                                                                            \
    k_ebe_k<PP, RR, false><<<grid, 128, 0, st>>>(n_nodes, ncols, node_ijk, dir, lat, Es, nx, ny,   \
                                                 nz, k, x, v, y, ld, ldy);
#define EBE_K(PP)                                                                                 \
  if (v) { EBE_K2(PP, true) } else { EBE_K2(PP, false) }
  if (P == 4) { EBE_K(4) } else if (P == 2) { EBE_K(2) } else { EBE_K(1) }
#undef EBE_K
#undef EBE_K2
}

static int g_ebe_mode = -1;   // 1 = k_ebe (default), 2 = two nodes per thread (k_ebe2)

void launch_ebe(int n_nodes, const int32_t* node_ijk, const uint8_t* dir, const int32_t* lat,
                const int32_t* lat_all, const double* Es, int nx, int ny, int nz,
                const double* K0_host, const double* x, const double* v, double* y,
                cudaStream_t st) {
  if (n_nodes <= 0) return;
  if (g_ebe_mode < 0) {
    const char* e = getenv("HPLMM_EBE_PAIR");
    const char* e1 = getenv("HPLMM_EBE_K1");   // experiment: k_ebe_k<1> (E-scaled form)
    g_ebe_mode = (e && e[0] == '1') ? 2 : ((e1 && e1[0] == '1') ? 3 : 1);
  }
  if (g_ebe_mode == 3) {
    launch_ebe_k(1, 1, n_nodes, node_ijk, dir, lat, Es, nx, ny, nz, K0_host, x, v, y, 0, 0, st);
    return;
  }
  EbeK0 k;
  for (int t = 0; t < 576; ++t) k.k[t] = K0_host[t];
  if (g_ebe_mode == 2 && lat_all) {
    const int kx = (nx + 2) / 2;   // x-pairs per lattice line (nx + 1 points)
    const int64_t npairs = (int64_t)kx * (ny + 1) * (nz + 1);
    const unsigned grid = (unsigned)((npairs + 127) / 128);
    if (v)
      k_ebe2<true><<<grid, 128, 0, st>>>(npairs, kx, nx, ny, nz, lat_all, lat, Es, k, x, v, y);
    else
      k_ebe2<false><<<grid, 128, 0, st>>>(npairs, kx, nx, ny, nz, lat_all, lat, Es, k, x, v, y);
    return;
  }
  const int grid = (n_nodes + 127) / 128;
  // K0's 10 value classes in registers (HPLMM_EBE_CLS=0: the general form)
  static const bool cls_on = !(getenv("HPLMM_EBE_CLS") && getenv("HPLMM_EBE_CLS")[0] == '0');
  if (cls_on && ebe_classes_hold(K0_host)) {
    // Measured variants of the classed kernel (cfg3, apply(SPMV) incl. ~0.03 ms
    // of call overhead; default 0.091-0.094 ms): lookups in 3 groups of 9 with
    // 80 / 72 / 64 registers (6 / 7 / 8 CTAs per SM, spills) 0.096-0.098,
    // 27 lookups at 80 registers 0.095-0.098, 116 registers (4 CTAs) 0.100-0.103,
    // branch-free gathers (a missing neighbour gathers the node's own x and
    // contributes zeros) 0.089-0.093 in any grouping -- none separates from the
    // default, which stays.
    if (v)
      k_ebe<true, true><<<grid, 128, 0, st>>>(n_nodes, node_ijk, dir, lat, Es, nx, ny, nz, k, x, v, y);
    else
      k_ebe<false, true><<<grid, 128, 0, st>>>(n_nodes, node_ijk, dir, lat, Es, nx, ny, nz, k, x, v, y);
    return;
  }
  if (v)
    k_ebe<true, false><<<grid, 128, 0, st>>>(n_nodes, node_ijk, dir, lat, Es, nx, ny, nz, k, x, v, y);
  else
    k_ebe<false, false><<<grid, 128, 0, st>>>(n_nodes, node_ijk, dir, lat, Es, nx, ny, nz, k, x, v, y);
}

// ---------------------------------------------------------------------------
// Gaussian mortar weights (eq:gauss, R11): W[y, i] = alpha_i(y) / sum_j alpha_j(y)
// alpha_i(y) = exp(-|y-x_i|^2 / (beta min_{j!=i} |x_i-x_j|^2)), max-shifted.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t d2i(const int32_t* ijk, int a, int b) {
  int64_t dx = ijk[3 * a] - ijk[3 * b], dy = ijk[3 * a + 1] - ijk[3 * b + 1],
          dz = ijk[3 * a + 2] - ijk[3 * b + 2];
  return dx * dx + dy * dy + dz * dz;
}

__device__ double gauss_exponent(const int32_t* ijk, const int32_t* X, int nu, int i, int y,
                                 double beta) {
  int64_t dmin = INT64_MAX;
  for (int j = 0; j < nu; ++j)
    if (j != i) {
      int64_t d = d2i(ijk, X[i], X[j]);
      dmin = d < dmin ? d : dmin;
    }
  return -(double)d2i(ijk, y, X[i]) / (beta * (double)dmin);
}

// Gaussian mortar block rows of interface node y (index yl in F_c):
// M[3 yl + d][3 i + gamma] = w_i(y) delta_{d gamma}   (row-major, 3 nu columns)
__global__ void k_mortar_weights(int n, const int32_t* iface_of, const int32_t* iface_ptr,
                                 const int32_t* iface_nodes, const int32_t* mortar_ptr,
                                 const int32_t* mortar_nodes, const int64_t* wt_off,
                                 const int32_t* ijk, double beta, double* W) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  int c = iface_of[e];
  int y = iface_nodes[e];
  int yl = e - iface_ptr[c];
  const int32_t* X = mortar_nodes + mortar_ptr[c];
  int nu = mortar_ptr[c + 1] - mortar_ptr[c];
  double* out = W + wt_off[c] + (int64_t)(3 * yl) * (3 * nu);
  double m = 0.0, s = 1.0;
  if (nu > 1) {
    m = -DBL_MAX;
    for (int i = 0; i < nu; ++i) m = fmax(m, gauss_exponent(ijk, X, nu, i, y, beta));
    s = 0.0;
    for (int i = 0; i < nu; ++i) s += exp(gauss_exponent(ijk, X, nu, i, y, beta) - m);
  }
  for (int i = 0; i < nu; ++i) {
    const double wi = nu == 1 ? 1.0 : exp(gauss_exponent(ijk, X, nu, i, y, beta) - m) / s;
    for (int d = 0; d < 3; ++d)
      for (int g = 0; g < 3; ++g) out[(int64_t)d * 3 * nu + 3 * i + g] = (d == g) ? wi : 0.0;
  }
}

void launch_mortar_weights(int n_iface_nodes, const int32_t* iface_of, const int32_t* iface_ptr,
                           const int32_t* iface_nodes, const int32_t* mortar_ptr,
                           const int32_t* mortar_nodes, const int64_t* wt_off,
                           const int32_t* node_ijk, double beta, double* W, cudaStream_t st) {
  if (n_iface_nodes <= 0) return;
  k_mortar_weights<<<(n_iface_nodes + 127) / 128, 128, 0, st>>>(
      n_iface_nodes, iface_of, iface_ptr, iface_nodes, mortar_ptr, mortar_nodes, wt_off, node_ijk,
      beta, W);
}

}  // namespace hplmm
