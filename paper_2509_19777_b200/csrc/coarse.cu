// Coarse space of hPLMM on the GPU (sm_100a, fp64).
//
// PAPER.md eq:mg_struct / eq:WQP, eq:reduced_defs (Q^o),
// eq:all_prolong (P = [B C; I O]).  W is absorbed: P^ columns live
// in the original DOF order.  Per grain g the non-zero rows of P^_B form the
// dense block B_g (|I_g| x k_g, row-major, padded to 64-row blocks) over the
// column set cols_g (R14, option B); the correction vector c^g is stored as the
// extra last column of the same block so that restriction and prolongation
// treat it uniformly (eq:col_cg, R15).  Interface rows of P^_B are the mortar
// weights Q^o (R12).
#include <cstdlib>

#include "kernels.cuh"

namespace hplmm {

__device__ __forceinline__ int grain_col_base(const DevCoarse& c, int g, int iface,
                                              const int32_t* mortar_ptr) {
  int base = 0;
  for (int t = c.giface_ptr[g]; t < c.giface_ptr[g + 1]; ++t) {
    int cc = c.giface[t];
    if (cc == iface) return base;
    base += 3 * (mortar_ptr[cc + 1] - mortar_ptr[cc]);
  }
  return -1;
}

// R_g = A^[I_g, iface] Q^o[:, cols_g]  (one thread per grain DOF row)
__global__ void k_build_R(DevCoarse c, int64_t nloc, const int32_t* lmap, const int32_t* row_s,
                          const int64_t* row_base, const int32_t* rp, const int32_t* col,
                          const double* val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nloc) return;
  int d = lmap[i];
  if (d < 0) return;
  int g = row_s[i >> 6];
  int64_t lr = i - 64 * row_base[g];
  int p = d / 3, r = d - 3 * p;
  int L = c.ld[g];
  double* R = c.R + c.b_off[g] + lr * L;
  for (int e = rp[p]; e < rp[p + 1]; ++e) {
    int q = col[e];
    int cf = c.node_iface[q];
    if (cf < 0) continue;
    int jb = grain_col_base(c, g, cf, c.mortar_ptr);
    if (jb < 0) continue;
    const int nq3 = 3 * (c.mortar_ptr[cf + 1] - c.mortar_ptr[cf]);
    // mortar block rows of node q (3 components): M[3 lq + d][col]
    const double* w = c.W + c.wt_off[cf] + (int64_t)(3 * c.node_local[q]) * nq3;
    const double* a = val + 9 * (int64_t)e + 3 * r;
    for (int col = 0; col < nq3; ++col) {
      const double t = a[0] * w[col] + a[1] * w[nq3 + col] + a[2] * w[2 * nq3 + col];
      R[jb + col] += t;
    }
  }
}

void launch_build_R(const DevCoarse& c, const DevBatch& gb, const int32_t* row_ptr,
                    const int32_t* col, const double* val, cudaStream_t st) {
  if (gb.nloc <= 0) return;
  k_build_R<<<(unsigned)((gb.nloc + 127) / 128), 128, 0, st>>>(c, gb.nloc, gb.lmap, gb.row_s,
                                                               gb.row_base, row_ptr, col, val);
}

// Y_g = A_g B_g + R_g  (overwrites R), one warp per grain DOF row
__global__ void k_grain_AB(DevCoarse c, int64_t nloc, const int32_t* lmap, const int32_t* row_s,
                           const int64_t* row_base, const int32_t* rp, const int32_t* col,
                           const double* val) {
  int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (i >= nloc) return;
  int d = lmap[i];
  if (d < 0) return;
  int g = row_s[i >> 6];
  int64_t lr = i - 64 * row_base[g];
  int p = d / 3, r = d - 3 * p;
  int L = c.ld[g];
  int k = L - 1;
  const double* Bg = c.B + c.b_off[g];
  double* Y = c.R + c.b_off[g] + lr * L;
  for (int j0 = 0; j0 < k; j0 += 32) {
    int j = j0 + lane;
    double acc = 0.0;
    for (int e = rp[p]; e < rp[p + 1]; ++e) {
      int q = col[e];
      if (c.node_iface[q] >= 0 || c.node_owner[q] != g) continue;
      int lq = c.node_local[q];
      const double* a = val + 9 * (int64_t)e + 3 * r;
      if (j < k)
        for (int cc = 0; cc < 3; ++cc) acc += a[cc] * Bg[(int64_t)(3 * lq + cc) * L + j];
    }
    if (j < k) Y[j] += acc;
  }
}

void launch_grain_AB(const DevCoarse& c, const DevBatch& gb, const int32_t* row_ptr,
                     const int32_t* col, const double* val, cudaStream_t st) {
  if (gb.nloc <= 0) return;
  int64_t th = 32 * gb.nloc;
  k_grain_AB<<<(unsigned)((th + 255) / 256), 256, 0, st>>>(c, gb.nloc, gb.lmap, gb.row_s,
                                                           gb.row_base, row_ptr, col, val);
}

// C_g = B_g^T Y_g (k_g x k_g); CTA per (grain, 8-row slab of C_g)
__global__ void k_grain_BtY(DevCoarse c, const int32_t* nb) {
  int g = blockIdx.x;
  int j1 = blockIdx.y * 8;
  int L = c.ld[g], k = L - 1;
  if (j1 >= k) return;
  int nrow = 64 * nb[g];
  const double* Bg = c.B + c.b_off[g];
  const double* Y = c.R + c.b_off[g];
  double* C = c.Cg + c.cg_off[g];
  for (int j2 = threadIdx.x; j2 < k; j2 += blockDim.x) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int row = 0; row < nrow; ++row) {
      double y = Y[(int64_t)row * L + j2];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j1 + u < k) acc[u] += Bg[(int64_t)row * L + j1 + u] * y;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j1 + u < k) C[(int64_t)(j1 + u) * k + j2] = acc[u];
  }
}

void launch_grain_BtY(const DevCoarse& c, const DevBatch& gb, cudaStream_t st) {
  if (c.n_grains <= 0 || c.max_k <= 0) return;
  dim3 grid(c.n_grains, (c.max_k + 7) / 8);
  k_grain_BtY<<<grid, 128, 0, st>>>(c, gb.nb);
}

// Interface-row part of S = P_B^T (A^ P_B):  for every interface DOF d,
//   S[k, :] += Q^o[d,k] * (A^[d,:] P_B)       (one CTA per interface; rows k
// of S belong to exactly one interface, so CTAs never share an entry)
// S entry (k, j) += v: dense row-major (lds > 0), or straight into the packed
// lower 64-tiles of the coarse batch (lds == 0; entries above the diagonal are
// dropped -- S is taken from its lower triangle either way, R16)
__device__ __forceinline__ void s_add(double* S, int64_t lds, int k, int j, double v) {
  if (lds > 0) {
    S[(int64_t)k * lds + j] += v;
  } else if (k >= j) {
    const int64_t I = k >> 6, J = j >> 6;
    S[(I * (I + 1) / 2 + J) * TILE + (k & 63) + 64 * (j & 63)] += v;
  }
}

__global__ void k_S_iface(DevCoarse c, const int32_t* rp, const int32_t* col, const double* val,
                          double* S, int64_t lds) {
  int cf = blockIdx.x;
  const int nu3 = 3 * (c.mortar_ptr[cf + 1] - c.mortar_ptr[cf]);
  int kbase = 3 * c.mortar_ptr[cf];
  for (int e0 = c.iface_ptr[cf]; e0 < c.iface_ptr[cf + 1]; ++e0) {
    int y = c.iface_nodes[e0];
    // rows 3 yl + gam of this interface's mortar block
    const double* My = c.W + c.wt_off[cf] + (int64_t)(3 * (e0 - c.iface_ptr[cf])) * nu3;
    for (int gam = 0; gam < 3; ++gam) {
      const double* wy = My + (int64_t)gam * nu3;   // wy[q]: coefficient of S row kbase + q
      for (int e = rp[y]; e < rp[y + 1]; ++e) {
        int q = col[e];
        const double* a = val + 9 * (int64_t)e + 3 * gam;
        int cq = c.node_iface[q];
        for (int c3 = 0; c3 < 3; ++c3) {
          double aa = a[c3];
          if (cq < 0) {                      // grain row of P_B (class G)
            int g = c.node_owner[q];
            int L = c.ld[g], k = L - 1;
            const double* Brow = c.B + c.b_off[g] + (int64_t)(3 * c.node_local[q] + c3) * L;
            const int32_t* cols = c.gcols + c.gcols_ptr[g];
            for (int t = threadIdx.x; t < nu3 * k; t += blockDim.x) {
              int i = t / k, j = t - i * k;
              if (wy[i] != 0.0) s_add(S, lds, kbase + i, cols[j], wy[i] * aa * Brow[j]);
            }
          } else {                           // interface row of P_B (Q^o)
            const int nq3 = 3 * (c.mortar_ptr[cq + 1] - c.mortar_ptr[cq]);
            const double* wq = c.W + c.wt_off[cq] + (int64_t)(3 * c.node_local[q] + c3) * nq3;
            int qbase = 3 * c.mortar_ptr[cq];
            for (int t = threadIdx.x; t < nu3 * nq3; t += blockDim.x) {
              int i = t / nq3, i2 = t - i * nq3;
              if (wy[i] != 0.0 && wq[i2] != 0.0)
                s_add(S, lds, kbase + i, qbase + i2, wy[i] * aa * wq[i2]);
            }
          }
          __syncthreads();
        }
      }
    }
  }
}

void launch_S_iface(const DevCoarse& c, const int32_t* row_ptr, const int32_t* col,
                    const double* val, double* S, int64_t lds, cudaStream_t st) {
  if (c.n_ifaces <= 0) return;
  k_S_iface<<<c.n_ifaces, 256, 0, st>>>(c, row_ptr, col, val, S, lds);
}

// Grain-row part: S[k, cols_g] += C_g[j_k, :] for g in G(k) ascending
__global__ void k_S_grain(DevCoarse c, double* S, int64_t lds) {
  int kk = blockIdx.x;
  if (kk >= c.Nm) return;
  for (int e = c.mcol_ptr[kk]; e < c.mcol_ptr[kk + 1]; ++e) {
    int g = c.mcol_g[e], jk = c.mcol_j[e];
    int k = c.ld[g] - 1;
    const double* C = c.Cg + c.cg_off[g] + (int64_t)jk * k;
    const int32_t* cols = c.gcols + c.gcols_ptr[g];
    for (int j = threadIdx.x; j < k; j += blockDim.x) s_add(S, lds, kk, cols[j], C[j]);
    __syncthreads();
  }
}

void launch_S_grain(const DevCoarse& c, double* S, int64_t lds, cudaStream_t st) {
  if (c.Nm <= 0) return;
  k_S_grain<<<c.Nm, 128, 0, st>>>(c, S, lds);
}

// ---------------------------------------------------------------------------
// Algebraic mortars (eq:algebra via the Remark P:356, reading R25): column q =
// 3i + gamma of interface c's block solves A~ x_free = -A^[free, (x_i, gamma)]
// on the interface's free (non-mortar) nodes; the constrained rows are 0/1.
// One pass per column q: k_alg_rhs writes the right-hand sides into the
// interface batch's xloc (its packed A~^-1 is then applied by the batched
// SYMV), k_alg_store scatters y_loc and the 0/1 rows into the blocks.
// ---------------------------------------------------------------------------
__global__ void k_alg_rhs(int q, int64_t nloc, const int32_t* __restrict__ lmap,
                          const int32_t* __restrict__ row_s, const int32_t* mortar_ptr,
                          const int32_t* mortar_nodes, const int32_t* rp,
                          const int32_t* col, const double* val, double* xloc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nloc) return;
  const int d = lmap[t];
  double v = 0.0;
  if (d >= 0) {
    const int c = row_s[t >> 6];
    const int nu = mortar_ptr[c + 1] - mortar_ptr[c];
    if (q < 3 * nu) {
      const int x = mortar_nodes[mortar_ptr[c] + q / 3], gam = q % 3;
      const int y = d / 3, r = d - 3 * y;
      for (int e = rp[y]; e < rp[y + 1]; ++e)
        if (col[e] == x) {
          v = -val[9 * (int64_t)e + 3 * r + gam];
          break;
        }
    }
  }
  xloc[t] = v;
}

// free rows from y_loc (interface batch local order = free nodes of F_c in
// ascending order, 3 DOFs each); constrained rows 0/1.  free_pos / con_pos:
// position of each free / mortar node within F_c.
__global__ void k_alg_store(int q, int C, const int32_t* mortar_ptr, const int32_t* free_ptr,
                            const int32_t* free_pos, const int32_t* con_pos,
                            const int64_t* row_base, const int64_t* wt_off,
                            const double* __restrict__ yloc, double* W) {
  const int c = blockIdx.x;
  if (c >= C) return;
  const int nu = mortar_ptr[c + 1] - mortar_ptr[c];
  const int nu3 = 3 * nu;
  if (q >= nu3) return;
  double* M = W + wt_off[c];
  const int nf = free_ptr[c + 1] - free_ptr[c];
  const double* y = yloc + 64 * row_base[c];
  for (int t = threadIdx.x; t < 3 * nf; t += blockDim.x) {
    const int f = free_pos[free_ptr[c] + t / 3];
    M[(int64_t)(3 * f + t % 3) * nu3 + q] = y[t];
  }
  for (int t = threadIdx.x; t < nu3; t += blockDim.x) {
    const int f = con_pos[mortar_ptr[c] + t / 3];
    M[(int64_t)(3 * f + t % 3) * nu3 + q] = (t == q) ? 1.0 : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Surface Algebraic mortars (mortar_kind = 2, reading R29): eq:algebra
// discretised on the voxel faces shared by the interface's two grains (Q1,
// 2x2 Gauss, tangential strain of all 3 components) plus a translation-free
// tie tau (eta_p - eta_q)^2 over the pattern couplings inside F_c.  Each
// interface's operator K_c (3|F| x 3|F|, dense, transient) is assembled by one
// CTA in a fixed order (faces one after the other, then the tie row by row),
// copied into the free-node packed tiles of the interface batch, and its
// constrained columns give the right-hand sides of the constrained solves.
// ---------------------------------------------------------------------------
// face stiffness for E = 1: local components (a, b, n) per node, corners
// (0,0), (1,0), (0,1), (1,1) of (a, b); K = sum_gp 1/4 B^T D B
__device__ __forceinline__ void surf_B(int col, double s, double t, double (&b)[5]) {
  const int k = col / 3, cmp = col % 3;
  const int da = k & 1, db = k >> 1;
  const double fa = da ? s : 1.0 - s, fb = db ? t : 1.0 - t;
  const double dA = (da ? 1.0 : -1.0) * fb, dB = fa * (db ? 1.0 : -1.0);
  for (int i = 0; i < 5; ++i) b[i] = 0.0;
  if (cmp == 0) { b[0] = dA; b[2] = dB; }
  else if (cmp == 1) { b[1] = dB; b[2] = dA; }
  else { b[3] = dA; b[4] = dB; }
}
__global__ void k_surf_K1(double nu, double* K1) {
  const int e = threadIdx.x;
  if (e >= 144) return;
  const int r = e / 12, c = e % 12;
  const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), mu = 1.0 / (2.0 * (1.0 + nu));
  const double D[5][5] = {{lam + 2 * mu, lam, 0, 0, 0}, {lam, lam + 2 * mu, 0, 0, 0},
                          {0, 0, mu, 0, 0}, {0, 0, 0, mu, 0}, {0, 0, 0, 0, mu}};
  const double g = 0.5 / sqrt(3.0);
  const double gp[2] = {0.5 - g, 0.5 + g};
  double acc = 0.0;
  for (int is = 0; is < 2; ++is)
    for (int it = 0; it < 2; ++it) {
      double br[5], bc[5];
      surf_B(r, gp[is], gp[it], br);
      surf_B(c, gp[is], gp[it], bc);
      double v = 0.0;
      for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) v += br[i] * D[i][j] * bc[j];
      acc += 0.25 * v;
    }
  K1[e] = acc;
}
// tau = TIE * mean(E over solid voxels) / (2 (1 + nu)); one block, fixed order
__global__ void k_surf_tau(int64_t nvox, const double* __restrict__ E,
                           const uint8_t* __restrict__ solid, double nu, double tie,
                           double* tau) {
  __shared__ double ss[256], sc[256];
  double a = 0.0, c = 0.0;
  for (int64_t v = threadIdx.x; v < nvox; v += blockDim.x)
    if (solid[v]) { a += E[v]; c += 1.0; }
  ss[threadIdx.x] = a;
  sc[threadIdx.x] = c;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      ss[threadIdx.x] += ss[threadIdx.x + o];
      sc[threadIdx.x] += sc[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *tau = tie * (ss[0] / sc[0]) / (2.0 * (1.0 + nu));
}
__global__ void __launch_bounds__(256) k_surf_assemble(
    const int32_t* __restrict__ iface_ptr, const int32_t* __restrict__ face_ptr,
    const int4* __restrict__ faces, const double* __restrict__ E, const double* __restrict__ K1,
    const int32_t* __restrict__ tie_ptr, const int32_t* __restrict__ tie_q,
    const double* __restrict__ tau_p, const int64_t* __restrict__ koff, double* Kbuf) {
  const int c = blockIdx.x, tid = threadIdx.x;
  const int e0 = iface_ptr[c], nF = iface_ptr[c + 1] - e0, n3 = 3 * nF;
  double* K = Kbuf + koff[c];
  for (int64_t e = tid; e < (int64_t)n3 * n3; e += blockDim.x) K[e] = 0.0;
  __syncthreads();
  for (int f = face_ptr[c]; f < face_ptr[c + 1]; ++f) {
    if (tid < 144) {
      const int4 nd = faces[2 * f], meta = faces[2 * f + 1];
      const int r = tid / 12, q = tid % 12;
      const int node[4] = {nd.x, nd.y, nd.z, nd.w};
      const int cm[3] = {meta.x & 3, (meta.x >> 2) & 3, (meta.x >> 4) & 3};
      const int row = 3 * node[r / 3] + cm[r % 3], col = 3 * node[q / 3] + cm[q % 3];
      const double Ef = 0.5 * (E[meta.y] + E[meta.z]);
      K[(int64_t)row * n3 + col] += Ef * K1[tid];
    }
    __syncthreads();
  }
  const double tau = *tau_p;
  for (int f = tid; f < nF; f += blockDim.x)
    for (int t = tie_ptr[e0 + f]; t < tie_ptr[e0 + f + 1]; ++t) {
      const int q = tie_q[t];
      for (int cc = 0; cc < 3; ++cc) {
        K[(int64_t)(3 * f + cc) * n3 + 3 * f + cc] += tau;
        K[(int64_t)(3 * f + cc) * n3 + 3 * q + cc] -= tau;
      }
    }
}
// free/free block of K_c -> the interface batch's packed tiles
__global__ void __launch_bounds__(256) k_surf_extract(
    int64_t ntiles, const int32_t* __restrict__ tile_s, const int32_t* __restrict__ tile_ij,
    const int32_t* __restrict__ iface_ptr, const int32_t* __restrict__ free_ptr,
    const int32_t* __restrict__ free_pos, const int64_t* __restrict__ koff,
    const double* __restrict__ Kbuf, double* tiles) {
  const int64_t t = blockIdx.x;
  if (t >= ntiles) return;
  const int c = tile_s[t], I = tile_ij[t] >> 16, J = tile_ij[t] & 0xffff;
  const int n3 = 3 * (iface_ptr[c + 1] - iface_ptr[c]);
  const int f0 = free_ptr[c], m3 = 3 * (free_ptr[c + 1] - f0);
  const double* K = Kbuf + koff[c];
  for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
    const int lr = TB * I + (e & 63), lc = TB * J + (e >> 6);
    if (lr < m3 && lc < m3) {
      const int row = 3 * free_pos[f0 + lr / 3] + lr % 3;
      const int col = 3 * free_pos[f0 + lc / 3] + lc % 3;
      tiles[t * TILE + e] = K[(int64_t)row * n3 + col];
    }
  }
}
// right-hand side of constrained column q: -K_c[free, (mortar q/3, component q%3)]
__global__ void k_surf_rhs(int q, int64_t nloc, const int32_t* __restrict__ row_s,
                           const int64_t* __restrict__ row_base,
                           const int32_t* __restrict__ iface_ptr,
                           const int32_t* __restrict__ mortar_ptr,
                           const int32_t* __restrict__ free_ptr,
                           const int32_t* __restrict__ free_pos,
                           const int32_t* __restrict__ con_pos, const int64_t* __restrict__ koff,
                           const double* __restrict__ Kbuf, double* xloc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nloc) return;
  const int c = row_s[t >> 6];
  const int64_t l = t - TB * row_base[c];
  const int f0 = free_ptr[c], m3 = 3 * (free_ptr[c + 1] - f0);
  const int nu3 = 3 * (mortar_ptr[c + 1] - mortar_ptr[c]);
  double v = 0.0;
  if (l < m3 && q < nu3) {
    const int n3 = 3 * (iface_ptr[c + 1] - iface_ptr[c]);
    const int row = 3 * free_pos[f0 + l / 3] + (int)(l % 3);
    const int col = 3 * con_pos[mortar_ptr[c] + q / 3] + q % 3;
    v = -Kbuf[koff[c] + (int64_t)row * n3 + col];
  }
  xloc[t] = v;
}

void launch_surf_operator(int C, const int32_t* iface_ptr, const int32_t* face_ptr,
                          const int4* faces, const double* E, const uint8_t* solid,
                          int64_t nvox, double nu, double tie, const int32_t* tie_ptr,
                          const int32_t* tie_q, const int64_t* koff, double* K1, double* tau,
                          double* Kbuf, cudaStream_t st) {
  if (C <= 0) return;
  k_surf_K1<<<1, 160, 0, st>>>(nu, K1);
  k_surf_tau<<<1, 256, 0, st>>>(nvox, E, solid, nu, tie, tau);
  k_surf_assemble<<<C, 256, 0, st>>>(iface_ptr, face_ptr, faces, E, K1, tie_ptr, tie_q, tau,
                                     koff, Kbuf);
}

void launch_surf_extract(const DevBatch& ab, const int32_t* iface_ptr, const int32_t* free_ptr,
                         const int32_t* free_pos, const int64_t* koff, const double* Kbuf,
                         cudaStream_t st) {
  if (ab.ntiles <= 0) return;
  k_surf_extract<<<(unsigned)ab.ntiles, 256, 0, st>>>(ab.ntiles, ab.tile_s, ab.tile_ij, iface_ptr,
                                                      free_ptr, free_pos, koff, Kbuf, ab.tiles);
}

void launch_surf_rhs(int q, const DevBatch& ab, const int32_t* iface_ptr,
                     const int32_t* mortar_ptr, const int32_t* free_ptr, const int32_t* free_pos,
                     const int32_t* con_pos, const int64_t* koff, const double* Kbuf,
                     cudaStream_t st) {
  if (ab.nloc <= 0) return;
  k_surf_rhs<<<(unsigned)((ab.nloc + 255) / 256), 256, 0, st>>>(
      q, ab.nloc, ab.row_s, ab.row_base, iface_ptr, mortar_ptr, free_ptr, free_pos, con_pos,
      koff, Kbuf, ab.xloc);
}

void launch_alg_rhs(int q, const DevBatch& ab, const int32_t* mortar_ptr,
                    const int32_t* mortar_nodes, const int32_t* rp, const int32_t* col,
                    const double* val, cudaStream_t st) {
  if (ab.nloc <= 0) return;
  k_alg_rhs<<<(unsigned)((ab.nloc + 255) / 256), 256, 0, st>>>(q, ab.nloc, ab.lmap, ab.row_s,
                                                               mortar_ptr, mortar_nodes, rp, col,
                                                               val, ab.xloc);
}

void launch_alg_store(int q, int C, const DevBatch& ab, const int32_t* mortar_ptr,
                      const int32_t* free_ptr, const int32_t* free_pos, const int32_t* con_pos,
                      const int64_t* wt_off, double* W, cudaStream_t st) {
  if (C <= 0) return;
  k_alg_store<<<C, 128, 0, st>>>(q, C, mortar_ptr, free_ptr, free_pos, con_pos, ab.row_base,
                                 wt_off, ab.yloc, W);
}

// ---------------------------------------------------------------------------
// Restriction r_c = P^T r.  Pass 1: per (grain, 128-row chunk) partial
// B_g^T r_g over all ld_g columns (coalesced row-major reads of B).  Pass 2:
// per mortar column k, fixed-order sum over the grains/chunks touching k plus
// the Q^o part; per grain the correction entry c_g^T r_g.
// ---------------------------------------------------------------------------
// 256 threads: warp w sums rows 8w .. 8w+7 of the 64-row chunk for the columns
// j = lane + 32 t (8 independent row loads in flight per column), then the 8
// warp partials of each column are added in warp order through shared memory.
constexpr int RS_MAXL = 640;   // columns kept in shared memory per pass
__global__ void __launch_bounds__(256) k_restrict_chunks(DevCoarse c, const int32_t* lmap,
                                                         const int64_t* row_base,
                                                         const double* __restrict__ r) {
  const int64_t ch = blockIdx.x;           // chunk = one 64-row block of a grain
  if (ch >= c.n_chunks) return;
  const int g = c.chunk_g[ch];
  const int r0 = c.chunk_r0[ch];
  const int L = c.ld[g];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* Bg = c.B + c.b_off[g] + (int64_t)(r0 + 8 * w) * L;
  const int32_t* lm = lmap + 64 * row_base[g];
  __shared__ double rv[64];
  __shared__ double part[8][RS_MAXL + 1];
  if (threadIdx.x < 64) {
    const int d = lm[r0 + threadIdx.x];
    rv[threadIdx.x] = d >= 0 ? r[d] : 0.0;
  }
  __syncthreads();
  double rr[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) rr[q] = rv[8 * w + q];
  double* out = c.tpart + c.chunk_t[ch];
  for (int j0 = 0; j0 < L; j0 += RS_MAXL) {
    const int jn = min(RS_MAXL, L - j0);
    for (int jj = lane; jj < jn; jj += 32) {
      const double* col = Bg + j0 + jj;
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldcs(col + (int64_t)q * L);
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) a = fma(v[q], rr[q], a);
      part[w][jj] = a;
    }
    __syncthreads();
    for (int jj = threadIdx.x; jj < jn; jj += blockDim.x) {
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) a += part[q][jj];
      out[j0 + jj] = a;
    }
    __syncthreads();
  }
}

// per grain: gpart[j] = sum over its 64-row chunks of tpart.  One CTA per (grain,
// 32-column tile): lane = column, warp w sums the chunks w, w + 8, ... (two
// interleaved partial sums), then warp 0 adds the 8 warp sums in order (fixed
// order; a single thread per column walking all ~100 chunks of a grain was a
// 26-step dependent load chain: 29 us per launch at cfg3)
__global__ void __launch_bounds__(256) k_restrict_grain(DevCoarse c) {
  const int g = blockIdx.x;
  const int L = c.ld[g];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.y * 32 + lane;
  const int c0 = c.chunk_ptr[g], c1 = c.chunk_ptr[g + 1];
  if (blockIdx.y * 32 >= L || c1 <= c0) return;
  __shared__ double red[8][32];
  const double* t = c.tpart + c.chunk_t[c0];
  const int nch = c1 - c0;
  double a0 = 0.0, a1 = 0.0;
  if (j < L) {
    int ch = w;
    for (; ch + 8 < nch; ch += 16) {
      a0 += t[(int64_t)ch * L + j];
      a1 += t[(int64_t)(ch + 8) * L + j];
    }
    if (ch < nch) a0 += t[(int64_t)ch * L + j];
  }
  red[w][lane] = a0 + a1;
  __syncthreads();
  if (w == 0 && j < L) {
    double a = red[0][lane];
#pragma unroll
    for (int q = 1; q < 8; ++q) a += red[q][lane];
    c.gpart[c.yext_off[g] + j] = a;
  }
}

// rm[k] = sum over grains of the pre-summed B_g^T r parts + the interface term
// Q^o[:, k]^T r.  RF_W warps per interface split its rows; each lane keeps the
// partial sums of all the interface's 3 nu mortar columns (r read once per
// row, not once per column), one transposing butterfly per warp, then the
// RF_W warp sums in order through shared memory (fixed order).  rc[g] =
// correction part.  NV = 3 nu rounded up to 16 / 32.
constexpr int RF_W = 4;
template <int NV>
__global__ void __launch_bounds__(256) k_restrict_final(DevCoarse c, const double* r, double* rm,
                                                        double* rc) {
  constexpr int IPB = 8 / RF_W;   // interfaces per 256-thread block
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wi = w / RF_W, wq = w % RF_W;
  const int nbi = (c.n_ifaces + IPB - 1) / IPB;
  __shared__ double red[8][NV];
  if ((int)blockIdx.x >= nbi) {   // correction parts
    const int g = ((int)blockIdx.x - nbi) * 256 + threadIdx.x;
    if (g < c.n_grains) rc[g] = c.Dc[g] != 0.0 ? c.gpart[c.yext_off[g] + c.ld[g] - 1] : 0.0;
    return;
  }
  const int cf = blockIdx.x * IPB + wi;
  const bool live = cf < c.n_ifaces;
  int nu3 = 0, kb = 0, e0 = 0, e1 = 0;
  const double* W = nullptr;
  if (live) {
    nu3 = 3 * (c.mortar_ptr[cf + 1] - c.mortar_ptr[cf]);
    kb = 3 * c.mortar_ptr[cf];
    W = c.W + c.wt_off[cf];
    e0 = c.iface_ptr[cf];
    e1 = c.iface_ptr[cf + 1];
  }
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  for (int e = e0 + wq * 32 + lane; e < e1; e += 32 * RF_W) {
    const double* ry = r + 3 * (int64_t)c.iface_nodes[e];
    const double r0 = ry[0], r1 = ry[1], r2 = ry[2];
    const double* wr = W + 3 * (int64_t)(e - e0) * nu3;
#pragma unroll
    for (int q = 0; q < NV; ++q)
      if (q < nu3) acc[q] += wr[q] * r0 + wr[nu3 + q] * r1 + wr[2 * nu3 + q] * r2;
  }
  int idx = 0, o = 16;
#pragma unroll
  for (int h = NV / 2; h >= 1; h >>= 1, o >>= 1) {
    const bool up = lane & o;
    if (up) idx += h;
#pragma unroll
    for (int t = 0; t < h; ++t) {
      const double send = up ? acc[t] : acc[h + t];
      const double keep = up ? acc[h + t] : acc[t];
      acc[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (; o > 0; o >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
  if ((lane & (32 / NV - 1)) == 0) red[w][idx] = acc[0];
  __syncthreads();
  if (live && wq == 0 && lane < nu3) {
    const int k = kb + lane;
    double a = red[wi * RF_W][lane];
#pragma unroll
    for (int t = 1; t < RF_W; ++t) a += red[wi * RF_W + t][lane];
    for (int e = c.mcol_ptr[k]; e < c.mcol_ptr[k + 1]; ++e)
      a += c.gpart[c.yext_off[c.mcol_g[e]] + c.mcol_j[e]];
    rm[k] = a;
  }
}

// generic form (any 3 nu, e.g. the full-cap case nu_c = |F_c|): RF_LPC lanes per
// mortar column.  rm[k] = sum over grains of the pre-summed B_g^T r parts + the interface term
// Q^o[:, k]^T r; RF_LPC lanes per column split the interface rows (fixed
// order: lane-strided partial sums, then a butterfly), rc[g] = correction part
constexpr int RF_LPC = 8;
__global__ void k_restrict_final_lpc(DevCoarse c, const int32_t* mortar_iface, const double* r,
                                 double* rm, double* rc) {
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int k = (int)(gt / RF_LPC), sl = (int)(gt % RF_LPC);
  double acc = 0.0;
  if (k < c.Nm) {
    const int m = k / 3;
    const int cf = mortar_iface[m];
    const int nu3 = 3 * (c.mortar_ptr[cf + 1] - c.mortar_ptr[cf]);
    const int q = k - 3 * c.mortar_ptr[cf];   // column of the interface block
    const double* w = c.W + c.wt_off[cf] + q;
    const int e0 = c.iface_ptr[cf], e1 = c.iface_ptr[cf + 1];
    for (int e = e0 + sl; e < e1; e += RF_LPC) {
      const int64_t row = 3 * (int64_t)(e - e0);
      const double* ry = r + 3 * (int64_t)c.iface_nodes[e];
      acc += w[row * nu3] * ry[0] + w[(row + 1) * nu3] * ry[1] + w[(row + 2) * nu3] * ry[2];
    }
  }
  // every lane of the warp takes part (the grid is a whole number of warps)
#pragma unroll
  for (int o = RF_LPC / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, RF_LPC);
  if (sl != 0) return;
  if (k < c.Nm) {
    for (int e = c.mcol_ptr[k]; e < c.mcol_ptr[k + 1]; ++e) {
      int g = c.mcol_g[e], j = c.mcol_j[e];
      acc += c.gpart[c.yext_off[g] + j];
    }
    rm[k] = acc;
  } else if (k < c.Nm + c.n_grains) {
    int g = k - c.Nm;
    double v = 0.0;
    if (c.Dc[g] != 0.0) v = c.gpart[c.yext_off[g] + c.ld[g] - 1];
    rc[g] = v;
  }
}

void launch_restrict(const DevCoarse& c, const double* r, double* rm, double* rc,
                     cudaStream_t st) {
  if (c.n_chunks > 0)
    k_restrict_chunks<<<(unsigned)c.n_chunks, 256, 0, st>>>(c, c.g_lmap, c.g_row_base, r);
  if (c.n_grains > 0)
    k_restrict_grain<<<dim3((unsigned)c.n_grains, (unsigned)((c.max_ld + 31) / 32)), 256, 0, st>>>(c);
  const int nb = (c.n_ifaces + 8 / RF_W - 1) / (8 / RF_W) + (c.n_grains + 255) / 256;
  if (nb > 0) {
    if (c.max_nu3 <= 16) k_restrict_final<16><<<nb, 256, 0, st>>>(c, r, rm, rc);
    else if (c.max_nu3 <= 32) k_restrict_final<32><<<nb, 256, 0, st>>>(c, r, rm, rc);
    else
      k_restrict_final_lpc<<<(unsigned)(((int64_t)(c.Nm + c.n_grains) * RF_LPC + 255) / 256), 256,
                             0, st>>>(c, c.mortar_iface, r, rm, rc);
  }
}

// ---------------------------------------------------------------------------
// Prolongation x = P_B y_m + sum_g c^g y_c[g]
// ---------------------------------------------------------------------------
__global__ void k_yext(DevCoarse c, const double* ym, const double* yc) {
  int g = blockIdx.x;
  int L = c.ld[g];
  const int32_t* cols = c.gcols + c.gcols_ptr[g];
  double* out = c.yext + c.yext_off[g];
  for (int j = threadIdx.x; j < L; j += blockDim.x)
    out[j] = (j < L - 1) ? ym[cols[j]] : (c.Dc[g] != 0.0 ? yc[g] : 0.0);
}

__global__ void __launch_bounds__(256) k_prolong(DevCoarse c, const int32_t* gpos,
                                                 const int32_t* row_s, const int64_t* row_base,
                                                 const double* __restrict__ ym,
                                                 double* __restrict__ x) {
  int64_t d = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (d >= c.n_dof) return;
  int gp = gpos[d];
  if (gp >= 0) {
    int g = row_s[gp >> 6];
    int64_t lr = gp - 64 * row_base[g];
    int L = c.ld[g];
    const double* Brow = c.B + c.b_off[g] + lr * L;
    const double* y = c.yext + c.yext_off[g];
    double acc = 0.0;
    for (int j = lane; j < L; j += 32) acc += __ldcs(Brow + j) * y[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) x[d] = acc;
  } else if (lane == 0) {
    int p = (int)(d / 3), gam = (int)(d - 3 * p);
    int cf = c.node_iface[p];
    const int nu3 = 3 * (c.mortar_ptr[cf + 1] - c.mortar_ptr[cf]);
    const double* w = c.W + c.wt_off[cf] + (int64_t)(3 * c.node_local[p] + gam) * nu3;
    int kb = 3 * c.mortar_ptr[cf];
    double acc = 0.0;
    for (int q = 0; q < nu3; ++q) acc += w[q] * ym[kb + q];
    x[d] = acc;
  }
}

// Grain rows in the grain batch's local order (B_g rows are contiguous): one
// CTA per 64-row block of a grain, each warp 8 rows at once (lane-strided
// coalesced row reads, 8 independent dot products in flight), 9-shuffle
// transpose reduction, scatter to x through lmap.  Interface rows separately.
constexpr int PR_ROWS = 8;
__global__ void __launch_bounds__(256) k_prolong_rows(DevCoarse c, const int32_t* __restrict__ lmap,
                                                      const int32_t* __restrict__ row_s,
                                                      const int64_t* __restrict__ row_base,
                                                      double* __restrict__ x) {
  const int64_t ch = blockIdx.x;
  const int g = row_s[ch];
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = c.ld[g];
  const int64_t lr0 = (ch - row_base[g]) * 64 + wp * PR_ROWS;   // local row of the grain
  const double* Bg = c.B + c.b_off[g] + lr0 * L;
  const double* y = c.yext + c.yext_off[g];
  const int32_t* lm = lmap + 64 * ch + wp * PR_ROWS;
  double a[PR_ROWS];
#pragma unroll
  for (int q = 0; q < PR_ROWS; ++q) a[q] = 0.0;
  for (int j = lane; j < L; j += 32) {
    const double yj = __ldg(y + j);
#pragma unroll
    for (int q = 0; q < PR_ROWS; ++q) a[q] = fma(__ldcs(Bg + (int64_t)q * L + j), yj, a[q]);
  }
#pragma unroll
  for (int h = 4, o = 16; h >= 1; h >>= 1, o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int t = 0; t < h; ++t) {
      double send = up ? a[t] : a[h + t];
      double keep = up ? a[h + t] : a[t];
      a[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  a[0] += __shfl_xor_sync(0xffffffffu, a[0], 2);
  a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
  const int q = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  if ((lane & 3) == 0) {
    const int d = lm[q];
    if (d >= 0) x[d] = a[0];
  }
}

__global__ void k_prolong_iface(DevCoarse c, const double* __restrict__ ym, double* __restrict__ x) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  int n3 = 3 * c.n_iface_nodes;
  if (e >= n3) return;
  int en = e / 3, gam = e - 3 * en;
  int cf = c.iface_of[en];
  const int nu3 = 3 * (c.mortar_ptr[cf + 1] - c.mortar_ptr[cf]);
  const double* w = c.W + c.wt_off[cf] + (int64_t)(3 * (en - c.iface_ptr[cf]) + gam) * nu3;
  int kb = 3 * c.mortar_ptr[cf];
  // two interleaved partial sums (fixed order): half the dependent FMA chain
  double a0 = 0.0, a1 = 0.0;
  int q = 0;
  for (; q + 1 < nu3; q += 2) {
    a0 += w[q] * ym[kb + q];
    a1 += w[q + 1] * ym[kb + q + 1];
  }
  if (q < nu3) a0 += w[q] * ym[kb + q];
  x[3 * (int64_t)c.iface_nodes[en] + gam] = a0 + a1;
}

static int g_prolong_mode = -1;

void launch_prolong(const DevCoarse& c, const double* ym, const double* yc, double* x,
                    cudaStream_t st) {
  if (g_prolong_mode < 0) {
    const char* e = getenv("HPLMM_PROLONG");
    g_prolong_mode = (e && e[0] == '0') ? 0 : 1;
  }
  if (c.n_grains > 0) k_yext<<<c.n_grains, 128, 0, st>>>(c, ym, yc);
  if (g_prolong_mode == 1) {
    if (c.n_chunks > 0)
      k_prolong_rows<<<(unsigned)c.n_chunks, 256, 0, st>>>(c, c.g_lmap, c.g_row_s, c.g_row_base, x);
    if (c.n_iface_nodes > 0)
      k_prolong_iface<<<(3 * c.n_iface_nodes + 255) / 256, 256, 0, st>>>(c, ym, x);
    return;
  }
  int64_t th = 32 * (int64_t)c.n_dof;
  k_prolong<<<(unsigned)((th + 255) / 256), 256, 0, st>>>(c, c.gpos, c.g_row_s, c.g_row_base, ym,
                                                          x);
}

__global__ void k_coarse_diag(int G, const double* rc, const double* Dc, double* yc) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  yc[g] = Dc[g] != 0.0 ? rc[g] / Dc[g] : 0.0;
}

void launch_coarse_diag(int G, const double* rc, const double* Dc, double* yc, cudaStream_t st) {
  if (G <= 0) return;
  k_coarse_diag<<<(G + 127) / 128, 128, 0, st>>>(G, rc, Dc, yc);
}

// c^g = A_g^-1 b^g is in the grain batch's yloc (b^g in xloc).  Keep it only if
// b^g != 0 exactly (R15); D_c[g] = b^g . c^g (R16).
__global__ void k_set_correction(DevCoarse c, const int32_t* nb, const int64_t* row_base,
                                 const double* xloc, const double* yloc) {
  int g = blockIdx.x;
  int n = 64 * nb[g];
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
  int keep = anynz;
  int L = c.ld[g];
  double* Bg = c.B + c.b_off[g] + (L - 1);
  for (int i = threadIdx.x; i < n; i += blockDim.x) Bg[(int64_t)i * L] = keep ? y[i] : 0.0;
  if (threadIdx.x == 0) c.Dc[g] = keep ? red[0] : 0.0;
}

void launch_set_correction(const DevCoarse& c, const DevBatch& gb, cudaStream_t st) {
  if (c.n_grains <= 0) return;
  k_set_correction<<<c.n_grains, 256, 0, st>>>(c, gb.nb, gb.row_base, gb.xloc, gb.yloc);
}

}  // namespace hplmm
