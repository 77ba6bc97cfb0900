// Device-side views and launchers of the batched supernodal factors.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "kernels.cuh"
#include "supernodal.h"

namespace hplmm {

// read-only view of one factored batch (device pointers)
struct SnDev {
  const int32_t* sub_n = nullptr;
  const int64_t* sub_base = nullptr;
  const int64_t *sub_fc0 = nullptr, *sub_fc1 = nullptr, *sub_bc0 = nullptr, *sub_bc1 = nullptr;
  const int32_t* gmap = nullptr;   // local position -> global DOF
  const int32_t *sn_w = nullptr, *sn_r = nullptr, *sn_p0 = nullptr, *sn_ldw = nullptr,
                *sn_ldf = nullptr;
  const int64_t* sn_rows_off = nullptr;
  const int32_t* rows = nullptr;
  const double* factor = nullptr;
};

// mode 0: x = in[gmap], out[base+p] = x (one RHS)
// mode 1: shape-vector columns of the grain batch: x[p][c] = in[b_off + bmap*L + c0 + c],
//         out[same] = -x  (L = ld[sub], columns [0, L-1))
// mode 2: several right-hand sides (multi-RHS solves): x[p][c] = in[c ldin + gmap],
//         c < ncols (0 beyond), out[(base+p) NRHS + c] = x[p][c] (interleaved)
struct SnIO {
  int mode = 0;
  int ncols = 1;
  int64_t ldin = 0;
  const double* in = nullptr;
  double* out = nullptr;
  const int32_t* bmap = nullptr;
  const int64_t* b_off = nullptr;
  const int32_t* ld = nullptr;
};

// per-CTA work: items = (subdomain, first RHS column); the CTA's chunk
// descriptors are materialised in traversal order (flags mark item bounds)
struct SnWork {
  int nblocks = 0;
  int cons = 16;                        // consumer warps per CTA (8 => 2 CTAs per SM)
  const int32_t* item_ptr = nullptr;
  const int32_t* item_sub = nullptr;
  const int32_t* item_c0 = nullptr;
  const int64_t* chunk_ptr = nullptr;   // [nblocks+1]
  const SnChunk* chunks = nullptr;      // flat, per CTA contiguous
  // x in global memory (xg != nullptr; used for NRHS > 1): per-CTA slice of
  // xg_stride doubles holding x (max_n even, NRHS interleaved); shared memory
  // then holds the factor ring, x_S of the current supernode (staged per part,
  // max_w) and x_R, so that the 8 x 2 shape fits several columns
  double* xg = nullptr;
  int64_t xg_stride = 0;
  int max_w = 0;
  // subtree-parallel items (split = true; one RHS, x in shared memory): a team
  // of `team` consecutive CTAs shares one subdomain, each member sweeping its
  // own subtree of the nested-dissection tree; x ranges of the common
  // ancestors travel through xbuf, ordered by the one-shot flags xflag (set by
  // the sender, cleared by the receiver).  A member writes out only the x
  // positions [item_lo, item_hi) it owns.  The launch is cooperative: all
  // CTAs are resident together (team = the largest team, for the report).
  bool split = false;
  int team = 1;
  int nteams = 0;                       // subdomains shared by a team
  const int32_t* item_lo = nullptr;
  const int32_t* item_hi = nullptr;
  double* xbuf = nullptr;
  int32_t* xflag = nullptr;
};

// numeric-factorisation view (device pointers)
struct SnNum {
  const int64_t *asm_ptr = nullptr, *asm_e = nullptr;
  const int32_t *asm_u = nullptr, *asm_v = nullptr;
  const int32_t *sn_w = nullptr, *sn_r = nullptr, *sn_parent = nullptr, *sn_ldw = nullptr,
                *sn_ldf = nullptr;
  const int64_t *sn_foff = nullptr, *rel_off = nullptr;
  const int64_t* rows_off = nullptr;
  const int32_t* rows = nullptr;
  const int32_t* rel = nullptr;
  const int64_t* front_off = nullptr;   // per supernode of the current wave
  double* pool = nullptr;
};

// one (subdomain, supernode) of a multi-RHS sweep step
struct SnMrItem {
  int g;          // subdomain
  int sn;         // supernode (global index)
  int n, k;       // subdomain DOFs, right-hand sides
  int64_t base;   // offset of the subdomain's local positions (gmap / lidx)
  int64_t xoff;   // X block of the subdomain (n x k col-major, ld n)
  int64_t toff;   // temporary (h x k col-major, ld h)
};

struct GemmProb {
  const double* A;
  const double* B;
  double* C;
  int m, n, k, lda, ldb, ldc;
  double alpha, beta;
  int transB;
  int transA;     // op(A) = A^T: A stored k x m (lda >= k)
};

// ring stages of a launch shape (cons consumer warps) for these subdomain sizes
int sn_solve_stages(int max_n, int max_r, int nrhs, int chunk, int cons, int max_w, bool xg);
void launch_sn_solve(const SnDev& d, const SnIO& io, const SnWork& wk, int nrhs, int max_n,
                     int max_r, int chunk, int cons, cudaStream_t st);
void launch_front_asm(const int32_t* list, int nlist, const SnNum& nm, const double* val,
                      cudaStream_t st);
void launch_front_ext(const int32_t* list, int nlist, const SnNum& nm, cudaStream_t st);
void launch_front_to_tiles(const DevBatch& b, const int32_t* list, const SnNum& nm,
                           cudaStream_t st);
void launch_tiles_to_finv(const DevBatch& b, const int32_t* list, int nlist, int max_w,
                          const SnNum& nm, double* factor, cudaStream_t st);
// xloc = b[lmap], yloc = ysn[gpos_sn[lmap] P + c] (P interleaved columns of a
// multi-RHS solve; P = 1, c = 0: one RHS)
void launch_sn_to_batch(int64_t nloc, const int32_t* lmap, const int32_t* gpos_sn, const double* b,
                        const double* ysn, double* xloc, double* yloc, cudaStream_t st, int P = 1,
                        int c = 0);
void launch_mr_io(int nitems, const SnMrItem* it, const int32_t* lidx, const int64_t* b_off,
                  const int32_t* ld, const double* R, double* X, double* B, int to_x,
                  cudaStream_t st);
void launch_mr_rows(int nitems, const SnMrItem* it, const SnNum& nm, const int32_t* sn_p0,
                    double* X, double* T, int mode, cudaStream_t st);
// rows headers of every supernode into the factor array
void launch_rows_to_factor(int nsn, const SnNum& nm, double* factor, cudaStream_t st);
void launch_gemm_batched(const GemmProb* probs, const int32_t* work, int nwork, cudaStream_t st);

}  // namespace hplmm
