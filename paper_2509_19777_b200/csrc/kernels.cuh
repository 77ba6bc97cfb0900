// Kernel launchers of libhplmm (internal).  All fp64, sm_100a.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace hplmm {

constexpr int TB = 64;              // dense tile edge (packed lower-tile storage)
constexpr int TILE = TB * TB;       // doubles per tile
constexpr int SWEEP_M = 2;          // pivot tiles per blocked sweep pass (dense.cu); setup buffers sized for it

// A batch of dense SPD subdomain matrices stored as packed lower 64x64 tiles
// (tile (I,J), J<=I, col-major; diagonal tiles full).  Used for the grain
// blocks A_g, the contact-grid blocks A^[zeta,zeta] and the coarse block S.
struct DevBatch {
  int nsub = 0;
  int max_nb = 0;
  int64_t ntiles = 0;     // sum nb(nb+1)/2
  int64_t nrows = 0;      // sum nb   (row blocks)
  int64_t nloc = 0;       // sum 64 nb (padded local entries)
  int32_t* nb = nullptr;          // [nsub]
  int32_t* ndof = nullptr;        // [nsub]
  int64_t* tile_base = nullptr;   // [nsub]
  int64_t* row_base = nullptr;    // [nsub]  (= loc_off / 64)
  int32_t* tile_s = nullptr;      // [ntiles]
  int32_t* tile_ij = nullptr;     // [ntiles] (I<<16)|J
  int32_t* row_s = nullptr;       // [nrows]
  int32_t* row_k = nullptr;       // [nrows]
  int32_t* lmap = nullptr;        // [nloc] global index or -1 (padding)
  double* tiles = nullptr;        // [ntiles*TILE]
  double* part_row = nullptr;     // [ntiles*64]
  double* part_col = nullptr;     // [ntiles*64]
  double* xloc = nullptr;         // [nloc]
  double* yloc = nullptr;         // [nloc]
  double* dinv = nullptr;         // [nsub*TILE]   (setup only)
  double* cbuf = nullptr;         // [nrows*TILE]  (setup only)
  double* wbuf = nullptr;         // [nrows*TILE]  (setup only)
  int32_t* err = nullptr;         // [1] first failing subdomain (INT_MAX = none)
};

// ---- FEM (fem.cu) ----------------------------------------------------------
void launch_element_K0(double* K0, double nu, cudaStream_t st);
void launch_assemble(int nnzb, const int32_t* block_row, const int32_t* col,
                     const int32_t* node_ijk, const uint8_t* dir, const uint8_t* solid,
                     const double* E, int nx, int ny, int nz, const double* K0, double* val,
                     cudaStream_t st);
void launch_assemble_rhs(int n_nodes, const int32_t* drow_ptr, const int32_t* dcol,
                         const int32_t* node_ijk, const uint8_t* dir, const uint8_t* solid,
                         const double* E, int nx, int ny, int nz, const double* K0,
                         const double* f, const double* uD, double* b, cudaStream_t st);
// y = A x            (v == nullptr)
// y = v - A x        (v != nullptr)
// max_row_blocks: largest row length in blocks (<= 27 on the voxel lattice
// selects the TMA streaming kernel); col and val need 16 bytes of tail padding.
void launch_spmv(int n_nodes, const int32_t* row_ptr, const int32_t* col, const double* val,
                 const double* x, const double* v, double* y, cudaStream_t st,
                 int max_row_blocks);
// Element-by-element A^ (operator_kind = 0; same y = A^ x / y = v - A^ x as
// launch_spmv).  lat: lattice point -> free node id, -1 for no node or a
// Dirichlet node; Es: E per voxel, 0 where void; K0_host: 576 doubles (host)
// multi-RHS blocks: P (1, 2, 4) columns at once, column c at x / v + c ld, y + c ldy
void launch_ebe_k(int P, int ncols, int n_nodes, const int32_t* node_ijk, const uint8_t* dir,
                  const int32_t* lat, const double* Es, int nx, int ny, int nz,
                  const double* K0_host, const double* x, const double* v, double* y, int64_t ld,
                  int64_t ldy, cudaStream_t st);
void launch_ebe(int n_nodes, const int32_t* node_ijk, const uint8_t* dir, const int32_t* lat,
                const int32_t* lat_all,
                const double* Es, int nx, int ny, int nz, const double* K0_host, const double* x,
                const double* v, double* y, cudaStream_t st);
void launch_mortar_weights(int n_iface_nodes, const int32_t* iface_of, const int32_t* iface_ptr,
                           const int32_t* iface_nodes, const int32_t* mortar_ptr,
                           const int32_t* mortar_nodes, const int64_t* wt_off,
                           const int32_t* node_ijk, double beta, double* W, cudaStream_t st);

// ---- dense batched local operators (dense.cu) --------------------------------
void launch_extract_local(const DevBatch& b, int nsub_nodes_total, const int32_t* sub_node_ptr,
                          const int32_t* sub_nodes, const int32_t* row_ptr, const int32_t* col,
                          const double* val, cudaStream_t st);
void launch_pad_identity(const DevBatch& b, cudaStream_t st);
// Sweep-operator inversion (packed tiles in place): A <- A^-1.
// Returns via b.err the first subdomain with a non-positive pivot.
void launch_sweep_invert(const DevBatch& b, cudaStream_t st);
// y_loc = A x_loc for every subdomain (x_loc gathered from x through lmap).
void launch_gather(const DevBatch& b, const double* x, cudaStream_t st);
void launch_symv(const DevBatch& b, cudaStream_t st);
void launch_symv_tiles(const DevBatch& b, cudaStream_t st);
void launch_symv_reduce(const DevBatch& b, cudaStream_t st);
// multi-RHS blocks: P-column SYMV (tiles streamed once; k_symv_tma<P>) and
// gather; column c at xk / yk + c nloc, partials at prk / pck + c ntiles 64
void launch_symv_k(const DevBatch& b, int P, int ncols, const double* xk, double* yk, double* prk,
                   double* pck, cudaStream_t st);
void launch_gather_k(const DevBatch& b, int ncols, const double* x, int64_t xld, double* xk,
                     cudaStream_t st);
// C = -(A^-1 X) for grain batch:  X row-major [64 nb x ld], cols [0,k)
void launch_symm_neg(const DevBatch& b, const int64_t* x_off, const int32_t* ld,
                     const int32_t* kcols, int max_kchunks, const double* X, double* B,
                     cudaStream_t st);
void launch_pack_dense(const DevBatch& b, const double* S, int64_t lds, cudaStream_t st);

// ---- coarse space (coarse.cu) ----------------------------------------------
struct DevCoarse {
  int n_grains = 0, n_ifaces = 0, Nm = 0;
  int n_dof = 0;
  int32_t* grain_node_ptr = nullptr;   // [G+1]  I_g nodes
  int32_t* grain_nodes = nullptr;
  int32_t* gcols_ptr = nullptr;        // [G+1]
  int32_t* gcols = nullptr;            // mortar DOF columns per grain
  int32_t* giface_ptr = nullptr;       // [G+1]
  int32_t* giface = nullptr;           // interfaces per grain (sorted)
  int32_t* ld = nullptr;               // [G] k_g + 1
  int max_ld = 0;                      // max over grains of ld
  int max_nu3 = 0;                     // max over interfaces of 3 nu_c
  int64_t* b_off = nullptr;            // [G] offset of B_g (row-major [64 nb_g x ld_g])
  double* B = nullptr;                 // shape vectors + correction column
  double* R = nullptr;                 // scratch R_g / Y_g (setup), same layout
  int32_t* iface_ptr = nullptr;        // [C+1]
  int32_t* iface_nodes = nullptr;
  int32_t* iface_of = nullptr;         // [n_iface_nodes] interface of each entry
  int n_iface_nodes = 0;
  int32_t* mortar_ptr = nullptr;       // [C+1]
  int64_t* wt_off = nullptr;           // [C]
  double* W = nullptr;                 // mortar weights
  int32_t* node_class = nullptr;
  int32_t* node_owner = nullptr;
  int32_t* node_iface = nullptr;
  int32_t* node_local = nullptr;       // index of a G/D node within I_g; of an
                                       // interface node within F_c
  // restriction bookkeeping
  int64_t n_chunks = 0;                // row chunks over all grains
  int32_t* chunk_g = nullptr;          // [n_chunks]
  int32_t* chunk_r0 = nullptr;         // [n_chunks] first DOF row
  int64_t* chunk_t = nullptr;          // [n_chunks] offset into tpart
  double* tpart = nullptr;             // partial B_g^T r per chunk (ld_g each)
  double* gpart = nullptr;             // per grain sum of its chunks (yext layout)
  int32_t* chunk_ptr = nullptr;        // [G+1] chunks of each grain
  int32_t* mcol_ptr = nullptr;         // [Nm+1] grains touching mortar column k
  int32_t* mcol_g = nullptr;           // grain
  int32_t* mcol_j = nullptr;           // local column in that grain
  double* yext = nullptr;              // per grain ld_g values (prolongation input)
  int64_t* yext_off = nullptr;         // [G]
  double* Dc = nullptr;                // [G] correction scalars (0 => no column)
  double* Cg = nullptr;                // [sum k_g^2] B_g^T Y_g (setup)
  int64_t* cg_off = nullptr;           // [G]
  int32_t* mortar_iface = nullptr;     // [N^m] interface of each mortar node
  int32_t* gpos = nullptr;             // [n_dof] position in the grain batch or -1
  const int32_t* g_lmap = nullptr;     // grain batch lmap / row_s / row_base
  const int32_t* g_row_s = nullptr;
  const int64_t* g_row_base = nullptr;
  int max_k = 0;                       // max_g k_g
};

void launch_build_R(const DevCoarse& c, const DevBatch& gb, const int32_t* row_ptr,
                    const int32_t* col, const double* val, cudaStream_t st);
void launch_grain_AB(const DevCoarse& c, const DevBatch& gb, const int32_t* row_ptr,
                     const int32_t* col, const double* val, cudaStream_t st);
void launch_grain_BtY(const DevCoarse& c, const DevBatch& gb, cudaStream_t st);
void launch_S_iface(const DevCoarse& c, const int32_t* row_ptr, const int32_t* col,
                    const double* val, double* S, int64_t lds, cudaStream_t st);
void launch_S_grain(const DevCoarse& c, double* S, int64_t lds, cudaStream_t st);
// Algebraic mortar blocks (column q of every interface block)
void launch_alg_rhs(int q, const DevBatch& ab, const int32_t* mortar_ptr,
                    const int32_t* mortar_nodes, const int32_t* rp, const int32_t* col,
                    const double* val, cudaStream_t st);
// surface Algebraic mortars (mortar_kind = 2): dense interface operators K_c
// (faces: 2 int4 per face = 4 local node positions | comps a,b,n (2 bits
// each), voxel ids of the two sides), their free/free tiles, constrained RHS
void launch_surf_operator(int C, const int32_t* iface_ptr, const int32_t* face_ptr,
                          const int4* faces, const double* E, const uint8_t* solid,
                          int64_t nvox, double nu, double tie, const int32_t* tie_ptr,
                          const int32_t* tie_q, const int64_t* koff, double* K1, double* tau,
                          double* Kbuf, cudaStream_t st);
void launch_surf_extract(const DevBatch& ab, const int32_t* iface_ptr, const int32_t* free_ptr,
                         const int32_t* free_pos, const int64_t* koff, const double* Kbuf,
                         cudaStream_t st);
void launch_surf_rhs(int q, const DevBatch& ab, const int32_t* iface_ptr,
                     const int32_t* mortar_ptr, const int32_t* free_ptr, const int32_t* free_pos,
                     const int32_t* con_pos, const int64_t* koff, const double* Kbuf,
                     cudaStream_t st);
void launch_alg_store(int q, int C, const DevBatch& ab, const int32_t* mortar_ptr,
                      const int32_t* free_ptr, const int32_t* free_pos, const int32_t* con_pos,
                      const int64_t* wt_off, double* W, cudaStream_t st);
// r_m (Nm) and r_c (G, correction part) from r (n_dof)
void launch_restrict(const DevCoarse& c, const double* r, double* rm, double* rc,
                     cudaStream_t st);
// x = P_B y_m + sum_g c_g y_c[g]
void launch_prolong(const DevCoarse& c, const double* ym, const double* yc, double* x,
                    cudaStream_t st);
void launch_coarse_diag(int G, const double* rc, const double* Dc, double* yc, cudaStream_t st);
// correction column from a grain-batch y_loc (c_g) and D_c = b_g . c_g
void launch_set_correction(const DevCoarse& c, const DevBatch& gb, cudaStream_t st);

// ---- coarse Cholesky factor and triangular solves (cholesky.cu) -----------
void launch_chol_factor(const DevBatch& b, double* linv, double* linvT, cudaStream_t st);
// y = L^-T L^-1 r  (r, y, zbuf: 64 nb doubles); epoch > every earlier epoch
void launch_chol_solve(const DevBatch& b, const double* linv, const double* linvT,
                       const double* r, double* zbuf, double* y, int* flags_fwd, int* flags_bwd,
                       int epoch, cudaStream_t st);

// ---- combine / scatter (dense.cu) -------------------------------------------
// out[d] = (a? a[d]:0) + (b? b[d]:0) + yloc_grain[gpos[d]] (if gpos>=0)
void launch_combine_grain(int n_dof, const int32_t* gpos, const double* yloc, const double* a,
                          const double* b, double* out, cudaStream_t st);
// out[d] = sum over cpos entries of yloc_contact (ascending subdomain)
void launch_sum_contact(int n_dof, const int32_t* cptr, const int32_t* cidx, const double* yloc,
                        double* out, cudaStream_t st);

// ---- per-device launch helpers (dense.cu) --------------------------------------
// Dynamic shared-memory opt-in of a kernel on the CURRENT device (function
// attributes belong to a device context: cached per (device, kernel),
// thread-safe) and the current device's SM count.
void set_max_dynamic_smem(const void* func, size_t bytes);
int device_sm_count();

// ---- Krylov (krylov.cu) ----------------------------------------------------
int krylov_blocks(int64_t n);
// doubles of a handle's Krylov partial-sum buffer (incl. its completion counter;
// allocate zeroed)
int64_t krylov_partial_doubles(int64_t n);
// partial[b*m + j] = sum over block b of V[j][i] * w[i], j < m; final[j] = sum_b
// cnt (optional, device): vector count = *cnt + 1 read by the kernels (m = its maximum)
void launch_multidot(int64_t n, int m, const double* V, int64_t ldv, const double* w,
                     double* partial, double* out, cudaStream_t st, const int* cnt = nullptr);
// w -= sum_j V[j] h[j]; optional: partial norm^2 of the updated w -> out_norm2
void launch_update(int64_t n, int m, const double* V, int64_t ldv, const double* h, double* w,
                   double* partial, double* out_norm2, cudaStream_t st,
                   const int* cnt = nullptr);
void launch_norm2(int64_t n, const double* x, double* partial, double* out, cudaStream_t st);
void launch_scale(int64_t n, const double* x, const double* s_dev, int invert, double* y,
                  cudaStream_t st);
// x += sum_j V[j] y[j]  (y on device)
void launch_combine_basis(int64_t n, int m, const double* V, int64_t ldv, const double* y,
                          double* x, cudaStream_t st);
void launch_axpy(int64_t n, double a, const double* x, double* y, cudaStream_t st);

// ---- multi-RHS blocks (multirhs.cu; NEXT #2) ----------------------------------
void launch_set_correction_k(const DevBatch& gb, int G, double* Ck, double* Dck, cudaStream_t st);
void launch_restrict_k(const DevCoarse& c, int P, const double* r, int64_t ldr, int ncols,
                       const double* Ck, int64_t ldc, const double* Dck, double* tk, double* gk,
                       double* rm, double* rc, cudaStream_t st);
void launch_prolong_k(const DevCoarse& c, int P, const double* ym, const double* yc,
                      const double* Dck, const double* Ck, int64_t ldc, int ncols, double* yk,
                      double* x, int64_t ldx, cudaStream_t st);
void launch_coarse_diag_k(int n, const double* rc, const double* Dck, double* yc, cudaStream_t st);
void launch_sum_contact_k(int n, int P, int ncols, const int32_t* cptr, const int32_t* cidx,
                          const double* yloc, double* out, int64_t ldo, cudaStream_t st);
void launch_combine_grain_k(int n, int P, int ncols, const int32_t* gpos, const double* yloc,
                            const double* a, const double* b, int64_t ld, double* out,
                            cudaStream_t st);

// ---- device-resident GMRES cycle (gmres.cu; graph-captured, R22) ------------
// Scalars of one solve, in device memory next to the small dense arrays.
struct GmresScalars {
  int j;           // Arnoldi step within the cycle (vectors V[0..j] exist)
  int total;       // Arnoldi steps of the solve
  int k;           // steps of the current cycle when it stopped
  int stop_inner;  // the cycle's step loop has ended
  int done;        // the solve has ended (converged, cap, or non-finite)
  int converged;
  int nonfinite;
  int m, maxit;
  int cycles;      // restart cycles started
  double bnorm, tol, relres;
};
struct GmresDev {
  GmresScalars* s;
  double *H, *g, *cs, *sn, *y, *hist;   // (m+1) x m (row-major, ld m), m+1, m, m, m, maxit
  const double* hb;                     // CGS2 dots: [0, m] pass 1, [m+1, 2m+1] pass 2, [2m+2] ||w||^2
  double* beta2;                        // ||r||^2 slot (= hb + 2(m+1))
};
// cycle start: g = beta e_1, j = 0, step loop on; V[0] = r / beta, vj = V[0]
void launch_gmres_cycle_init(const GmresDev& d, unsigned long long inner, int64_t n, const double* r,
                             double* V, double* vj, cudaStream_t st);
// after CGS2 of step j: Givens update of H(:, j), g; history; stop test; then
// V[j+1] = w / ||w|| and vj = V[j+1] unless the step loop stops
void launch_gmres_step_end(const GmresDev& d, unsigned long long inner, int64_t n, const double* w,
                           double* V, int64_t ldv, double* vj, cudaStream_t st);
// cycle end, part 1: y = H(0:k, 0:k)^-1 g, out = sum_{j<k} V[j] y[j]
void launch_gmres_combine(const GmresDev& d, int64_t n, const double* V, int64_t ldv, double* out,
                          cudaStream_t st);
// cycle end, part 2: relres from beta2; done / converged / non-finite; loop flag
void launch_gmres_cycle_end(const GmresDev& d, unsigned long long outer, cudaStream_t st);

// ---- ILU(0) base smoother (ilu.cu) -----------------------------------------
// Block ILU(0) factor of A^ in its own BSR layout (row_ptr/col of A^):
// L_IK below the diagonal, A~_IJ above, A~_II^-1 on it.  Rows are processed
// in level order (ord_f / ord_b) by sync-free kernels (epoch-stamped flags,
// atomic tickets with a host-tracked running base).
struct IluDev {
  int n = 0;                                   // block rows
  const int32_t* row_ptr = nullptr;
  const int32_t* col = nullptr;
  const int32_t* diag = nullptr;               // position of block (I,I)
  const int32_t* ord_f = nullptr;              // rows by forward level
  const int32_t* ord_b = nullptr;              // rows by backward level
  double* val = nullptr;                       // nnzb*9 factor values
  int* flag_f = nullptr;                       // factorisation epoch stamps
  double* ybuf = nullptr;                      // forward-sweep output (sentinel between sweeps)
  int epoch_f = 0;
  unsigned long long* ticket = nullptr;
  unsigned long long ticket_base = 0;
  int* err = nullptr;                          // first row with a singular pivot
  int levels_f = 0, levels_b = 0;
};
// val must hold A^'s values on entry
void launch_ilu_factor(IluDev& f, cudaStream_t st);
// x = U^-1 L^-1 r  (r and x distinct, neither is ybuf); ybuf must hold the
// all-ones sentinel on entry and holds it again on exit
void launch_ilu_solve(IluDev& f, const double* r, double* x, cudaStream_t st);
// out = a + b (a may be null: out = b)
void launch_lincomb(int64_t n, const double* a, const double* b, double* out, cudaStream_t st);

}  // namespace hplmm
