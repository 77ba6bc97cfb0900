// libhplmm C ABI: handle, device state, setup / solve / apply orchestration.
// See include/hplmm.h for the contract and DESIGN.md for the data layout.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "hplmm_internal.h"
#include "kernels.cuh"
#include "sn_setup.h"

using namespace hplmm;

namespace {

thread_local std::string g_last_error;

constexpr int kSnLeaf = 32;                          // ND leaf size (nodes)
constexpr double kSurfaceTie = 0.1;                  // R29 tie (x mean shear modulus)
static int sn_leaf() {   // HPLMM_SN_LEAF overrides (ordering experiments)
  static const int v = getenv("HPLMM_SN_LEAF") ? std::max(4, atoi(getenv("HPLMM_SN_LEAF"))) : kSnLeaf;
  return v;
}
constexpr int64_t kSnPoolBytes = (int64_t)4 << 30;   // frontal matrices per wave

struct HError {
  hplmm_status st;
  std::string msg;
};

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw HError{e_ == cudaErrorMemoryAllocation ? HPLMM_ERR_OOM : HPLMM_ERR_CUDA,       \
                   std::string(#call) + ": " + cudaGetErrorString(e_)};                   \
  } while (0)

enum KernelClass {
  KC_SYMV_GRAIN = 0, KC_SYMV_CONTACT = 1, KC_SYMV_COARSE = 2, KC_SN_GRAIN = 3, KC_SN_CONTACT = 4,
  KC_ILU = 5, KC_EBE = 6, KC_BSR = 7, KC_N = 8
};

}  // namespace

struct hplmm_handle {
  HostSetup hs;
  int device = -1;
  cudaStream_t st = 0;
  bool assembled = false, setup_done = false, rhs_set = false;
  hplmm_report rep{};
  std::vector<void*> allocs;
  std::vector<void*> setup_allocs;

  // mesh / matrix
  int n_nodes = 0, n_dof = 0;
  int64_t nnzb = 0;
  int max_row_blocks = 0;
  int32_t *d_row_ptr = nullptr, *d_col = nullptr, *d_block_row = nullptr, *d_drow_ptr = nullptr,
          *d_dcol = nullptr, *d_ijk = nullptr;
  uint8_t *d_dir = nullptr, *d_solid = nullptr;
  double *d_E = nullptr, *d_K0 = nullptr, *d_val = nullptr, *d_b = nullptr, *d_f = nullptr,
         *d_uD = nullptr;

  // subdomains
  DevBatch gb, cb, sb, sS;  // grain, contact, coarse inverse, coarse S (refinement)
  double* d_ym = nullptr;
  int32_t *d_gnode_ptr = nullptr, *d_gnodes = nullptr, *d_cnode_ptr = nullptr,
          *d_cnodes = nullptr;
  int32_t *d_cptr = nullptr, *d_cidx = nullptr;
  DevCoarse co;
  std::vector<int32_t> h_corr;   // grains with a correction column (after set_rhs)
  double* d_Sdense = nullptr;
  int64_t lds = 0;
  std::vector<int32_t> h_ld, h_nbg;

  // work vectors
  double *d_in = nullptr, *d_out = nullptr, *d_y = nullptr, *d_r1 = nullptr, *d_z1 = nullptr,
         *d_t = nullptr, *d_rm = nullptr, *d_rc = nullptr, *d_yc = nullptr, *d_x = nullptr,
         *d_u = nullptr, *d_bb = nullptr;
  double *d_V = nullptr, *d_partial = nullptr, *d_hbuf = nullptr;
  double* h_hh = nullptr;   // pinned host copy of the Arnoldi step's dots
  int hh_cap = 0;

  // device-resident solve: one CUDA graph per handle (two nested WHILE
  // conditional nodes: restart cycles around Arnoldi steps), gmres.cu
  cudaGraph_t solve_graph = nullptr;
  cudaGraphExec_t solve_exec = nullptr;
  cudaStream_t cap_st = nullptr;
  GmresDev gdev{};
  GmresScalars* h_gs = nullptr;   // pinned host mirror of the solve's scalars
  double* h_ghist = nullptr;      // pinned host copy of the history
  double *d_vj = nullptr, *d_w = nullptr;
  int64_t graph_launches_pre = 0, graph_launches_cycle = 0, graph_launches_step = 0;
  bool graph_failed = false;

  // multi-RHS batches (hplmm_solve_many, multirhs.cu): K <= 4 columns of
  // stride ldv; per-column Krylov bases; per-RHS correction columns Ck / Dck
  int64_t co_ct = 0, co_yo = 0;      // sizes of the restriction partials / grain coarse values
  int64_t co_off = 0, co_cg = 0;     // doubles of B / R and of the Cg scratch (hplmm_refresh_coarse)
  struct Multi {
    int K = 0;
    double *B = nullptr, *X = nullptr, *vin = nullptr, *y = nullptr, *r1 = nullptr, *z1 = nullptr,
           *t = nullptr, *u = nullptr, *w = nullptr, *V = nullptr;
    double *Ck = nullptr, *Dck = nullptr, *tk = nullptr, *gk = nullptr, *yk = nullptr, *rm = nullptr,
           *rc = nullptr, *ym = nullptr, *yc = nullptr, *snc = nullptr, *sng = nullptr;
    double *hb = nullptr, *partial = nullptr, *h_hb = nullptr;
    // block coarse solve (S^-1 streamed once for the block; null: per column)
    double *cx = nullptr, *cy = nullptr, *cpr = nullptr, *cpc = nullptr;
  } mr;
  int64_t ldv = 0;
  int Vcap = 0;

  // profiling of the dominant kernel (packed SYMV tiles)
  bool profile = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_pending;
  double kc_ms[KC_N] = {};
  int64_t kc_launches[KC_N] = {};

  // coarse Cholesky (coarse_solver == 1)
  double *d_linv = nullptr, *d_linvT = nullptr, *d_zc = nullptr;
  int *d_cflag_f = nullptr, *d_cflag_b = nullptr;
  int coarse_epoch = 0;
  bool chol() const { return hs.opt.coarse_solver == 1; }
  void coarse_apply(DevBatch& b) {   // b.yloc = S^-1 b.xloc
    if (chol()) {
      launch_chol_solve(b, d_linv, d_linvT, b.xloc, d_zc, b.yloc, d_cflag_f, d_cflag_b,
                        ++coarse_epoch, st);
      launches += 2;
    } else {
      symv(b, KC_SYMV_COARSE);
    }
  }

  // supernodal local factors (local_factor == 1)
  SnBatch sg, sc;                       // grains, contact grids
  int32_t* d_gpos_sn = nullptr;         // global DOF -> position in sg.yloc (or -1)
  int32_t *d_cptr_sn = nullptr, *d_cidx_sn = nullptr;   // DOF -> positions in sc.yloc
  int nsm = 148;
  bool sparse() const { return hs.opt.local_factor == 1; }
  int64_t launches = 0;

  // ILU(0) base smoother (smoother == 1) and the n_st-stage buffers
  IluDev ilu;
  double *d_ls_u = nullptr, *d_ls_t0 = nullptr, *d_ls_t1 = nullptr, *d_ls_acc = nullptr;
  bool ilu_smoother() const { return hs.opt.smoother == 1; }

  // element-by-element A^ (operator_kind = 0, own assembly only)
  bool ebe = false, matrix_external = false;
  int32_t* d_lat_ebe = nullptr;
  int32_t* d_lat_all = nullptr;   // lattice -> node id (Dirichlet included) or -1
  double* d_Es = nullptr;
  double K0h[576];

  size_t alloc_bytes = 0, alloc_peak = 0;
  template <class T>
  T* dalloc(size_t n, bool setup_only = false) {
    void* p = nullptr;
    if (n == 0) n = 1;
    static const bool dbg = getenv("HPLMM_DEBUG_ALLOC") != nullptr;
    if (dbg && n * sizeof(T) > ((size_t)256 << 20))
      fprintf(stderr, "hplmm alloc %.3f GB (%s), total %.3f GB\n", n * sizeof(T) / 1e9,
              setup_only ? "setup" : "kept", (alloc_bytes + n * sizeof(T)) / 1e9);
    cudaError_t e = cudaMalloc(&p, n * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw HError{HPLMM_ERR_OOM, "cudaMalloc of " + std::to_string(n * sizeof(T)) + " bytes: " +
                                      cudaGetErrorString(e)};
    }
    (setup_only ? setup_allocs : allocs).push_back(p);
    alloc_bytes += n * sizeof(T);
    alloc_peak = std::max(alloc_peak, alloc_bytes);
    return (T*)p;
  }
  template <class T>
  T* upload(const std::vector<T>& v, bool setup_only = false) {
    T* p = dalloc<T>(v.size(), setup_only);
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return p;
  }
  void free_setup() {
    for (void* p : setup_allocs) cudaFree(p);
    setup_allocs.clear();
    alloc_bytes = 0;   // approximate after the setup-only buffers are released
  }
  ~hplmm_handle() {
    if (device >= 0) {
      cudaSetDevice(device);
      cudaDeviceSynchronize();
      for (void* p : allocs) cudaFree(p);
      free_setup();
      if (h_hh) cudaFreeHost(h_hh);
      if (mr.h_hb) cudaFreeHost(mr.h_hb);
      if (h_gs) cudaFreeHost(h_gs);
      if (h_ghist) cudaFreeHost(h_ghist);
      if (solve_exec) cudaGraphExecDestroy(solve_exec);
      if (solve_graph) cudaGraphDestroy(solve_graph);
      if (cap_st) cudaStreamDestroy(cap_st);
      for (auto e : ev_pool) cudaEventDestroy(e);
      for (auto& e : ev_pending) {
        cudaEventDestroy(e.second.first);
        cudaEventDestroy(e.second.second);
      }
    }
  }

  // ---- profiled launches of the dominant kernel --------------------------
  void symv(DevBatch& b, int kc) {
    if (profile && b.ntiles > 0) {
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0, st));
      launch_symv_tiles(b, st);
      CK(cudaEventRecord(e1, st));
      ev_pending.push_back({kc, {e0, e1}});
    } else {
      launch_symv_tiles(b, st);
    }
    launch_symv_reduce(b, st);
    launches += 2;
  }
  void sn_solve(SnBatch& b, const double* in, int kc) {
    if (profile && b.work.nblocks > 0) {
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0, st));
      sn_apply(b, in, st);
      CK(cudaEventRecord(e1, st));
      ev_pending.push_back({kc, {e0, e1}});
    } else {
      sn_apply(b, in, st);
    }
    launches += 1;
  }
  void flush_profile() {
    for (auto& e : ev_pending) {
      float ms = 0.f;
      CK(cudaEventSynchronize(e.second.second));
      CK(cudaEventElapsedTime(&ms, e.second.first, e.second.second));
      kc_ms[e.first] += ms;
      kc_launches[e.first] += 1;
      cudaEventDestroy(e.second.first);
      cudaEventDestroy(e.second.second);
    }
    ev_pending.clear();
  }
};

namespace {

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

hplmm_status fail(const HError& e) {
  g_last_error = e.msg;
  return e.st;
}

// Build a packed-tile batch over subdomains given by node lists (DOFs 3n+c)
// or, for the coarse block, one subdomain of `ndof_override` identity DOFs.
void build_batch(hplmm_handle* h, DevBatch& b, const std::vector<int32_t>& ptr,
                 const std::vector<int32_t>& nodes, int ndof_override, bool setup_buffers,
                 bool with_tiles = true, bool transient = false) {
  int nsub = ndof_override >= 0 ? 1 : (int)ptr.size() - 1;
  std::vector<int32_t> nb(nsub), ndof(nsub);
  std::vector<int64_t> tile_base(nsub), row_base(nsub);
  int64_t nt = 0, nr = 0;
  int maxnb = 0;
  for (int s = 0; s < nsub; ++s) {
    ndof[s] = ndof_override >= 0 ? ndof_override : 3 * (ptr[s + 1] - ptr[s]);
    nb[s] = (ndof[s] + TB - 1) / TB;
    tile_base[s] = nt;
    row_base[s] = nr;
    nt += (int64_t)nb[s] * (nb[s] + 1) / 2;
    nr += nb[s];
    maxnb = std::max(maxnb, nb[s]);
  }
  std::vector<int32_t> tile_s(nt), tile_ij(nt), row_s(nr), row_k(nr), lmap(nr * TB, -1);
  for (int s = 0; s < nsub; ++s) {
    int64_t t = tile_base[s];
    for (int I = 0; I < nb[s]; ++I) {
      row_s[row_base[s] + I] = s;
      row_k[row_base[s] + I] = I;
      for (int J = 0; J <= I; ++J, ++t) {
        tile_s[t] = s;
        tile_ij[t] = (I << 16) | J;
      }
    }
    for (int i = 0; i < ndof[s]; ++i)
      lmap[row_base[s] * TB + i] =
          ndof_override >= 0 ? i : 3 * nodes[ptr[s] + i / 3] + (i % 3);
  }
  b.nsub = nsub;
  b.max_nb = maxnb;
  b.ntiles = nt;
  b.nrows = nr;
  b.nloc = nr * TB;
  b.nb = h->upload(nb, transient);
  b.ndof = h->upload(ndof, transient);
  b.tile_base = h->upload(tile_base, transient);
  b.row_base = h->upload(row_base, transient);
  b.tile_s = h->upload(tile_s, transient);
  b.tile_ij = h->upload(tile_ij, transient);
  b.row_s = h->upload(row_s, transient);
  b.row_k = h->upload(row_k, transient);
  b.lmap = h->upload(lmap, transient);
  b.xloc = h->dalloc<double>((size_t)b.nloc, transient);
  b.yloc = h->dalloc<double>((size_t)b.nloc, transient);
  b.err = h->dalloc<int32_t>(1, transient);
  if (!with_tiles) return;   // layout only (supernodal mode: B_g row layout, lmap)
  b.tiles = h->dalloc<double>((size_t)nt * TILE, transient);
  b.part_row = h->dalloc<double>((size_t)nt * TB, transient);
  b.part_col = h->dalloc<double>((size_t)nt * TB, transient);
  if (setup_buffers) {
    b.dinv = h->dalloc<double>((size_t)nsub * TILE * SWEEP_M * SWEEP_M, true);
    b.cbuf = h->dalloc<double>((size_t)nr * TILE * SWEEP_M, true);
    b.wbuf = h->dalloc<double>((size_t)nr * TILE * SWEEP_M, true);
  }
}

void check_batch_err(hplmm_handle* h, DevBatch& b, int offset, bool coarse) {
  int32_t e = INT_MAX;
  CK(cudaMemcpyAsync(&e, b.err, sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (e != INT_MAX) {
    h->rep.err_index = offset + e;
    if (coarse) throw HError{HPLMM_ERR_SINGULAR_COARSE, "non-positive pivot in the coarse matrix S"};
    throw HError{HPLMM_ERR_SINGULAR_LOCAL,
                 "non-positive pivot in local subdomain " + std::to_string(offset + e)};
  }
}

double elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e-3;
}

// NVTX range for the profiler timelines (ncu --nvtx, nsys): setup phases,
// each solve, each Arnoldi step
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

struct HandleAlloc : DevAlloc {
  hplmm_handle* h;
  explicit HandleAlloc(hplmm_handle* hh) : h(hh) {}
  void* alloc(size_t bytes, bool setup_only) override {
    return h->dalloc<char>(bytes, setup_only);
  }
};

struct Timer {
  cudaEvent_t a, b;
  cudaStream_t st;
  explicit Timer(cudaStream_t s) : st(s) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
  }
  double stop() {
    cudaEventRecord(b, st);
    return elapsed(a, b);
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

// copy `n` doubles from host-or-device `src` to device `dst`
void to_device(hplmm_handle* h, double* dst, const double* src, int64_t n) {
  CK(cudaMemcpyAsync(dst, src, n * sizeof(double),
                     is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->st));
}
void from_device(hplmm_handle* h, double* dst, const double* src, int64_t n) {
  CK(cudaMemcpyAsync(dst, src, n * sizeof(double),
                     is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->st));
}

// copy `n` elements of a host-or-device array to a host vector
template <class T>
std::vector<T> host_copy(const T* p, int64_t n) {
  std::vector<T> v((size_t)n);
  if (n == 0) return v;
  if (is_device_ptr(p)) CK(cudaMemcpy(v.data(), p, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost));
  else std::memcpy(v.data(), p, (size_t)n * sizeof(T));
  return v;
}
void require_device(hplmm_handle* h) {
  if (h->device < 0) throw HError{HPLMM_ERR_STATE, "no device bound: call hplmm_assemble first"};
  CK(cudaSetDevice(h->device));
}

// ---------------------------------------------------------------------------
// ILU(0) base smoother setup (smoother == 1; R26): level schedules of the
// forward and backward elimination DAGs of A^'s block pattern (host, integer),
// then the block factorisation on the device.
void setup_ilu(hplmm_handle* h) {
  const HostSetup& hs = h->hs;
  const int n = h->n_nodes;
  const std::vector<int32_t>& rp = hs.row_ptr;
  const std::vector<int32_t>& ci = hs.col_idx;
  std::vector<int32_t> diag(n), lf(n, 0), lb(n, 0);
  int nlf = 0, nlb = 0;
  for (int I = 0; I < n; ++I) {
    int d = -1, l = 0;
    for (int e = rp[I]; e < rp[I + 1]; ++e) {
      if (ci[e] == I) d = e;
      else if (ci[e] < I) l = std::max(l, lf[ci[e]] + 1);
    }
    if (d < 0) throw HError{HPLMM_ERR_ARG, "ILU(0): row " + std::to_string(I) + " has no diagonal block"};
    diag[I] = d;
    lf[I] = l;
    nlf = std::max(nlf, l + 1);
  }
  for (int I = n - 1; I >= 0; --I) {
    int l = 0;
    for (int e = diag[I] + 1; e < rp[I + 1]; ++e) l = std::max(l, lb[ci[e]] + 1);
    lb[I] = l;
    nlb = std::max(nlb, l + 1);
  }
  auto order = [n](const std::vector<int32_t>& lev, int nl) {   // stable counting sort
    std::vector<int32_t> cnt(nl + 1, 0), ord(n);
    for (int I = 0; I < n; ++I) cnt[lev[I] + 1]++;
    for (int l = 0; l < nl; ++l) cnt[l + 1] += cnt[l];
    for (int I = 0; I < n; ++I) ord[cnt[lev[I]]++] = I;
    return ord;
  };
  IluDev& f = h->ilu;
  f.n = n;
  f.row_ptr = h->d_row_ptr;
  f.col = h->d_col;
  f.diag = h->upload(diag);
  f.ord_f = h->upload(order(lf, nlf));
  f.ord_b = h->upload(order(lb, nlb));
  f.levels_f = nlf;
  f.levels_b = nlb;
  f.val = h->dalloc<double>((size_t)h->nnzb * 9);
  f.flag_f = h->dalloc<int>(n);
  f.ticket = h->dalloc<unsigned long long>(1);
  f.ybuf = h->dalloc<double>((size_t)3 * n);
  CK(cudaMemsetAsync(f.ybuf, 0xff, (size_t)24 * n, h->st));
  f.err = h->dalloc<int>(1);
  CK(cudaMemsetAsync(f.flag_f, 0, (size_t)n * 4, h->st));
  CK(cudaMemsetAsync(f.ticket, 0, 8, h->st));
  const int big = INT_MAX;
  CK(cudaMemcpyAsync(f.err, &big, 4, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(f.val, h->d_val, (size_t)h->nnzb * 72, cudaMemcpyDeviceToDevice, h->st));
  launch_ilu_factor(f, h->st);
  CK(cudaGetLastError());
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, f.err, 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (bad != INT_MAX)
    throw HError{HPLMM_ERR_SINGULAR_LOCAL,
                 "ILU(0): singular or non-finite pivot block at node " + std::to_string(bad)};
  h->rep.local_bytes += (int64_t)h->nnzb * 72;
}

// ---------------------------------------------------------------------------
// operator applications (all on device vectors of length n_dof)
// ---------------------------------------------------------------------------
// y = A^ x (v null) or v - A^ x from the stored blocks; profiled as KC_BSR
void bsr_spmv(hplmm_handle* h, const double* x, const double* v, double* y) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (h->profile) {
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, h->st));
  }
  launch_spmv(h->n_nodes, h->d_row_ptr, h->d_col, h->d_val, x, v, y, h->st, h->max_row_blocks);
  if (h->profile) {
    CK(cudaEventRecord(e1, h->st));
    h->ev_pending.push_back({KC_BSR, {e0, e1}});
  }
}

void op_spmv(hplmm_handle* h, const double* x, const double* v, double* y) {
  if (h->ebe) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (h->profile) {
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0, h->st));
    }
    launch_ebe(h->n_nodes, h->d_ijk, h->d_dir, h->d_lat_ebe, h->d_lat_all, h->d_Es, h->hs.nx, h->hs.ny,
               h->hs.nz, h->K0h, x, v, y, h->st);
    if (h->profile) {
      CK(cudaEventRecord(e1, h->st));
      h->ev_pending.push_back({KC_EBE, {e0, e1}});
    }
  } else {
    bsr_spmv(h, x, v, y);
  }
  h->launches++;
}

// y_c = A^ x_c (v == nullptr) or v_c - A^ x_c for ncols columns (x, v stride
// ld; y stride ldy): one element-by-element launch for the block (lookups and
// moduli shared by the columns), else the stored blocks per column
void op_spmv_k(hplmm_handle* h, int ncols, const double* x, const double* v, double* y,
               int64_t ld, int64_t ldy) {
  if (h->ebe) {
    const int P = ncols > 2 ? 4 : ncols;
    launch_ebe_k(P, ncols, h->n_nodes, h->d_ijk, h->d_dir, h->d_lat_ebe, h->d_Es, h->hs.nx,
                 h->hs.ny, h->hs.nz, h->K0h, x, v, y, ld, ldy, h->st);
    h->launches++;
    return;
  }
  for (int c = 0; c < ncols; ++c) op_spmv(h, x + c * ld, v ? v + c * ld : nullptr, y + c * ldy);
}

void op_mzeta(hplmm_handle* h, const double* in, double* out) {
  if (h->ilu_smoother())
    throw HError{HPLMM_ERR_STATE, "M_zeta / M_CG: contact grids are not built with smoother = 1"};
  if (h->sparse()) {
    h->sn_solve(h->sc, in, KC_SN_CONTACT);
    launch_sum_contact(h->n_dof, h->d_cptr_sn, h->d_cidx_sn, h->sc.yloc, out, h->st);
    h->launches += 1;
    return;
  }
  launch_gather(h->cb, in, h->st);
  h->symv(h->cb, KC_SYMV_CONTACT);
  launch_sum_contact(h->n_dof, h->d_cptr, h->d_cidx, h->cb.yloc, out, h->st);
  h->launches += 2;
}

// out = a + b + M_g^-1 in
void op_mgrain(hplmm_handle* h, const double* in, const double* a, const double* b, double* out) {
  if (h->sparse()) {
    h->sn_solve(h->sg, in, KC_SN_GRAIN);
    launch_combine_grain(h->n_dof, h->d_gpos_sn, h->sg.yloc, a, b, out, h->st);
    h->launches += 1;
    return;
  }
  launch_gather(h->gb, in, h->st);
  h->symv(h->gb, KC_SYMV_GRAIN);
  launch_combine_grain(h->n_dof, h->co.gpos, h->gb.yloc, a, b, out, h->st);
  h->launches += 2;
}

// y_m = S^-1 r_m by the packed inverse; optional refinement y += S^-1 (r - S y)
const double* op_coarse(hplmm_handle* h, const double* rm) {
  launch_gather(h->sb, rm, h->st);
  h->coarse_apply(h->sb);
  h->launches += 1;
  if (!h->hs.opt.coarse_refine || h->co.Nm == 0) return h->sb.yloc;
  const int Nm = h->co.Nm;
  CK(cudaMemcpyAsync(h->d_ym, h->sb.yloc, (size_t)Nm * 8, cudaMemcpyDeviceToDevice, h->st));
  launch_gather(h->sS, h->d_ym, h->st);
  h->symv(h->sS, KC_SYMV_COARSE);
  launch_gather(h->sb, rm, h->st);
  launch_axpy(h->sb.nloc, -1.0, h->sS.yloc, h->sb.xloc, h->st);
  h->coarse_apply(h->sb);
  launch_axpy(Nm, 1.0, h->sb.yloc, h->d_ym, h->st);
  h->launches += 4;
  return h->d_ym;
}

void op_mg(hplmm_handle* h, const double* in, double* out) {
  launch_restrict(h->co, in, h->d_rm, h->d_rc, h->st);
  const double* ym = op_coarse(h, h->d_rm);
  launch_coarse_diag(h->co.n_grains, h->d_rc, h->co.Dc, h->d_yc, h->st);
  launch_prolong(h->co, ym, h->d_yc, out, h->st);
  h->launches += 6;
}

// M_CG^-1: z1 = M_zeta^-1 in ; out = z1 + M_g^-1 (in - A z1)   (eq:local_smoother_CG)
void op_mcg(hplmm_handle* h, const double* in, double* out) {
  op_mzeta(h, in, h->d_z1);
  op_spmv(h, h->d_z1, in, h->d_t);
  op_mgrain(h, h->d_t, h->d_z1, nullptr, out);
}

// M_ILU^-1 (R27): out = U^-1 L^-1 in
void op_milu(hplmm_handle* h, const double* in, double* out) {
  if (h->profile) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, h->st));
    launch_ilu_solve(h->ilu, in, out, h->st);
    CK(cudaEventRecord(e1, h->st));
    h->ev_pending.push_back({KC_ILU, {e0, e1}});
  } else {
    launch_ilu_solve(h->ilu, in, out, h->st);
  }
  h->launches += 2;
}

// out = (y ? y : 0) + M_L^-1 r, n_st stages of the base smoother in the order
// of eq:local_smoother (R28): t_1 = r, u_i = M_l^-1 t_i, t_{i+1} = t_i - A^ u_i
void op_ml(hplmm_handle* h, const double* r, const double* y, double* out) {
  const int nst = h->hs.opt.n_st;
  if (!h->ilu_smoother() && nst == 1) {   // M_CG, fused: out = y + z1 + M_g^-1 (r - A z1)
    op_mzeta(h, r, h->d_z1);
    op_spmv(h, h->d_z1, r, h->d_t);
    op_mgrain(h, h->d_t, y, h->d_z1, out);
    return;
  }
  if (h->ilu_smoother() && nst == 1) {
    if (!y) { op_milu(h, r, out); return; }
    op_milu(h, r, h->d_ls_u);
    launch_lincomb(h->n_dof, y, h->d_ls_u, out, h->st);
    h->launches += 1;
    return;
  }
  const double* t = r;
  double* tb[2] = {h->d_ls_t0, h->d_ls_t1};
  for (int i = 0; i < nst; ++i) {
    double* u = h->d_ls_u;
    if (h->ilu_smoother()) {
      op_milu(h, t, u);
    } else {                               // u = M_CG^-1 t
      op_mzeta(h, t, h->d_z1);
      op_spmv(h, h->d_z1, t, h->d_t);
      op_mgrain(h, h->d_t, h->d_z1, nullptr, u);
    }
    // acc = (i == 0 ? y : acc) + u, written to out at the last stage
    double* acc = (i + 1 == nst) ? out : h->d_ls_acc;
    launch_lincomb(h->n_dof, i == 0 ? y : h->d_ls_acc, u, acc, h->st);
    h->launches += 1;
    if (i + 1 < nst) {
      op_spmv(h, u, t, tb[i & 1]);         // t_{i+1} = t_i - A^ u_i
      t = tb[i & 1];
    }
  }
}

// M^-1: y = M_G^-1 in ; r1 = in - A y ; out = y + M_L^-1 r1     (eq:multi_precond)
void op_minv(hplmm_handle* h, const double* in, double* out) {
  op_mg(h, in, h->d_y);
  op_spmv(h, h->d_y, in, h->d_r1);
  op_ml(h, h->d_r1, h->d_y, out);
}

void do_set_rhs(hplmm_handle* h, const double* b_dev) {
  Timer t(h->st);
  if (h->sparse()) {
    h->sn_solve(h->sg, b_dev, KC_SN_GRAIN);
    launch_sn_to_batch(h->gb.nloc, h->gb.lmap, h->d_gpos_sn, b_dev, h->sg.yloc, h->gb.xloc,
                       h->gb.yloc, h->st);
    h->launches += 1;
  } else {
    launch_gather(h->gb, b_dev, h->st);
    h->symv(h->gb, KC_SYMV_GRAIN);
    h->launches += 1;
  }
  launch_set_correction(h->co, h->gb, h->st);
  h->launches += 1;
  std::vector<double> Dc(h->co.n_grains);
  if (h->co.n_grains)
    CK(cudaMemcpyAsync(Dc.data(), h->co.Dc, Dc.size() * sizeof(double), cudaMemcpyDeviceToHost,
                       h->st));
  CK(cudaStreamSynchronize(h->st));
  h->h_corr.clear();
  for (int g = 0; g < h->co.n_grains; ++g)
    if (Dc[g] != 0.0) h->h_corr.push_back(g);
  h->rep.n_coarse = h->co.Nm + (int)h->h_corr.size();
  h->rhs_set = true;
  h->rep.t_rhs_s = t.stop();
}

// ---------------------------------------------------------------------------
// Multi-RHS: up to 4 right-hand sides in
// lockstep GMRES(m); every streamed operator is applied to the whole block.
// ---------------------------------------------------------------------------
constexpr int kMaxBlock = 4;

bool multi_eligible(hplmm_handle* h) {
  // rhs_block = 0 (automatic): blocks of 4, unless the one-RHS local solves
  // form CTA teams (a batch with few subdomains) -- the block solves do not, and
  // four team solves are then faster (cfg2: 0.109 vs 0.127 s for 4 load cases)
  const int rb = h->hs.opt.rhs_block;
  const bool teams = h->sg.work.split || h->sc.work.split;
  return h->sparse() && !h->ilu_smoother() && h->hs.opt.n_st == 1 && (rb > 1 || (rb == 0 && !teams));
}

void multi_alloc(hplmm_handle* h) {
  auto& M = h->mr;
  if (M.K) return;
  if (!h->ldv) h->ldv = ((int64_t)h->n_dof + 31) / 32 * 32;   // as hplmm_solve sets it
  const int m = h->hs.opt.restart;
  const int64_t ld = h->ldv;
  const int K = kMaxBlock;
  const int G = h->co.n_grains, Nm = h->co.Nm;
  M.K = K;
  for (double** p : {&M.B, &M.X, &M.vin, &M.y, &M.r1, &M.z1, &M.t, &M.u, &M.w})
    *p = h->dalloc<double>((size_t)K * ld);
  M.V = h->dalloc<double>((size_t)K * (m + 1) * ld);
  M.Ck = h->dalloc<double>((size_t)K * std::max<int64_t>(h->gb.nloc, 1));
  M.Dck = h->dalloc<double>((size_t)K * std::max(G, 1));
  M.tk = h->dalloc<double>((size_t)K * std::max<int64_t>(h->co_ct, 1));
  M.gk = h->dalloc<double>((size_t)K * std::max<int64_t>(h->co_yo, 1));
  M.yk = h->dalloc<double>((size_t)K * std::max<int64_t>(h->co_yo, 1));
  M.rm = h->dalloc<double>((size_t)K * std::max(Nm, 1));
  M.ym = h->dalloc<double>((size_t)K * std::max(Nm, 1));
  M.rc = h->dalloc<double>((size_t)K * std::max(G, 1));
  M.yc = h->dalloc<double>((size_t)K * std::max(G, 1));
  M.snc = h->dalloc<double>((size_t)K * std::max<int64_t>(h->sc.n_loc, 1));
  M.sng = h->dalloc<double>((size_t)K * std::max<int64_t>(h->sg.n_loc, 1));
  const int hbn = 2 * (m + 1) + 8;
  M.hb = h->dalloc<double>((size_t)K * hbn);
  // block SYMV buffers when the coarse solve is the plain S^-1 apply and the
  // per-column partials take < 1/8 of the free memory (else per column)
  if (!h->chol() && !h->hs.opt.coarse_refine && h->sb.ntiles > 0) {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    const size_t need = (size_t)K * 8 * (2 * h->sb.nloc + 2 * h->sb.ntiles * 64);
    if (need < fr / 8) {
      M.cx = h->dalloc<double>((size_t)K * h->sb.nloc);
      M.cy = h->dalloc<double>((size_t)K * h->sb.nloc);
      M.cpr = h->dalloc<double>((size_t)K * h->sb.ntiles * 64);
      M.cpc = h->dalloc<double>((size_t)K * h->sb.ntiles * 64);
    }
  }
  M.partial = h->dalloc<double>((size_t)krylov_partial_doubles(h->n_dof));
  CK(cudaMemsetAsync(M.partial, 0, (size_t)krylov_partial_doubles(h->n_dof) * 8, h->st));
  CK(cudaMallocHost(&M.h_hb, (size_t)K * hbn * 8));
}

// out = M_G^-1 in for ncols columns (eq:mg_struct with each column's own C)
void op_mg_k(hplmm_handle* h, int ncols, const double* in, double* out) {
  auto& M = h->mr;
  const int P = ncols > 2 ? 4 : ncols;
  const int Nm = h->co.Nm, G = h->co.n_grains;
  const int64_t ld = h->ldv;
  launch_restrict_k(h->co, P, in, ld, ncols, M.Ck, h->gb.nloc, M.Dck, M.tk, M.gk, M.rm, M.rc, h->st);
  if (Nm > 0 && M.cx) {   // S^-1 applied to the block in one pass over its tiles
    launch_gather_k(h->sb, ncols, M.rm, Nm, M.cx, h->st);
    launch_symv_k(h->sb, P, ncols, M.cx, M.cy, M.cpr, M.cpc, h->st);
    CK(cudaMemcpy2DAsync(M.ym, (size_t)Nm * 8, M.cy, (size_t)h->sb.nloc * 8, (size_t)Nm * 8,
                         (size_t)ncols, cudaMemcpyDeviceToDevice, h->st));
    h->launches += 3;
  } else {
    for (int c = 0; c < ncols; ++c) {
      if (Nm <= 0) break;
      const double* ymc = op_coarse(h, M.rm + (int64_t)c * Nm);
      CK(cudaMemcpyAsync(M.ym + (int64_t)c * Nm, ymc, (size_t)Nm * 8, cudaMemcpyDeviceToDevice,
                         h->st));
    }
  }
  launch_coarse_diag_k(ncols * G, M.rc, M.Dck, M.yc, h->st);
  launch_prolong_k(h->co, P, M.ym, M.yc, M.Dck, M.Ck, h->gb.nloc, ncols, M.yk, out, ld, h->st);
  h->launches += 7;
}

// out = M_zeta^-1 in, P columns per supernodal launch (factor streamed once)
void op_mzeta_k(hplmm_handle* h, int ncols, const double* in, double* out) {
  HandleAlloc ha(h);
  const int P = sn_multi_width(h->sc, ha, h->st, h->nsm, ncols);
  if (P == 0) throw HError{HPLMM_ERR_ARG, "multi-RHS contact solve does not fit shared memory"};
  const int64_t ld = h->ldv;
  for (int c0 = 0; c0 < ncols; c0 += P) {
    const int nc = std::min(P, ncols - c0);
    sn_apply_multi(h->sc, P, in + c0 * ld, ld, nc, h->mr.snc, h->st);
    launch_sum_contact_k(h->n_dof, P, nc, h->d_cptr_sn, h->d_cidx_sn, h->mr.snc, out + c0 * ld, ld,
                         h->st);
    h->launches += 2;
  }
}

// out = a + b + M_g^-1 in (a, b optional), P columns per supernodal launch
void op_mgrain_k(hplmm_handle* h, int ncols, const double* in, const double* a, const double* b,
                 double* out) {
  HandleAlloc ha(h);
  const int P = sn_multi_width(h->sg, ha, h->st, h->nsm, ncols);
  if (P == 0) throw HError{HPLMM_ERR_ARG, "multi-RHS grain solve does not fit shared memory"};
  const int64_t ld = h->ldv;
  for (int c0 = 0; c0 < ncols; c0 += P) {
    const int nc = std::min(P, ncols - c0);
    sn_apply_multi(h->sg, P, in + c0 * ld, ld, nc, h->mr.sng, h->st);
    launch_combine_grain_k(h->n_dof, P, nc, h->d_gpos_sn, h->mr.sng, a ? a + c0 * ld : nullptr,
                           b ? b + c0 * ld : nullptr, ld, out + c0 * ld, h->st);
    h->launches += 2;
  }
}

// out = M^-1 in for ncols columns (eq:multi_precond, M_L = M_CG, n_st = 1)
void op_minv_k(hplmm_handle* h, int ncols, const double* in, double* out) {
  auto& M = h->mr;
  const int64_t ld = h->ldv;
  op_mg_k(h, ncols, in, M.y);
  op_spmv_k(h, ncols, M.y, in, M.r1, ld, ld);
  op_mzeta_k(h, ncols, M.r1, M.z1);
  op_spmv_k(h, ncols, M.z1, M.r1, M.t, ld, ld);
  op_mgrain_k(h, ncols, M.t, M.y, M.z1, out);
}

// correction columns of the block's right-hand sides (eq:col_cg, R15, R16):
// c_g = A_g^-1 b_g for all columns by one block grain solve
void set_rhs_k(hplmm_handle* h, int ncols, const double* B) {
  auto& M = h->mr;
  HandleAlloc ha(h);
  const int P = sn_multi_width(h->sg, ha, h->st, h->nsm, ncols);
  if (P == 0) throw HError{HPLMM_ERR_ARG, "multi-RHS grain solve does not fit shared memory"};
  for (int c0 = 0; c0 < ncols; c0 += P) {
    const int nc = std::min(P, ncols - c0);
    sn_apply_multi(h->sg, P, B + c0 * h->ldv, h->ldv, nc, M.sng, h->st);
    h->launches++;
    for (int c = c0; c < c0 + nc; ++c) {
      launch_sn_to_batch(h->gb.nloc, h->gb.lmap, h->d_gpos_sn, B + c * h->ldv, M.sng, h->gb.xloc,
                         h->gb.yloc, h->st, P, c - c0);
      launch_set_correction_k(h->gb, h->co.n_grains, M.Ck + c * h->gb.nloc,
                              M.Dck + (int64_t)c * h->co.n_grains, h->st);
      h->launches += 2;
    }
  }
}

// Lockstep GMRES(m) (R22) on ncols <= 4 columns of Bd (device, stride ldv):
// each column runs its own Arnoldi process and Givens rotations exactly as
// hplmm_solve's host loop; the operator applications of a step are batched.
// A cycle ends when every column still iterating has stopped (converged,
// happy breakdown, cap) or reached m; columns that stopped earlier wait.
void solve_block(hplmm_handle* h, int ncols, double tol, hplmm_report* reps) {
  auto& M = h->mr;
  cudaStream_t st = h->st;
  const int n = h->n_dof, m = h->hs.opt.restart, maxit = h->hs.opt.max_iter;
  const int64_t ld = h->ldv;
  const int hbn = 2 * (m + 1) + 8;
  // ||b_c||
  for (int c = 0; c < ncols; ++c)
    launch_norm2(n, M.B + c * ld, M.partial, M.hb + (int64_t)c * hbn + 2 * (m + 1), st);
  std::vector<double> bn(ncols), bn2(ncols);
  CK(cudaMemcpyAsync(M.h_hb, M.hb, (size_t)ncols * hbn * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int c = 0; c < ncols; ++c) {
    bn2[c] = M.h_hb[(int64_t)c * hbn + 2 * (m + 1)];
    bn[c] = std::sqrt(bn2[c]);
  }
  set_rhs_k(h, ncols, M.B);
  CK(cudaMemsetAsync(M.X, 0, (size_t)ncols * ld * 8, st));
  CK(cudaMemcpyAsync(M.r1, M.B, (size_t)ncols * ld * 8, cudaMemcpyDeviceToDevice, st));
  struct Col {
    std::vector<double> H, cs, sn, g;
    int total = 0, k = 0;
    bool done = false, conv = false, active = false;
    double beta2 = 0, relres = 1.0;
  };
  std::vector<Col> col(ncols);
  for (int c = 0; c < ncols; ++c) {
    col[c].H.assign((size_t)(m + 1) * m, 0.0);
    col[c].cs.assign(m, 0.0);
    col[c].sn.assign(m, 0.0);
    col[c].g.assign(m + 1, 0.0);
    col[c].beta2 = bn2[c];
    if (bn[c] == 0.0) {
      col[c].done = col[c].conv = true;
      col[c].relres = 0.0;
    }
  }
  double* r = M.r1;   // residual block (the cycle start vectors), overwritten per cycle
  std::vector<double> hbuf;
  while (true) {
    bool any = false;
    for (int c = 0; c < ncols; ++c) {
      Col& C = col[c];
      C.active = !C.done;
      if (!C.active) continue;
      any = true;
      std::fill(C.H.begin(), C.H.end(), 0.0);
      std::fill(C.g.begin(), C.g.end(), 0.0);
      C.g[0] = std::sqrt(C.beta2);
      C.k = 0;
      // V_c[0] = r_c / beta_c (norm^2 in the column's hb slot)
      CK(cudaMemcpyAsync(M.hb + (int64_t)c * hbn + 2 * (m + 1), &C.beta2, 8, cudaMemcpyHostToDevice,
                         st));
      launch_scale(n, r + c * ld, M.hb + (int64_t)c * hbn + 2 * (m + 1), 1,
                   M.V + (int64_t)c * (m + 1) * ld, st);
    }
    if (!any) break;
    for (int j = 0; j < m; ++j) {
      bool stepping = false;
      for (int c = 0; c < ncols; ++c) stepping |= col[c].active;
      if (!stepping) break;
      // u_c = M^-1 v_j,c (block; columns not iterating carry zeros), w_c = A u_c
      for (int c = 0; c < ncols; ++c) {
        if (col[c].active)
          CK(cudaMemcpyAsync(M.vin + c * ld, M.V + ((int64_t)c * (m + 1) + j) * ld, (size_t)n * 8,
                             cudaMemcpyDeviceToDevice, st));
        else
          CK(cudaMemsetAsync(M.vin + c * ld, 0, (size_t)n * 8, st));
      }
      op_minv_k(h, ncols, M.vin, M.u);
      // w_c = A u_c for the whole block into V_c[j + 1] (columns not iterating
      // have u_c = 0: their slot j + 1 > their last step is not used)
      op_spmv_k(h, ncols, M.u, nullptr, M.V + (int64_t)(j + 1) * ld, ld, (int64_t)(m + 1) * ld);
      for (int c = 0; c < ncols; ++c) {
        if (!col[c].active) continue;
        double* V = M.V + (int64_t)c * (m + 1) * ld;
        double* w = V + (j + 1) * ld;
        double* hb = M.hb + (int64_t)c * hbn;
        launch_multidot(n, j + 1, V, ld, w, M.partial, hb, st);
        launch_update(n, j + 1, V, ld, hb, w, nullptr, nullptr, st);
        launch_multidot(n, j + 1, V, ld, w, M.partial, hb + (m + 1), st);
        launch_update(n, j + 1, V, ld, hb + (m + 1), w, M.partial, hb + 2 * (m + 1), st);
        h->launches += 7;
      }
      CK(cudaMemcpyAsync(M.h_hb, M.hb, (size_t)ncols * hbn * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int c = 0; c < ncols; ++c) {
        Col& C = col[c];
        if (!C.active) continue;
        const double* hh = M.h_hb + (int64_t)c * hbn;
        const double hn = std::sqrt(hh[2 * (m + 1)]);
        std::vector<double> cv(j + 2);
        for (int i = 0; i <= j; ++i) cv[i] = hh[i] + hh[m + 1 + i];
        cv[j + 1] = hn;
        for (int i = 0; i < j; ++i) {
          const double tq = C.cs[i] * cv[i] + C.sn[i] * cv[i + 1];
          cv[i + 1] = -C.sn[i] * cv[i] + C.cs[i] * cv[i + 1];
          cv[i] = tq;
        }
        const double den = std::hypot(cv[j], cv[j + 1]);
        C.cs[j] = cv[j] / den;
        C.sn[j] = cv[j + 1] / den;
        cv[j] = den;
        C.g[j + 1] = -C.sn[j] * C.g[j];
        C.g[j] = C.cs[j] * C.g[j];
        for (int i = 0; i <= j; ++i) C.H[(size_t)i * m + j] = cv[i];
        C.total++;
        C.k = j + 1;
        const double est = std::fabs(C.g[j + 1]) / bn[c];
        if (!std::isfinite(est)) throw HError{HPLMM_ERR_NONFINITE, "non-finite GMRES residual"};
        if (hn == 0.0 || est < tol || C.total >= maxit) {
          C.active = false;   // this column's cycle ends here
        } else {
          double* V = M.V + (int64_t)c * (m + 1) * ld;
          launch_scale(n, V + (j + 1) * ld, M.hb + (int64_t)c * hbn + 2 * (m + 1), 1,
                       V + (j + 1) * ld, st);
          h->launches++;
        }
      }
    }
    // cycle end: x_c += M^-1 (V_c y_c), r_c = b_c - A x_c for every column that iterated
    for (int c = 0; c < ncols; ++c) {
      Col& C = col[c];
      if (C.done) {
        CK(cudaMemsetAsync(M.vin + c * ld, 0, (size_t)n * 8, st));
        continue;
      }
      std::vector<double> y(C.k);
      for (int i = C.k - 1; i >= 0; --i) {
        double s = C.g[i];
        for (int l = i + 1; l < C.k; ++l) s -= C.H[(size_t)i * m + l] * y[l];
        y[i] = s / C.H[(size_t)i * m + i];
      }
      double* hb = M.hb + (int64_t)c * hbn;
      CK(cudaMemcpyAsync(hb, y.data(), C.k * 8, cudaMemcpyHostToDevice, st));
      CK(cudaMemsetAsync(M.vin + c * ld, 0, (size_t)n * 8, st));
      launch_combine_basis(n, C.k, M.V + (int64_t)c * (m + 1) * ld, ld, hb, M.vin + c * ld, st);
      h->launches++;
    }
    op_minv_k(h, ncols, M.vin, M.u);
    for (int c = 0; c < ncols; ++c) {
      if (col[c].done) continue;
      launch_axpy(n, 1.0, M.u + c * ld, M.X + c * ld, st);
      op_spmv(h, M.X + c * ld, M.B + c * ld, r + c * ld);
      launch_norm2(n, r + c * ld, M.partial, M.hb + (int64_t)c * hbn + 2 * (m + 1), st);
      h->launches += 3;
    }
    CK(cudaMemcpyAsync(M.h_hb, M.hb, (size_t)ncols * hbn * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int c = 0; c < ncols; ++c) {
      Col& C = col[c];
      if (C.done) continue;
      C.beta2 = M.h_hb[(int64_t)c * hbn + 2 * (m + 1)];
      C.relres = std::sqrt(C.beta2) / bn[c];
      if (!std::isfinite(C.relres)) throw HError{HPLMM_ERR_NONFINITE, "non-finite true residual"};
      if (C.relres < tol) C.done = C.conv = true;
      else if (C.total >= maxit) C.done = true;
    }
  }
  for (int c = 0; c < ncols; ++c) {
    hplmm_report& R = reps[c];
    R = h->rep;
    R.iterations = col[c].total;
    R.converged = col[c].conv ? 1 : 0;
    R.hist_len = 0;
    R.final_true_relres = col[c].relres;
  }
}

// ---------------------------------------------------------------------------
// Device-resident solve (R22 on the GPU, gmres.cu).  The graph is
//   WHILE (outer: restart cycles) {
//     cycle init: g = beta e1, V0 = r / beta
//     WHILE (inner: Arnoldi steps) {
//       u = M^-1 v_j ; w = A^ u ; CGS2 (j read on the device) ; Givens,
//       history, stop test ; v_{j+1} = w / ||w||
//     }
//     y = H^-1 g ; x += M^-1 (V y) ; r = b - A^ x ; restart test
//   }
// captured once per handle on a private stream (every pointer is a handle
// buffer), launched once per solve.  Used when the kernels of a step take no
// per-call host state: M_CG smoother (ILU(0) sweeps carry a host ticket base)
// and the explicit coarse inverse (the Cholesky sweeps carry a host epoch);
// profiling (CUDA events around kernels) also selects the host loop.
bool graph_eligible(hplmm_handle* h) {
  static const bool off = [] {
    const char* e = getenv("HPLMM_GRAPH");
    return e && e[0] == '0';
  }();
  return !off && !h->hs.opt.host_loop && !h->graph_failed && !h->profile && !h->ilu_smoother() &&
         !h->chol();
}

void build_solve_graph(hplmm_handle* h) {
  const int n = h->n_dof;
  const int m = h->hs.opt.restart;
  const int maxit = h->hs.opt.max_iter;
  if (!h->d_vj) {
    h->d_vj = h->dalloc<double>((size_t)h->ldv);
    h->d_w = h->dalloc<double>((size_t)h->ldv);
    // scalars | H (m+1) x m | g m+1 | cs m | sn m | y m | hist maxit
    const size_t nd = (size_t)(m + 1) * m + (m + 1) + 3 * (size_t)m + maxit;
    char* base = h->dalloc<char>(256 + nd * 8);
    GmresDev& d = h->gdev;
    d.s = (GmresScalars*)base;
    double* p = (double*)(base + 256);
    d.H = p; p += (size_t)(m + 1) * m;
    d.g = p; p += m + 1;
    d.cs = p; p += m;
    d.sn = p; p += m;
    d.y = p; p += m;
    d.hist = p;
    d.hb = h->d_hbuf;
    d.beta2 = h->d_hbuf + 2 * (m + 1);
    CK(cudaMallocHost(&h->h_gs, sizeof(GmresScalars)));
    CK(cudaMallocHost(&h->h_ghist, (size_t)maxit * 8));
  }
  if (!h->cap_st) CK(cudaStreamCreateWithFlags(&h->cap_st, cudaStreamNonBlocking));
  const GmresDev& d = h->gdev;
  cudaGraph_t G = nullptr;
  CK(cudaGraphCreate(&G, 0));
  cudaStream_t user = h->st;
  const int64_t launches0 = h->launches;
  try {
    cudaGraphConditionalHandle outer, inner;
    CK(cudaGraphConditionalHandleCreate(&outer, G, 1, cudaGraphCondAssignDefault));
    CK(cudaGraphConditionalHandleCreate(&inner, G, 1, 0));
    cudaGraphNodeParams po{};
    po.type = cudaGraphNodeTypeConditional;
    po.conditional.handle = outer;
    po.conditional.type = cudaGraphCondTypeWhile;
    po.conditional.size = 1;
    cudaGraphNode_t n_outer;
    CK(cudaGraphAddNode(&n_outer, G, nullptr, 0, &po));
    cudaGraph_t body1 = po.conditional.phGraph_out[0];
    cudaStream_t cs = h->cap_st;
    h->st = cs;
    double* V = h->d_V;
    // (1) cycle start, captured into the outer body
    CK(cudaStreamBeginCaptureToGraph(cs, body1, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    launch_gmres_cycle_init(d, inner, n, h->d_r1, V, h->d_vj, cs);
    cudaStreamCaptureStatus cst;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    CK(cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &ndeps));
    std::vector<cudaGraphNode_t> dv(deps, deps + ndeps);
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(cs, &tmp));
    // (2) the Arnoldi step loop
    cudaGraphNodeParams pi{};
    pi.type = cudaGraphNodeTypeConditional;
    pi.conditional.handle = inner;
    pi.conditional.type = cudaGraphCondTypeWhile;
    pi.conditional.size = 1;
    cudaGraphNode_t n_inner;
    CK(cudaGraphAddNode(&n_inner, body1, dv.data(), dv.size(), &pi));
    cudaGraph_t body2 = pi.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(cs, body2, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const int64_t l_step0 = h->launches;
    op_minv(h, h->d_vj, h->d_u);
    op_spmv(h, h->d_u, nullptr, h->d_w);
    launch_multidot(n, m, V, h->ldv, h->d_w, h->d_partial, h->d_hbuf, cs, &d.s->j);
    launch_update(n, m, V, h->ldv, h->d_hbuf, h->d_w, nullptr, nullptr, cs, &d.s->j);
    launch_multidot(n, m, V, h->ldv, h->d_w, h->d_partial, h->d_hbuf + (m + 1), cs, &d.s->j);
    launch_update(n, m, V, h->ldv, h->d_hbuf + (m + 1), h->d_w, h->d_partial, d.beta2, cs, &d.s->j);
    launch_gmres_step_end(d, inner, n, h->d_w, V, h->ldv, h->d_vj, cs);
    h->launches += 9;
    h->graph_launches_step = h->launches - l_step0;
    CK(cudaStreamEndCapture(cs, &tmp));
    // (3) cycle end, captured into the outer body after the step loop
    CK(cudaStreamBeginCaptureToGraph(cs, body1, &n_inner, nullptr, 1, cudaStreamCaptureModeThreadLocal));
    const int64_t l_cyc0 = h->launches;
    launch_gmres_combine(d, n, V, h->ldv, h->d_in, cs);
    op_minv(h, h->d_in, h->d_u);
    launch_axpy(n, 1.0, h->d_u, h->d_x, cs);
    op_spmv(h, h->d_x, h->d_bb, h->d_r1);   // r = b - A^ x
    launch_norm2(n, h->d_r1, h->d_partial, d.beta2, cs);
    launch_gmres_cycle_end(d, outer, cs);
    h->launches += 7;
    h->graph_launches_cycle = h->launches - l_cyc0 + 2;   // + the cycle start
    CK(cudaStreamEndCapture(cs, &tmp));
    h->st = user;
    CK(cudaGraphInstantiate(&h->solve_exec, G, 0));
    h->solve_graph = G;
  } catch (...) {
    h->st = user;
    cudaStreamCaptureStatus cst;
    if (cudaStreamIsCapturing(h->cap_st, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
      cudaGraph_t junk;
      cudaStreamEndCapture(h->cap_st, &junk);
    }
    cudaGetLastError();
    cudaGraphDestroy(G);
    h->launches = launches0;
    throw;
  }
  h->launches = launches0;
}

}  // namespace

// ===========================================================================
extern "C" {

void hplmm_default_options(hplmm_options* o) {
  if (!o) return;
  o->n_mortar = 4;
  o->beta = 4.0;
  o->contact_h = 1;
  o->restart = 50;
  o->max_iter = 300;
  o->n_st = 1;
  o->coarse_refine = 0;
  o->local_factor = 1;
  o->coarse_solver = 0;
  o->mortar_kind = 0;
  o->smoother = 0;
  o->operator_kind = 0;
  o->sn_shape = 0;
  o->sn_split = 0;
  o->host_loop = 0;
  o->rhs_block = 0;
}

const char* hplmm_last_error(void) { return g_last_error.c_str(); }

hplmm_status hplmm_create(const hplmm_problem* prob, const hplmm_options* opt,
                          hplmm_handle** out) {
  if (!out) { g_last_error = "hplmm_create: out is NULL"; return HPLMM_ERR_ARG; }
  *out = nullptr;
  hplmm_options dflt;
  if (!opt) {   // NULL options = the defaults
    hplmm_default_options(&dflt);
    opt = &dflt;
  }
  auto t0 = std::chrono::steady_clock::now();
  hplmm_handle* h = new hplmm_handle();
  std::string err;
  if (!host_setup(prob, opt, h->hs, err)) {
    delete h;
    g_last_error = err;
    return HPLMM_ERR_ARG;
  }
  HostSetup& hs = h->hs;
  h->n_nodes = hs.n_nodes;
  h->n_dof = 3 * hs.n_nodes;
  h->nnzb = (int64_t)hs.col_idx.size();
  h->rep.n_nodes = hs.n_nodes;
  h->rep.nnzb = h->nnzb;
  h->rep.n_grains = hs.n_grains;
  h->rep.n_interfaces = hs.n_ifaces();
  h->rep.n_mortar_dofs = 3 * hs.n_mortar_nodes();
  h->rep.n_coarse = h->rep.n_mortar_dofs;
  h->rep.err_index = -1;
  h->rep.t_host_setup_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = h;
  return HPLMM_OK;
}

hplmm_status hplmm_assemble(hplmm_handle* h, int32_t device, void* stream) {
  if (!h) { g_last_error = "null handle"; return HPLMM_ERR_ARG; }
  try {
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw HError{HPLMM_ERR_CUDA, "no CUDA device available (there is no CPU fallback)"};
    }
    if (h->device >= 0 && h->device != device)
      throw HError{HPLMM_ERR_STATE, "handle already bound to another device"};
    CK(cudaSetDevice(device));
    h->device = device;
    h->st = (cudaStream_t)stream;
    HostSetup& hs = h->hs;
    Timer t(h->st);
    if (!h->d_val) {
      std::vector<int32_t> brow(h->nnzb);
      for (int p = 0; p < h->n_nodes; ++p)
        for (int e2 = hs.row_ptr[p]; e2 < hs.row_ptr[p + 1]; ++e2) brow[e2] = p;
      h->d_row_ptr = h->upload(hs.row_ptr);
      {
        std::vector<int32_t> colp(hs.col_idx);
        colp.resize(colp.size() + 4, 0);   // tail padding for 16-byte TMA granules
        h->d_col = h->upload(colp);
        h->max_row_blocks = 0;
        for (int p = 0; p < h->n_nodes; ++p)
          h->max_row_blocks = std::max(h->max_row_blocks, hs.row_ptr[p + 1] - hs.row_ptr[p]);
      }
      h->d_block_row = h->upload(brow);
      h->d_drow_ptr = h->upload(hs.drow_ptr);
      h->d_dcol = h->upload(hs.dcol);
      h->d_ijk = h->upload(hs.node_ijk);
      h->d_dir = h->upload(hs.dir);
      h->d_solid = h->upload(hs.solid);
      h->d_E = h->upload(hs.E);
      h->d_f = h->upload(hs.f);
      h->d_uD = h->upload(hs.u_D);
      h->d_K0 = h->dalloc<double>(576);
      h->d_val = h->dalloc<double>((size_t)h->nnzb * 9 + 4);  // +pad: SpMV vector loads
      h->d_b = h->dalloc<double>(h->n_dof);
    }
    launch_element_K0(h->d_K0, hs.nu, h->st);
    launch_assemble((int)h->nnzb, h->d_block_row, h->d_col, h->d_ijk, h->d_dir, h->d_solid,
                    h->d_E, hs.nx, hs.ny, hs.nz, h->d_K0, h->d_val, h->st);
    launch_assemble_rhs(h->n_nodes, h->d_drow_ptr, h->d_dcol, h->d_ijk, h->d_dir, h->d_solid,
                        h->d_E, hs.nx, hs.ny, hs.nz, h->d_K0, h->d_f, h->d_uD, h->d_b, h->st);
    CK(cudaGetLastError());
    h->rep.t_assemble_s = t.stop();
    CK(cudaStreamSynchronize(h->st));
    h->assembled = true;
    return HPLMM_OK;
  } catch (const HError& e) {
    return fail(e);
  }
}

hplmm_status hplmm_set_matrix(hplmm_handle* h, const double* val, void* stream) {
  if (!h || !val) { g_last_error = "null argument"; return HPLMM_ERR_ARG; }
  try {
    if (!h->assembled) throw HError{HPLMM_ERR_STATE, "hplmm_set_matrix before hplmm_assemble"};
    if (h->setup_done) throw HError{HPLMM_ERR_STATE, "hplmm_set_matrix after hplmm_setup"};
    require_device(h);
    h->st = (cudaStream_t)stream;
    to_device(h, h->d_val, val, h->nnzb * 9);
    h->matrix_external = true;   // A^ no longer the voxel assembly: stored blocks only
    CK(cudaStreamSynchronize(h->st));
    return HPLMM_OK;
  } catch (const HError& e) {
    return fail(e);
  }
}

hplmm_status hplmm_setup_bsr(const hplmm_bsr* A, const hplmm_problem* geom,
                             const hplmm_options* opt, int32_t device, void* stream,
                             hplmm_handle** out) {
  if (!out) { g_last_error = "hplmm_setup_bsr: out is NULL"; return HPLMM_ERR_ARG; }
  *out = nullptr;
  if (!A || !geom || !A->row_ptr || !A->col_idx || !A->val || A->n_nodes <= 0 || A->nnzb <= 0) {
    g_last_error = "hplmm_setup_bsr: null matrix / geometry or empty matrix";
    return HPLMM_ERR_ARG;
  }
  hplmm_handle* h = nullptr;
  hplmm_status s = hplmm_create(geom, opt, &h);
  if (s != HPLMM_OK) return s;
  try {
    const HostSetup& hs = h->hs;
    if (A->n_nodes != h->n_nodes)
      throw HError{HPLMM_ERR_ARG, "hplmm_setup_bsr: A has " + std::to_string(A->n_nodes) +
                                      " block rows, the geometry defines " +
                                      std::to_string(h->n_nodes) + " nodes (R3)"};
    if (A->nnzb != h->nnzb)
      throw HError{HPLMM_ERR_ARG, "hplmm_setup_bsr: A has " + std::to_string(A->nnzb) +
                                      " blocks, the geometry's pattern (R4) has " +
                                      std::to_string(h->nnzb)};
    if (A->node_ijk) {
      const std::vector<int32_t> ijk = host_copy(A->node_ijk, 3 * (int64_t)A->n_nodes);
      for (int p = 0; p < h->n_nodes; ++p)
        for (int c = 0; c < 3; ++c)
          if (ijk[3 * p + c] != hs.node_ijk[3 * p + c])
            throw HError{HPLMM_ERR_ARG, "hplmm_setup_bsr: node " + std::to_string(p) +
                                            " is not the geometry's node in lattice-key order (R3)"};
    }
    const std::vector<int32_t> rp = host_copy(A->row_ptr, (int64_t)A->n_nodes + 1);
    const std::vector<int32_t> ci = host_copy(A->col_idx, A->nnzb);
    for (int p = 0; p <= h->n_nodes; ++p)
      if (rp[p] != hs.row_ptr[p])
        throw HError{HPLMM_ERR_ARG, "hplmm_setup_bsr: row_ptr differs from the geometry's pattern "
                                    "at block row " + std::to_string(p > 0 ? p - 1 : 0) + " (R4)"};
    for (int p = 0; p < h->n_nodes; ++p)
      for (int e = rp[p]; e < rp[p + 1]; ++e)
        if (ci[e] != hs.col_idx[e])
          throw HError{HPLMM_ERR_ARG, "hplmm_setup_bsr: col_idx differs from the geometry's "
                                      "pattern in block row " + std::to_string(p) + " (R4)"};
  } catch (const HError& e) {
    delete h;
    return fail(e);
  }
  if ((s = hplmm_assemble(h, device, stream)) != HPLMM_OK ||
      (s = hplmm_set_matrix(h, A->val, stream)) != HPLMM_OK ||
      (s = hplmm_setup(h, stream)) != HPLMM_OK) {
    const std::string msg = g_last_error;
    delete h;
    g_last_error = msg;
    return s;
  }
  *out = h;
  return HPLMM_OK;
}

hplmm_status hplmm_assemble_bsr(const hplmm_problem* prob, int32_t device, hplmm_bsr** A,
                                double** b) {
  if (!A || !b) { g_last_error = "hplmm_assemble_bsr: null output"; return HPLMM_ERR_ARG; }
  *A = nullptr;
  *b = nullptr;
  hplmm_handle* h = nullptr;
  hplmm_status s = hplmm_create(prob, nullptr, &h);
  if (s != HPLMM_OK) return s;
  if ((s = hplmm_assemble(h, device, nullptr)) != HPLMM_OK) {
    const std::string msg = g_last_error;
    delete h;
    g_last_error = msg;
    return s;
  }
  hplmm_bsr* M = (hplmm_bsr*)std::calloc(1, sizeof(hplmm_bsr));
  const int n = h->n_nodes;
  const int64_t nb = h->nnzb;
  int32_t* rp = (int32_t*)std::malloc((size_t)(n + 1) * 4);
  int32_t* ci = (int32_t*)std::malloc((size_t)nb * 4);
  int32_t* ijk = (int32_t*)std::malloc((size_t)n * 12);
  double* val = (double*)std::malloc((size_t)nb * 72);
  double* bb = (double*)std::malloc((size_t)n * 24);
  if (!M || !rp || !ci || !ijk || !val || !bb) {
    std::free(M); std::free(rp); std::free(ci); std::free(ijk); std::free(val); std::free(bb);
    delete h;
    g_last_error = "hplmm_assemble_bsr: host allocation failed";
    return HPLMM_ERR_OOM;
  }
  std::memcpy(rp, h->hs.row_ptr.data(), (size_t)(n + 1) * 4);
  std::memcpy(ci, h->hs.col_idx.data(), (size_t)nb * 4);
  std::memcpy(ijk, h->hs.node_ijk.data(), (size_t)n * 12);
  cudaError_t e1 = cudaMemcpy(val, h->d_val, (size_t)nb * 72, cudaMemcpyDeviceToHost);
  cudaError_t e2 = cudaMemcpy(bb, h->d_b, (size_t)n * 24, cudaMemcpyDeviceToHost);
  delete h;
  M->n_nodes = n;
  M->nnzb = nb;
  M->row_ptr = rp;
  M->col_idx = ci;
  M->val = val;
  M->node_ijk = ijk;
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    hplmm_free_bsr(M, bb);
    g_last_error = "hplmm_assemble_bsr: device-to-host copy failed";
    return HPLMM_ERR_CUDA;
  }
  *A = M;
  *b = bb;
  return HPLMM_OK;
}

void hplmm_free_bsr(hplmm_bsr* A, double* b) {
  if (A) {
    std::free((void*)A->row_ptr);
    std::free((void*)A->col_idx);
    std::free((void*)A->val);
    std::free((void*)A->node_ijk);
    std::free(A);
  }
  std::free(b);
}

hplmm_status hplmm_setup(hplmm_handle* h, void* stream) {
  if (!h) { g_last_error = "null handle"; return HPLMM_ERR_ARG; }
  try {
    if (!h->assembled) throw HError{HPLMM_ERR_STATE, "hplmm_setup before hplmm_assemble"};
    if (h->setup_done) throw HError{HPLMM_ERR_STATE, "hplmm_setup called twice"};
    require_device(h);
    h->st = (cudaStream_t)stream;
    HostSetup& hs = h->hs;
    const int G = hs.n_grains, C = hs.n_ifaces(), N = h->n_nodes;
    const int Nm = 3 * hs.n_mortar_nodes();

    // ---------------- fine operator (operator_kind) ------------------------
    {
      const char* e = getenv("HPLMM_EBE");   // HPLMM_EBE=0: stored blocks (A/B)
      h->ebe = hs.opt.operator_kind == 0 && !h->matrix_external && !(e && e[0] == '0');
      h->rep.fine_operator = h->ebe ? 0 : 1;
      if (h->ebe) {
        const int64_t nvox = (int64_t)hs.nx * hs.ny * hs.nz;
        std::vector<double> Es(nvox);
        for (int64_t v = 0; v < nvox; ++v) Es[v] = hs.solid[v] ? hs.E[v] : 0.0;
        std::vector<int32_t> lat(hs.lat_id.size());
        for (size_t k = 0; k < lat.size(); ++k) {
          const int32_t q = hs.lat_id[k];
          lat[k] = (q < 0 || hs.dir[q]) ? -1 : q;
        }
        h->d_Es = h->upload(Es);
        h->d_lat_ebe = h->upload(lat);
        h->d_lat_all = h->upload(hs.lat_id);
        CK(cudaMemcpyAsync(h->K0h, h->d_K0, sizeof(h->K0h), cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
      }
    }

    // ---------------- host bookkeeping -----------------------------------
    std::vector<int32_t> node_local(N, -1);
    for (int g = 0; g < G; ++g)
      for (int e = hs.grain_ptr[g]; e < hs.grain_ptr[g + 1]; ++e)
        node_local[hs.grain_nodes[e]] = e - hs.grain_ptr[g];
    for (int c = 0; c < C; ++c)
      for (int e = hs.iface_ptr[c]; e < hs.iface_ptr[c + 1]; ++e)
        node_local[hs.iface_nodes[e]] = e - hs.iface_ptr[c];

    // ---------------- batches --------------------------------------------
    const bool sparse = h->sparse();
    build_batch(h, h->gb, hs.grain_ptr, hs.grain_nodes, -1, true, !sparse);
    const bool ilu = h->ilu_smoother();
    if (!sparse && !ilu) build_batch(h, h->cb, hs.contact_ptr, hs.contact_nodes, -1, true);
    build_batch(h, h->sb, {}, {}, Nm, true);
    int64_t lb = (h->gb.ntiles + h->cb.ntiles) * (int64_t)TILE * 8;
    h->rep.local_bytes = lb;
    h->rep.coarse_bytes = h->sb.ntiles * (int64_t)TILE * 8 * (hs.opt.coarse_refine ? 2 : 1);

    // grain positions and contact reverse map
    std::vector<int32_t> nbg(G), gpos(h->n_dof, -1);
    {
      int64_t rb = 0;
      for (int g = 0; g < G; ++g) {
        int nd = 3 * (hs.grain_ptr[g + 1] - hs.grain_ptr[g]);
        nbg[g] = (nd + TB - 1) / TB;
        for (int i = 0; i < nd; ++i)
          gpos[3 * hs.grain_nodes[hs.grain_ptr[g] + i / 3] + i % 3] = (int32_t)(rb * TB + i);
        rb += nbg[g];
      }
    }
    h->h_nbg = nbg;
    {
      std::vector<int32_t> cnt(h->n_dof + 1, 0);
      int64_t rb = 0;
      std::vector<int64_t> crb(C);
      for (int c = 0; c < C; ++c) {
        crb[c] = rb;
        int nd = 3 * (hs.contact_ptr[c + 1] - hs.contact_ptr[c]);
        for (int i = 0; i < nd; ++i) cnt[3 * hs.contact_nodes[hs.contact_ptr[c] + i / 3] + i % 3 + 1]++;
        rb += (nd + TB - 1) / TB;
      }
      for (int d = 0; d < h->n_dof; ++d) cnt[d + 1] += cnt[d];
      std::vector<int32_t> idx(cnt[h->n_dof]), fill(cnt.begin(), cnt.end() - 1);
      for (int c = 0; c < C; ++c) {
        int nd = 3 * (hs.contact_ptr[c + 1] - hs.contact_ptr[c]);
        for (int i = 0; i < nd; ++i) {
          int d = 3 * hs.contact_nodes[hs.contact_ptr[c] + i / 3] + i % 3;
          idx[fill[d]++] = (int32_t)(crb[c] * TB + i);
        }
      }
      h->d_cptr = h->upload(cnt);
      h->d_cidx = h->upload(idx);
    }

    // coarse bookkeeping
    DevCoarse& co = h->co;
    co.n_grains = G;
    co.n_ifaces = C;
    co.Nm = Nm;
    co.n_dof = h->n_dof;
    std::vector<int32_t> ld(G), mortar_iface(hs.n_mortar_nodes());
    std::vector<int64_t> b_off(G), wt_off(C), yext_off(G), cg_off(G), chunk_t(h->gb.nrows);
    int64_t off = 0, yo = 0, co2 = 0, ct = 0;
    int maxk = 0;
    for (int g = 0; g < G; ++g) {
      int k = hs.gcols_ptr[g + 1] - hs.gcols_ptr[g];
      maxk = std::max(maxk, k);
      ld[g] = k + 1;
      b_off[g] = off;
      off += (int64_t)TB * nbg[g] * ld[g];
      yext_off[g] = yo;
      yo += ld[g];
      cg_off[g] = co2;
      co2 += (int64_t)k * k;
    }
    {
      int64_t rb = 0;
      for (int g = 0; g < G; ++g)
        for (int I = 0; I < nbg[g]; ++I, ++rb) {
          chunk_t[rb] = ct;
          ct += ld[g];
        }
    }
    int64_t wo = 0;
    for (int c = 0; c < C; ++c) {
      wt_off[c] = wo;
      int nu = hs.mortar_ptr[c + 1] - hs.mortar_ptr[c];
      wo += (int64_t)9 * (hs.iface_ptr[c + 1] - hs.iface_ptr[c]) * nu;   // 3|F| x 3nu block
      for (int m = hs.mortar_ptr[c]; m < hs.mortar_ptr[c + 1]; ++m) mortar_iface[m] = c;
    }
    std::vector<int32_t> mcol_ptr(Nm + 1, 0), mcol_g, mcol_j;
    for (int g = 0; g < G; ++g)
      for (int e = hs.gcols_ptr[g]; e < hs.gcols_ptr[g + 1]; ++e) mcol_ptr[hs.gcols[e] + 1]++;
    for (int k = 0; k < Nm; ++k) mcol_ptr[k + 1] += mcol_ptr[k];
    mcol_g.resize(mcol_ptr[Nm]);
    mcol_j.resize(mcol_ptr[Nm]);
    {
      std::vector<int32_t> fill(mcol_ptr.begin(), mcol_ptr.end() - 1);
      for (int g = 0; g < G; ++g)
        for (int e = hs.gcols_ptr[g]; e < hs.gcols_ptr[g + 1]; ++e) {
          int k = hs.gcols[e];
          mcol_g[fill[k]] = g;
          mcol_j[fill[k]++] = e - hs.gcols_ptr[g];
        }
    }
    std::vector<int32_t> chunk_ptr(G + 1, 0);
    for (int g = 0; g < G; ++g) chunk_ptr[g + 1] = chunk_ptr[g] + nbg[g];
    h->h_ld = ld;
    co.grain_node_ptr = h->upload(hs.grain_ptr);
    co.grain_nodes = h->upload(hs.grain_nodes);
    co.gcols_ptr = h->upload(hs.gcols_ptr);
    co.gcols = h->upload(hs.gcols);
    co.giface_ptr = h->upload(hs.giface_ptr);
    co.giface = h->upload(hs.giface);
    co.ld = h->upload(ld);
    co.max_ld = ld.empty() ? 0 : *std::max_element(ld.begin(), ld.end());
    co.max_nu3 = 0;
    for (size_t cf = 0; cf + 1 < hs.mortar_ptr.size(); ++cf)
      co.max_nu3 = std::max(co.max_nu3, 3 * (hs.mortar_ptr[cf + 1] - hs.mortar_ptr[cf]));
    co.b_off = h->upload(b_off);
    co.B = h->dalloc<double>(std::max<int64_t>(off, 1));
    co.R = h->dalloc<double>(std::max<int64_t>(off, 1), true);
    co.iface_ptr = h->upload(hs.iface_ptr);
    co.iface_nodes = h->upload(hs.iface_nodes);
    co.mortar_ptr = h->upload(hs.mortar_ptr);
    co.wt_off = h->upload(wt_off);
    co.W = h->dalloc<double>(std::max<int64_t>(wo, 1));
    co.node_class = h->upload(hs.node_class);
    co.node_owner = h->upload(hs.node_owner);
    co.node_iface = h->upload(hs.node_iface);
    co.node_local = h->upload(node_local);
    co.n_chunks = h->gb.nrows;
    co.chunk_g = h->gb.row_s;
    {
      std::vector<int32_t> r0(h->gb.nrows);
      int64_t rb = 0;
      for (int g = 0; g < G; ++g)
        for (int I = 0; I < nbg[g]; ++I) r0[rb++] = TB * I;
      co.chunk_r0 = h->upload(r0);
    }
    co.chunk_t = h->upload(chunk_t);
    co.tpart = h->dalloc<double>(std::max<int64_t>(ct, 1));
    co.chunk_ptr = h->upload(chunk_ptr);
    co.mcol_ptr = h->upload(mcol_ptr);
    co.mcol_g = h->upload(mcol_g);
    co.mcol_j = h->upload(mcol_j);
    co.yext = h->dalloc<double>(std::max<int64_t>(yo, 1));
    co.gpart = h->dalloc<double>(std::max<int64_t>(yo, 1));
    co.yext_off = h->upload(yext_off);
    h->co_ct = ct;
    h->co_off = off;
    h->co_cg = co2;
    h->co_yo = yo;
    co.Dc = h->dalloc<double>(std::max(G, 1));
    co.Cg = h->dalloc<double>(std::max<int64_t>(co2, 1), true);
    co.cg_off = h->upload(cg_off);
    co.mortar_iface = h->upload(mortar_iface);
    co.gpos = h->upload(gpos);
    co.g_lmap = h->gb.lmap;
    co.g_row_s = h->gb.row_s;
    co.g_row_base = h->gb.row_base;
    co.max_k = maxk;
    h->rep.prolong_nnz = off + wo / 3;   // Q^o entries with a nonzero (Gaussian) pattern
    CK(cudaMemsetAsync(co.B, 0, std::max<int64_t>(off, 1) * 8, h->st));
    CK(cudaMemsetAsync(co.R, 0, std::max<int64_t>(off, 1) * 8, h->st));
    CK(cudaMemsetAsync(co.Dc, 0, std::max(G, 1) * 8, h->st));

    // node lists for extraction
    h->d_gnode_ptr = h->upload(hs.grain_ptr);
    h->d_gnodes = h->upload(hs.grain_nodes);
    h->d_cnode_ptr = h->upload(hs.contact_ptr);
    h->d_cnodes = h->upload(hs.contact_nodes);

    // work vectors
    int nd = h->n_dof;
    for (double** p : {&h->d_in, &h->d_out, &h->d_y, &h->d_r1, &h->d_z1, &h->d_t, &h->d_x,
                       &h->d_u, &h->d_bb})
      *p = h->dalloc<double>(nd);
    h->d_rm = h->dalloc<double>(std::max(Nm, 1));
    h->d_ym = h->dalloc<double>(std::max(Nm, 1));
    h->d_rc = h->dalloc<double>(std::max(G, 1));
    h->d_yc = h->dalloc<double>(std::max(G, 1));
    CK(cudaMemsetAsync(h->d_rm, 0, std::max(Nm, 1) * 8, h->st));

    // ---------------- T_ML: local inversions / factorisations ------------
    Nvtx nv_ml("hplmm_setup:T_ML");
    Timer tl(h->st);
    int32_t big = INT_MAX;
    HandleAlloc halloc(h);
    CK(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, h->device));
    if (sparse) {
      std::string err;
      static const bool dbg = getenv("HPLMM_DEBUG") != nullptr;
      auto wall = [&]() {
        if (dbg) CK(cudaStreamSynchronize(h->st));
        return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
      };
      double t0 = wall();
      // 1 = automatic, teams allowed (sn_solve_cfg)
      const int shape = hs.opt.sn_shape ? hs.opt.sn_shape : (hs.opt.sn_split >= 0 ? 1 : 0);
      // experiments: per-batch launch shape (HPLMM_SN_SHAPE_G / _C = 8 | 16)
      const int shape_g = getenv("HPLMM_SN_SHAPE_G") ? atoi(getenv("HPLMM_SN_SHAPE_G")) : shape;
      const int shape_c = getenv("HPLMM_SN_SHAPE_C") ? atoi(getenv("HPLMM_SN_SHAPE_C")) : shape;
      // experiments: x of the one-RHS solves in global memory (-1 = automatic per batch)
      const int xg_all = getenv("HPLMM_SN_XG") ? atoi(getenv("HPLMM_SN_XG")) : -1;
      const int xg_g = getenv("HPLMM_SN_XG_G") ? atoi(getenv("HPLMM_SN_XG_G")) : xg_all;
      const int xg_c = getenv("HPLMM_SN_XG_C") ? atoi(getenv("HPLMM_SN_XG_C")) : xg_all;
      // the contact-grid analysis (host) runs on its own thread while the grain
      // batch is analysed, uploaded and its factorisation is queued on the GPU
      std::string err_c;
      bool ok_c = true;
      std::thread th_c;
      if (!ilu)
        th_c = std::thread([&] {
          ok_c = sn_analyse(hs, hs.contact_ptr, hs.contact_nodes, sn_leaf(), h->sc.sym, err_c, h->nsm,
                            shape_c, xg_c);
        });
      struct Joiner {
        std::thread& t;
        ~Joiner() { if (t.joinable()) t.join(); }
      } joiner{th_c};
      if (getenv("HPLMM_SN_OVERLAP") && getenv("HPLMM_SN_OVERLAP")[0] == '0' && th_c.joinable())
        th_c.join();   // experiments: the two analyses one after the other
      if (!sn_analyse(hs, hs.grain_ptr, hs.grain_nodes, sn_leaf(), h->sg.sym, err, h->nsm, shape_g, xg_g))
        throw HError{HPLMM_ERR_ARG, "supernodal analysis: " + err};
      double t1 = wall();
      try {
        h->sg.sym.split = hs.opt.sn_split;
        sn_upload(h->sg, halloc, h->st, h->nsm);
        double t2 = wall();
        sn_factor(h->sg, h->d_val, halloc, h->st, kSnPoolBytes);
        double t3 = wall();
        if (dbg)
          fprintf(stderr, "hplmm T_ML: grain analyse %.3f s, upload %.3f s, grain factor %.3f s\n", t1 - t0,
                  t2 - t1, t3 - t2);
        if (th_c.joinable()) th_c.join();
        if (!ok_c) throw HError{HPLMM_ERR_ARG, "supernodal analysis: " + err_c};
        double t4 = wall();
        if (!ilu) {
          h->sc.sym.split = hs.opt.sn_split;
          sn_upload(h->sc, halloc, h->st, h->nsm);
        }
        h->rep.sn_shape_grain = h->sg.work.cons;
        h->rep.sn_shape_contact = ilu ? 0 : h->sc.work.cons;
        h->rep.sn_teams_grain = h->sg.work.nteams;
        h->rep.sn_teams_contact = ilu ? 0 : h->sc.work.nteams;
        h->rep.sn_team_max = std::max(h->sg.work.team, ilu ? 1 : h->sc.work.team);
        h->rep.sn_xg_grain = h->sg.sym.xg1 ? 1 : 0;
        h->rep.sn_xg_contact = (!ilu && h->sc.sym.xg1) ? 1 : 0;
        if (!ilu) try {
          sn_factor(h->sc, h->d_val, halloc, h->st, kSnPoolBytes);
          if (dbg)
            fprintf(stderr, "hplmm T_ML: wait for the contact analysis %.3f s, contact upload + factor %.3f s\n",
                    t4 - t3, wall() - t4);
        } catch (SnError& e) {
          e.sub += G;   // contact grids are numbered after the grains
          throw;
        }
      } catch (const SnError& e) {
        h->rep.err_index = e.sub;
        throw HError{(hplmm_status)e.status, e.msg + " " + std::to_string(e.sub)};
      }
      h->rep.local_bytes = 8 * (h->sg.sym.factor_doubles + h->sc.sym.factor_doubles);
      // maps of the local (elimination-order) solutions back to global DOFs
      std::vector<int32_t> gpos(h->n_dof, -1);
      for (size_t p = 0; p < h->sg.sym.gmap.size(); ++p) gpos[h->sg.sym.gmap[p]] = (int32_t)p;
      h->d_gpos_sn = h->upload(gpos);
      std::vector<int32_t> cnt(h->n_dof + 1, 0);
      for (int32_t d : h->sc.sym.gmap) cnt[d + 1]++;
      for (int d = 0; d < h->n_dof; ++d) cnt[d + 1] += cnt[d];
      std::vector<int32_t> idx(cnt[h->n_dof]), fill(cnt.begin(), cnt.end() - 1);
      for (size_t p = 0; p < h->sc.sym.gmap.size(); ++p) idx[fill[h->sc.sym.gmap[p]]++] = (int32_t)p;
      h->d_cptr_sn = h->upload(cnt);
      h->d_cidx_sn = h->upload(idx);
      CK(cudaMemcpyAsync(h->sb.err, &big, 4, cudaMemcpyHostToDevice, h->st));
      CK(cudaMemsetAsync(h->sb.tiles, 0, (size_t)h->sb.ntiles * TILE * 8, h->st));
    } else {
      for (DevBatch* b : {&h->gb, &h->cb, &h->sb}) {
        if (b == &h->cb && ilu) continue;
        CK(cudaMemsetAsync(b->tiles, 0, (size_t)b->ntiles * TILE * 8, h->st));
        CK(cudaMemcpyAsync(b->err, &big, 4, cudaMemcpyHostToDevice, h->st));
      }
      launch_extract_local(h->gb, hs.grain_ptr.back(), h->d_gnode_ptr, h->d_gnodes, h->d_row_ptr,
                           h->d_col, h->d_val, h->st);
      launch_pad_identity(h->gb, h->st);
      launch_sweep_invert(h->gb, h->st);
      if (!ilu) {
        launch_extract_local(h->cb, hs.contact_ptr.back(), h->d_cnode_ptr, h->d_cnodes,
                             h->d_row_ptr, h->d_col, h->d_val, h->st);
        launch_pad_identity(h->cb, h->st);
        launch_sweep_invert(h->cb, h->st);
      }
      CK(cudaGetLastError());
      check_batch_err(h, h->gb, 0, false);
      if (!ilu) check_batch_err(h, h->cb, G, false);
    }
    if (ilu) setup_ilu(h);
    if (ilu || hs.opt.n_st > 1)
      for (double** p : {&h->d_ls_u, &h->d_ls_t0, &h->d_ls_t1, &h->d_ls_acc})
        *p = h->dalloc<double>(h->n_dof);
    h->rep.t_setup_local_s = tl.stop();

    // ---------------- T_MG: mortars, P_B, S, S^-1 -------------------------
    Nvtx nv_mg("hplmm_setup:T_MG");
    Timer tc(h->st);
    static const bool dbg_mg = getenv("HPLMM_DEBUG") != nullptr;
    double tmg = 0;
    auto mg_mark = [&](const char* what) {   // phase wall times under HPLMM_DEBUG
      if (!dbg_mg) return;
      CK(cudaStreamSynchronize(h->st));
      const double now =
          std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
      if (tmg > 0) fprintf(stderr, "hplmm T_MG: %-22s %.3f s\n", what, now - tmg);
      tmg = now;
    };
    mg_mark("start");
    {
      std::vector<int32_t> iface_of(hs.iface_nodes.size());
      for (int c = 0; c < C; ++c)
        for (int e = hs.iface_ptr[c]; e < hs.iface_ptr[c + 1]; ++e) iface_of[e] = c;
      int32_t* d_iface_of = h->upload(iface_of);
      co.iface_of = d_iface_of;
      co.n_iface_nodes = (int)iface_of.size();
      int32_t* d_mortar_nodes = h->upload(hs.mortar_nodes);
      if (hs.opt.mortar_kind == 0) {
        launch_mortar_weights((int)iface_of.size(), d_iface_of, co.iface_ptr, co.iface_nodes,
                              co.mortar_ptr, d_mortar_nodes, co.wt_off, h->d_ijk, hs.opt.beta,
                              co.W, h->st);
      } else {
        // Algebraic mortars: batch of SPD interface blocks A~ = A^[free, free]
        // (free = interface nodes that are not mortar nodes), inverted by the
        // packed-tile sweep, applied to the 3 nu_c constraint columns
        std::vector<int32_t> free_ptr(C + 1, 0), free_nodes, free_pos, con_pos;
        int maxq = 0;
        for (int c = 0; c < C; ++c) {
          std::vector<int32_t> X(hs.mortar_nodes.begin() + hs.mortar_ptr[c],
                                 hs.mortar_nodes.begin() + hs.mortar_ptr[c + 1]);
          maxq = std::max(maxq, 3 * (int)X.size());
          std::sort(X.begin(), X.end());
          for (int e = hs.iface_ptr[c]; e < hs.iface_ptr[c + 1]; ++e) {
            const int y = hs.iface_nodes[e];
            if (!std::binary_search(X.begin(), X.end(), y)) {
              free_nodes.push_back(y);
              free_pos.push_back(e - hs.iface_ptr[c]);
            }
          }
          free_ptr[c + 1] = (int32_t)free_nodes.size();
        }
        for (int m = 0; m < hs.n_mortar_nodes(); ++m) {
          const int c = mortar_iface[m], x = hs.mortar_nodes[m];
          const int* F = hs.iface_nodes.data() + hs.iface_ptr[c];
          const int nF = hs.iface_ptr[c + 1] - hs.iface_ptr[c];
          con_pos.push_back((int32_t)(std::lower_bound(F, F + nF, x) - F));
        }
        DevBatch ab;
        build_batch(h, ab, free_ptr, free_nodes, -1, true, true, /*transient=*/true);
        int32_t big2 = INT_MAX;
        CK(cudaMemsetAsync(ab.tiles, 0, (size_t)ab.ntiles * TILE * 8, h->st));
        CK(cudaMemcpyAsync(ab.err, &big2, 4, cudaMemcpyHostToDevice, h->st));
        int32_t* d_free_ptr = h->upload(free_ptr);
        int32_t* d_free_pos = h->upload(free_pos);
        int32_t* d_con_pos = h->upload(con_pos);
        const bool surf = hs.opt.mortar_kind == 2;
        int64_t* d_koff = nullptr;
        double* d_Kbuf = nullptr;
        if (surf) {
          // Surface reading (R29): faces shared by the pair's grains with all
          // four nodes on the interface, in the oracle's order (array axis z,
          // y, x; voxels lexicographic), and the pattern couplings inside F_c
          const int nx = hs.nx, ny = hs.ny, nz = hs.nz;
          const int64_t nx1 = nx + 1, ny1 = ny + 1;
          std::vector<std::vector<int4>> fc(C);
          const int comp_of_axis[3] = {2, 1, 0};
          const int dims[3] = {nz, ny, nx};
          for (int ax = 0; ax < 3; ++ax) {
            int o[2], oi = 0;
            for (int a = 0; a < 3; ++a)
              if (a != ax) o[oi++] = a;
            for (int k = 0; k < nz; ++k)
              for (int j = 0; j < ny; ++j)
                for (int i = 0; i < nx; ++i) {
                  int v1c[3] = {k, j, i};
                  if (v1c[ax] + 1 >= dims[ax]) continue;
                  int v2c[3] = {k, j, i};
                  v2c[ax] += 1;
                  const int64_t v1 = i + (int64_t)nx * (j + (int64_t)ny * k);
                  const int64_t v2 = v2c[2] + (int64_t)nx * (v2c[1] + (int64_t)ny * v2c[0]);
                  if (!hs.solid[v1] || !hs.solid[v2]) continue;
                  const int ga = hs.grain[v1], gb = hs.grain[v2];
                  if (ga == gb) continue;
                  int nodes[4], q = 0;
                  for (int db = 0; db < 2; ++db)
                    for (int da = 0; da < 2; ++da) {
                      int c3[3] = {v2c[0], v2c[1], v2c[2]};
                      c3[o[0]] += da;
                      c3[o[1]] += db;
                      nodes[q++] = hs.lat_id[c3[2] + nx1 * (c3[1] + ny1 * c3[0])];
                    }
                  const int cf = nodes[0] >= 0 ? hs.node_iface[nodes[0]] : -1;
                  if (cf < 0) continue;
                  const int p1 = std::min(ga, gb), p2 = std::max(ga, gb);
                  if (hs.iface_pair[2 * cf] != p1 || hs.iface_pair[2 * cf + 1] != p2) continue;
                  bool all = true;
                  int pos[4];
                  const int* F = hs.iface_nodes.data() + hs.iface_ptr[cf];
                  const int nF = hs.iface_ptr[cf + 1] - hs.iface_ptr[cf];
                  for (int t = 0; t < 4 && all; ++t) {
                    all = nodes[t] >= 0 && hs.node_iface[nodes[t]] == cf;
                    if (all) pos[t] = (int)(std::lower_bound(F, F + nF, nodes[t]) - F);
                  }
                  if (!all) continue;
                  const int code = comp_of_axis[o[0]] | (comp_of_axis[o[1]] << 2) |
                                   (comp_of_axis[ax] << 4);
                  fc[cf].push_back(make_int4(pos[0], pos[1], pos[2], pos[3]));
                  fc[cf].push_back(make_int4(code, (int)v1, (int)v2, 0));
                }
          }
          std::vector<int32_t> face_ptr(C + 1, 0);
          std::vector<int4> faces;
          for (int c = 0; c < C; ++c) {
            faces.insert(faces.end(), fc[c].begin(), fc[c].end());
            face_ptr[c + 1] = (int32_t)(faces.size() / 2);
          }
          std::vector<int32_t> tie_ptr(hs.iface_nodes.size() + 1, 0), tie_q;
          std::vector<int64_t> koff(C + 1, 0);
          for (int c = 0; c < C; ++c) {
            const int* F = hs.iface_nodes.data() + hs.iface_ptr[c];
            const int nF = hs.iface_ptr[c + 1] - hs.iface_ptr[c];
            for (int f = 0; f < nF; ++f) {
              const int y = F[f];
              for (int e = hs.row_ptr[y]; e < hs.row_ptr[y + 1]; ++e) {
                const int qn = hs.col_idx[e];
                if (qn == y || hs.node_iface[qn] != c) continue;
                tie_q.push_back((int32_t)(std::lower_bound(F, F + nF, qn) - F));
              }
              tie_ptr[hs.iface_ptr[c] + f + 1] = (int32_t)tie_q.size();
            }
            koff[c + 1] = koff[c] + (int64_t)(3 * nF) * (3 * nF);
          }
          d_koff = h->upload(koff, true);
          d_Kbuf = h->dalloc<double>((size_t)std::max<int64_t>(koff[C], 1), true);
          double* d_K1 = h->dalloc<double>(144, true);
          double* d_tau = h->dalloc<double>(1, true);
          launch_surf_operator(C, co.iface_ptr, h->upload(face_ptr, true),
                               reinterpret_cast<const int4*>(h->upload(
                                   std::vector<int32_t>(reinterpret_cast<int32_t*>(faces.data()),
                                                        reinterpret_cast<int32_t*>(faces.data()) +
                                                            4 * faces.size()),
                                   true)),
                               h->d_E, h->d_solid, (int64_t)hs.nx * hs.ny * hs.nz, hs.nu,
                               kSurfaceTie, h->upload(tie_ptr, true), h->upload(tie_q, true),
                               d_koff, d_K1, d_tau, d_Kbuf, h->st);
          launch_surf_extract(ab, co.iface_ptr, d_free_ptr, d_free_pos, d_koff, d_Kbuf, h->st);
        } else {
          launch_extract_local(ab, free_ptr.back(), d_free_ptr, h->upload(free_nodes),
                               h->d_row_ptr, h->d_col, h->d_val, h->st);
        }
        launch_pad_identity(ab, h->st);
        launch_sweep_invert(ab, h->st);
        CK(cudaGetLastError());
        check_batch_err(h, ab, 0, false);
        for (int q = 0; q < maxq; ++q) {
          if (surf)
            launch_surf_rhs(q, ab, co.iface_ptr, co.mortar_ptr, d_free_ptr, d_free_pos, d_con_pos,
                            d_koff, d_Kbuf, h->st);
          else
            launch_alg_rhs(q, ab, co.mortar_ptr, d_mortar_nodes, h->d_row_ptr, h->d_col,
                           h->d_val, h->st);
          launch_symv(ab, h->st);
          launch_alg_store(q, C, ab, co.mortar_ptr, d_free_ptr, d_free_pos, d_con_pos, co.wt_off,
                           co.W, h->st);
        }
        CK(cudaGetLastError());
      }
    }
    mg_mark("mortars");
    launch_build_R(co, h->gb, h->d_row_ptr, h->d_col, h->d_val, h->st);
    {
      std::vector<int32_t> kc(G);
      for (int g = 0; g < G; ++g) kc[g] = ld[g] - 1;
      if (sparse)
      {
        // R serves as the workspace of the multi-RHS sweep; rebuild it for S
        sn_shape_vectors(h->sg, halloc, h->st, h->nsm, kc, co.b_off, co.ld, co.R, co.B,
                         std::max<int64_t>(off, 1));
        CK(cudaMemsetAsync(co.R, 0, std::max<int64_t>(off, 1) * 8, h->st));
        launch_build_R(co, h->gb, h->d_row_ptr, h->d_col, h->d_val, h->st);
      }
      else
        launch_symm_neg(h->gb, co.b_off, co.ld, h->upload(kc), (maxk + TB - 1) / TB, co.R, co.B,
                        h->st);
    }
    mg_mark("shape vectors");
    launch_grain_AB(co, h->gb, h->d_row_ptr, h->d_col, h->d_val, h->st);
    launch_grain_BtY(co, h->gb, h->st);
    mg_mark("grain A B, B^T Y");
    int64_t npS = (int64_t)TB * h->sb.max_nb;
    // small S: dense copy kept for export (HPLMM_ART_S); large S (cfg5: 67 GB
    // dense) is assembled straight into the packed lower tiles
    bool keepS = (npS * npS * 8) <= (int64_t)512 << 20;
    if (keepS) {
      h->lds = npS;
      h->d_Sdense = h->dalloc<double>(std::max<int64_t>(npS * npS, 1));
      CK(cudaMemsetAsync(h->d_Sdense, 0, std::max<int64_t>(npS * npS, 1) * 8, h->st));
      launch_S_iface(co, h->d_row_ptr, h->d_col, h->d_val, h->d_Sdense, npS, h->st);
      launch_S_grain(co, h->d_Sdense, npS, h->st);
      launch_pack_dense(h->sb, h->d_Sdense, npS, h->st);
    } else {
      h->lds = 0;
      h->d_Sdense = nullptr;
      CK(cudaMemsetAsync(h->sb.tiles, 0, (size_t)h->sb.ntiles * TILE * 8, h->st));
      launch_S_iface(co, h->d_row_ptr, h->d_col, h->d_val, h->sb.tiles, 0, h->st);
      launch_S_grain(co, h->sb.tiles, 0, h->st);
    }
    launch_pad_identity(h->sb, h->st);
    mg_mark("S assembly");
    if (hs.opt.coarse_refine) {
      h->sS = h->sb;
      h->sS.tiles = h->dalloc<double>((size_t)h->sb.ntiles * TILE);
      h->sS.xloc = h->dalloc<double>((size_t)h->sb.nloc);
      h->sS.yloc = h->dalloc<double>((size_t)h->sb.nloc);
      CK(cudaMemcpyAsync(h->sS.tiles, h->sb.tiles, (size_t)h->sb.ntiles * TILE * 8,
                         cudaMemcpyDeviceToDevice, h->st));
    }
    if (h->chol()) {
      const int nbS = h->sb.max_nb;
      h->d_linv = h->dalloc<double>((size_t)std::max(nbS, 1) * TILE);
      h->d_linvT = h->dalloc<double>((size_t)std::max(nbS, 1) * TILE);
      h->d_zc = h->dalloc<double>((size_t)std::max(nbS, 1) * TB);
      h->d_cflag_f = h->dalloc<int>(std::max(nbS, 1));
      h->d_cflag_b = h->dalloc<int>(std::max(nbS, 1));
      CK(cudaMemsetAsync(h->d_cflag_f, 0, std::max(nbS, 1) * 4, h->st));
      CK(cudaMemsetAsync(h->d_cflag_b, 0, std::max(nbS, 1) * 4, h->st));
      h->coarse_epoch = 0;
      launch_chol_factor(h->sb, h->d_linv, h->d_linvT, h->st);
    } else {
      launch_sweep_invert(h->sb, h->st);
    }
    CK(cudaGetLastError());
    check_batch_err(h, h->sb, 0, true);
    mg_mark("coarse inversion");
    h->rep.t_setup_coarse_s = tc.stop();
    CK(cudaStreamSynchronize(h->st));
    h->free_setup();
    h->gb.dinv = h->gb.cbuf = h->gb.wbuf = nullptr;
    h->cb.dinv = h->cb.cbuf = h->cb.wbuf = nullptr;
    h->sb.dinv = h->sb.cbuf = h->sb.wbuf = nullptr;
    h->sS.dinv = h->sS.cbuf = h->sS.wbuf = nullptr;
    co.R = nullptr;
    co.Cg = nullptr;
    h->setup_done = true;
    return HPLMM_OK;
  } catch (const SnError& e) {
    h->rep.err_index = e.sub;
    return fail(HError{(hplmm_status)e.status, e.msg});
  } catch (const HError& e) {
    return fail(e);
  }
}

hplmm_status hplmm_update_moduli(hplmm_handle* h, const double* E, void* stream) {
  if (!h || !E) { g_last_error = "null argument"; return HPLMM_ERR_ARG; }
  try {
    if (!h->setup_done) throw HError{HPLMM_ERR_STATE, "hplmm_update_moduli before hplmm_setup"};
    if (h->matrix_external)
      throw HError{HPLMM_ERR_STATE, "hplmm_update_moduli: A^ was supplied by the caller (no voxel moduli)"};
    if (!h->sparse() || h->ilu_smoother())
      throw HError{HPLMM_ERR_STATE,
                   "hplmm_update_moduli needs local_factor = 1 (supernodal) and smoother = 0 (M_CG)"};
    require_device(h);
    h->st = (cudaStream_t)stream;
    HostSetup& hs = h->hs;
    const int64_t nvox = (int64_t)hs.nx * hs.ny * hs.nz;
    for (int64_t v = 0; v < nvox; ++v)
      if (hs.solid[v] && !(E[v] > 0) )
        throw HError{HPLMM_ERR_ARG, "hplmm_update_moduli: E <= 0 in solid voxel " + std::to_string(v)};
    Timer t(h->st);
    hs.E.assign(E, E + nvox);
    CK(cudaMemcpyAsync(h->d_E, hs.E.data(), (size_t)nvox * 8, cudaMemcpyHostToDevice, h->st));
    if (h->d_Es) {
      std::vector<double> Es(nvox);
      for (int64_t v = 0; v < nvox; ++v) Es[v] = hs.solid[v] ? hs.E[v] : 0.0;
      CK(cudaMemcpyAsync(h->d_Es, Es.data(), (size_t)nvox * 8, cudaMemcpyHostToDevice, h->st));
      CK(cudaStreamSynchronize(h->st));   // Es is a local
    }
    // A^ values and b^ from the new moduli (same pattern, R4)
    launch_assemble((int)h->nnzb, h->d_block_row, h->d_col, h->d_ijk, h->d_dir, h->d_solid,
                    h->d_E, hs.nx, hs.ny, hs.nz, h->d_K0, h->d_val, h->st);
    launch_assemble_rhs(h->n_nodes, h->d_drow_ptr, h->d_dcol, h->d_ijk, h->d_dir, h->d_solid,
                        h->d_E, hs.nx, hs.ny, hs.nz, h->d_K0, h->d_f, h->d_uD, h->d_b, h->st);
    CK(cudaGetLastError());
    // numeric refactorisation of every grain and contact-grid block with the
    // symbolic analysis, factor layout and work lists of hplmm_setup
    HandleAlloc halloc(h);
    try {
      sn_factor(h->sg, h->d_val, halloc, h->st, kSnPoolBytes);
      try {
        sn_factor(h->sc, h->d_val, halloc, h->st, kSnPoolBytes);
      } catch (SnError& e) {
        e.sub += hs.n_grains;
        throw;
      }
    } catch (const SnError& e) {
      h->rep.err_index = e.sub;
      h->free_setup();
      throw HError{(hplmm_status)e.status, e.msg + " " + std::to_string(e.sub)};
    }
    CK(cudaGetLastError());
    h->rep.t_update_s = t.stop();
    CK(cudaStreamSynchronize(h->st));
    h->free_setup();
    h->rhs_set = false;   // the correction columns follow the new A_g (eq:col_cg)
    return HPLMM_OK;
  } catch (const HError& e) {
    return fail(e);
  }
}

hplmm_status hplmm_refresh_coarse(hplmm_handle* h, void* stream) {
  if (!h) { g_last_error = "null handle"; return HPLMM_ERR_ARG; }
  try {
    if (!h->setup_done) throw HError{HPLMM_ERR_STATE, "hplmm_refresh_coarse before hplmm_setup"};
    const HostSetup& hs = h->hs;
    if (!h->sparse() || h->ilu_smoother() || h->chol() || hs.opt.coarse_refine ||
        hs.opt.mortar_kind != 0)
      throw HError{HPLMM_ERR_STATE,
                   "hplmm_refresh_coarse needs local_factor = 1, smoother = 0, coarse_solver = 0, "
                   "coarse_refine = 0 and Gaussian mortars (whose weights do not depend on A^)"};
    require_device(h);
    h->st = (cudaStream_t)stream;
    DevCoarse& co = h->co;
    const int G = hs.n_grains;
    Timer t(h->st);
    HandleAlloc halloc(h);
    const int64_t off = std::max<int64_t>(h->co_off, 1);
    // the setup-only scratch of the T_MG phases, again
    co.R = h->dalloc<double>(off, true);
    co.Cg = h->dalloc<double>(std::max<int64_t>(h->co_cg, 1), true);
    h->sb.dinv = h->dalloc<double>((size_t)std::max(h->sb.nsub, 1) * TILE * SWEEP_M * SWEEP_M, true);
    h->sb.cbuf = h->dalloc<double>((size_t)std::max<int64_t>(h->sb.nrows, 1) * TILE * SWEEP_M, true);
    h->sb.wbuf = h->dalloc<double>((size_t)std::max<int64_t>(h->sb.nrows, 1) * TILE * SWEEP_M, true);
    auto drop = [&]() {
      h->free_setup();
      co.R = co.Cg = nullptr;
      h->sb.dinv = h->sb.cbuf = h->sb.wbuf = nullptr;
    };
    try {
      const int32_t big = INT_MAX;
      CK(cudaMemcpyAsync(h->sb.err, &big, 4, cudaMemcpyHostToDevice, h->st));
      CK(cudaMemsetAsync(co.B, 0, off * 8, h->st));
      CK(cudaMemsetAsync(co.R, 0, off * 8, h->st));
      // shape vectors B_g = -A_g^-1 A^[I_g,:] Q^o[:, cols_g] (eq:col_pk) with the current factors
      launch_build_R(co, h->gb, h->d_row_ptr, h->d_col, h->d_val, h->st);
      std::vector<int32_t> kc(G);
      for (int g = 0; g < G; ++g) kc[g] = h->h_ld[g] - 1;
      sn_shape_vectors(h->sg, halloc, h->st, h->nsm, kc, co.b_off, co.ld, co.R, co.B, off);
      CK(cudaMemsetAsync(co.R, 0, off * 8, h->st));
      launch_build_R(co, h->gb, h->d_row_ptr, h->d_col, h->d_val, h->st);
      // S = P_B^T A^ P_B (eq:mg_struct, R16) and its inverse (R17)
      launch_grain_AB(co, h->gb, h->d_row_ptr, h->d_col, h->d_val, h->st);
      launch_grain_BtY(co, h->gb, h->st);
      CK(cudaMemsetAsync(h->sb.tiles, 0, (size_t)h->sb.ntiles * TILE * 8, h->st));
      if (h->d_Sdense) {
        const int64_t npS = h->lds;
        CK(cudaMemsetAsync(h->d_Sdense, 0, std::max<int64_t>(npS * npS, 1) * 8, h->st));
        launch_S_iface(co, h->d_row_ptr, h->d_col, h->d_val, h->d_Sdense, npS, h->st);
        launch_S_grain(co, h->d_Sdense, npS, h->st);
        launch_pack_dense(h->sb, h->d_Sdense, npS, h->st);
      } else {
        launch_S_iface(co, h->d_row_ptr, h->d_col, h->d_val, h->sb.tiles, 0, h->st);
        launch_S_grain(co, h->sb.tiles, 0, h->st);
      }
      launch_pad_identity(h->sb, h->st);
      launch_sweep_invert(h->sb, h->st);
      CK(cudaGetLastError());
      check_batch_err(h, h->sb, 0, true);
    } catch (const SnError& e) {
      drop();
      throw HError{(hplmm_status)e.status, e.msg};
    } catch (const HError&) {
      drop();
      throw;
    }
    h->rep.t_setup_coarse_s = t.stop();
    CK(cudaStreamSynchronize(h->st));
    drop();
    h->rhs_set = false;   // the correction column sits in B's last column (R15)
    return HPLMM_OK;
  } catch (const HError& e) {
    return fail(e);
  }
}

hplmm_status hplmm_set_rhs(hplmm_handle* h, const double* b, void* stream) {
  if (!h || !b) { g_last_error = "null argument"; return HPLMM_ERR_ARG; }
  try {
    if (!h->setup_done) throw HError{HPLMM_ERR_STATE, "hplmm_set_rhs before hplmm_setup"};
    require_device(h);
    h->st = (cudaStream_t)stream;
    to_device(h, h->d_bb, b, h->n_dof);
    do_set_rhs(h, h->d_bb);
    CK(cudaGetLastError());
    return HPLMM_OK;
  } catch (const HError& e) {
    return fail(e);
  }
}

hplmm_status hplmm_apply(hplmm_handle* h, int32_t op, const double* in, double* out,
                         void* stream) {
  if (!h || !in || !out) { g_last_error = "null argument"; return HPLMM_ERR_ARG; }
  try {
    require_device(h);
    h->st = (cudaStream_t)stream;
    if (op == HPLMM_OP_SPMV || op == HPLMM_OP_SPMV_BSR) {
      if (!h->assembled) throw HError{HPLMM_ERR_STATE, "apply(SPMV) before assemble"};
    } else if (!h->setup_done) {
      throw HError{HPLMM_ERR_STATE, "apply before hplmm_setup"};
    }
    if ((op == HPLMM_OP_MG || op == HPLMM_OP_MINV || op == HPLMM_OP_RESTRICT ||
         op == HPLMM_OP_PROLONG) && !h->rhs_set)
      throw HError{HPLMM_ERR_STATE, "apply(MG/MINV/RESTRICT/PROLONG) needs hplmm_set_rhs"};
    int nd = h->n_dof;
    double* din = h->d_in;
    double* dout = h->d_out;
    if ((op == HPLMM_OP_SPMV || op == HPLMM_OP_SPMV_BSR) && !din) {  // before setup: temporary buffers
      din = h->dalloc<double>(nd);
      dout = h->dalloc<double>(nd);
      h->d_in = din;
      h->d_out = dout;
    }
    int nin = (op == HPLMM_OP_PROLONG) ? h->rep.n_coarse : nd;
    int nout = (op == HPLMM_OP_RESTRICT) ? h->rep.n_coarse : nd;
    const int Nm = h->co.Nm;
    if (op == HPLMM_OP_COARSE) {
      to_device(h, h->d_rm, in, Nm);
      const double* ym = op_coarse(h, h->d_rm);
      from_device(h, out, ym, Nm);
      CK(cudaStreamSynchronize(h->st));
      h->flush_profile();
      return HPLMM_OK;
    }
    if (op == HPLMM_OP_PROLONG) {
      std::vector<double> hin(nin), yc(std::max(h->co.n_grains, 1), 0.0);
      if (is_device_ptr(in)) CK(cudaMemcpy(hin.data(), in, nin * 8, cudaMemcpyDeviceToHost));
      else std::memcpy(hin.data(), in, nin * 8);
      for (size_t j = 0; j < h->h_corr.size(); ++j) yc[h->h_corr[j]] = hin[Nm + j];
      CK(cudaMemcpyAsync(h->d_rm, hin.data(), std::max(Nm, 0) * 8, cudaMemcpyHostToDevice, h->st));
      CK(cudaMemcpyAsync(h->d_yc, yc.data(), yc.size() * 8, cudaMemcpyHostToDevice, h->st));
      launch_prolong(h->co, h->d_rm, h->d_yc, dout, h->st);
    } else {
      to_device(h, din, in, nin);
      switch (op) {
        case HPLMM_OP_SPMV: op_spmv(h, din, nullptr, dout); break;
        case HPLMM_OP_SPMV_BSR:
          bsr_spmv(h, din, nullptr, dout);
          h->launches++;
          break;
        case HPLMM_OP_MG: op_mg(h, din, dout); break;
        case HPLMM_OP_MZETA: op_mzeta(h, din, dout); break;
        case HPLMM_OP_MGRAIN: op_mgrain(h, din, nullptr, nullptr, dout); break;
        case HPLMM_OP_MCG: op_mcg(h, din, dout); break;
        case HPLMM_OP_MINV: op_minv(h, din, dout); break;
        case HPLMM_OP_MILU:
          if (!h->ilu_smoother()) throw HError{HPLMM_ERR_STATE, "MILU needs smoother = 1"};
          op_milu(h, din, dout);
          break;
        case HPLMM_OP_ML: op_ml(h, din, nullptr, dout); break;
        case HPLMM_OP_RESTRICT: {
          launch_restrict(h->co, din, h->d_rm, h->d_rc, h->st);
          std::vector<double> rm(std::max(Nm, 0)), rc(std::max(h->co.n_grains, 1));
          CK(cudaMemcpyAsync(rm.data(), h->d_rm, Nm * 8, cudaMemcpyDeviceToHost, h->st));
          CK(cudaMemcpyAsync(rc.data(), h->d_rc, h->co.n_grains * 8, cudaMemcpyDeviceToHost, h->st));
          CK(cudaStreamSynchronize(h->st));
          std::vector<double> o(nout);
          std::copy(rm.begin(), rm.end(), o.begin());
          for (size_t j = 0; j < h->h_corr.size(); ++j) o[Nm + j] = rc[h->h_corr[j]];
          if (is_device_ptr(out)) CK(cudaMemcpy(out, o.data(), nout * 8, cudaMemcpyHostToDevice));
          else std::memcpy(out, o.data(), nout * 8);
          return HPLMM_OK;
        }
        default: throw HError{HPLMM_ERR_ARG, "unknown op"};
      }
    }
    CK(cudaGetLastError());
    from_device(h, out, dout, nout);
    CK(cudaStreamSynchronize(h->st));
    h->flush_profile();
    return HPLMM_OK;
  } catch (const HError& e) {
    return fail(e);
  }
}

hplmm_status hplmm_apply_many(hplmm_handle* h, int32_t op, int32_t ncols, const double* in,
                              int64_t ldin, double* out, int64_t ldout, void* stream) {
  if (!h || !in || !out) { g_last_error = "null argument"; return HPLMM_ERR_ARG; }
  try {
    if (op != HPLMM_OP_MZETA && op != HPLMM_OP_MGRAIN && op != HPLMM_OP_MCG && op != HPLMM_OP_SPMV)
      throw HError{HPLMM_ERR_ARG, "apply_many: op must be SPMV, MZETA, MGRAIN or MCG"};
    if (ncols < 1 || ncols > kMaxBlock) throw HError{HPLMM_ERR_ARG, "apply_many: ncols must be 1..4"};
    if (!h->setup_done) throw HError{HPLMM_ERR_STATE, "apply_many before hplmm_setup"};
    if (!h->sparse() || h->ilu_smoother())
      throw HError{HPLMM_ERR_STATE, "apply_many needs local_factor = 1 and smoother = 0"};
    const int n = h->n_dof;
    if (ldin < n || ldout < n) throw HError{HPLMM_ERR_ARG, "apply_many: ld < n_dof"};
    require_device(h);
    h->st = (cudaStream_t)stream;
    multi_alloc(h);
    auto& M = h->mr;
    const int64_t ld = h->ldv;
    for (int c = 0; c < ncols; ++c) to_device(h, M.vin + c * ld, in + c * ldin, n);
    if (op == HPLMM_OP_SPMV) {
      op_spmv_k(h, ncols, M.vin, nullptr, M.u, ld, ld);
    } else if (op == HPLMM_OP_MZETA) {
      op_mzeta_k(h, ncols, M.vin, M.u);
    } else if (op == HPLMM_OP_MGRAIN) {
      op_mgrain_k(h, ncols, M.vin, nullptr, nullptr, M.u);
    } else {   // M_CG: z1 = M_zeta^-1 v ; u = z1 + M_g^-1 (v - A z1)
      op_mzeta_k(h, ncols, M.vin, M.z1);
      op_spmv_k(h, ncols, M.z1, M.vin, M.t, ld, ld);
      op_mgrain_k(h, ncols, M.t, M.z1, nullptr, M.u);
    }
    CK(cudaGetLastError());
    for (int c = 0; c < ncols; ++c) from_device(h, out + c * ldout, M.u + c * ld, n);
    CK(cudaStreamSynchronize(h->st));
    return HPLMM_OK;
  } catch (const HError& e) {
    return fail(e);
  }
}

hplmm_status hplmm_solve(hplmm_handle* h, const double* b, double tol, double* x,
                         hplmm_report* report, double* hist, int32_t hist_cap, void* stream) {
  if (!h || !b || !x) { g_last_error = "null argument"; return HPLMM_ERR_ARG; }
  try {
    if (!h->setup_done) throw HError{HPLMM_ERR_STATE, "hplmm_solve before hplmm_setup"};
    if (!(tol > 0)) throw HError{HPLMM_ERR_ARG, "tol must be > 0"};
    require_device(h);
    h->st = (cudaStream_t)stream;
    cudaStream_t st = h->st;
    const int n = h->n_dof;
    const int m = h->hs.opt.restart;
    const int maxit = h->hs.opt.max_iter;
    h->launches = 0;
    if (h->Vcap < m + 1) {
      h->ldv = ((int64_t)n + 31) / 32 * 32;
      h->d_V = h->dalloc<double>((size_t)(m + 1) * h->ldv);
      h->d_partial = h->dalloc<double>((size_t)krylov_partial_doubles(n));
        CK(cudaMemsetAsync(h->d_partial, 0, (size_t)krylov_partial_doubles(n) * 8, h->st));
      h->d_hbuf = h->dalloc<double>(2 * (m + 1) + 8);
      h->Vcap = m + 1;
    }
    Nvtx nv_solve("hplmm_solve");
    Timer tt(st);
    double* dB = h->d_bb;
    to_device(h, dB, b, n);
    // ||b||
    double* hb = h->d_hbuf;
    launch_norm2(n, dB, h->d_partial, hb + 2 * (m + 1), st);
    h->launches += 2;
    double bn2 = 0;
    CK(cudaMemcpyAsync(&bn2, hb + 2 * (m + 1), 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double bnorm = std::sqrt(bn2);
    double* dx = h->d_x;
    CK(cudaMemsetAsync(dx, 0, (size_t)n * 8, st));
    int total = 0, hl = 0;
    bool conv = false;
    double relres = 1.0;
    hplmm_status status = HPLMM_OK;
    if (bnorm == 0.0) {
      conv = true;
      relres = 0.0;
    } else {
      do_set_rhs(h, dB);   // correction columns for this RHS (R15)
      // r = b (x0 = 0)
      CK(cudaMemcpyAsync(h->d_r1, dB, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
      bool graph = graph_eligible(h);
      if (graph && !h->solve_exec) {
        try {
          build_solve_graph(h);
        } catch (const HError& e) {
          h->graph_failed = true;   // fall back to the host-driven loop below
          graph = false;
          if (getenv("HPLMM_DEBUG")) fprintf(stderr, "hplmm: solve graph unavailable: %s\n", e.msg.c_str());
        }
      }
      if (graph) {
        GmresScalars& s0 = *h->h_gs;
        s0 = GmresScalars{};
        s0.m = m;
        s0.maxit = maxit;
        s0.bnorm = bnorm;
        s0.tol = tol;
        CK(cudaMemcpyAsync(h->gdev.s, &s0, sizeof(GmresScalars), cudaMemcpyHostToDevice, st));
        CK(cudaGraphLaunch(h->solve_exec, st));
        CK(cudaMemcpyAsync(h->h_gs, h->gdev.s, sizeof(GmresScalars), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(h->h_ghist, h->gdev.hist, (size_t)maxit * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const GmresScalars& s1 = *h->h_gs;
        if (s1.nonfinite) throw HError{HPLMM_ERR_NONFINITE, "non-finite GMRES residual"};
        total = s1.total;
        conv = s1.converged != 0;
        relres = s1.relres;
        hl = total;
        if (hist)
          for (int i = 0; i < std::min(total, hist_cap); ++i) hist[i] = h->h_ghist[i];
        h->launches += h->graph_launches_cycle * s1.cycles + h->graph_launches_step * total;
      }
      std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1);
      // the per-step Hessenberg column comes back through pinned memory
      if (h->hh_cap < 2 * (m + 1) + 1) {
        if (h->h_hh) cudaFreeHost(h->h_hh);
        CK(cudaMallocHost(&h->h_hh, (size_t)(2 * (m + 1) + 1) * 8));
        h->hh_cap = 2 * (m + 1) + 1;
      }
      double* hh = h->h_hh;
      double beta2 = bn2;
      while (!graph) {
        double beta = std::sqrt(beta2);
        // V0 = r / beta
        double* V = h->d_V;
        launch_scale(n, h->d_r1, hb + 2 * (m + 1), 1, V, st);
        h->launches++;
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int k = 0;
        for (int j = 0; j < m; ++j) {
          Nvtx nv_step("arnoldi_step");
          double* vj = V + j * h->ldv;
          double* w = V + (j + 1) * h->ldv;
          op_minv(h, vj, h->d_u);
          op_spmv(h, h->d_u, nullptr, w);
          // CGS2
          launch_multidot(n, j + 1, V, h->ldv, w, h->d_partial, hb, st);
          launch_update(n, j + 1, V, h->ldv, hb, w, nullptr, nullptr, st);
          launch_multidot(n, j + 1, V, h->ldv, w, h->d_partial, hb + (m + 1), st);
          launch_update(n, j + 1, V, h->ldv, hb + (m + 1), w, h->d_partial, hb + 2 * (m + 1), st);
          h->launches += 7;
          CK(cudaMemcpyAsync(hh, hb, (2 * (m + 1) + 1) * 8, cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          double hn = std::sqrt(hh[2 * (m + 1)]);
          std::vector<double> col(j + 2);
          for (int i = 0; i <= j; ++i) col[i] = hh[i] + hh[m + 1 + i];
          col[j + 1] = hn;
          for (int i = 0; i < j; ++i) {
            double t = cs[i] * col[i] + sn[i] * col[i + 1];
            col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
            col[i] = t;
          }
          double den = std::hypot(col[j], col[j + 1]);
          cs[j] = col[j] / den;
          sn[j] = col[j + 1] / den;
          col[j] = den;
          col[j + 1] = 0.0;
          g[j + 1] = -sn[j] * g[j];
          g[j] = cs[j] * g[j];
          for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = col[i];
          total++;
          k = j + 1;
          double est = std::fabs(g[j + 1]) / bnorm;
          if (!std::isfinite(est)) throw HError{HPLMM_ERR_NONFINITE, "non-finite GMRES residual"};
          if (hist && hl < hist_cap) hist[hl] = est;
          hl++;
          if (hn == 0.0 || est < tol || total >= maxit) break;
          // v_{j+1} = w / hn
          launch_scale(n, w, hb + 2 * (m + 1), 1, w, st);
          h->launches++;
        }
        // y = H^-1 g ; x += M^-1 (V y)
        std::vector<double> y(k);
        for (int i = k - 1; i >= 0; --i) {
          double s = g[i];
          for (int l = i + 1; l < k; ++l) s -= H[(size_t)i * m + l] * y[l];
          y[i] = s / H[(size_t)i * m + i];
        }
        CK(cudaMemcpyAsync(hb, y.data(), k * 8, cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(h->d_in, 0, (size_t)n * 8, st));
        launch_combine_basis(n, k, V, h->ldv, hb, h->d_in, st);
        op_minv(h, h->d_in, h->d_u);
        launch_axpy(n, 1.0, h->d_u, dx, st);
        op_spmv(h, dx, dB, h->d_r1);  // r = b - A x
        launch_norm2(n, h->d_r1, h->d_partial, hb + 2 * (m + 1), st);
        h->launches += 4;
        CK(cudaMemcpyAsync(&beta2, hb + 2 * (m + 1), 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        relres = std::sqrt(beta2) / bnorm;
        if (!std::isfinite(relres)) throw HError{HPLMM_ERR_NONFINITE, "non-finite true residual"};
        if (relres < tol) { conv = true; break; }
        if (total >= maxit) break;
      }
      if (!conv) status = HPLMM_NOT_CONVERGED;
    }
    from_device(h, x, dx, n);
    CK(cudaGetLastError());
    h->rep.t_solve_s = tt.stop();
    CK(cudaStreamSynchronize(st));
    h->flush_profile();
    h->rep.iterations = total;
    h->rep.converged = conv ? 1 : 0;
    h->rep.hist_len = std::min(hl, hist_cap);
    h->rep.final_true_relres = relres;
    h->rep.kernel_launches = h->launches;
    if (report) *report = h->rep;
    return status;
  } catch (const HError& e) {
    return fail(e);
  }
}

hplmm_status hplmm_solve_many(hplmm_handle* h, int32_t nrhs, const double* B, double tol,
                              double* X, hplmm_report* reports, void* stream) {
  if (!h || !B || !X || nrhs < 0) { g_last_error = "null argument"; return HPLMM_ERR_ARG; }
  const int64_t n = 3 * (int64_t)h->hs.n_nodes;
  hplmm_status worst = HPLMM_OK;
  if (nrhs > 1 && h->setup_done && multi_eligible(h)) {
    try {
      if (!(tol > 0)) throw HError{HPLMM_ERR_ARG, "tol must be > 0"};
      require_device(h);
      h->st = (cudaStream_t)stream;
      const int m = h->hs.opt.restart;
      if (h->Vcap < m + 1) {
        h->ldv = ((int64_t)n + 31) / 32 * 32;
        h->d_V = h->dalloc<double>((size_t)(m + 1) * h->ldv);
        h->d_partial = h->dalloc<double>((size_t)krylov_partial_doubles(n));
        CK(cudaMemsetAsync(h->d_partial, 0, (size_t)krylov_partial_doubles(n) * 8, h->st));
        h->d_hbuf = h->dalloc<double>(2 * (m + 1) + 8);
        h->Vcap = m + 1;
      }
      multi_alloc(h);
      const int blk = h->hs.opt.rhs_block == 0 ? kMaxBlock : std::min(kMaxBlock, (int)h->hs.opt.rhs_block);
      const bool bdev = is_device_ptr(B), xdev = is_device_ptr(X);
      for (int c0 = 0; c0 < nrhs; c0 += blk) {
        const int nc = std::min(blk, nrhs - c0);
        Timer tt(h->st);
        h->launches = 0;
        for (int c = 0; c < nc; ++c)
          CK(cudaMemcpyAsync(h->mr.B + c * h->ldv, B + (c0 + c) * n, n * 8,
                             bdev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->st));
        std::vector<hplmm_report> reps(nc);
        solve_block(h, nc, tol, reps.data());
        for (int c = 0; c < nc; ++c)
          CK(cudaMemcpyAsync(X + (c0 + c) * n, h->mr.X + c * h->ldv, n * 8,
                             xdev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->st));
        const double ts = tt.stop();
        CK(cudaStreamSynchronize(h->st));
        for (int c = 0; c < nc; ++c) {
          reps[c].t_solve_s = ts;
          reps[c].kernel_launches = h->launches;
          if (reports) reports[c0 + c] = reps[c];
          const hplmm_status s = reps[c].converged ? HPLMM_OK : HPLMM_NOT_CONVERGED;
          if (s > worst) worst = s;
        }
        h->rep = reps[nc - 1];
      }
      return worst;
    } catch (const HError& e) {
      return fail(e);
    }
  }
  for (int32_t i = 0; i < nrhs; ++i) {
    hplmm_report rep{};
    const hplmm_status st = hplmm_solve(h, B + i * n, tol, X + i * n, &rep, nullptr, 0, stream);
    if (reports) reports[i] = rep;
    if (st < 0) return st;
    if (st > worst) worst = st;
  }
  return worst;
}

hplmm_status hplmm_export(hplmm_handle* h, int32_t art, void* buf, int64_t cap, int64_t* len) {
  if (!h || !len) { g_last_error = "null argument"; return HPLMM_ERR_ARG; }
  try {
    HostSetup& hs = h->hs;
    const void* src = nullptr;
    int64_t n = 0, esz = 4;
    bool dev = false;
    std::vector<int32_t> tmp;
    switch (art) {
      case HPLMM_ART_NODE_KEY: src = hs.node_key.data(); n = hs.node_key.size(); esz = 8; break;
      case HPLMM_ART_ROW_PTR: src = hs.row_ptr.data(); n = hs.row_ptr.size(); break;
      case HPLMM_ART_COL_IDX: src = hs.col_idx.data(); n = hs.col_idx.size(); break;
      case HPLMM_ART_NODE_CLASS: src = hs.node_class.data(); n = hs.node_class.size(); break;
      case HPLMM_ART_NODE_IFACE: src = hs.node_iface.data(); n = hs.node_iface.size(); break;
      case HPLMM_ART_NODE_OWNER: src = hs.node_owner.data(); n = hs.node_owner.size(); break;
      case HPLMM_ART_IFACE_PTR: src = hs.iface_ptr.data(); n = hs.iface_ptr.size(); break;
      case HPLMM_ART_IFACE_NODES: src = hs.iface_nodes.data(); n = hs.iface_nodes.size(); break;
      case HPLMM_ART_CONTACT_PTR: src = hs.contact_ptr.data(); n = hs.contact_ptr.size(); break;
      case HPLMM_ART_CONTACT_NODES: src = hs.contact_nodes.data(); n = hs.contact_nodes.size(); break;
      case HPLMM_ART_MORTAR_PTR: src = hs.mortar_ptr.data(); n = hs.mortar_ptr.size(); break;
      case HPLMM_ART_MORTAR_NODES: src = hs.mortar_nodes.data(); n = hs.mortar_nodes.size(); break;
      case HPLMM_ART_GRAIN_COLS_PTR: src = hs.gcols_ptr.data(); n = hs.gcols_ptr.size(); break;
      case HPLMM_ART_GRAIN_COLS: src = hs.gcols.data(); n = hs.gcols.size(); break;
      case HPLMM_ART_VAL:
        if (!h->assembled) throw HError{HPLMM_ERR_STATE, "VAL before assemble"};
        src = h->d_val; n = h->nnzb * 9; esz = 8; dev = true; break;
      case HPLMM_ART_RHS:
        if (!h->assembled) throw HError{HPLMM_ERR_STATE, "RHS before assemble"};
        src = h->d_b; n = h->n_dof; esz = 8; dev = true; break;
      case HPLMM_ART_S: {
        if (!h->setup_done || !h->d_Sdense) throw HError{HPLMM_ERR_STATE, "S not available"};
        int Nm = h->co.Nm;
        n = (int64_t)Nm * Nm;
        *len = n;
        if (!buf) return HPLMM_OK;
        if (cap < n * 8) throw HError{HPLMM_ERR_ARG, "buffer too small"};
        require_device(h);
        CK(cudaMemcpy2D(buf, Nm * 8, h->d_Sdense, h->lds * 8, Nm * 8, Nm, cudaMemcpyDeviceToHost));
        return HPLMM_OK;
      }
      case HPLMM_ART_MORTAR_W: {
        if (!h->setup_done) throw HError{HPLMM_ERR_STATE, "weights before setup"};
        int64_t wo = 0;
        for (int c = 0; c < hs.n_ifaces(); ++c)
          wo += (int64_t)9 * (hs.iface_ptr[c + 1] - hs.iface_ptr[c]) *
                (hs.mortar_ptr[c + 1] - hs.mortar_ptr[c]);
        src = h->co.W; n = wo; esz = 8; dev = true; break;
      }
      case HPLMM_ART_ILU:
        if (!h->setup_done || !h->ilu.val) throw HError{HPLMM_ERR_STATE, "ILU factor not built"};
        src = h->ilu.val; n = h->nnzb * 9; esz = 8; dev = true; break;
      default: throw HError{HPLMM_ERR_ARG, "unknown artifact"};
    }
    *len = n;
    if (!buf) return HPLMM_OK;
    if (cap < n * esz) throw HError{HPLMM_ERR_ARG, "buffer too small"};
    if (dev) {
      require_device(h);
      CK(cudaMemcpy(buf, src, n * esz, cudaMemcpyDeviceToHost));
    } else if (n) {
      std::memcpy(buf, src, n * esz);
    }
    return HPLMM_OK;
  } catch (const HError& e) {
    return fail(e);
  }
}

hplmm_status hplmm_get_report(hplmm_handle* h, hplmm_report* r) {
  if (!h || !r) { g_last_error = "null argument"; return HPLMM_ERR_ARG; }
  *r = h->rep;
  return HPLMM_OK;
}

// Profiling of the dominant kernel (packed SYMV tiles): CUDA events around
// each launch on the launch stream; stats accumulate until reset.
hplmm_status hplmm_profile(hplmm_handle* h, int32_t enable, int32_t reset) {
  if (!h) { g_last_error = "null handle"; return HPLMM_ERR_ARG; }
  h->profile = enable != 0;
  if (reset)
    for (int k = 0; k < KC_N; ++k) { h->kc_ms[k] = 0; h->kc_launches[k] = 0; }
  return HPLMM_OK;
}

// kernel: 0 grain SYMV tiles, 1 contact SYMV tiles, 2 coarse SYMV tiles.
// bytes = packed-tile bytes streamed per launch (32 KiB per tile).
hplmm_status hplmm_kernel_stats(hplmm_handle* h, int32_t kernel, double* total_ms,
                                int64_t* launches, int64_t* tile_bytes) {
  if (!h || kernel < 0 || kernel >= KC_N) { g_last_error = "bad argument"; return HPLMM_ERR_ARG; }
  if (total_ms) *total_ms = h->kc_ms[kernel];
  if (launches) *launches = h->kc_launches[kernel];
  if (kernel == KC_EBE) {   // y = A^ x form: x, y, node coords + flag, lattice map, moduli
    const HostSetup& hs = h->hs;
    if (tile_bytes)
      *tile_bytes = 16 * (int64_t)h->n_dof + 13 * (int64_t)h->n_nodes +
                    4 * (int64_t)(hs.nx + 1) * (hs.ny + 1) * (hs.nz + 1) +
                    8 * (int64_t)hs.nx * hs.ny * hs.nz;
    return HPLMM_OK;
  }
  if (kernel == KC_BSR) {   // y = A^ x form: 72 B values + 4 B column per block, row_ptr, x, y
    if (tile_bytes) *tile_bytes = 76 * h->nnzb + 4 * (int64_t)h->n_nodes + 16 * (int64_t)h->n_dof;
    return HPLMM_OK;
  }
  if (kernel == KC_ILU) {   // every stored block once per apply (L in fwd, U + D in bwd)
    if (tile_bytes) *tile_bytes = h->ilu.val ? h->nnzb * 72 : 0;
    return HPLMM_OK;
  }
  if (kernel >= KC_SN_GRAIN) {
    if (tile_bytes) *tile_bytes = kernel == KC_SN_GRAIN ? h->sg.solve_bytes : h->sc.solve_bytes;
    return HPLMM_OK;
  }
  DevBatch* b = kernel == 0 ? &h->gb : (kernel == 1 ? &h->cb : &h->sb);
  if (tile_bytes) *tile_bytes = b->ntiles * (int64_t)TILE * 8;
  return HPLMM_OK;
}

void hplmm_destroy(hplmm_handle* h) { delete h; }

}  // extern "C"
