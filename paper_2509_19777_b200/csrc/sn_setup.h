// Host-side management of a batch of supernodal local factors (internal).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "supernodal.h"
#include "supernodal_dev.cuh"

namespace hplmm {

struct SnError {
  int status;          // hplmm_status value
  std::string msg;
  int sub = -1;        // failing subdomain (singular local factor)
};

// device allocator of the owning handle (setup_only buffers are freed at the
// end of hplmm_setup)
struct DevAlloc {
  virtual void* alloc(size_t bytes, bool setup_only) = 0;
  virtual ~DevAlloc() = default;
};

struct SnBatch {
  SnSymbolic sym;
  SnDev dev;
  SnWork work;                 // one CTA per SM, LPT over subdomains (apply)
  double* factor = nullptr;
  double* yloc = nullptr;      // solution in local (elimination) order, [n_loc]
  int64_t n_loc = 0;
  int64_t solve_bytes = 0;     // factor bytes streamed by one batch solve
  SnWork mwork[3];             // multi-RHS solves: work lists for NRHS = 1, 2, 4 (built lazily)
  int mstate[3] = {0, 0, 0};   // 0 not built, 1 ready, -1 does not fit shared memory
  int32_t *d_sub_n = nullptr, *d_gmap = nullptr, *d_lidx = nullptr, *d_sn_w = nullptr,
          *d_sn_r = nullptr, *d_sn_p0 = nullptr, *d_sn_ldw = nullptr, *d_sn_ldf = nullptr,
          *d_rows = nullptr;
  int64_t *d_sub_base = nullptr, *d_sub_fc0 = nullptr, *d_sub_fc1 = nullptr,
          *d_sub_bc0 = nullptr, *d_sub_bc1 = nullptr, *d_sn_rows_off = nullptr;
};

void sn_upload(SnBatch& B, DevAlloc& A, cudaStream_t st, int nsm);
void sn_build_work(SnBatch& B, DevAlloc& A, cudaStream_t st, int nblocks, int nrhs,
                   const std::vector<int32_t>* ncols, SnWork& wk, int force_cons = 0,
                   bool allow_split = false);
// numeric factorisation; throws SnError (status -4 + subdomain) on a
// non-positive pivot.  pool_budget: bytes of frontal matrices per wave.
void sn_factor(SnBatch& B, const double* d_val, DevAlloc& A, cudaStream_t st,
               int64_t pool_budget);
// yloc = A_s^-1 in[gmap] for every subdomain of the batch
void sn_apply(const SnBatch& B, const double* in, cudaStream_t st);
// Several right-hand sides at once (the factor streams once per launch):
// largest P in {4, 2, 1}, P <= k, whose solve fits shared memory for this batch
int sn_multi_width(SnBatch& B, DevAlloc& A, cudaStream_t st, int nsm, int k);
// out[(base + p) P + c] = (A_s^-1 in_c[gmap])_p for c < ncols <= P; in_c = in + c ldin
void sn_apply_multi(const SnBatch& B, int P, const double* in, int64_t ldin, int ncols, double* out,
                    cudaStream_t st);
// B_g[:, 0:k_g] = -A_g^-1 R_g[:, 0:k_g] (grain batch, gb row layout)
// (R is overwritten: it serves as the workspace; rb_doubles = size of R and B)
void sn_shape_vectors(SnBatch& B, DevAlloc& A, cudaStream_t st, int nsm,
                      const std::vector<int32_t>& kcols, const int64_t* d_b_off,
                      const int32_t* d_ld, double* R, double* Bout, int64_t rb_doubles);

}  // namespace hplmm
