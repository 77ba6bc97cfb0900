// Device-resident GMRES(m) cycle control (reading R22): the Givens
// update, residual estimate, stop test, back substitution and restart test of
// hplmm_solve run on the GPU, so that a whole solve -- every Arnoldi step and
// every restart cycle -- is ONE CUDA-graph launch with two nested WHILE
// conditional nodes (api.cu: build_solve_graph) and one host synchronisation
// at the end.  The arithmetic mirrors the host loop of api.cu operation by
// operation (same formulas, same order), so both paths compute the same
// iterates up to the rounding of hypot.
//
// The small dense state (H, g, Givens cosines/sines, y: <= 513 x 512 doubles)
// is touched by a single thread: O(j) work per step, latency not bandwidth.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace hplmm {

__global__ void k_gmres_cycle_init(GmresDev d, cudaGraphConditionalHandle inner) {
  GmresScalars* s = d.s;
  const double beta = sqrt(*d.beta2);
  for (int i = 0; i <= s->m; ++i) d.g[i] = 0.0;
  d.g[0] = beta;
  s->j = 0;
  s->k = 0;
  s->stop_inner = 0;
  s->cycles += 1;
  cudaGraphSetConditional(inner, 1u);
}

// y = x / sqrt(*s2) for the cycle's first basis vector, twice (V[0] and vj)
__global__ void k_scale_first(int64_t n, const double* __restrict__ x, const double* __restrict__ s2,
                              double* __restrict__ y0, double* __restrict__ y1) {
  const double f = 1.0 / sqrt(s2[0]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i] * f;
    y0[i] = v;
    y1[i] = v;
  }
}

void launch_gmres_cycle_init(const GmresDev& d, unsigned long long inner, int64_t n, const double* r,
                             double* V, double* vj, cudaStream_t st) {
  k_gmres_cycle_init<<<1, 1, 0, st>>>(d, (cudaGraphConditionalHandle)inner);
  k_scale_first<<<krylov_blocks(n), 256, 0, st>>>(n, r, d.beta2, V, vj);
}

// one thread: the host loop's Givens step (api.cu) on the device
__global__ void k_gmres_givens(GmresDev d, cudaGraphConditionalHandle inner) {
  GmresScalars* s = d.s;
  const int m = s->m, j = s->j;
  const double* hb = d.hb;
  const double hn = sqrt(hb[2 * (m + 1)]);
  double* H = d.H;
  // column j of H in place: CGS2 coefficients h1 + h2, then the previous rotations
  for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = hb[i] + hb[m + 1 + i];
  double below = hn;   // entry j+1 of the column (never stored: rotated to 0)
  for (int i = 0; i < j; ++i) {
    const double a = H[(size_t)i * m + j], b = H[(size_t)(i + 1) * m + j];
    H[(size_t)i * m + j] = d.cs[i] * a + d.sn[i] * b;
    H[(size_t)(i + 1) * m + j] = -d.sn[i] * a + d.cs[i] * b;
  }
  const double cj = H[(size_t)j * m + j];
  const double den = hypot(cj, below);
  d.cs[j] = cj / den;
  d.sn[j] = below / den;
  H[(size_t)j * m + j] = den;
  d.g[j + 1] = -d.sn[j] * d.g[j];
  d.g[j] = d.cs[j] * d.g[j];
  const double est = fabs(d.g[j + 1]) / s->bnorm;
  const int total = s->total + 1;
  s->total = total;
  s->k = j + 1;
  s->j = j + 1;
  int stop = 0;
  if (!isfinite(est)) {
    s->nonfinite = 1;
    s->done = 1;
    stop = 1;
  } else {
    if (total - 1 < s->maxit) d.hist[total - 1] = est;
    stop = (hn == 0.0 || est < s->tol || total >= s->maxit || j + 1 >= m) ? 1 : 0;
  }
  s->stop_inner = stop;
  cudaGraphSetConditional(inner, stop ? 0u : 1u);
}

// V[j+1] = w / ||w||, vj = V[j+1] (skipped when the step loop stops); the
// same scale factor as the host loop's k_scale (1 / sqrt(||w||^2))
__global__ void k_scale_next(int64_t n, const GmresScalars* __restrict__ s,
                             const double* __restrict__ w2, const double* __restrict__ w,
                             double* __restrict__ V, int64_t ldv, double* __restrict__ vj) {
  if (s->stop_inner) return;
  const double f = 1.0 / sqrt(w2[0]);
  double* v = V + (int64_t)s->j * ldv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double t = w[i] * f;
    v[i] = t;
    vj[i] = t;
  }
}

void launch_gmres_step_end(const GmresDev& d, unsigned long long inner, int64_t n, const double* w,
                           double* V, int64_t ldv, double* vj, cudaStream_t st) {
  k_gmres_givens<<<1, 1, 0, st>>>(d, (cudaGraphConditionalHandle)inner);
  k_scale_next<<<krylov_blocks(n), 256, 0, st>>>(n, d.s, d.beta2, w, V, ldv, vj);
}

// y = H(0:k, 0:k)^-1 g(0:k) by back substitution (the host loop's order)
__global__ void k_gmres_backsolve(GmresDev d) {
  const GmresScalars* s = d.s;
  const int m = s->m, k = s->k;
  for (int i = k - 1; i >= 0; --i) {
    double t = d.g[i];
    for (int l = i + 1; l < k; ++l) t -= d.H[(size_t)i * m + l] * d.y[l];
    d.y[i] = t / d.H[(size_t)i * m + i];
  }
}

// out = sum_{j<k} V[j] y[j] (j ascending, fma chain from 0: bitwise the host
// loop's memset + k_combine_basis)
__global__ void k_gmres_combine(int64_t n, const GmresScalars* __restrict__ s,
                                const double* __restrict__ V, int64_t ldv,
                                const double* __restrict__ y, double* __restrict__ out) {
  __shared__ double ys[513];
  const int k = s->k;
  for (int j = threadIdx.x; j < k; j += blockDim.x) ys[j] = y[j];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < k; ++j) acc = fma(V[j * ldv + i], ys[j], acc);
    out[i] = acc;
  }
}

void launch_gmres_combine(const GmresDev& d, int64_t n, const double* V, int64_t ldv, double* out,
                          cudaStream_t st) {
  k_gmres_backsolve<<<1, 1, 0, st>>>(d);
  k_gmres_combine<<<krylov_blocks(n), 256, 0, st>>>(n, d.s, V, ldv, d.y, out);
}

// after x += M^-1 (V y) and r = b - A^ x, ||r||^2 in *beta2: the restart test
__global__ void k_gmres_cycle_end(GmresDev d, cudaGraphConditionalHandle outer) {
  GmresScalars* s = d.s;
  const double relres = sqrt(*d.beta2) / s->bnorm;
  s->relres = relres;
  if (s->done) {                        // non-finite estimate inside the cycle
  } else if (!isfinite(relres)) {
    s->nonfinite = 1;
    s->done = 1;
  } else if (relres < s->tol) {
    s->converged = 1;
    s->done = 1;
  } else if (s->total >= s->maxit) {
    s->done = 1;
  }
  cudaGraphSetConditional(outer, s->done ? 0u : 1u);
}

void launch_gmres_cycle_end(const GmresDev& d, unsigned long long outer, cudaStream_t st) {
  k_gmres_cycle_end<<<1, 1, 0, st>>>(d, (cudaGraphConditionalHandle)outer);
}

}  // namespace hplmm
