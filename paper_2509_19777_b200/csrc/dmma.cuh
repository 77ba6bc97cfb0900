// FP64 tensor-core (DMMA) tile products for the setup phase (sm_100a:
// mma.sync.aligned.m8n8k4 .f64, SASS DMMA.8x8x4).  256-thread CTAs.
#pragma once

namespace hplmm {

// ---------------------------------------------------------------------------
// 64x64 tile product on the FP64 tensor cores: mma.sync m8n8k4 .f64 (SASS DMMA.8x8x4).
// Warp w owns rows (w>>1)*16 .. +16 and columns (w&1)*32 .. +32 of the 64x64
// result: 2 x 4 fragments of 8x8, two accumulators each per thread.
// Accumulator t = (mi*4 + ni)*2 + i holds element
//   (r, c) = ((w>>1)*16 + mi*8 + lane/4,  (w&1)*32 + ni*8 + (lane%4)*2 + i).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// acc += A B over K = kdim (multiple of 4) with A(r,k) = As[k*lda + r], B(k,c) = Bs[k*ldb + c]
__device__ __forceinline__ void tile_dmma(const double* __restrict__ As, int lda,
                                          const double* __restrict__ Bs, int ldb, int kdim,
                                          double (&acc)[16]) {
  const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 7;
  const int g = lane >> 2, q = lane & 3;
  const int mb = (w >> 1) * 16, nb = (w & 1) * 32;
#pragma unroll 4
  for (int k0 = 0; k0 < kdim; k0 += 4) {
    const double* Ak = As + (k0 + q) * lda + mb + g;
    const double* Bk = Bs + (k0 + q) * ldb + nb + g;
    const double a0 = Ak[0], a1 = Ak[8];
    double b[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bk[ni * 8];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      dmma_884(acc[ni * 2], acc[ni * 2 + 1], a0, b[ni]);
      dmma_884(acc[8 + ni * 2], acc[8 + ni * 2 + 1], a1, b[ni]);
    }
  }
}
__device__ __forceinline__ void dmma_rc(int t, int& r, int& c) {
  const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 7;
  const int mi = t >> 3, ni = (t >> 1) & 3, i = t & 1;
  r = (w >> 1) * 16 + mi * 8 + (lane >> 2);
  c = (w & 1) * 32 + ni * 8 + (lane & 3) * 2 + i;
}


bool use_dmma();   // HPLMM_DMMA=0 selects the FP64 FMA kernels (comparison)

}  // namespace hplmm
