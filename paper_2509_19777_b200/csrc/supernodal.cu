// Batched supernodal block-LDL^T local factors (sm_100a, fp64): numeric
// multifrontal factorisation (setup, T_ML) and the TMA-streamed solve that
// applies every grain / contact-grid inverse in the hot path (eq:Mg_Mz).
// See supernodal.h for the algebra and the layout.
#include <algorithm>
#include <vector>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "dmma.cuh"
#include "kernels.cuh"
#include "supernodal.h"
#include "supernodal_dev.cuh"
#include "tma.cuh"

namespace hplmm {

// ===========================================================================
// Solve: one persistent CTA per SM walks its list of (subdomain, RHS column
// chunk) items.  The subdomain's right-hand side lives in shared memory
// (x[p*NRHS + c], p = elimination position); the factor streams through a
// ring of 32-KiB stages filled by 1-D TMA bulk copies issued by one producer
// lane, following the static chunk schedule (forward then backward chunks of
// each item).  All SN_CONS consumer warps take part in every chunk:
//   W fwd  : acc_i += W[i,j] x_S[j]  (thread per row i; col-major => conflict
//            free), at the end of the part x_R[i] -= acc_i
//   F fwd  : acc_i += Finv[i,j] x_S[j], at the end x_S = acc (two barriers)
//   W bwd  : warp per column j: x_S[j] -= sum_i W[i,j] x_R[i]
// A stage is released (empty mbarrier, count SN_CONS) as soon as every warp
// has read it; the producer runs ahead across supernode and item boundaries.
// ===========================================================================
constexpr int SN_MAXST = 16;
// per-CTA start / end %globaltimer of the last launch (flags & 16; experiments)
__device__ unsigned long long g_sn_cta_t[2 * 4096];
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// per-warp phase timing of k_sn_solve (printf for a few CTAs when flags & 2);
// compiled out unless built with -DHPLMM_SN_PROF=1
#ifndef HPLMM_SN_PROF
#define HPLMM_SN_PROF 0
#endif

// one-shot flags of the subtree-parallel exchange steps
__device__ __forceinline__ void flag_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int flag_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int CONS>
struct SnT {
  static constexpr int NT = 32 * CONS;                  // consumer threads
  static constexpr int LGNT = CONS == 16 ? 9 : (CONS == 8 ? 8 : (CONS == 4 ? 7 : 5));
  static_assert((1 << LGNT) == NT, "power-of-two consumer threads");
  static constexpr int MAXQ = 4;                        // double2 row pairs per thread
  static_assert(MAXQ * 2 * 256 >= SN_MAX_WR, "row coverage at TG = 256");
};

template <int NT>
__device__ __forceinline__ void cons_sync() {
  asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
}

// Row-parallel layout of a part with h rows: row pairs are spread over TG
// threads (a power of two >= 32), the SN_NT consumer threads form G = SN_NT/TG
// groups and group g takes the chunk columns jj == g (mod G), so every chunk
// keeps all consumer warps busy whatever the aspect ratio of the panel.
struct RowLayout {
  int TG, G, g, t, lg;
  // lgc = log2(TG) - 5, precomputed on the host per part (chunk descriptor,
  // TG <= 512), capped at the CTA's consumer thread count NT = 2^lgnt
  __device__ __forceinline__ RowLayout(int lgc, int tid, int lgnt) {
    lg = min(lgc + 5, lgnt);
    TG = 1 << lg;
    G = 1 << (lgnt - lg);
    g = tid >> lg;
    t = tid & (TG - 1);
  }
  // row-pair slots per thread for h rows
  __device__ __forceinline__ int nq(int h) const { return (h + 2 * TG - 1) >> (lg + 1); }
};

// effective row-group code of a part with h rows: the host's (TG >= h/8), or
// for NRHS > 1 the smallest TG >= the host's whose row pairs fit MAXQ per
// thread and whose group-reduction scratch (G - 1) h NRHS fits one stage
template <int NRHS, int MAXQ>
__device__ __forceinline__ int sn_lg(int lgc, int h, int lgnt, int stage_doubles) {
  if (NRHS == 1) return lgc;
  int lg = min(lgc + 5, lgnt);
  while (lg < lgnt && ((h + (2 << lg) - 1) >> (lg + 1) > MAXQ ||
                       (int64_t)((1 << (lgnt - lg)) - 1) * h * NRHS > stage_doubles))
    ++lg;
  return lg - 5;
}

// acc[q][e][c] += sum over this group's chunk columns of col[2(t + q TG) + e] * x_S
// Columns are taken four at a time (all loads issued before the FMAs, two
// accumulator sets) so that a warp keeps several shared-memory loads in flight.
template <int NQ, int NRHS, int MAXQ>
__device__ __forceinline__ void sn_rows(const double* __restrict__ st, int ld, int nc, int h,
                                        const double* __restrict__ xcol, const RowLayout& L,
                                        double (&acc)[MAXQ][2][NRHS]) {
  // columns per step (register budget: NQ row pairs x NRHS accumulators)
  constexpr int U0 = NQ == 1 ? 4 : (NQ == 2 ? 2 : 1);
  constexpr int U = NRHS == 1 ? U0 : (NQ == 1 ? 2 : 1);
  double acc2[NQ][2][NRHS];
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int c = 0; c < NRHS; ++c) acc2[q][e][c] = 0.0;
  int jj = L.g;
  const int G = L.G;
  for (; jj + (U - 1) * G < nc; jj += U * G) {
    double xv[U][NRHS];
    double2 a[U][NQ];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (NRHS % 2 == 0) {   // x rows are 16-byte aligned: paired loads
#pragma unroll
        for (int c = 0; c < NRHS; c += 2) {
          const double2 t = *reinterpret_cast<const double2*>(xcol + (jj + u * G) * NRHS + c);
          xv[u][c] = t.x;
          xv[u][c + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int c = 0; c < NRHS; ++c) xv[u][c] = xcol[(jj + u * G) * NRHS + c];
      }
      const double* cu = st + (size_t)(jj + u * G) * ld;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int i = 2 * (L.t + q * L.TG);
        // NRHS == 1: rows >= h are read unconditionally (whatever follows in
        // shared memory; sn_tail_doubles keeps a guard after the ring) into
        // accumulator rows that are never used -- no predicate, no zeroing
        if (NRHS == 1) a[u][q] = *reinterpret_cast<const double2*>(cu + i);
        else a[u][q] = i < h ? *reinterpret_cast<const double2*>(cu + i) : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int c = 0; c < NRHS; ++c) {
          if (u & 1) {
            acc2[q][0][c] = fma(a[u][q].x, xv[u][c], acc2[q][0][c]);
            acc2[q][1][c] = fma(a[u][q].y, xv[u][c], acc2[q][1][c]);
          } else {
            acc[q][0][c] = fma(a[u][q].x, xv[u][c], acc[q][0][c]);
            acc[q][1][c] = fma(a[u][q].y, xv[u][c], acc[q][1][c]);
          }
        }
  }
  for (; jj < nc; jj += G) {
    double xa[NRHS];
#pragma unroll
    for (int c = 0; c < NRHS; ++c) xa[c] = xcol[jj * NRHS + c];
    const double* ca = st + (size_t)jj * ld;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = 2 * (L.t + q * L.TG);
      if (NRHS == 1 || i < h) {
        const double2 a = *reinterpret_cast<const double2*>(ca + i);
#pragma unroll
        for (int c = 0; c < NRHS; ++c) {
          acc[q][0][c] = fma(a.x, xa[c], acc[q][0][c]);
          acc[q][1][c] = fma(a.y, xa[c], acc[q][1][c]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int c = 0; c < NRHS; ++c) acc[q][e][c] += acc2[q][e][c];
}

// group partials -> group 0 (fixed order g = 0..G-1), through smem scratch
// scratch[c (G - 1) h + (g - 1) h + row]: (G - 1) h NRHS <= 8 NT (TG >= h/8; NRHS > 1:
// TG >= h/2) doubles, i.e. within one 32-KiB stage for NT <= 512
template <int NRHS, int MAXQ, int NT>
__device__ __forceinline__ void sn_group_reduce(const RowLayout& L, int h, double* scratch,
                                                double (&acc)[MAXQ][2][NRHS]) {
  // component-major (c, g - 1, row): consecutive rows of one RHS are adjacent
  // doubles, so the group's row-parallel writes and reads are bank-conflict free
  const int stride = h;
  const size_t cstride = (size_t)(L.G - 1) * h;
  if (L.g > 0) {
#pragma unroll
    for (int q = 0; q < MAXQ; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = 2 * (L.t + q * L.TG) + e;
        if (i < h)
#pragma unroll
          for (int c = 0; c < NRHS; ++c)
            scratch[(size_t)c * cstride + (size_t)(L.g - 1) * stride + i] = acc[q][e][c];
      }
  }
  cons_sync<NT>();
  if (L.g == 0) {
    for (int gg = 1; gg < L.G; ++gg)
#pragma unroll
      for (int q = 0; q < MAXQ; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 2 * (L.t + q * L.TG) + e;
          if (i < h)
#pragma unroll
            for (int c = 0; c < NRHS; ++c)
              acc[q][e][c] += scratch[(size_t)c * cstride + (size_t)(gg - 1) * stride + i];
        }
  }
}

// Backward W part chunk: x_S[j] -= W[:, j]^T x_R for the chunk's nc columns
// (column-major, ld), LPC lanes split the rows of a column; each lane group
// takes CB columns at once, so one x_R load serves CB columns, and the
// CB x NRHS sums are reduced over the group by a transposing butterfly (each
// halving step keeps half of the sums: NV - 1 + log2(LPC / NV) shuffles for
// NV = CB NRHS sums instead of NV log2(LPC)).  xo[j NRHS + c] receives the
// update of column j (0 <= j < nc) for right-hand side c; x_R is
// component-major, xr[c rpad + i] (lanes read consecutive rows: conflict-free).
template <int LPC, int NRHS, int CONS>
__device__ __forceinline__ void sn_wbwd(const double* __restrict__ st, int ld, int r, int nc,
                                        const double* __restrict__ xr, int rpad, double* xo,
                                        int warp, int lane) {
  constexpr int CB = NRHS == 1 ? 4 : (NRHS == 2 ? 4 : 2);   // NV <= 8 <= LPC
  constexpr int NV = CB * NRHS;
  static_assert(NV <= LPC, "one sum per lane after the halving steps");
  constexpr int CPW = 32 / LPC;                  // lane groups per warp
  const int sl = lane & (LPC - 1), cl = lane / LPC;
  for (int jw = warp * CPW * CB; jw < nc; jw += CONS * CPW * CB) {
    const int jb = jw + cl * CB;                 // first column of the lane group
    double sum[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) sum[v] = 0.0;
    if (jb < nc) {
      const double* col[CB];
#pragma unroll
      for (int b = 0; b < CB; ++b) col[b] = st + (size_t)min(jb + b, nc - 1) * ld;   // clamped
#pragma unroll 2
      for (int i = 2 * sl; i < r; i += 2 * LPC) {
        double2 xa[NRHS];
#pragma unroll
        for (int c = 0; c < NRHS; ++c) xa[c] = *reinterpret_cast<const double2*>(xr + c * rpad + i);
#pragma unroll
        for (int b = 0; b < CB; ++b) {
          const double2 a = *reinterpret_cast<const double2*>(col[b] + i);
#pragma unroll
          for (int c = 0; c < NRHS; ++c)
            sum[b * NRHS + c] = fma(a.x, xa[c].x, fma(a.y, xa[c].y, sum[b * NRHS + c]));
        }
      }
    }
    int idx = 0, o = LPC / 2;
#pragma unroll
    for (int h = NV / 2; h >= 1; h >>= 1, o >>= 1) {
      const bool up = sl & o;
      if (up) idx += h;
#pragma unroll
      for (int t = 0; t < h; ++t) {
        const double send = up ? sum[t] : sum[h + t];
        const double keep = up ? sum[h + t] : sum[t];
        sum[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
#pragma unroll
    for (; o > 0; o >>= 1) sum[0] += __shfl_xor_sync(0xffffffffu, sum[0], o);
    const int b = idx / NRHS, c = idx - b * NRHS;
    if ((sl & (LPC / NV - 1)) == 0 && jb + b < nc) xo[(jb + b) * NRHS + c] -= sum[0];
  }
}

template <int NRHS, int CONS, int CPS, bool XG, bool SPLIT>
__global__ void __launch_bounds__(32 * (CONS + 1), CPS)
    k_sn_solve(SnDev d, SnIO io, SnWork wk, int stages, int stage_doubles, int max_n, int max_r,
               int flags) {
  extern __shared__ __align__(128) unsigned char sn_smem[];
  __shared__ __align__(8) uint64_t full[SN_MAXST], empty[SN_MAXST];
  double* ring = reinterpret_cast<double*>(sn_smem);
  // x (elimination order, NRHS interleaved) and x_R of the current backward
  // part (16-B aligned): after the ring in shared memory, or (XG) in the
  // CTA's slice of global memory (L1/L2-resident; only the ring in smem)
  double* x = XG ? wk.xg + (size_t)blockIdx.x * wk.xg_stride : ring + (size_t)stages * stage_doubles;
  // XG: x_S of the current supernode staged in shared memory (forward: read by
  // its W and F parts; backward: updated by its W part, written back at the end)
  double* xs = ring + (size_t)stages * stage_doubles;
  double* xr = XG ? xs + (size_t)((wk.max_w + 1) & ~1) * NRHS : x + (size_t)((max_n + 1) & ~1) * NRHS;
  const int rpad = (max_r + 3) & ~1;   // x_R: NRHS component-major rows of rpad doubles
  constexpr int SN_NT = SnT<CONS>::NT, SN_CONS = CONS;
  static_assert(NRHS == 1 || XG, "several right-hand sides keep x in global memory");
  static_assert(!SPLIT || (NRHS == 1 && !XG), "subtree-parallel items: one RHS, x in shared memory");
  // row pairs per thread: up to 4 for one RHS (TG >= h/8); with several RHS
  // at most 2 (sn_lg widens TG): h <= 2048 with 16 warps, h <= 1024 with 8
  // (sn_build_work keeps taller parts off the 8-warp shape) -- a smaller
  // accumulator array keeps the multi-RHS solve free of register spills
  constexpr int SN_MAXQ = (NRHS == 1 || CONS < 8) ? SnT<CONS>::MAXQ : (CONS == 8 ? 1 : 2);
  constexpr int SN_LGNT = SnT<CONS>::LGNT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t k0 = wk.chunk_ptr[blockIdx.x], k1 = wk.chunk_ptr[blockIdx.x + 1];
  // optional per-warp phase timing (flags & 2; printed for a few CTAs)
  const bool prof = HPLMM_SN_PROF && (flags & 2) && (blockIdx.x % 37 == 0);
  long long t_wait = 0, t_sync = 0;
  long long t_kind[6] = {0, 0, 0, 0, 0, 0}, n_kind[6] = {0, 0, 0, 0, 0, 0};
  const long long t_start = prof ? clock64() : 0;
#define PSYNC()                                        \
  do {                                                 \
    const long long ts_ = prof ? clock64() : 0;        \
    cons_sync<SN_NT>();                                       \
    if (prof) t_sync += clock64() - ts_;               \
  } while (0)
  const SnChunk* __restrict__ ch = wk.chunks;
  if ((flags & 16) && threadIdx.x == 0 && blockIdx.x < 4096) g_sn_cta_t[2 * blockIdx.x] = globaltimer();
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SN_CONS);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == SN_CONS) {
    // producer warp: lanes prefetch 32 chunk descriptors, lane 0 issues the
    // ring loads; the chunk PD ahead of the one being loaded is prefetched
    // into L2 by its own lane (a bulk L2 prefetch), so that a ring slot, once
    // released, refills from L2 instead of waiting a DRAM latency.  PD = 2
    // (flags bit 12 set: PD = (flags >> 8) & 15, 0 = off).  Measured at cfg3
    // (contact / grain solve): no prefetch 1.94 / 1.32 ms, PD = 1 1.81 / 1.24,
    // PD = 2 1.82 / 1.24, 4 1.82 / 1.25, 6 1.84 / 1.26
    const int pd = (flags & 0x1000) ? ((flags >> 8) & 15) : 1;
    const uint64_t pol = policy_evict_first();
    int s = 0;
    uint32_t ph = 0;
    int64_t k = 0;
    for (int64_t kb = k0; kb < k1; kb += 32) {
      int64_t off = 0;
      int bytes = 0;
      if (kb + lane < k1) {
        off = ch[kb + lane].off;
        bytes = ch[kb + lane].bytes & 0xffffff;
      }
      const int cnt = (int)min((int64_t)32, k1 - kb);
      if (kb > k0 && lane < pd && lane < cnt && (!SPLIT || bytes > 0))
        bulk_prefetch_l2(d.factor + off, (uint32_t)bytes);
      for (int j = 0; j < cnt; ++j) {
        const int64_t o = __shfl_sync(0xffffffffu, off, j);
        const int b = __shfl_sync(0xffffffffu, bytes, j);
        if (pd > 0 && lane == j + pd && lane < cnt && (!SPLIT || bytes > 0))
          bulk_prefetch_l2(d.factor + off, (uint32_t)bytes);
        if (SPLIT && b == 0) continue;   // exchange step: no factor data, no ring slot
        if (lane == 0) {
          if (k >= stages) {
            const long long tw = prof ? clock64() : 0;
            if (flags & 8) mbar_wait_sleep(&empty[s], ph ^ 1);
            else mbar_wait(&empty[s], ph ^ 1);
            if (prof) t_wait += clock64() - tw;
          }
          mbar_expect_tx(&full[s], (uint32_t)b);
          bulk_g2s_hint(ring + (size_t)s * stage_doubles, d.factor + o, (uint32_t)b, &full[s],
                        pol);
        }
        if (++s == stages) { s = 0; ph ^= 1; }
        ++k;
      }
    }
    if (prof && lane == 0)
      printf("sn_prof cta %d producer: total %lld empty-wait %lld chunks %lld\n", blockIdx.x,
             clock64() - t_start, t_wait, (long long)(k1 - k0));
    return;
  }
  const int tid = threadIdx.x;
  double acc[SN_MAXQ][2][NRHS];
  // row positions of a W part whose row list came in its first chunk (group-0
  // threads keep the rows they scatter to at the part's end)
  int prow[SN_MAXQ][2];
  bool rows_held = false;
  int item = wk.item_ptr[blockIdx.x] - 1;
  int n = 0, rc0 = 0, sub = 0;
  int64_t base = 0;
  int s = 0;
  uint32_t ph = 0;
  // descriptor of the next chunk is loaded one chunk ahead
  int4 dn0 = make_int4(0, 0, 0, 0), dn1 = make_int4(0, 0, 0, 0);
  if (k0 < k1) {
    dn0 = __ldg(reinterpret_cast<const int4*>(ch + k0));
    dn1 = __ldg(reinterpret_cast<const int4*>(ch + k0) + 1);
  }
  for (int64_t kk = k0; kk < k1; ++kk) {
    // SnChunk = {off (2 ints), bytes, info | p0, w, r, sub}
    const int info = dn0.w, p0 = dn1.x, w = dn1.y, r = dn1.z, csub = dn1.w;
    const int lgc = (dn0.z >> 24) & 15;
    if (kk + 1 < k1) {
      dn0 = __ldg(reinterpret_cast<const int4*>(ch + kk + 1));
      dn1 = __ldg(reinterpret_cast<const int4*>(ch + kk + 1) + 1);
    }
    const int cc0 = info & 0xfff, nc = ((info >> 12) & 0xfff) + 1, kind = (info >> 24) & 7;
    const bool last = info & SN_INFO_LAST;
    if (info & SN_INFO_FIRST_ITEM) {
      // ---- gather the right-hand side (4 independent loads per thread in flight)
      ++item;
      sub = csub;
      n = d.sub_n[sub];
      base = d.sub_base[sub];
      rc0 = wk.item_c0[item];
      if (io.mode == 2) {
        for (int p = tid; p < n; p += SN_NT) {
          const int64_t gd = __ldg(d.gmap + base + p);
#pragma unroll
          for (int c = 0; c < NRHS; ++c) x[p * NRHS + c] = c < io.ncols ? io.in[c * io.ldin + gd] : 0.0;
        }
      } else if (io.mode == 0) {
        for (int q0 = tid; q0 < n; q0 += 4 * SN_NT) {
          double v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int p = q0 + u * SN_NT;
            v[u] = p < n ? io.in[__ldg(d.gmap + base + p)] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (q0 + u * SN_NT < n) x[q0 + u * SN_NT] = v[u];
        }
      } else {
        const int L = io.ld[sub];
        const int ncr = min(NRHS, L - 1 - rc0);
        const double* R = io.in + io.b_off[sub];
        for (int p = tid; p < n; p += SN_NT) {
          const int64_t row = (int64_t)io.bmap[base + p] * L + rc0;
#pragma unroll
          for (int c = 0; c < NRHS; ++c) x[p * NRHS + c] = c < ncr ? R[row + c] : 0.0;
        }
      }
      PSYNC();
    }
    if (SPLIT && kind >= SN_XSEND) {
      // exchange step of a subtree-parallel item (no ring slot): p0 / w = the x
      // range, SnChunk::off = its offset in the exchange buffer, r = flag
      double* xb = wk.xbuf + ch[kk].off;
      if (kind == SN_XZERO) {
        for (int e = tid; e < w; e += SN_NT) x[p0 + e] = 0.0;
        PSYNC();
      } else if (kind == SN_XSEND) {
        for (int e = tid; e < w; e += SN_NT) __stcg(xb + e, x[p0 + e]);
        __threadfence();
        PSYNC();
        if (tid == 0) flag_release(wk.xflag + r, 1);
      } else {
        if (tid == 0) {
          while (flag_acquire(wk.xflag + r) == 0) {}
          wk.xflag[r] = 0;   // one-shot: the sender sets it again in the next launch
        }
        PSYNC();
        if (cc0 & 1) {
          for (int e = tid; e < w; e += SN_NT) x[p0 + e] += __ldcg(xb + e);
        } else {
          for (int e = tid; e < w; e += SN_NT) x[p0 + e] = __ldcg(xb + e);
        }
        PSYNC();
      }
    } else {
    {
      const long long tw = prof ? clock64() : 0;
      if (flags & 1) mbar_wait_sleep(&full[s], ph);
      else mbar_wait(&full[s], ph);
      if (prof) t_wait += clock64() - tw;
    }
    const double* st = ring + (size_t)s * stage_doubles;
    const int cs = s;
    if (flags & 4) {   // streaming-only probe: no compute (results invalid)
      if (++s == stages) { s = 0; ph ^= 1; }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[cs]);
      continue;
    }
    const long long t_k0 = prof ? clock64() : 0;
    if (++s == stages) { s = 0; ph ^= 1; }
    const int rd = (info & SN_INFO_ROWS) ? (int)sn_rows_doubles(r) : 0;   // row-list prefix
    if (kind == SN_W_FWD || kind == SN_F_FWD) {
      // row-parallel gemv on a column chunk: W_S, F_SS^-1
      const int h = kind == SN_W_FWD ? r : w;
      const int ld = h + (h & 1);
      const RowLayout L(sn_lg<NRHS, SN_MAXQ>(lgc, h, SN_LGNT, stage_doubles), tid, SN_LGNT);
      if (rd) {   // W_S part with its row list in front: group 0 keeps its rows
        const int32_t* rows = reinterpret_cast<const int32_t*>(st);
        if (L.g == 0) {
#pragma unroll
          for (int q = 0; q < SN_MAXQ; ++q)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 2 * (L.t + q * L.TG) + e;
              prow[q][e] = i < r ? rows[i] : -1;
            }
        }
        rows_held = true;
        st += rd;
      }
      if (cc0 == 0) {
#pragma unroll
        for (int q = 0; q < SN_MAXQ; ++q)
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int cr = 0; cr < NRHS; ++cr) acc[q][e][cr] = 0.0;
        if (XG && (kind == SN_W_FWD || r == 0)) {
          // first forward chunk of S: stage x_S (w consecutive positions from p0)
          const double* src = x + (size_t)p0 * NRHS;
          for (int e = tid; e < w * NRHS; e += SN_NT) xs[e] = src[e];
          PSYNC();
        }
      }
      const double* xcol = XG ? xs + (size_t)cc0 * NRHS : x + (size_t)(p0 + cc0) * NRHS;
      const int nq = L.nq(h);
      if (nq <= 1) sn_rows<1, NRHS, SN_MAXQ>(st, ld, nc, h, xcol, L, acc);
      else if (nq == 2 || SN_MAXQ == 2) sn_rows<2, NRHS, SN_MAXQ>(st, ld, nc, h, xcol, L, acc);
      else if constexpr (SN_MAXQ >= 4) {
        if (nq == 3) sn_rows<3, NRHS, SN_MAXQ>(st, ld, nc, h, xcol, L, acc);
        else sn_rows<4, NRHS, SN_MAXQ>(st, ld, nc, h, xcol, L, acc);
      }
      if (!(last && L.G > 1)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cs]);
      }
      if (last) {
        if (L.G > 1) {
          // the stage just read serves as the scratch of the group reduction
          // (from its base: a row-list prefix is already held in registers);
          // it is released once group 0 has read the partials
          double* scratch = ring + (size_t)cs * stage_doubles;
          PSYNC();
          sn_group_reduce<NRHS, SN_MAXQ, SN_NT>(L, h, scratch, acc);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[cs]);
        }
        if (kind == SN_W_FWD) {
          if (rows_held) {   // x_R -= W_S x_S (else a ROWS_FWD chunk follows)
            if (L.g == 0) {
#pragma unroll
              for (int q = 0; q < SN_MAXQ; ++q)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const int pr = prow[q][e];
                  if (pr >= 0) {
#pragma unroll
                    for (int cr = 0; cr < NRHS; ++cr) x[pr * NRHS + cr] -= acc[q][e][cr];
                  }
                }
            }
            rows_held = false;
          }
        } else {
          if (L.G == 1) PSYNC();   // every thread is done reading x_S
          if (L.g == 0) {
#pragma unroll
            for (int q = 0; q < SN_MAXQ; ++q)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int i = 2 * (L.t + q * L.TG) + e;
                if (i < w) {
#pragma unroll
                  for (int cr = 0; cr < NRHS; ++cr) x[(p0 + i) * NRHS + cr] = acc[q][e][cr];
                }
              }
          }
          PSYNC();
        }
      }
    } else if (kind == SN_ROWS_FWD) {
      // x_R -= W_S x_S (summed over the W part by group 0; rows are distinct)
      const RowLayout L(sn_lg<NRHS, SN_MAXQ>(lgc, r, SN_LGNT, stage_doubles), tid, SN_LGNT);
      const int32_t* rows = reinterpret_cast<const int32_t*>(st);
      if (L.g == 0) {
#pragma unroll
        for (int q = 0; q < SN_MAXQ; ++q)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = 2 * (L.t + q * L.TG) + e;
            if (i < r) {
              const int pr = rows[i];
#pragma unroll
              for (int cr = 0; cr < NRHS; ++cr) x[pr * NRHS + cr] -= acc[q][e][cr];
            }
          }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[cs]);
    } else if (kind == SN_ROWS_BWD) {
      // stage x_R contiguously (read by every column of the W part)
      const int32_t* rows = reinterpret_cast<const int32_t*>(st);
      for (int i = tid; i < r; i += SN_NT) {
        const int pr = rows[i];
#pragma unroll
        for (int cr = 0; cr < NRHS; ++cr) xr[cr * rpad + i] = x[pr * NRHS + cr];
      }
      if ((r & 1) && tid < NRHS) xr[tid * rpad + r] = 0.0;
      if (XG) {
        const double* src = x + (size_t)p0 * NRHS;
        for (int e = tid; e < w * NRHS; e += SN_NT) xs[e] = src[e];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[cs]);
      PSYNC();
    } else {  // SN_W_BWD: x_S[j] -= W[:,j] . x_R, LPC lanes per column
      if (rd) {   // the row list came first in this chunk: stage x_R as ROWS_BWD does
        const int32_t* rows = reinterpret_cast<const int32_t*>(st);
        for (int i = tid; i < r; i += SN_NT) {
          const int pr = rows[i];
#pragma unroll
          for (int cr = 0; cr < NRHS; ++cr) xr[cr * rpad + i] = x[pr * NRHS + cr];
        }
        if ((r & 1) && tid < NRHS) xr[tid * rpad + r] = 0.0;
        if (XG) {   // and x_S of S (updated in shared memory, written back at the end)
          const double* src = x + (size_t)p0 * NRHS;
          for (int e = tid; e < w * NRHS; e += SN_NT) xs[e] = src[e];
        }
        PSYNC();
        st += rd;
      }
      const int ld = r + (r & 1);
      double* xo = XG ? xs + (size_t)cc0 * NRHS : x + (size_t)(p0 + cc0) * NRHS;
      if (r > 256) sn_wbwd<32, NRHS, SN_CONS>(st, ld, r, nc, xr, rpad, xo, warp, lane);
      else if (r > 128) sn_wbwd<16, NRHS, SN_CONS>(st, ld, r, nc, xr, rpad, xo, warp, lane);
      else sn_wbwd<8, NRHS, SN_CONS>(st, ld, r, nc, xr, rpad, xo, warp, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[cs]);
      if (last) {
        PSYNC();
        if (XG) {   // x_S of S is final: back to x
          double* dst = x + (size_t)p0 * NRHS;
          for (int e = tid; e < w * NRHS; e += SN_NT) dst[e] = xs[e];
          PSYNC();
        }
      }
    }
    if (prof && kind < 6) {
      t_kind[kind] += clock64() - t_k0;
      n_kind[kind]++;
    }
    }   // factor chunk
    if (info & SN_INFO_LAST_ITEM) {
      PSYNC();
      // ---- write the solution
      if (io.mode == 2) {
        for (int p = tid; p < n * NRHS; p += SN_NT) io.out[base * NRHS + p] = x[p];
      } else if (io.mode == 0) {
        if (SPLIT) {   // the x positions this team member owns
          const int hi = wk.item_hi[item];
          for (int p = wk.item_lo[item] + tid; p < hi; p += SN_NT) io.out[base + p] = x[p];
        } else {
          for (int p = tid; p < n; p += SN_NT) io.out[base + p] = x[p];
        }
      } else {
        const int L = io.ld[sub];
        const int ncr = min(NRHS, L - 1 - rc0);
        double* B = io.out + io.b_off[sub];
        for (int p = tid; p < n; p += SN_NT) {
          const int64_t row = (int64_t)io.bmap[base + p] * L + rc0;
#pragma unroll
          for (int c = 0; c < NRHS; ++c)
            if (c < ncr) B[row + c] = -x[p * NRHS + c];
        }
      }
      PSYNC();
    }
  }
  if (flags & 16) {
    cons_sync<SN_NT>();
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_sn_cta_t[2 * blockIdx.x + 1] = globaltimer();
  }
  if (prof && lane == 0)
    printf("sn_prof cta %d warp %d: total %lld full-wait %lld sync %lld | Wf %lld/%lld Ff %lld/%lld "
           "Wb %lld/%lld Rf %lld/%lld Rb %lld/%lld\n", blockIdx.x, warp, clock64() - t_start,
           t_wait, t_sync, t_kind[0], n_kind[0], t_kind[1], n_kind[1], t_kind[2], n_kind[2],
           t_kind[3], n_kind[3], t_kind[4], n_kind[4]);
}
#undef PSYNC
// shared memory: ring (stages x chunk) | x (max_n even, NRHS) | x_R / scratch
// x_S (max_n) and x_R (max_r) after the ring; at least SN_GUARD doubles, the
// largest row overrun of an unpredicated sn_rows read (2 TG - 1, TG <= 256)
constexpr int SN_GUARD = 512;
// x and x_R in global memory (SnWork::xg): always for several right-hand
// sides; for one, per batch (SnSymbolic::xg1, sn_pick_xg)
bool sn_xg(int nrhs, bool xg1) { return nrhs > 1 || xg1; }
// One right-hand side: x of the whole subdomain in shared memory is what makes
// the sweep fast while two 8-warp CTAs per SM fit next to it with chunks of
// >= 32 KiB (cfg3: 1.70 vs 2.11 ms with x in global memory).  When x is too
// large for that -- the batch would run 16 x 1 (cfg4 / cfg5 grains, x up to
// 12 k DOF) or 8 x 2 on 16-24 KiB chunks (their contact grids) -- x moves to
// the CTA's global slice (L1/L2-resident, x_S staged per supernode as for
// several RHS) and the batch keeps 8 x 2 with ~50 KiB chunks: cfg4 solve
// 0.697 -> 0.638 s.  mode: -1 automatic, 0 / 1 forced (HPLMM_SN_XG, _G, _C).
bool sn_pick_xg(int nitems, int nsm, int max_n, int max_r, int shape, int max_w, int mode) {
  if (mode >= 0) return mode > 0;
  const int cs = sn_pick_chunk(nitems, nsm, max_n, max_r, shape, max_w, false);
  const int cfg_s = sn_solve_cfg(nitems, nsm, max_n, max_r, 1, cs, shape, max_w, false);
  if (cfg_s == 8 && cs >= 4096) return false;
  if (cfg_s != 8 && nitems < 2 * nsm) return false;   // few subdomains: 16 x 1 is the shape anyway
  const int cx = sn_pick_chunk(nitems, nsm, max_n, max_r, shape, max_w, true);
  const int cfg_x = sn_solve_cfg(nitems, nsm, max_n, max_r, 1, cx, shape, max_w, true);
  return cfg_x == 8 && (cfg_s != 8 || cx > cs);
}
int64_t sn_xg_stride(int max_n, int nrhs) { return (int64_t)((max_n + 1) & ~1) * nrhs; }
// shared memory after the ring: x (or, XG, x_S of one supernode) then x_R
static size_t sn_tail_doubles(int max_n, int max_r, int nrhs, int max_w, bool xg) {
  const int xs = xg ? max_w : max_n;
  const size_t t = (size_t)(((xs + 1) & ~1) + ((max_r + 3) & ~1)) * nrhs;
  return t < SN_GUARD ? SN_GUARD : t;
}

// Launch shape of the solve: 16 consumer warps x 1 CTA per SM, or 8 x 2 (two
// independent item streams per SM; better latency hiding when there are at
// least two items per CTA).  shape: 0 = automatic from the item count
// (HPLMM_SN_CFG=16|8 forces one for experiments), 8 / 16 = the handle's
// hplmm_options.sn_shape (falls back to automatic when it does not fit); 1 =
// automatic with subtree-parallel teams allowed (sn_split >= 0): one RHS takes
// 8 x 2 whenever it fits -- teams turn few subdomains into many items, and
// twice the CTAs let the scheduler cut deeper (cfg2: 0.0352 -> 0.0292 s).

int sn_solve_cfg(int nitems, int nsm, int max_n, int max_r, int nrhs, int chunk, int shape,
                 int max_w, bool xg) {
  static int env_forced = -1;
  if (env_forced < 0) {
    const char* e = getenv("HPLMM_SN_CFG");
    env_forced = e ? atoi(e) : 0;
  }
  const bool teams = shape == 1 && nrhs == 1;
  if (shape == 1) shape = 0;
  const int forced = shape ? shape : env_forced;
  // the group-reduction scratch must fit one stage: (G - 1) h NRHS doubles, with
  // TG >= h/8 for one RHS (<= 8 x consumer threads) and TG >= h/2 for several
  // (sn_lg: <= 2 x consumer threads x NRHS)
  auto scratch = [nrhs](int nt) { return nrhs == 1 ? 8 * nt : 2 * nt * nrhs; };
  const bool fit8 = sn_solve_stages(max_n, max_r, nrhs, chunk, 8, max_w, xg) >= 2 && chunk >= scratch(256);
  const bool fit16 = sn_solve_stages(max_n, max_r, nrhs, chunk, 16, max_w, xg) >= 2 && chunk >= scratch(512);
  if (forced == 4 && sn_solve_stages(max_n, max_r, nrhs, chunk, 4, max_w, xg) >= 2 && chunk >= scratch(128))
    return 4;
  if (forced == 8 && fit8) return 8;
  if (forced == 16 && fit16) return 16;
  if (fit8 && (nitems >= 2 * nsm || (teams && !forced))) return 8;
  if (fit16) return 16;
  return 0;   // does not fit
}

// CTAs per SM of a consumer-warp count; HPLMM_SN_CPS1 (experiment): 8 warps x 1 CTA
static bool cps1_8() {
  static const int v = getenv("HPLMM_SN_CPS1") ? 1 : 0;
  return v;
}
int sn_cfg_cps(int cons) { return cons == 16 ? 1 : (cons == 8 && cps1_8() ? 1 : 2); }
static int cfg_cps(int cons) { return sn_cfg_cps(cons); }

// Chunk size of a batch's solve stream: 32 KiB when the batch runs 8 warps x 2
// CTAs per SM; a batch that needs 16 x 1 (few subdomains, or x_S too large for
// two CTAs) streams 64 KiB (else 48 KiB) chunks -- half the per-chunk
// overhead for its 16 consumer warps (cfg5 grain / contact solves -13% / -8%).
// HPLMM_SN_CHUNK overrides.
int sn_pick_chunk(int nitems, int nsm, int max_n, int max_r, int shape, int max_w, bool xg) {
  if (getenv("HPLMM_SN_CHUNK")) return sn_chunk_doubles();
  const int base = sn_chunk_doubles();
  if (sn_solve_cfg(nitems, nsm, max_n, max_r, 1, base, shape, max_w, xg) == 8) {
    // the largest chunk (2 KiB steps) that keeps two 8-warp CTAs per SM with
    // two stages: the solve's cost is per chunk more than per byte (cfg3
    // contact batch: 32 KiB 1.79 ms, 36 KiB 1.74 ms, 38 KiB 1.70 ms)
    int best = base;
    for (int c = base + 256; c <= SN_CHUNK_DOUBLES_MAX; c += 256) {
      if (sn_solve_cfg(nitems, nsm, max_n, max_r, 1, c, shape, max_w, xg) != 8) break;
      best = c;
    }
    return best;
  }
  // enough subdomains for 8 x 2 but x_S leaves no room for two 32-KiB stages:
  // smaller chunks keep the 8 x 2 shape (far cheaper per byte than 16 x 1)
  for (int c : {3072, 2048})
    if (c < base && sn_solve_cfg(nitems, nsm, max_n, max_r, 1, c, shape, max_w, xg) == 8) return c;
  for (int c : {SN_CHUNK_DOUBLES_MAX, 6144})
    if (c > base && sn_solve_stages(max_n, max_r, 1, c, 16, max_w, xg) >= 2) return c;
  return base;
}

int sn_solve_stages(int max_n, int max_r, int nrhs, int chunk, int cons, int max_w, bool xg) {
  const int p = cfg_cps(cons);
  const long avail =
      (226L * 1024) / p - 1024 - (long)sn_tail_doubles(max_n, max_r, nrhs, max_w, xg) * 8;
  return (int)std::min<long>(SN_MAXST, avail / ((long)chunk * 8));
}

template <int NRHS, int CONS, int CPS, bool XG>
static void sn_solve_launch_x(const SnDev& d, const SnIO& io, const SnWork& wk, int stages,
                              int chunk, int max_n, int max_r, size_t smem, cudaStream_t st) {
  static int flags = -1;
  if (flags < 0) {
    const char* e = getenv("HPLMM_SN_FLAGS");
    flags = e ? atoi(e) : 0;
  }
  if constexpr (NRHS == 1 && !XG) {
    if (wk.split) {
      // subtree-parallel items: a team's members wait for each other, so all
      // CTAs must be resident together: a cooperative launch (fails loudly when
      // they cannot be); HPLMM_SN_TEAM_LAUNCH=0: a plain launch (experiments)
      static const int mode = getenv("HPLMM_SN_TEAM_LAUNCH") ? atoi(getenv("HPLMM_SN_TEAM_LAUNCH")) : 1;
      set_max_dynamic_smem((const void*)k_sn_solve<1, CONS, CPS, false, true>, smem);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)wk.nblocks);
      cfg.blockDim = dim3(32 * (CONS + 1));
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = mode == 0 ? 0 : 1;
      cudaLaunchKernelEx(&cfg, k_sn_solve<1, CONS, CPS, false, true>, d, io, wk, stages, chunk,
                         max_n, max_r, flags);
      return;
    }
  }
  set_max_dynamic_smem((const void*)k_sn_solve<NRHS, CONS, CPS, XG, false>, smem);
  k_sn_solve<NRHS, CONS, CPS, XG, false><<<wk.nblocks, 32 * (CONS + 1), smem, st>>>(
      d, io, wk, stages, chunk, max_n, max_r, flags);
  if ((flags & 16) && wk.nblocks <= 4096) {   // experiment: per-CTA finish-time quantiles
    static unsigned long long h[2 * 4096];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_sn_cta_t, sizeof(unsigned long long) * 2 * wk.nblocks);
    unsigned long long t0 = ~0ull, t1 = 0;
    std::vector<double> end(wk.nblocks), dur(wk.nblocks);
    for (int b = 0; b < wk.nblocks; ++b) { t0 = std::min(t0, h[2 * b]); t1 = std::max(t1, h[2 * b + 1]); }
    for (int b = 0; b < wk.nblocks; ++b) {
      end[b] = (h[2 * b + 1] - t0) * 1e-3;
      dur[b] = (h[2 * b + 1] - h[2 * b]) * 1e-3;
    }
    std::sort(end.begin(), end.end());
    std::sort(dur.begin(), dur.end());
    auto q = [&](const std::vector<double>& v, double f) { return v[(size_t)(f * (v.size() - 1))]; };
    fprintf(stderr, "sn_solve ctas %d span %.1f us | end q10 %.1f q50 %.1f q90 %.1f max %.1f | dur q10 %.1f q50 %.1f q90 %.1f max %.1f\n",
            wk.nblocks, (t1 - t0) * 1e-3, q(end, .1), q(end, .5), q(end, .9), end.back(), q(dur, .1),
            q(dur, .5), q(dur, .9), dur.back());
  }
}

template <int NRHS, int CONS, int CPS>
static void sn_solve_launch(const SnDev& d, const SnIO& io, const SnWork& wk, int stages,
                            int chunk, int max_n, int max_r, size_t smem, cudaStream_t st) {
  // several right-hand sides always keep x in global memory (sn_build_work
  // allocates the slices whenever sn_xg says so)
  if constexpr (NRHS > 1) {
    sn_solve_launch_x<NRHS, CONS, CPS, true>(d, io, wk, stages, chunk, max_n, max_r, smem, st);
  } else {
    if (wk.xg) sn_solve_launch_x<NRHS, CONS, CPS, true>(d, io, wk, stages, chunk, max_n, max_r, smem, st);
    else sn_solve_launch_x<NRHS, CONS, CPS, false>(d, io, wk, stages, chunk, max_n, max_r, smem, st);
  }
}

template <int CONS, int CPS>
static void sn_launch_nrhs(const SnDev& d, const SnIO& io, const SnWork& wk, int nrhs, int stages,
                           int chunk, int max_n, int max_r, size_t smem, cudaStream_t st) {
  if (nrhs == 1) sn_solve_launch<1, CONS, CPS>(d, io, wk, stages, chunk, max_n, max_r, smem, st);
  else if (nrhs == 2) sn_solve_launch<2, CONS, CPS>(d, io, wk, stages, chunk, max_n, max_r, smem, st);
  else sn_solve_launch<4, CONS, CPS>(d, io, wk, stages, chunk, max_n, max_r, smem, st);
}

void launch_sn_solve(const SnDev& d, const SnIO& io, const SnWork& wk, int nrhs, int max_n,
                     int max_r, int chunk, int cons, cudaStream_t st) {
  if (wk.nblocks <= 0) return;
  const bool xg = wk.xg != nullptr;
  const int stages = sn_solve_stages(max_n, max_r, nrhs, chunk, cons, wk.max_w, xg);
  const size_t smem = ((size_t)stages * chunk + sn_tail_doubles(max_n, max_r, nrhs, wk.max_w, xg)) * 8;
  static const bool dbg = getenv("HPLMM_DEBUG") != nullptr;
  static int printed = 0;
  if (dbg && printed < 4) {
    ++printed;
    fprintf(stderr, "hplmm sn_solve: blocks %d cons %d nrhs %d max_n %d max_r %d chunk %d stages %d smem %zu\n",
            wk.nblocks, cons, nrhs, max_n, max_r, chunk, stages, smem);
  }
  if (cons == 4) sn_launch_nrhs<4, 2>(d, io, wk, nrhs, stages, chunk, max_n, max_r, smem, st);
  else if (cons == 8 && cps1_8()) sn_launch_nrhs<8, 1>(d, io, wk, nrhs, stages, chunk, max_n, max_r, smem, st);
  else if (cons == 8) sn_launch_nrhs<8, 2>(d, io, wk, nrhs, stages, chunk, max_n, max_r, smem, st);
  else sn_launch_nrhs<16, 1>(d, io, wk, nrhs, stages, chunk, max_n, max_r, smem, st);
}

// grain-batch layout views of a supernodal grain solve (for the per-RHS
// correction columns, eq:col_cg): xloc = b[lmap], yloc = y_sn[gpos_sn[lmap]]
__global__ void k_sn_to_batch(int64_t nloc, const int32_t* __restrict__ lmap,
                              const int32_t* __restrict__ gpos_sn, const double* __restrict__ b,
                              const double* __restrict__ ysn, double* __restrict__ xloc,
                              double* __restrict__ yloc, int P, int c) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nloc) return;
  const int d = lmap[i];
  xloc[i] = d >= 0 ? b[d] : 0.0;
  yloc[i] = d >= 0 ? ysn[(int64_t)gpos_sn[d] * P + c] : 0.0;
}

void launch_sn_to_batch(int64_t nloc, const int32_t* lmap, const int32_t* gpos_sn, const double* b,
                        const double* ysn, double* xloc, double* yloc, cudaStream_t st, int P,
                        int c) {
  if (nloc <= 0) return;
  k_sn_to_batch<<<(unsigned)((nloc + 255) / 256), 256, 0, st>>>(nloc, lmap, gpos_sn, b, ysn, xloc,
                                                                 yloc, P, c);
}

// ===========================================================================
// Numeric factorisation (multifrontal, level by level over the batch)
// ===========================================================================
// F (h x h col-major, zeroed) <- A^ blocks with a column node in S
__global__ void k_front_asm(const int32_t* __restrict__ list, int nlist, const int64_t* asm_ptr,
                            const int64_t* asm_e, const int32_t* asm_u, const int32_t* asm_v,
                            const int32_t* sn_w, const int32_t* sn_r, const int64_t* front_off,
                            const double* __restrict__ val, double* __restrict__ pool) {
  const int sn = list[blockIdx.x];
  const int h = sn_w[sn] + sn_r[sn];
  double* F = pool + front_off[sn];
  for (int64_t t = asm_ptr[sn] + threadIdx.x; t < asm_ptr[sn + 1]; t += blockDim.x) {
    const int64_t e = asm_e[t];
    const int fu = asm_u[t], fv = asm_v[t];
    const double* blk = val + 9 * e;   // A[v][u] (row node v in S, column node u)
    if (fu == fv) {
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) F[(3 * fu + i) + (int64_t)(3 * fv + j) * h] = blk[3 * i + j];
    } else {
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          const double a = blk[3 * j + i];   // A[u][v](i,j) = A[v][u](j,i)
          F[(3 * fu + i) + (int64_t)(3 * fv + j) * h] = a;
          F[(3 * fv + j) + (int64_t)(3 * fu + i) * h] = a;
        }
    }
  }
}

// parent front += U_child (extend-add through the child's relative indices)
__global__ void k_front_ext(const int32_t* __restrict__ list, const int32_t* sn_w,
                            const int32_t* sn_r, const int32_t* sn_parent, const int64_t* rel_off,
                            const int32_t* rel, const int64_t* front_off, double* pool) {
  const int c = list[blockIdx.x];
  const int wc = sn_w[c], rc = sn_r[c], hc = wc + rc;
  const int par = sn_parent[c];
  const int hp = sn_w[par] + sn_r[par];
  const double* Fc = pool + front_off[c];
  double* Fp = pool + front_off[par];
  const int32_t* rl = rel + rel_off[c];
  const int64_t tot = (int64_t)rc * rc;
  for (int64_t t = threadIdx.x; t < tot; t += blockDim.x) {
    const int i = (int)(t % rc), j = (int)(t / rc);
    const int pi = 3 * rl[i / 3] + i % 3, pj = 3 * rl[j / 3] + j % 3;
    Fp[pi + (int64_t)pj * hp] += Fc[(wc + i) + (int64_t)(wc + j) * hc];
  }
}

// F_SS -> packed 64-tiles of the level batch (lower tiles, col-major)
__global__ void k_front_to_tiles(int64_t ntiles, const int32_t* __restrict__ tile_s,
                                 const int32_t* __restrict__ tile_ij,
                                 const int32_t* __restrict__ list, const int32_t* sn_w,
                                 const int32_t* sn_r, const int64_t* front_off,
                                 const double* __restrict__ pool, double* __restrict__ tiles) {
  const int64_t t = blockIdx.x;
  if (t >= ntiles) return;
  const int ls = tile_s[t], ij = tile_ij[t];
  const int I = ij >> 16, J = ij & 0xffff;
  const int sn = list[ls];
  const int w = sn_w[sn], h = w + sn_r[sn];
  const double* F = pool + front_off[sn];
  double* T = tiles + t * TILE;
  for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
    const int a = e & 63, b = e >> 6;
    const int i = TB * I + a, j = TB * J + b;
    T[e] = (i < w && j < w) ? F[i + (int64_t)j * h] : 0.0;
  }
}

// inverse tiles -> Finv (w x w col-major, ld ldf) in the factor storage
__global__ void k_tiles_to_finv(int nlist, const int32_t* __restrict__ list,
                                const int64_t* __restrict__ tile_base, const int32_t* __restrict__ nb,
                                const int32_t* sn_w, const int32_t* sn_r, const int32_t* sn_ldw,
                                const int32_t* sn_ldf, const int64_t* sn_foff,
                                const double* __restrict__ tiles, double* __restrict__ factor) {
  const int ls = blockIdx.y;
  const int sn = list[ls];
  const int w = sn_w[sn], ldf = sn_ldf[sn];
  double* Fi = factor + sn_foff[sn] + sn_rows_doubles(sn_r[sn]) + (int64_t)sn_ldw[sn] * w;
  const int64_t tot = (int64_t)w * w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % w), j = (int)(t / w);
    const int ii = i >= j ? i : j, jj = i >= j ? j : i;
    const int I = ii / TB, J = jj / TB;
    const int64_t tix = tile_base[ls] + (int64_t)I * (I + 1) / 2 + J;
    Fi[i + (int64_t)j * ldf] = tiles[tix * TILE + (ii % TB) + TB * (jj % TB)];
  }
}

// Batched FP64 GEMM  C = alpha op(A) op(B) + beta C  (col-major), 64x64 output
// tiles, BK = 16 through shared memory; FP64 tensor cores (DMMA m8n8k4) or
// 4x4 FMA outputs per thread.
template <bool DMMA>
__global__ void __launch_bounds__(256) k_gemm_batched(const GemmProb* __restrict__ probs,
                                                      const int32_t* __restrict__ work) {
  const int p = work[3 * blockIdx.x], ti = work[3 * blockIdx.x + 1], tj = work[3 * blockIdx.x + 2];
  const GemmProb g = probs[p];
  constexpr int LD = 72;   // smem row stride (bank spread of the DMMA fragments)
  __shared__ double As[16 * LD];
  __shared__ double Bs[16 * LD];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = ti * 64, j0 = tj * 64;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (int k0 = 0; k0 < g.k; k0 += 16) {
    for (int e = threadIdx.x; e < 1024; e += 256) {
      const int r = e & 63, kk = e >> 6;
      const int gi = i0 + r, gk = k0 + kk;
      As[kk * LD + r] = (gi < g.m && gk < g.k)
                            ? (g.transA ? g.A[gk + (int64_t)gi * g.lda] : g.A[gi + (int64_t)gk * g.lda])
                            : 0.0;
      const int gj = j0 + r;
      double bv = 0.0;
      if (gj < g.n && gk < g.k) bv = g.transB ? g.B[gj + (int64_t)gk * g.ldb] : g.B[gk + (int64_t)gj * g.ldb];
      Bs[kk * LD + r] = bv;
    }
    __syncthreads();
    if (DMMA) {
      tile_dmma(As, LD, Bs, LD, 16, acc);
    } else {
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q] = As[kk * LD + tx + 16 * q];
          b[q] = Bs[kk * LD + ty + 16 * q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[q * 4 + u] = fma(a[q], b[u], acc[q * 4 + u]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    int r, c;
    if (DMMA) {
      dmma_rc(q, r, c);
    } else {
      r = tx + 16 * (q >> 2);
      c = ty + 16 * (q & 3);
    }
    const int gi = i0 + r, gj = j0 + c;
    if (gi < g.m && gj < g.n) {
      double* cp = g.C + gi + (int64_t)gj * g.ldc;
      *cp = g.beta == 0.0 ? g.alpha * acc[q] : fma(g.alpha, acc[q], g.beta * *cp);
    }
  }
}

void launch_front_asm(const int32_t* list, int nlist, const SnNum& nm, const double* val,
                      cudaStream_t st) {
  if (nlist <= 0) return;
  k_front_asm<<<nlist, 128, 0, st>>>(list, nlist, nm.asm_ptr, nm.asm_e, nm.asm_u, nm.asm_v,
                                     nm.sn_w, nm.sn_r, nm.front_off, val, nm.pool);
}
void launch_front_ext(const int32_t* list, int nlist, const SnNum& nm, cudaStream_t st) {
  if (nlist <= 0) return;
  k_front_ext<<<nlist, 256, 0, st>>>(list, nm.sn_w, nm.sn_r, nm.sn_parent, nm.rel_off, nm.rel,
                                     nm.front_off, nm.pool);
}
void launch_front_to_tiles(const DevBatch& b, const int32_t* list, const SnNum& nm,
                           cudaStream_t st) {
  if (b.ntiles <= 0) return;
  k_front_to_tiles<<<(unsigned)b.ntiles, 256, 0, st>>>(b.ntiles, b.tile_s, b.tile_ij, list,
                                                       nm.sn_w, nm.sn_r, nm.front_off, nm.pool,
                                                       b.tiles);
}
void launch_tiles_to_finv(const DevBatch& b, const int32_t* list, int nlist, int max_w,
                          const SnNum& nm, double* factor, cudaStream_t st) {
  if (nlist <= 0) return;
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(64, ((int64_t)max_w * max_w + 255) / 256)),
            (unsigned)nlist);
  k_tiles_to_finv<<<grid, 256, 0, st>>>(nlist, list, b.tile_base, b.nb, nm.sn_w, nm.sn_r,
                                        nm.sn_ldw, nm.sn_ldf, nm.sn_foff, b.tiles, factor);
}
// ---------------------------------------------------------------------------
// multi-RHS sweeps (shape vectors): X (n x k col-major per subdomain, elimination
// order) gathered from / written to the grain-batch row layout of R / B, and the
// row gathers/scatters between GEMM steps.  One CTA per step item.
// ---------------------------------------------------------------------------
__global__ void k_mr_io(int nitems, const SnMrItem* __restrict__ it, const int32_t* __restrict__ lidx,
                        const int64_t* __restrict__ b_off, const int32_t* __restrict__ ld,
                        const double* __restrict__ R, double* __restrict__ X,
                        double* __restrict__ B, int to_x) {
  const SnMrItem m = it[blockIdx.x];
  const int L = ld[m.g];
  const int64_t tot = (int64_t)m.n * m.k;
  for (int64_t t = threadIdx.x; t < tot; t += blockDim.x) {
    const int p = (int)(t % m.n), c = (int)(t / m.n);
    const int64_t row = b_off[m.g] + (int64_t)lidx[m.base + p] * L + c;
    if (to_x) X[m.xoff + t] = R[row];
    else B[row] = -X[m.xoff + t];
  }
}

// mode 0: X[rows] -= T   mode 1: T = X[rows]   mode 2: X[p0 + i] = T (i < w)
__global__ void k_mr_rows(const SnMrItem* __restrict__ it, const int32_t* __restrict__ rows,
                          const int64_t* __restrict__ rows_off, const int32_t* __restrict__ sn_r,
                          const int32_t* __restrict__ sn_w, const int32_t* __restrict__ sn_p0,
                          double* __restrict__ X, double* __restrict__ T, int mode) {
  const SnMrItem m = it[blockIdx.x];
  const int h = mode == 2 ? sn_w[m.sn] : sn_r[m.sn];
  const int p0 = sn_p0[m.sn];
  const int32_t* rw = rows + rows_off[m.sn];
  const int64_t tot = (int64_t)h * m.k;
  for (int64_t t = threadIdx.x; t < tot; t += blockDim.x) {
    const int i = (int)(t % h), c = (int)(t / h);
    const int64_t xi = m.xoff + (int64_t)c * m.n + (mode == 2 ? p0 + i : rw[i]);
    const int64_t ti = m.toff + t;
    if (mode == 0) X[xi] -= T[ti];
    else if (mode == 1) T[ti] = X[xi];
    else X[xi] = T[ti];
  }
}

void launch_mr_io(int nitems, const SnMrItem* it, const int32_t* lidx, const int64_t* b_off,
                  const int32_t* ld, const double* R, double* X, double* B, int to_x,
                  cudaStream_t st) {
  if (nitems <= 0) return;
  k_mr_io<<<nitems, 256, 0, st>>>(nitems, it, lidx, b_off, ld, R, X, B, to_x);
}
void launch_mr_rows(int nitems, const SnMrItem* it, const SnNum& nm, const int32_t* sn_p0,
                    double* X, double* T, int mode, cudaStream_t st) {
  if (nitems <= 0) return;
  k_mr_rows<<<nitems, 256, 0, st>>>(it, nm.rows, nm.rows_off, nm.sn_r, nm.sn_w, sn_p0, X, T, mode);
}

__global__ void k_rows_to_factor(int nsn, const int32_t* sn_r, const int64_t* sn_foff,
                                 const int64_t* rows_off, const int32_t* rows, double* factor) {
  const int sn = blockIdx.x;
  if (sn >= nsn) return;
  const int r = sn_r[sn];
  int32_t* dst = reinterpret_cast<int32_t*>(factor + sn_foff[sn]);
  const int rp = (int)(2 * sn_rows_doubles(r));
  for (int i = threadIdx.x; i < rp; i += blockDim.x) dst[i] = i < r ? rows[rows_off[sn] + i] : 0;
}

void launch_rows_to_factor(int nsn, const SnNum& nm, double* factor, cudaStream_t st) {
  if (nsn <= 0) return;
  k_rows_to_factor<<<nsn, 128, 0, st>>>(nsn, nm.sn_r, nm.sn_foff, nm.rows_off, nm.rows, factor);
}

void launch_gemm_batched(const GemmProb* probs, const int32_t* work, int nwork, cudaStream_t st) {
  if (nwork <= 0) return;
  if (use_dmma()) k_gemm_batched<true><<<nwork, 256, 0, st>>>(probs, work);
  else k_gemm_batched<false><<<nwork, 256, 0, st>>>(probs, work);
}

}  // namespace hplmm
