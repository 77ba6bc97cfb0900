// Batched supernodal block-LDL^T factors of the local subdomain matrices
// (grain blocks A^{g}_{g} and contact-grid blocks A^[zeta,zeta], eq:Mg_Mz /
// eq:permute_blk_2) -- SURVEY §8(f) NEXT #1.  Internal (not part of the ABI).
//
// Ordering: geometric nested dissection of each subdomain's node set on the
// voxel lattice (a plane of nodes separates the two halves because A^ couples
// only nodes within Chebyshev distance 1).  Every ND tree node (leaf set or
// separator plane) is one supernode S with w = 3|S| columns; its row structure
// R = struct(S) (r = 3|R| rows) follows from the node graph by the usual
// symbolic elimination.  Elimination of S from its frontal matrix
//     F = [F_SS F_SR; F_RS F_RR]
// gives (block LDL^T with SPD diagonal blocks)
//     W_S = F_RS F_SS^-1,   U_S = F_RR - W_S F_RS^T  (passed to the parent),
// and a solve A_s x = b is
//     forward  (postorder):         b_R -= W_S b_S ;  b_S <- F_SS^-1 b_S
//     backward (reverse postorder): x_S -= W_S^T x_R
// so the factor is W_S (r x w) and F_SS^-1 (w x w), both col-major; a solve
// streams W_S twice (forward gemv, backward column dot products) and F_SS^-1
// once: 2 r w + w^2 doubles per supernode.  (A transposed copy of W_S made the
// backward sweep a row-parallel gemv as well, measured no faster, and cost a
// third more memory -- cfg5 does not fit with it.)
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "hplmm_internal.h"

namespace hplmm {

constexpr int SN_CHUNK_DOUBLES_MAX = 8192;   // largest TMA chunk (64 KiB)
int sn_chunk_doubles();                          // chunk size in use (4096)
constexpr int SN_MAX_WR = 2048;          // max w and max r (DOFs) per supernode

// chunk kinds of the solve stream (forward per S: W_FWD.., ROWS_FWD, F_FWD..;
// backward per S: ROWS_BWD, W_BWD..).  ROWS chunks carry the supernode's row
// list (int32) so the scatter/gather of x_R never waits on a global load.
enum SnChunkKind : int32_t {
  SN_W_FWD = 0, SN_F_FWD = 1, SN_W_BWD = 2, SN_ROWS_FWD = 3, SN_ROWS_BWD = 4,
  // subtree-parallel solves (a subdomain shared by a team of CTAs, sn_build_work):
  // exchange steps without factor data (bytes = 0: no ring slot).  p0 / w = the
  // x positions [p0, p0 + w), off = offset of the range in the exchange
  // buffer, r = flag index, c0 bit 0 (XRECV) = add (else assign)
  SN_XSEND = 5, SN_XRECV = 6, SN_XZERO = 7
};

// one TMA chunk of the solve stream, denormalised so that the consumer needs
// exactly one (prefetched) descriptor load per chunk
struct SnChunk {
  int64_t off;     // first double of the chunk in the factor array
  int32_t bytes;   // [0,24): bytes (multiple of 16); [24,28): log2(TG) - 5, the
                   // row-pair thread-group size of the part (see k_sn_solve)
  int32_t info;    // c0 [0,12) | (ncols-1) [12,24) | kind [24,27) | last-of-part [27]
                   // | first-of-item [28] | last-of-item [29] | rows prefix [30]
  int32_t p0;      // first local DOF of S
  int32_t w, r;    // supernode width / struct rows
  int32_t sub;     // subdomain
};
constexpr int SN_INFO_LAST = 1 << 27, SN_INFO_FIRST_ITEM = 1 << 28, SN_INFO_LAST_ITEM = 1 << 29;
// [30]: the chunk starts with the supernode's row list (rows header, then the
// first W_S columns): the first W_FWD / W_BWD chunk of a part carries the rows
// that a separate ROWS_FWD / ROWS_BWD chunk would otherwise bring
constexpr int SN_INFO_ROWS = 1 << 30;

// rows header of a supernode in the factor array: r int32 padded to 16 bytes
#ifdef __CUDACC__
#define SN_HD __host__ __device__
#else
#define SN_HD
#endif
SN_HD inline int64_t sn_rows_doubles(int r) { return (int64_t)((r + 3) / 4) * 2; }

struct SnSymbolic {
  int nsub = 0, nsn = 0;
  int max_n = 0, max_w = 0, max_r = 0, n_levels = 0, max_children = 0;
  int chunk_doubles = 0;                   // TMA chunk (stage) size of the schedule
  int shape = 0;                           // launch shape asked for (0 auto, 8, 16)
  int split = 0;                           // hplmm_options.sn_split (0 auto, -1 off, 1..3 levels)
  bool xg1 = false;                        // one-RHS solves keep x in global memory (sn_pick_xg)
  // per subdomain
  std::vector<int32_t> sub_n;              // DOFs
  std::vector<int64_t> sub_base;           // offset of its local positions
  std::vector<int32_t> sub_sn0, sub_sn1;   // supernode range (postorder)
  std::vector<int64_t> sub_fc0, sub_fc1;   // forward chunk range
  std::vector<int64_t> sub_bc0, sub_bc1;   // backward chunk range
  std::vector<int64_t> sub_fbytes;         // factor bytes streamed by one solve
  std::vector<int32_t> gmap;               // [sum n] global DOF of each local position
  std::vector<int32_t> lidx;               // [sum n] DOF index in the subdomain's node list
  // per supernode
  std::vector<int32_t> sn_w, sn_r, sn_p0, sn_ldw, sn_ldf, sn_level, sn_parent, sn_sub,
      sn_child_rank;
  std::vector<int64_t> sn_rows_off, sn_foff;
  // chunk ranges of each supernode in `chunks`: forward [sn_fcb, sn_fce),
  // backward [sn_bcb, sn_bce) (empty for r = 0); within a subdomain the
  // forward ranges ascend and the backward ranges descend with the supernode
  std::vector<int64_t> sn_fcb, sn_fce, sn_bcb, sn_bce;
  std::vector<int32_t> rows;               // struct rows: local DOF positions (ascending)
  std::vector<SnChunk> chunks;             // per subdomain: [fc0,fc1) forward, [bc0,bc1) backward
  int64_t factor_doubles = 0;              // layout per S: [rows][W_S: ldw x w][F_SS^-1: ldf x w]
  // numeric setup: A-blocks scattered into each front, child -> parent maps
  std::vector<int64_t> asm_ptr;            // [nsn+1]
  std::vector<int64_t> asm_e;              // BSR block index (row node v in S, col node u)
  std::vector<int32_t> asm_u, asm_v;       // front node index of u (row) and v (col)
  std::vector<int64_t> rel_off;            // [nsn+1] per supernode as a child
  std::vector<int32_t> rel;                // front node index in the parent
};

// Symbolic analysis of the subdomains given as ascending node lists
// (CSR ptr/nodes).  leaf = max nodes of an ND leaf.  Returns false + err on
// a supernode wider than SN_MAX_WR.
// nsm: SMs of the device (the chunk size of the solve stream depends on the
// launch shape, sn_pick_chunk)
bool sn_analyse(const HostSetup& hs, const std::vector<int32_t>& ptr,
                const std::vector<int32_t>& nodes, int leaf, SnSymbolic& out, std::string& err,
                int nsm = 148, int shape = 0, int xg_mode = -1);
// shape: 0 = automatic, 8 = 8 consumer warps x 2 CTAs per SM, 16 = 16 x 1
int sn_pick_chunk(int nitems, int nsm, int max_n, int max_r, int shape, int max_w, bool xg);
// x of a one-RHS solve in global memory for this batch? (mode: -1 automatic, 0 / 1 forced)
bool sn_pick_xg(int nitems, int nsm, int max_n, int max_r, int shape, int max_w, int mode);
int sn_cfg_cps(int cons);   // CTAs per SM of a launch shape
// consumer warps per CTA (8: two CTAs per SM; 16: one), 0 if the subdomain
// vectors do not fit in shared memory with >= 2 ring stages
int sn_solve_cfg(int nitems, int nsm, int max_n, int max_r, int nrhs, int chunk, int shape,
                 int max_w, bool xg);
// x of the solve in global memory (per-CTA slices of sn_xg_stride doubles)
bool sn_xg(int nrhs, bool xg1);
int64_t sn_xg_stride(int max_n, int nrhs);

}  // namespace hplmm
