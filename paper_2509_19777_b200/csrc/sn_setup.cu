// Host orchestration of the batched supernodal factors: upload of the
// symbolic data, LPT work lists, and the level-by-level multifrontal numeric
// factorisation (setup, T_ML) -- see supernodal.h.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <queue>

#include "sn_setup.h"

namespace hplmm {

namespace {

#define SN_CK(call)                                                            \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) throw SnError{-2, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

template <class T>
T* up(DevAlloc& A, const std::vector<T>& v, cudaStream_t st, bool setup_only = false) {
  T* p = (T*)A.alloc(std::max<size_t>(v.size(), 1) * sizeof(T), setup_only);
  if (!v.empty()) SN_CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return p;
}

// LPT: items with weights -> nb bins; returns CSR (ptr per bin) over item ids
void lpt(const std::vector<int64_t>& wgt, int nb, std::vector<int32_t>& ptr,
         std::vector<int32_t>& ids) {
  std::vector<int32_t> ord(wgt.size());
  for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int32_t)i;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return wgt[a] > wgt[b]; });
  using P = std::pair<int64_t, int>;
  std::priority_queue<P, std::vector<P>, std::greater<P>> q;
  for (int b = 0; b < nb; ++b) q.push({0, b});
  std::vector<std::vector<int32_t>> bins(nb);
  for (int i : ord) {
    P t = q.top();
    q.pop();
    bins[t.second].push_back(i);
    q.push({t.first + wgt[i], t.second});
  }
  ptr.assign(nb + 1, 0);
  ids.clear();
  for (int b = 0; b < nb; ++b) {
    std::sort(bins[b].begin(), bins[b].end());
    ids.insert(ids.end(), bins[b].begin(), bins[b].end());
    ptr[b + 1] = (int32_t)ids.size();
  }
}

}  // namespace

// LPT cost of a subdomain: bytes streamed + gather/scatter + a fixed cost per
// chunk in byte equivalents (the solve's per-chunk overhead).  Measured at
// cfg3 (contact / grain solve): 0 -> 1.975 / 1.346 ms, 16 KiB -> 1.938 / 1.327,
// 32 KiB -> 1.925 / 1.313, >= 64 KiB -> 1.918 / 1.305 (plateau).  HPLMM_SN_WGT
// overrides.
static int64_t sn_chunk_cost() {
  static const int64_t v = getenv("HPLMM_SN_WGT") ? atoll(getenv("HPLMM_SN_WGT")) : 65536;
  return v;
}

// ---------------------------------------------------------------------------
// Subtree-parallel items.  When a batch has too few subdomains to fill the
// CTAs evenly (cfg2: 64 grains on 148 SMs), the largest ones are shared by a
// team of 2^L consecutive CTAs: the top L levels of the nested-dissection tree
// are cut, every team member sweeps one subtree, and the separators above the
// cut are handled by the member that owns the rightmost subtree below them.
// Forward: a member accumulates its updates of the common ancestors' x in
// rows it zeroed at the start; at each tree node the left subtree's owner
// sends those rows to the node's owner (XSEND / XRECV add), which then
// eliminates the separator.  Backward: the node's owner sends the solved
// ancestor rows to the left owner (XRECV assign) before both descend.
// ---------------------------------------------------------------------------
namespace {

struct TeamOp {
  int member;
  int kind;        // 0 FWD [a,b), 1 BWD [a,b), SN_XSEND / SN_XRECV / SN_XZERO
  int a = 0, b = 0;       // supernode range (FWD / BWD)
  int lo = 0, cnt = 0;    // x range (exchange steps)
  int xch = 0;            // exchange index within the team (flag, buffer slot)
  bool add = false;
};

struct Team {
  int members = 0;
  std::vector<TeamOp> ops;            // a valid global order (sends before their receives)
  std::vector<int32_t> lo, hi;        // owned x range per member
  std::vector<int64_t> finish;        // modelled finish time per member (byte equivalents)
  std::vector<int64_t> xoff;          // exchange buffer offset per exchange (doubles)
  int64_t xdoubles = 0;
};

struct TeamBuilder {
  const SnSymbolic& s;
  const std::vector<int64_t>&pf, &pb;   // prefix sums of forward / backward supernode costs
  const std::vector<std::vector<int>>& kids;
  const std::vector<int>& start;        // first supernode of each supernode's subtree
  Team& T;
  std::vector<std::pair<int, int>> anc;  // ancestor chains (supernode ranges), innermost last
  int64_t xcost;                         // an exchange step in byte equivalents
  std::vector<std::pair<std::pair<int, int>, int>> anc_owner;   // the same chains with their owners

  struct Node {
    int ca = 0, cb = 0;   // separator chain [ca, cb)
    int la = 0, lb = 0;   // leaf: supernode range
    int left = -1, right = -1;
    int owner = -1;
  };
  std::vector<Node> nodes;

  int64_t wrange(int a, int b) const { return (pf[b] - pf[a]) + (pb[b] - pb[a]); }
  int plo(int a) const { return s.sn_p0[a]; }
  int phi(int b) const { return s.sn_p0[b - 1] + s.sn_w[b - 1]; }

  // split tree over the forest `roots` (ascending, contiguous subtrees)
  int build(const std::vector<int>& roots, int depth) {
    Node nd;
    const int ra = start[roots.front()], rb = roots.back() + 1;
    std::vector<int> parts = roots;
    nd.ca = nd.cb = rb;
    if (depth > 0 && parts.size() == 1) {   // a tree: peel the separator chain
      int v = parts[0];
      nd.cb = v + 1;
      while (kids[v].size() == 1) v = kids[v][0];
      nd.ca = v;
      parts = kids[v];
    }
    if (depth == 0 || parts.size() < 2) {
      nd.ca = nd.cb = 0;
      nd.la = ra;
      nd.lb = rb;
      nd.owner = T.members++;
      nodes.push_back(nd);
      return (int)nodes.size() - 1;
    }
    // balanced contiguous cut of the parts
    int64_t tot = 0, acc = 0, best = INT64_MAX;
    for (int c : parts) tot += wrange(start[c], c + 1);
    size_t cut = 1;
    for (size_t j = 1; j < parts.size(); ++j) {
      acc += wrange(start[parts[j - 1]], parts[j - 1] + 1);
      const int64_t dev = std::llabs(2 * acc - tot);
      if (dev < best) { best = dev; cut = j; }
    }
    const std::vector<int> L(parts.begin(), parts.begin() + cut), R(parts.begin() + cut, parts.end());
    nd.left = build(L, depth - 1);
    nd.right = build(R, depth - 1);
    nd.owner = nodes[nd.right].owner;
    nodes.push_back(nd);
    return (int)nodes.size() - 1;
  }

  void emit(TeamOp op) { T.ops.push_back(op); }

  // x ranges of the chain of node v (if any) and of its ancestors
  std::vector<std::pair<int, int>> up_ranges(const Node& nd) const {
    std::vector<std::pair<int, int>> r;
    if (nd.cb > nd.ca) r.push_back({plo(nd.ca), phi(nd.cb)});
    for (size_t i = anc.size(); i-- > 0;) r.push_back({plo(anc[i].first), phi(anc[i].second)});
    return r;
  }
  void exchange(int from, int to, const std::vector<std::pair<int, int>>& rg, bool add) {
    for (auto& q : rg) {
      const int x = (int)T.xoff.size();
      T.xoff.push_back(T.xdoubles);
      T.xdoubles += (q.second - q.first + 1) & ~1;
      emit({from, SN_XSEND, 0, 0, q.first, q.second - q.first, x, false});
      emit({to, SN_XRECV, 0, 0, q.first, q.second - q.first, x, add});
    }
  }
  void fwd(int v) {
    const Node nd = nodes[v];
    if (nd.left < 0) {
      // rows of the common ancestors this member does not own start at zero
      for (auto& c : anc_owner)
        if (c.second != nd.owner) emit({nd.owner, SN_XZERO, 0, 0, plo(c.first.first), phi(c.first.second) - plo(c.first.first), 0, false});
      emit({nd.owner, 0, nd.la, nd.lb});
      return;
    }
    const bool chain = nd.cb > nd.ca;
    if (chain) { anc.push_back({nd.ca, nd.cb}); anc_owner.push_back({{nd.ca, nd.cb}, nd.owner}); }
    fwd(nd.left);
    fwd(nd.right);
    if (chain) { anc.pop_back(); anc_owner.pop_back(); }
    exchange(nodes[nd.left].owner, nd.owner, up_ranges(nd), true);
    if (chain) emit({nd.owner, 0, nd.ca, nd.cb});
  }
  void bwd(int v) {
    const Node nd = nodes[v];
    if (nd.left < 0) {
      emit({nd.owner, 1, nd.la, nd.lb});
      return;
    }
    const bool chain = nd.cb > nd.ca;
    if (chain) emit({nd.owner, 1, nd.ca, nd.cb});
    exchange(nd.owner, nodes[nd.left].owner, up_ranges(nd), false);
    if (chain) anc.push_back({nd.ca, nd.cb});
    bwd(nd.right);
    bwd(nd.left);
    if (chain) anc.pop_back();
  }
  void owned(int v) {
    const Node& nd = nodes[v];
    if (nd.left < 0) {
      T.lo[nd.owner] = plo(nd.la);
      T.hi[nd.owner] = phi(nd.lb);
      return;
    }
    owned(nd.left);
    owned(nd.right);
    if (nd.cb > nd.ca) T.hi[nd.owner] = phi(nd.cb);   // the chain follows the right subtree
  }
  void model() {
    std::vector<int64_t> t(T.members, 0), ready(T.xoff.size(), 0);
    for (const TeamOp& op : T.ops) {
      if (op.kind == 0) t[op.member] += pf[op.b] - pf[op.a];
      else if (op.kind == 1) t[op.member] += pb[op.b] - pb[op.a];
      else if (op.kind == SN_XSEND) { t[op.member] += xcost / 4; ready[op.xch] = t[op.member]; }
      else if (op.kind == SN_XRECV) t[op.member] = std::max(t[op.member], ready[op.xch]) + xcost;
    }
    T.finish = t;
  }
};

}  // namespace

// tree levels that may be cut: hplmm_options.sn_split (0: automatic = 3, or
// HPLMM_SN_SPLIT for experiments; -1: off)
static int sn_split_levels(int opt) {
  static const int env = getenv("HPLMM_SN_SPLIT") ? atoi(getenv("HPLMM_SN_SPLIT")) : 3;
  const int v = opt < 0 ? 0 : (opt > 0 ? opt : env);
  return std::max(0, std::min(3, v));
}

void sn_build_work(SnBatch& B, DevAlloc& A, cudaStream_t st, int nblocks, int nrhs,
                   const std::vector<int32_t>* ncols, SnWork& wk, int force_cons, bool allow_split) {
  const SnSymbolic& s = B.sym;
  const bool setup_only = ncols != nullptr;
  const bool xg = sn_xg(nrhs, s.xg1);   // x in the CTA's global slice
  std::vector<int64_t> wgt;
  std::vector<int32_t> isub, ic0;
  for (int g = 0; g < s.nsub; ++g) {
    const int nc = ncols ? (*ncols)[g] : 1;
    for (int c0 = 0; c0 < nc; c0 += nrhs) {
      isub.push_back(g);
      ic0.push_back(c0);
      wgt.push_back(s.sub_fbytes[g] + 8 * (int64_t)s.sub_n[g] * 64 +
                    sn_chunk_cost() * ((s.sub_fc1[g] - s.sub_fc0[g]) + (s.sub_bc1[g] - s.sub_bc0[g])));
    }
  }
  wk.cons = force_cons ? force_cons
                       : sn_solve_cfg((int)isub.size(), nblocks, s.max_n, s.max_r, nrhs,
                                      s.chunk_doubles, s.shape, s.max_w, xg);
  // several right-hand sides: the 8-warp CTAs hold at most 2 row pairs of
  // every column per thread (k_sn_solve SN_MAXQ), i.e. parts of <= 1024 rows
  if (nrhs > 1 && wk.cons == 8 && std::max(s.max_w, s.max_r) > 512) wk.cons = 16;
  if (wk.cons == 0)
    throw SnError{-1, "subdomain of " + std::to_string(s.max_n) +
                          " DOFs does not fit the supernodal solve's shared memory"};
  nblocks *= sn_cfg_cps(wk.cons);
  if (const char* e = getenv("HPLMM_SN_CTAS")) nblocks = std::max(1, atoi(e));   // experiments
  const int nslots = nblocks;
  nblocks = std::max(1, std::min<int>(nblocks, (int)isub.size()));
  const bool dbg = getenv("HPLMM_DEBUG") != nullptr;

  // ---- subtree-parallel teams for the largest items (one RHS, main solve only)
  const int Lmax = (allow_split && nrhs == 1 && !ncols && !xg && !isub.empty()) ? sn_split_levels(s.split) : 0;
  std::vector<int32_t> ord(wgt.size());
  for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int32_t)i;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return wgt[a] > wgt[b]; });
  std::vector<int64_t> pf, pb;
  std::vector<std::vector<int>> kids;
  std::vector<int> start;
  if (Lmax > 0) {
    pf.assign(s.nsn + 1, 0);
    pb.assign(s.nsn + 1, 0);
    kids.assign(s.nsn, {});
    start.resize(s.nsn);
    for (int k = 0; k < s.nsn; ++k) {
      int64_t f = 0, b = 0;
      for (int64_t c = s.sn_fcb[k]; c < s.sn_fce[k]; ++c) f += (s.chunks[c].bytes & 0xffffff) + sn_chunk_cost();
      for (int64_t c = s.sn_bcb[k]; c < s.sn_bce[k]; ++c) b += (s.chunks[c].bytes & 0xffffff) + sn_chunk_cost();
      pf[k + 1] = pf[k] + f;
      pb[k + 1] = pb[k] + b;
      start[k] = k;
      if (s.sn_parent[k] >= 0) kids[s.sn_parent[k]].push_back(k);
    }
    for (int k = 0; k < s.nsn; ++k)
      for (int c : kids[k]) start[k] = std::min(start[k], start[c]);
  }
  // an exchange step in byte equivalents (~2.5 us of one CTA's stream); HPLMM_SN_XCOST (experiments)
  static const int64_t xcost = getenv("HPLMM_SN_XCOST") ? atoll(getenv("HPLMM_SN_XCOST")) : 65536;
  auto make_team = [&](int g, int L, Team& T) {
    TeamBuilder tb{s, pf, pb, kids, start, T, {}, xcost};
    std::vector<int> roots;
    for (int k = s.sub_sn0[g]; k < s.sub_sn1[g]; ++k)
      if (s.sn_parent[k] < 0) roots.push_back(k);
    const int root = tb.build(roots, L);
    T.lo.assign(T.members, 0);
    T.hi.assign(T.members, 0);
    tb.owned(root);
    tb.fwd(root);
    tb.bwd(root);
    tb.model();
    for (int m = 0; m < T.members; ++m) T.finish[m] += 8 * (int64_t)s.sub_n[g] * 64;
  };
  // level[i] = tree levels cut for item i (0: one CTA).  Teams take consecutive
  // CTAs in item-weight order and come first in their CTAs; the other items
  // are spread by LPT over all CTAs (teams' CTAs start with their modelled
  // finish time).
  const int nitems = (int)ord.size();
  std::vector<int> level(nitems, 0);
  std::vector<std::vector<Team>> cache(nitems);   // per item: teams by level - 1
  auto team_of = [&](int i, int L) -> const Team& {
    auto& c = cache[i];
    if ((int)c.size() < L) c.resize(L);
    if (c[L - 1].members == 0) make_team(isub[i], L, c[L - 1]);
    return c[L - 1];
  };
  struct Eval { int64_t ms; int nb; int argmax; };
  // LPT of the unsplit items (weight order) onto bins with initial loads
  auto evaluate = [&](const std::vector<int>& lv, std::vector<std::vector<int32_t>>* bins,
                      std::vector<int>* cta_item) -> Eval {
    int nteam = 0, nrest = 0;
    for (int i = 0; i < nitems; ++i) {
      if (lv[i] > 0) nteam += team_of(i, lv[i]).members;
      else ++nrest;
    }
    if (nteam > nslots) return {INT64_MAX, 0, -1};
    const int nb = std::max(1, std::max(nteam, std::min(nslots, nteam + nrest)));
    std::vector<int64_t> load(nb, 0);
    if (cta_item) cta_item->assign(nb, -1);
    int b0 = 0;
    for (int k = 0; k < nitems; ++k) {
      const int i = ord[k];
      if (lv[i] == 0) continue;
      const Team& T = team_of(i, lv[i]);
      for (int m = 0; m < T.members; ++m) {
        load[b0 + m] = T.finish[m];
        if (cta_item) (*cta_item)[b0 + m] = i;
      }
      b0 += T.members;
    }
    if (bins) bins->assign(nb, {});
    using P = std::pair<int64_t, int>;
    std::priority_queue<P, std::vector<P>, std::greater<P>> q;
    for (int b = 0; b < nb; ++b) q.push({load[b], b});
    for (int k = 0; k < nitems; ++k) {
      const int i = ord[k];
      if (lv[i] > 0) continue;
      P t = q.top();
      q.pop();
      if (bins) (*bins)[t.second].push_back(i);
      load[t.second] = t.first + wgt[i];
      q.push({load[t.second], t.second});
    }
    const int am = (int)(std::max_element(load.begin(), load.end()) - load.begin());
    return {load[am], nb, am};
  };
  const int64_t ms0 = evaluate(level, nullptr, nullptr).ms;
  if (dbg && nitems > nslots && nitems <= 2 * nslots) {
    // fold bound: the nslots bins hold one or two items; the 2 (n - k) smallest
    // are paired largest-with-smallest
    const int k = nslots, np = nitems - k;
    int64_t fb = wgt[ord[0]];
    for (int t = 0; t < np; ++t) fb = std::max(fb, wgt[ord[nitems - 2 * np + t]] + wgt[ord[nitems - 1 - t]]);
    double tot = 0;
    for (int64_t w : wgt) tot += (double)w;
    fprintf(stderr, "hplmm sn work: LPT makespan %.4f of the mean, fold (<= 2 per CTA) %.4f\n",
            ms0 / (tot / k), fb / (tot / k));
  }
  int64_t best_ms = ms0;
  if (Lmax > 0 && s.split > 0) {
    // forced (hplmm_options.sn_split = L > 0; tests, experiments): every item,
    // largest first, is cut as deep as it can be (<= L levels) while CTAs last
    int used = nitems;
    for (int k = 0; k < nitems; ++k) {
      const int i = ord[k];
      for (int L = Lmax; L >= 1; --L) {
        const int m = team_of(i, L).members;
        if (m >= 2 && used - 1 + m <= nslots) {
          level[i] = L;
          used += m - 1;
          break;
        }
      }
    }
    best_ms = evaluate(level, nullptr, nullptr).ms;
  } else if (Lmax > 0) {
    // (1) the S largest items at a uniform level L
    std::vector<int> best = level;
    for (int L = 1; L <= Lmax; ++L) {
      std::vector<int> lv(nitems, 0);
      for (int S = 1; S <= nitems; ++S) {
        const int i = ord[S - 1];
        if (team_of(i, L).members < 2) break;   // cannot be cut
        lv[i] = L;
        const Eval e = evaluate(lv, nullptr, nullptr);
        if (e.ms == INT64_MAX) break;           // out of CTAs
        if (e.ms < best_ms) { best_ms = e.ms; best = lv; }
      }
    }
    level = best;
    // (2) greedy: cut the item that sets the makespan one level deeper while it helps
    for (int it = 0; it < 4 * nslots; ++it) {
      std::vector<std::vector<int32_t>> bins;
      std::vector<int> cta_item;
      const Eval e = evaluate(level, &bins, &cta_item);
      int i = cta_item[e.argmax];
      if (!bins[e.argmax].empty() && (i < 0 || wgt[bins[e.argmax][0]] > team_of(i, level[i]).finish[0]))
        i = bins[e.argmax][0];   // the largest unsplit item of that CTA
      if (i < 0 || level[i] >= Lmax) break;
      std::vector<int> lv = level;
      lv[i]++;
      if (team_of(i, lv[i]).members <= (level[i] ? team_of(i, level[i]).members : 1)) break;
      const Eval e2 = evaluate(lv, nullptr, nullptr);
      if (e2.ms >= best_ms) break;
      best_ms = e2.ms;
      level = lv;
    }
    // HPLMM_SN_SPLIT_GAIN (experiments): least modelled gain in percent
    static const double gain = getenv("HPLMM_SN_SPLIT_GAIN") ? atof(getenv("HPLMM_SN_SPLIT_GAIN")) : 5.0;
    if (dbg)
      fprintf(stderr, "hplmm sn work: modelled makespan with teams %.3f of the unsplit one\n",
              (double)best_ms / (double)ms0);
    if ((double)best_ms >= (1.0 - gain / 100.0) * (double)ms0) {   // not worth the exchange steps
      std::fill(level.begin(), level.end(), 0);
      best_ms = ms0;
    }
  }
  std::vector<std::vector<int32_t>> bins;
  std::vector<int> cta_item;
  const Eval ev = evaluate(level, &bins, &cta_item);
  nblocks = ev.nb;
  int nsplit = 0, max_team = 1;
  for (int i = 0; i < nitems; ++i)
    if (level[i] > 0) {
      ++nsplit;
      max_team = std::max(max_team, team_of(i, level[i]).members);
    }
  if (dbg) {
    double tot = 0;
    for (int64_t w : wgt) tot += (double)w;
    fprintf(stderr, "hplmm sn work: %zu items on %d CTAs, max/mean CTA weight %.3f (unsplit %.3f), largest item %.3f "
            "of the mean; %d items shared by teams of up to %d CTAs\n", wgt.size(), nblocks,
            ev.ms / (tot / nblocks), ms0 / (tot / nblocks), nitems ? (double)wgt[ord[0]] / (tot / nblocks) : 0.0,
            nsplit, max_team);
  }
  // team member index of each CTA
  std::vector<int> cta_member(nblocks, 0);
  for (int b = 0, m = 0; b < nblocks; ++b) {
    m = (b > 0 && cta_item[b] >= 0 && cta_item[b] == cta_item[b - 1]) ? m + 1 : 0;
    cta_member[b] = m;
  }
  std::vector<int32_t> ptr(nblocks + 1, 0), sub, c0, ilo, ihi;
  std::vector<int64_t> cptr(nblocks + 1, 0);
  std::vector<SnChunk> flat;
  int64_t xtot = 0;
  int nflags = 0;
  auto xchunk = [&](int g, int kind, int lo, int cnt, int64_t off, int flag, bool add) {
    SnChunk ch;
    ch.off = off;
    ch.bytes = 0;
    ch.info = (add ? 1 : 0) | (kind << 24);
    ch.p0 = lo;
    ch.w = cnt;
    ch.r = flag;
    ch.sub = g;
    flat.push_back(ch);
  };
  for (int b = 0; b < nblocks; ++b) {
    if (cta_item[b] >= 0) {
      const Team& T = team_of(cta_item[b], level[cta_item[b]]);
      const int m = cta_member[b], g = isub[cta_item[b]];
      const size_t first = flat.size();
      for (const TeamOp& op : T.ops) {
        if (op.member != m) continue;
        if (op.kind == 0) {
          flat.insert(flat.end(), s.chunks.begin() + s.sn_fcb[op.a], s.chunks.begin() + s.sn_fce[op.b - 1]);
        } else if (op.kind == 1) {
          flat.insert(flat.end(), s.chunks.begin() + s.sn_bcb[op.b - 1], s.chunks.begin() + s.sn_bce[op.a]);
        } else {
          xchunk(g, op.kind, op.lo, op.cnt, op.kind == SN_XZERO ? 0 : xtot + T.xoff[op.xch],
                 op.kind == SN_XZERO ? 0 : nflags + op.xch, op.add);
        }
      }
      flat[first].info |= SN_INFO_FIRST_ITEM;
      flat.back().info |= SN_INFO_LAST_ITEM;
      sub.push_back(g);
      c0.push_back(0);
      ilo.push_back(T.lo[m]);
      ihi.push_back(T.hi[m]);
      if (m == T.members - 1) {
        xtot += T.xdoubles;
        nflags += (int)T.xoff.size();
      }
    }
    std::sort(bins[b].begin(), bins[b].end());
    for (int id : bins[b]) {
      const int g = isub[id];
      const size_t first = flat.size();
      flat.insert(flat.end(), s.chunks.begin() + s.sub_fc0[g], s.chunks.begin() + s.sub_fc1[g]);
      flat.insert(flat.end(), s.chunks.begin() + s.sub_bc0[g], s.chunks.begin() + s.sub_bc1[g]);
      flat[first].info |= SN_INFO_FIRST_ITEM;
      flat.back().info |= SN_INFO_LAST_ITEM;
      sub.push_back(g);
      c0.push_back(ic0[id]);
      ilo.push_back(0);
      ihi.push_back(s.sub_n[g]);
    }
    ptr[b + 1] = (int32_t)sub.size();
    cptr[b + 1] = (int64_t)flat.size();
  }
  wk.nblocks = isub.empty() ? 0 : nblocks;
  wk.item_ptr = up(A, ptr, st, setup_only);
  wk.item_sub = up(A, sub, st, setup_only);
  wk.item_c0 = up(A, c0, st, setup_only);
  wk.chunk_ptr = up(A, cptr, st, setup_only);
  wk.chunks = up(A, flat, st, setup_only);
  wk.xg = nullptr;
  wk.xg_stride = 0;
  wk.max_w = s.max_w;
  wk.split = nsplit > 0;
  wk.team = max_team;
  wk.nteams = nsplit;
  if (wk.split) {
    wk.item_lo = up(A, ilo, st, setup_only);
    wk.item_hi = up(A, ihi, st, setup_only);
    wk.xbuf = (double*)A.alloc(std::max<int64_t>(xtot, 2) * 8, setup_only);
    wk.xflag = (int32_t*)A.alloc(std::max(nflags, 1) * 4, setup_only);
    SN_CK(cudaMemsetAsync(wk.xflag, 0, std::max(nflags, 1) * 4, st));
  }
  if (xg && wk.nblocks > 0) {
    wk.xg_stride = sn_xg_stride(s.max_n, nrhs);
    wk.xg = (double*)A.alloc((size_t)wk.nblocks * wk.xg_stride * 8, setup_only);
  }
}

void sn_upload(SnBatch& B, DevAlloc& A, cudaStream_t st, int nsm) {
  const SnSymbolic& s = B.sym;
  B.d_sub_n = up(A, s.sub_n, st);
  B.d_sub_base = up(A, s.sub_base, st);
  B.d_sub_fc0 = up(A, s.sub_fc0, st);
  B.d_sub_fc1 = up(A, s.sub_fc1, st);
  B.d_sub_bc0 = up(A, s.sub_bc0, st);
  B.d_sub_bc1 = up(A, s.sub_bc1, st);
  B.d_gmap = up(A, s.gmap, st);
  B.d_lidx = up(A, s.lidx, st);
  B.d_sn_w = up(A, s.sn_w, st);
  B.d_sn_r = up(A, s.sn_r, st);
  B.d_sn_p0 = up(A, s.sn_p0, st);
  B.d_sn_ldw = up(A, s.sn_ldw, st);
  B.d_sn_ldf = up(A, s.sn_ldf, st);
  B.d_sn_rows_off = up(A, s.sn_rows_off, st);
  B.d_rows = up(A, s.rows, st);
  B.factor = (double*)A.alloc(std::max<int64_t>(s.factor_doubles, 2) * 8, false);
  // zero padding rows (ld is even; the solve reads row pairs)
  SN_CK(cudaMemsetAsync(B.factor, 0, std::max<int64_t>(s.factor_doubles, 2) * 8, st));
  B.n_loc = s.sub_base.empty() ? 0 : s.sub_base.back() + s.sub_n.back();
  B.yloc = (double*)A.alloc(std::max<int64_t>(B.n_loc, 1) * 8, false);
  B.dev.sub_n = B.d_sub_n;
  B.dev.sub_base = B.d_sub_base;
  B.dev.sub_fc0 = B.d_sub_fc0;
  B.dev.sub_fc1 = B.d_sub_fc1;
  B.dev.sub_bc0 = B.d_sub_bc0;
  B.dev.sub_bc1 = B.d_sub_bc1;
  B.dev.gmap = B.d_gmap;
  B.dev.sn_w = B.d_sn_w;
  B.dev.sn_r = B.d_sn_r;
  B.dev.sn_p0 = B.d_sn_p0;
  B.dev.sn_ldw = B.d_sn_ldw;
  B.dev.sn_ldf = B.d_sn_ldf;
  B.dev.sn_rows_off = B.d_sn_rows_off;
  B.dev.rows = B.d_rows;
  B.dev.factor = B.factor;
  B.solve_bytes = 0;
  for (int64_t b : s.sub_fbytes) B.solve_bytes += b;
  sn_build_work(B, A, st, nsm, 1, nullptr, B.work, 0, true);
}

void sn_apply(const SnBatch& B, const double* in, cudaStream_t st) {
  SnIO io;
  io.mode = 0;
  io.in = in;
  io.out = B.yloc;
  launch_sn_solve(B.dev, io, B.work, 1, B.sym.max_n, B.sym.max_r, B.sym.chunk_doubles,
                  B.work.cons, st);
}

static int p_slot(int P) { return P == 4 ? 2 : (P == 2 ? 1 : 0); }

// The larger x_S of P columns forces the 16-warp x 1-CTA shape at cfg3
// (profiles/r02_ncu_sn_solve_nrhs4_cfg3.txt): latency-bound (barrier and
// shared-load stalls).  Measured, 4 load cases at cfg3: the whole block
// solve takes 0.703 s with the P = 4 / 2 solves and 0.734 s with one-column
// solves (P = 1, 8 x 2) -- so any shape is taken (HPLMM_MULTI_8X2_ONLY=1
// restricts P > 1 to the 8 x 2 shape).
int sn_multi_width(SnBatch& B, DevAlloc& A, cudaStream_t st, int nsm, int k) {
  static const bool any_shape = getenv("HPLMM_MULTI_8X2_ONLY") == nullptr;
  for (int P : {4, 2, 1}) {
    if (P > k && P > 1) continue;
    int& s = B.mstate[p_slot(P)];
    if (s == 0) {
      try {
        SnWork& wk = B.mwork[p_slot(P)];
        sn_build_work(B, A, st, nsm, P, nullptr, wk);
        s = (P == 1 || wk.cons == 8 || any_shape) ? 1 : -1;
      } catch (const SnError&) {
        s = -1;
      }
    }
    if (s == 1) return P;
  }
  return 0;
}

void sn_apply_multi(const SnBatch& B, int P, const double* in, int64_t ldin, int ncols, double* out,
                    cudaStream_t st) {
  SnIO io;
  io.mode = 2;
  io.in = in;
  io.ldin = ldin;
  io.ncols = ncols;
  io.out = out;
  const SnWork& wk = B.mwork[p_slot(P)];
  launch_sn_solve(B.dev, io, wk, P, B.sym.max_n, B.sym.max_r, B.sym.chunk_doubles, wk.cons, st);
}

// ---------------------------------------------------------------------------
// numeric factorisation
// ---------------------------------------------------------------------------
void sn_factor(SnBatch& B, const double* d_val, DevAlloc& A, cudaStream_t st, int64_t pool_budget) {
  const SnSymbolic& s = B.sym;
  if (s.nsn == 0) return;
  SnNum nm;
  nm.asm_ptr = up(A, s.asm_ptr, st, true);
  nm.asm_e = up(A, s.asm_e, st, true);
  nm.asm_u = up(A, s.asm_u, st, true);
  nm.asm_v = up(A, s.asm_v, st, true);
  nm.sn_w = B.d_sn_w;
  nm.sn_r = B.d_sn_r;
  nm.sn_parent = up(A, s.sn_parent, st, true);
  nm.sn_ldw = B.d_sn_ldw;
  nm.sn_ldf = B.d_sn_ldf;
  nm.sn_foff = up(A, s.sn_foff, st, true);
  nm.rel_off = up(A, s.rel_off, st, true);
  nm.rel = up(A, s.rel, st, true);
  nm.rows_off = B.d_sn_rows_off;
  nm.rows = B.d_rows;
  launch_rows_to_factor(s.nsn, nm, B.factor, st);
  int64_t* d_front_off = (int64_t*)A.alloc((size_t)s.nsn * 8, true);
  nm.front_off = d_front_off;

  // waves of consecutive subdomains whose fronts fit the pool budget
  std::vector<int64_t> fbytes(s.nsub, 0);
  for (int g = 0; g < s.nsub; ++g)
    for (int k = s.sub_sn0[g]; k < s.sub_sn1[g]; ++k) {
      int64_t h = s.sn_w[k] + s.sn_r[k];
      fbytes[g] += h * h * 8;
    }
  std::vector<std::pair<int, int>> waves;
  int64_t maxwave = 0;
  for (int g0 = 0; g0 < s.nsub;) {
    int64_t tot = 0;
    int g1 = g0;
    while (g1 < s.nsub && (g1 == g0 || tot + fbytes[g1] <= pool_budget)) tot += fbytes[g1++];
    waves.push_back({g0, g1});
    maxwave = std::max(maxwave, tot);
    g0 = g1;
  }
  double* pool = (double*)A.alloc(std::max<int64_t>(maxwave, 8), true);
  nm.pool = pool;

  // per-level scratch sizes (max over waves)
  std::vector<int64_t> front_off(s.nsn, 0);
  int64_t max_list = 1, max_tiles = 1, max_rows = 1, max_work = 1;
  for (auto& wv : waves) {
    std::vector<int64_t> ntl(s.n_levels, 0), nrw(s.n_levels, 0), nls(s.n_levels, 0), nwk(s.n_levels, 0);
    for (int k = s.sub_sn0[wv.first]; k < s.sub_sn1[wv.second - 1]; ++k) {
      int L = s.sn_level[k];
      int nb = (s.sn_w[k] + TB - 1) / TB;
      ntl[L] += (int64_t)nb * (nb + 1) / 2;
      nrw[L] += nb;
      nls[L]++;
      int64_t tr = (s.sn_r[k] + 63) / 64, tw = (s.sn_w[k] + 63) / 64;
      nwk[L] += std::max(tr * tw, tr * tr);
    }
    for (int L = 0; L < s.n_levels; ++L) {
      max_list = std::max(max_list, nls[L]);
      max_tiles = std::max(max_tiles, ntl[L]);
      max_rows = std::max(max_rows, nrw[L]);
      max_work = std::max(max_work, nwk[L]);
    }
  }
  DevBatch lb;
  lb.tiles = (double*)A.alloc((size_t)max_tiles * TILE * 8, true);
  lb.dinv = (double*)A.alloc((size_t)max_list * TILE * SWEEP_M * SWEEP_M * 8, true);
  lb.cbuf = (double*)A.alloc((size_t)max_rows * TILE * SWEEP_M * 8, true);
  lb.wbuf = (double*)A.alloc((size_t)max_rows * TILE * SWEEP_M * 8, true);
  lb.err = (int32_t*)A.alloc(4, true);
  int32_t* d_nb = (int32_t*)A.alloc(max_list * 4, true);
  int32_t* d_ndof = (int32_t*)A.alloc(max_list * 4, true);
  int64_t* d_tile_base = (int64_t*)A.alloc(max_list * 8, true);
  int64_t* d_row_base = (int64_t*)A.alloc(max_list * 8, true);
  int32_t* d_tile_s = (int32_t*)A.alloc(max_tiles * 4, true);
  int32_t* d_tile_ij = (int32_t*)A.alloc(max_tiles * 4, true);
  int32_t* d_row_s = (int32_t*)A.alloc(max_rows * 4, true);
  int32_t* d_row_k = (int32_t*)A.alloc(max_rows * 4, true);
  int32_t* d_list = (int32_t*)A.alloc(max_list * 4, true);
  int32_t* d_clist = (int32_t*)A.alloc(max_list * 4 * std::max(1, s.max_children), true);
  GemmProb* d_probs = (GemmProb*)A.alloc(max_list * sizeof(GemmProb), true);
  int32_t* d_work = (int32_t*)A.alloc(max_work * 12, true);

  auto h2d = [&](void* dst, const void* src, size_t bytes) {
    if (bytes) SN_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
  };
  for (auto& wv : waves) {
    const int k0 = s.sub_sn0[wv.first], k1 = s.sub_sn1[wv.second - 1];
    int64_t off = 0;
    for (int k = k0; k < k1; ++k) {
      front_off[k] = off;
      int64_t h = s.sn_w[k] + s.sn_r[k];
      off += h * h;
    }
    h2d(d_front_off + k0, front_off.data() + k0, (size_t)(k1 - k0) * 8);
    SN_CK(cudaMemsetAsync(pool, 0, (size_t)std::max<int64_t>(off, 1) * 8, st));
    for (int L = 0; L < s.n_levels; ++L) {
      std::vector<int32_t> list;
      for (int k = k0; k < k1; ++k)
        if (s.sn_level[k] == L) list.push_back(k);
      if (list.empty()) continue;
      const int nl = (int)list.size();
      h2d(d_list, list.data(), nl * 4);
      launch_front_asm(d_list, nl, nm, d_val, st);
      for (int rank = 0; rank < s.max_children; ++rank) {
        std::vector<int32_t> cl;
        for (int k = k0; k < k1; ++k)
          if (s.sn_parent[k] >= 0 && s.sn_child_rank[k] == rank && s.sn_level[s.sn_parent[k]] == L)
            cl.push_back(k);
        if (cl.empty()) continue;
        int32_t* dcl = d_clist + (size_t)rank * max_list;
        h2d(dcl, cl.data(), cl.size() * 4);
        launch_front_ext(dcl, (int)cl.size(), nm, st);
      }
      // F_SS^-1 by the packed-tile sweep (SPD, no pivoting)
      std::vector<int32_t> nb(nl), nd(nl), tile_s, tile_ij, row_s, row_k;
      std::vector<int64_t> tile_base(nl), row_base(nl);
      int64_t nt = 0, nr = 0;
      int maxnb = 0, maxw = 0;
      for (int i = 0; i < nl; ++i) {
        nd[i] = s.sn_w[list[i]];
        nb[i] = (nd[i] + TB - 1) / TB;
        maxnb = std::max(maxnb, nb[i]);
        maxw = std::max(maxw, nd[i]);
        tile_base[i] = nt;
        row_base[i] = nr;
        for (int I = 0; I < nb[i]; ++I) {
          row_s.push_back(i);
          row_k.push_back(I);
          for (int J = 0; J <= I; ++J) {
            tile_s.push_back(i);
            tile_ij.push_back((I << 16) | J);
          }
        }
        nt += (int64_t)nb[i] * (nb[i] + 1) / 2;
        nr += nb[i];
      }
      h2d(d_nb, nb.data(), nl * 4);
      h2d(d_ndof, nd.data(), nl * 4);
      h2d(d_tile_base, tile_base.data(), nl * 8);
      h2d(d_row_base, row_base.data(), nl * 8);
      h2d(d_tile_s, tile_s.data(), tile_s.size() * 4);
      h2d(d_tile_ij, tile_ij.data(), tile_ij.size() * 4);
      h2d(d_row_s, row_s.data(), row_s.size() * 4);
      h2d(d_row_k, row_k.data(), row_k.size() * 4);
      lb.nsub = nl;
      lb.max_nb = maxnb;
      lb.ntiles = nt;
      lb.nrows = nr;
      lb.nb = d_nb;
      lb.ndof = d_ndof;
      lb.tile_base = d_tile_base;
      lb.row_base = d_row_base;
      lb.tile_s = d_tile_s;
      lb.tile_ij = d_tile_ij;
      lb.row_s = d_row_s;
      lb.row_k = d_row_k;
      int32_t big = INT_MAX;
      h2d(lb.err, &big, 4);
      launch_front_to_tiles(lb, d_list, nm, st);
      launch_pad_identity(lb, st);
      launch_sweep_invert(lb, st);
      launch_tiles_to_finv(lb, d_list, nl, maxw, nm, B.factor, st);
      SN_CK(cudaGetLastError());
      int32_t bad = INT_MAX;
      SN_CK(cudaMemcpyAsync(&bad, lb.err, 4, cudaMemcpyDeviceToHost, st));
      SN_CK(cudaStreamSynchronize(st));
      if (bad != INT_MAX)
        throw SnError{-4, "non-positive pivot in the supernodal factor of local subdomain",
                      s.sn_sub[list[bad]]};
      // W = F_RS F_SS^-1 ; F_RR -= W F_RS^T
      for (int phase = 0; phase < 2; ++phase) {
        std::vector<GemmProb> probs;
        std::vector<int32_t> work;
        for (int i = 0; i < nl; ++i) {
          const int k = list[i];
          const int w = s.sn_w[k], r = s.sn_r[k], h = w + r;
          if (r == 0) continue;
          double* F = pool + front_off[k];
          double* W = B.factor + s.sn_foff[k] + sn_rows_doubles(r);
          const double* Fi = W + (int64_t)s.sn_ldw[k] * w;
          GemmProb g;
          if (phase == 0) {
            g = GemmProb{F + w, Fi, W, r, w, w, h, s.sn_ldf[k], s.sn_ldw[k], 1.0, 0.0, 0, 0};
          } else {
            g = GemmProb{W, F + w, F + w + (int64_t)w * h, r, r, w, s.sn_ldw[k], h, h, -1.0, 1.0, 1, 0};
          }
          const int p = (int)probs.size();
          probs.push_back(g);
          for (int ti = 0; ti < (g.m + 63) / 64; ++ti)
            for (int tj = 0; tj < (g.n + 63) / 64; ++tj) {
              work.push_back(p);
              work.push_back(ti);
              work.push_back(tj);
            }
        }
        if (probs.empty()) continue;
        h2d(d_probs, probs.data(), probs.size() * sizeof(GemmProb));
        h2d(d_work, work.data(), work.size() * 4);
        launch_gemm_batched(d_probs, d_work, (int)(work.size() / 3), st);
        SN_CK(cudaGetLastError());
      }
    }
  }
  SN_CK(cudaStreamSynchronize(st));
}

// shape vectors B_g = -A_g^-1 R_g (eq:col_pk) through the supernodal factor,
// as a level-3 multi-RHS sweep: step t handles the t-th supernode (postorder)
// of every grain at once with batched GEMMs
//   forward : T = W_S X_S ; X_R -= T ; T = F_SS^-1 X_S ; X_S = T
//   backward: T = X_R ; X_S -= W_S^T T
// (sequential within a grain, so deterministic; all k_g columns at once).
void sn_shape_vectors(SnBatch& B, DevAlloc& A, cudaStream_t st, int nsm,
                      const std::vector<int32_t>& kcols, const int64_t* d_b_off,
                      const int32_t* d_ld, double* R, double* Bout, int64_t rb_doubles) {
  (void)nsm;
  const SnSymbolic& s = B.sym;
  const int G = s.nsub;
  std::vector<int64_t> xoff(G, 0);
  int64_t xtot = 0, tmax = 0;
  int maxsteps = 0;
  for (int g = 0; g < G; ++g) {
    xoff[g] = xtot;
    xtot += (int64_t)s.sub_n[g] * kcols[g];
    maxsteps = std::max(maxsteps, s.sub_sn1[g] - s.sub_sn0[g]);
  }
  if (xtot == 0) return;
  // X (elimination order, n x k per grain) lives in R's memory: R is first
  // copied into B's storage (same row layout; its zero padding rows and zero
  // correction column are what B needs there), X is gathered from that copy,
  // and the result is written back into B with the sign of eq:col_pk
  if (xtot > rb_doubles) throw SnError{-1, "shape-vector workspace larger than R"};
  SN_CK(cudaMemcpyAsync(Bout, R, (size_t)rb_doubles * 8, cudaMemcpyDeviceToDevice, st));
  double* X = R;
  // temporaries: per grain max_S h_S x k_g, reused by every step
  std::vector<int64_t> toff(G, 0);
  for (int g = 0; g < G; ++g) {
    int hmax = 0;
    for (int k = s.sub_sn0[g]; k < s.sub_sn1[g]; ++k) hmax = std::max(hmax, std::max(s.sn_w[k], s.sn_r[k]));
    toff[g] = tmax;
    tmax += (int64_t)hmax * kcols[g];
  }
  double* T = (double*)A.alloc((size_t)std::max<int64_t>(tmax, 1) * 8, true);
  int32_t* d_p0 = B.d_sn_p0;
  SnNum nm;
  nm.sn_w = B.d_sn_w;
  nm.sn_r = B.d_sn_r;
  nm.rows = B.d_rows;
  nm.rows_off = B.d_sn_rows_off;

  // items: one per grain for IO, one per (grain, supernode) per step
  std::vector<SnMrItem> io_items, items;
  std::vector<int64_t> step_ptr(maxsteps + 1, 0);
  for (int g = 0; g < G; ++g)
    if (kcols[g] > 0) io_items.push_back(SnMrItem{g, -1, s.sub_n[g], kcols[g], s.sub_base[g], xoff[g], 0});
  for (int t = 0; t < maxsteps; ++t) {
    for (int g = 0; g < G; ++g) {
      const int k = s.sub_sn0[g] + t;
      if (kcols[g] == 0 || k >= s.sub_sn1[g]) continue;
      items.push_back(SnMrItem{g, k, s.sub_n[g], kcols[g], s.sub_base[g], xoff[g], toff[g]});
    }
    step_ptr[t + 1] = (int64_t)items.size();
  }
  SnMrItem* d_io = up(A, io_items, st, true);
  SnMrItem* d_items = up(A, items, st, true);
  // GEMM problems per item: 0 = W X_S, 1 = F^-1 X_S, 2 = X_S -= W^T T
  std::vector<GemmProb> probs(items.size() * 3);
  for (size_t q = 0; q < items.size(); ++q) {
    const SnMrItem& m = items[q];
    const int k = m.sn, w = s.sn_w[k], r = s.sn_r[k];
    const double* W = B.factor + s.sn_foff[k] + sn_rows_doubles(r);
    const double* F = W + (int64_t)s.sn_ldw[k] * w;
    double* XS = X + m.xoff + s.sn_p0[k];
    double* Tm = T + m.toff;
    probs[3 * q + 0] = GemmProb{W, XS, Tm, r, m.k, w, s.sn_ldw[k], m.n, std::max(r, 1), 1.0, 0.0, 0, 0};
    probs[3 * q + 1] = GemmProb{F, XS, Tm, w, m.k, w, s.sn_ldf[k], m.n, w, 1.0, 0.0, 0, 0};
    // X_S -= W_S^T T  (transA)
    probs[3 * q + 2] = GemmProb{W, Tm, XS, w, m.k, r, s.sn_ldw[k], std::max(r, 1), m.n, -1.0, 1.0, 0, 1};
  }
  GemmProb* d_probs = up(A, probs, st, true);
  // tile work lists per (step, kind)
  std::vector<int32_t> work;
  std::vector<int64_t> wptr;   // [(t * 3 + kind) + 1]
  wptr.push_back(0);
  for (int t = 0; t < maxsteps; ++t)
    for (int kind = 0; kind < 3; ++kind) {
      for (int64_t q = step_ptr[t]; q < step_ptr[t + 1]; ++q) {
        const GemmProb& gp = probs[3 * q + kind];
        if (gp.m == 0 || gp.n == 0 || gp.k == 0) continue;
        for (int ti = 0; ti < (gp.m + 63) / 64; ++ti)
          for (int tj = 0; tj < (gp.n + 63) / 64; ++tj) {
            work.push_back((int32_t)(3 * q + kind));
            work.push_back(ti);
            work.push_back(tj);
          }
      }
      wptr.push_back((int64_t)work.size() / 3);
    }
  int32_t* d_work = up(A, work, st, true);
  auto gemm = [&](int t, int kind) {
    const int64_t a = wptr[t * 3 + kind], b = wptr[t * 3 + kind + 1];
    if (b > a) launch_gemm_batched(d_probs, d_work + 3 * a, (int)(b - a), st);
  };
  launch_mr_io((int)io_items.size(), d_io, B.d_lidx, d_b_off, d_ld, Bout, X, nullptr, 1, st);
  for (int t = 0; t < maxsteps; ++t) {
    const int n = (int)(step_ptr[t + 1] - step_ptr[t]);
    const SnMrItem* it = d_items + step_ptr[t];
    gemm(t, 0);                                        // T = W_S X_S
    launch_mr_rows(n, it, nm, d_p0, X, T, 0, st);      // X_R -= T
    gemm(t, 1);                                        // T = F^-1 X_S
    launch_mr_rows(n, it, nm, d_p0, X, T, 2, st);      // X_S = T
  }
  for (int t = maxsteps - 1; t >= 0; --t) {
    const int n = (int)(step_ptr[t + 1] - step_ptr[t]);
    const SnMrItem* it = d_items + step_ptr[t];
    launch_mr_rows(n, it, nm, d_p0, X, T, 1, st);      // T = X_R
    gemm(t, 2);                                        // X_S -= W^T T
  }
  launch_mr_io((int)io_items.size(), d_io, B.d_lidx, d_b_off, d_ld, nullptr, X, Bout, 0, st);
  SN_CK(cudaGetLastError());
}

}  // namespace hplmm
