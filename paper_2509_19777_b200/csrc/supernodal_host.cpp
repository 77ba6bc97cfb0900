// Host symbolic analysis of the batched supernodal local factors (see
// supernodal.h): geometric nested dissection per subdomain, supernode row
// structures, factor layout, TMA chunk schedule, numeric assembly maps.
// Subdomains are analysed in parallel (std::thread) and concatenated in order,
// so the result is deterministic.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <thread>

#include "supernodal.h"

namespace hplmm {

namespace {

struct LocalSn {
  std::vector<int32_t> members;   // local node ids (ascending)
  int parent = -1;
};

struct SubResult {
  bool ok = true;
  std::string err;
  int n_nodes = 0;
  std::vector<int32_t> order;                       // local node ids in elimination order
  std::vector<LocalSn> sns;                         // postorder
  std::vector<std::vector<int32_t>> st;             // struct (node positions) per supernode
  std::vector<int32_t> level;
  // assembly entries per supernode
  std::vector<std::vector<int64_t>> ae;
  std::vector<std::vector<int32_t>> au, av;
  std::vector<std::vector<int32_t>> rel;            // per supernode (as child)
};

// separator choice (HPLMM_SN_SEP: 0 = median plane of the longest axis,
// 1 = fewest-node balanced plane, default); HPLMM_SN_SEPBAL = balance bound (%)
int sep_mode() {
  static const int v = getenv("HPLMM_SN_SEP") ? atoi(getenv("HPLMM_SN_SEP")) : 1;
  return v;
}
int sep_bal() {
  static const int v = getenv("HPLMM_SN_SEPBAL") ? atoi(getenv("HPLMM_SN_SEPBAL")) : 42;
  return v;
}
#define SEP_BAL sep_bal()

class NdBuilder {
 public:
  NdBuilder(const int32_t* ijk, const std::vector<int32_t>& gnodes, int leaf)
      : ijk_(ijk), g_(gnodes), leaf_(leaf) {}
  std::vector<LocalSn> sns;

  // returns the roots of the subtree built over `ids` (local node ids)
  std::vector<int> build(std::vector<int32_t> ids) {
    if (ids.empty()) return {};
    int lo[3], hi[3];
    for (int c = 0; c < 3; ++c) { lo[c] = INT32_MAX; hi[c] = INT32_MIN; }
    for (int a : ids)
      for (int c = 0; c < 3; ++c) {
        int v = ijk_[3 * (int64_t)g_[a] + c];
        lo[c] = std::min(lo[c], v);
        hi[c] = std::max(hi[c], v);
      }
    int ax = 0;
    for (int c = 1; c < 3; ++c)
      if (hi[c] - lo[c] > hi[ax] - lo[ax]) ax = c;
    if ((int)ids.size() <= leaf_ || hi[ax] - lo[ax] < 2) return {leaf(std::move(ids))};
    int m = 0;
    if (sep_mode() == 0) {   // r01: median plane of the longest axis
      std::vector<int> vals(ids.size());
      for (size_t i = 0; i < ids.size(); ++i) vals[i] = ijk_[3 * (int64_t)g_[ids[i]] + ax];
      std::vector<int> sorted = vals;
      std::nth_element(sorted.begin(), sorted.begin() + sorted.size() / 2, sorted.end());
      m = sorted[sorted.size() / 2];
      m = std::max(lo[ax] + 1, std::min(hi[ax] - 1, m));
    } else {
      // r02: over every axis whose extent is at least half the longest, the
      // lattice plane with the fewest nodes among those leaving at least
      // SEP_BAL of the nodes on each side (a porous subdomain's planes differ
      // in solid fraction; a smaller separator means less fill: fewer factor
      // bytes and smaller fronts); ties -> longer axis, then nearer the median
      const int64_t N = (int64_t)ids.size();
      const int ax0 = ax;
      int64_t best = INT64_MAX, best_dev = INT64_MAX;
      for (int c = 0; c < 3; ++c) {
        if (hi[c] - lo[c] < 2 || 2 * (hi[c] - lo[c]) < hi[ax0] - lo[ax0]) continue;
        std::vector<int64_t> cnt(hi[c] - lo[c] + 1, 0);
        for (int a : ids) cnt[ijk_[3 * (int64_t)g_[a] + c] - lo[c]]++;
        int64_t below = 0;
        for (int v = 0; v <= hi[c] - lo[c]; ++v) {
          const int64_t above = N - below - cnt[v];
          if (v >= 1 && v <= hi[c] - lo[c] - 1 && below * 100 >= SEP_BAL * N && above * 100 >= SEP_BAL * N) {
            const int64_t dev = std::llabs(2 * below + cnt[v] - N);
            const int64_t score = cnt[v];
            if (score < best || (score == best && c == ax0 && dev < best_dev)) {
              best = score;
              best_dev = dev;
              ax = c;
              m = lo[c] + v;
            }
          }
          below += cnt[v];
        }
      }
      if (best == INT64_MAX) {   // no plane meets the balance bound: median
        std::vector<int> vals(ids.size());
        for (size_t i = 0; i < ids.size(); ++i) vals[i] = ijk_[3 * (int64_t)g_[ids[i]] + ax];
        std::nth_element(vals.begin(), vals.begin() + vals.size() / 2, vals.end());
        m = std::max(lo[ax] + 1, std::min(hi[ax] - 1, vals[vals.size() / 2]));
      }
    }
    std::vector<int> vals(ids.size());
    for (size_t i = 0; i < ids.size(); ++i) vals[i] = ijk_[3 * (int64_t)g_[ids[i]] + ax];
    std::vector<int32_t> L, R, S;
    for (size_t i = 0; i < ids.size(); ++i)
      (vals[i] < m ? L : (vals[i] > m ? R : S)).push_back(ids[i]);
    std::vector<int> roots = build(std::move(L));
    std::vector<int> rr = build(std::move(R));
    roots.insert(roots.end(), rr.begin(), rr.end());
    if (S.empty()) return roots;   // halves are not coupled: a forest
    int s = leaf(std::move(S));
    for (int c : roots) sns[c].parent = s;
    return {s};
  }

 private:
  int leaf(std::vector<int32_t> ids) {
    std::sort(ids.begin(), ids.end());
    sns.push_back(LocalSn{std::move(ids), -1});
    return (int)sns.size() - 1;
  }
  const int32_t* ijk_;
  const std::vector<int32_t>& g_;
  int leaf_;
};

void analyse_one(const HostSetup& hs, const int32_t* gn, int m, int leaf, std::vector<int32_t>& g2l,
                 SubResult& res) {
  std::vector<int32_t> gnodes(gn, gn + m);
  for (int a = 0; a < m; ++a) g2l[gnodes[a]] = a;
  // local adjacency (includes self)
  std::vector<int32_t> aptr(m + 1, 0), adj;
  std::vector<int64_t> aeidx;
  for (int a = 0; a < m; ++a) {
    int v = gnodes[a];
    for (int e = hs.row_ptr[v]; e < hs.row_ptr[v + 1]; ++e) {
      int l = g2l[hs.col_idx[e]];
      if (l >= 0) {
        adj.push_back(l);
        aeidx.push_back(e);
      }
    }
    aptr[a + 1] = (int32_t)adj.size();
  }
  NdBuilder nd(hs.node_ijk.data(), gnodes, leaf);
  std::vector<int32_t> all(m);
  std::iota(all.begin(), all.end(), 0);
  nd.build(all);
  res.sns = std::move(nd.sns);
  const int ns = (int)res.sns.size();
  std::vector<int32_t> pos(m), first(ns), last(ns);
  int p = 0;
  for (int s = 0; s < ns; ++s) {
    first[s] = p;
    for (int a : res.sns[s].members) {
      pos[a] = p++;
      res.order.push_back(a);
    }
    last[s] = p - 1;
  }
  res.n_nodes = m;
  std::vector<std::vector<int>> kids(ns);
  for (int s = 0; s < ns; ++s)
    if (res.sns[s].parent >= 0) kids[res.sns[s].parent].push_back(s);
  res.st.assign(ns, {});
  res.level.assign(ns, 0);
  res.ae.assign(ns, {});
  res.au.assign(ns, {});
  res.av.assign(ns, {});
  res.rel.assign(ns, {});
  for (int s = 0; s < ns; ++s) {
    std::vector<int32_t> st;
    for (int a : res.sns[s].members)
      for (int e = aptr[a]; e < aptr[a + 1]; ++e)
        if (pos[adj[e]] > last[s]) st.push_back(pos[adj[e]]);
    int lev = 0;
    for (int c : kids[s]) {
      for (int q : res.st[c])
        if (q > last[s]) st.push_back(q);
      lev = std::max(lev, res.level[c] + 1);
    }
    std::sort(st.begin(), st.end());
    st.erase(std::unique(st.begin(), st.end()), st.end());
    res.st[s] = std::move(st);
    res.level[s] = lev;
    if (3 * (int)res.sns[s].members.size() > SN_MAX_WR || 3 * (int)res.st[s].size() > SN_MAX_WR) {
      res.ok = false;
      res.err = "supernode wider than " + std::to_string(SN_MAX_WR) + " DOFs";
      break;
    }
    // front node index of a position q (member or struct row)
    auto fidx = [&](int q) -> int {
      if (q >= first[s] && q <= last[s]) return q - first[s];
      auto it = std::lower_bound(res.st[s].begin(), res.st[s].end(), q);
      if (it == res.st[s].end() || *it != q) return -1;
      return (int)res.sns[s].members.size() + (int)(it - res.st[s].begin());
    };
    for (int a : res.sns[s].members)
      for (int e = aptr[a]; e < aptr[a + 1]; ++e) {
        int q = pos[adj[e]];
        if (q < pos[a]) continue;
        res.ae[s].push_back(aeidx[e]);
        res.au[s].push_back(fidx(q));
        res.av[s].push_back(fidx(pos[a]));
      }
    for (int c : kids[s])
      for (int q : res.st[c]) {
        int f = fidx(q);
        if (f < 0) {
          res.ok = false;
          res.err = "supernodal structure not closed under the elimination tree";
          break;
        }
        res.rel[c].push_back(f);
      }
  }
  for (int a = 0; a < m; ++a) g2l[gnodes[a]] = -1;
}

}  // namespace

int sn_chunk_doubles() {
  static int v = [] {
    const char* e = getenv("HPLMM_SN_CHUNK");
    int c = e ? atoi(e) : 4096;
    // >= 2048: the group-reduction scratch of the solve (8 x consumer threads
    // doubles) lives in one stage; 16-warp CTAs need 4096 (sn_solve_cfg)
    if (c < 2048) c = 2048;
    c &= ~1;
    if (c > SN_CHUNK_DOUBLES_MAX) c = SN_CHUNK_DOUBLES_MAX;
    return c;
  }();
  return v;
}

bool sn_analyse(const HostSetup& hs, const std::vector<int32_t>& ptr,
                const std::vector<int32_t>& nodes, int leaf, SnSymbolic& o, std::string& err, int nsm, int shape,
                int xg_mode) {
  const int nsub = (int)ptr.size() - 1;
  std::vector<SubResult> res(std::max(nsub, 0));
  unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::atomic<int> next{0};
  auto work = [&]() {
    std::vector<int32_t> g2l(hs.n_nodes, -1);
    for (int s; (s = next.fetch_add(1)) < nsub;)
      analyse_one(hs, nodes.data() + ptr[s], ptr[s + 1] - ptr[s], leaf, g2l, res[s]);
  };
  static const bool dbg = getenv("HPLMM_DEBUG") != nullptr;
  auto now = [] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t0 = now();
  std::vector<std::thread> th;
  for (unsigned t = 0; t + 1 < nth; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  const double t1 = now();

  o = SnSymbolic();
  o.nsub = nsub;
  for (int s = 0; s < nsub; ++s)
    if (!res[s].ok) {
      err = "subdomain " + std::to_string(s) + ": " + res[s].err;
      return false;
    }
  // pass 1 (serial, per subdomain): offsets of every concatenated array
  std::vector<int64_t> o_loc(nsub + 1, 0), o_sn(nsub + 1, 0), o_rows(nsub + 1, 0),
      o_asm(nsub + 1, 0), o_rel(nsub + 1, 0), o_f(nsub + 1, 0);
  for (int s = 0; s < nsub; ++s) {
    const SubResult& r = res[s];
    int64_t nr = 0, na = 0, nl = 0, nf = 0;
    for (size_t k = 0; k < r.sns.size(); ++k) {
      const int w = 3 * (int)r.sns[k].members.size(), rr = 3 * (int)r.st[k].size();
      nr += rr;
      na += (int64_t)r.ae[k].size();
      nl += (int64_t)r.rel[k].size();
      nf += sn_rows_doubles(rr) + (int64_t)(rr + (rr & 1)) * w + (int64_t)(w + (w & 1)) * w;
    }
    o_loc[s + 1] = o_loc[s] + 3 * (int64_t)r.n_nodes;
    o_sn[s + 1] = o_sn[s] + (int64_t)r.sns.size();
    o_rows[s + 1] = o_rows[s] + nr;
    o_asm[s + 1] = o_asm[s] + na;
    o_rel[s + 1] = o_rel[s] + nl;
    o_f[s + 1] = o_f[s] + nf;
  }
  const int64_t NS = o_sn[nsub];
  o.nsn = (int)NS;
  o.sub_n.resize(nsub);
  o.sub_base.resize(nsub);
  o.sub_sn0.resize(nsub);
  o.sub_sn1.resize(nsub);
  o.gmap.resize(o_loc[nsub]);
  o.lidx.resize(o_loc[nsub]);
  o.rows.resize(o_rows[nsub]);
  o.asm_e.resize(o_asm[nsub]);
  o.asm_u.resize(o_asm[nsub]);
  o.asm_v.resize(o_asm[nsub]);
  o.rel.resize(o_rel[nsub]);
  for (auto* v : {&o.sn_w, &o.sn_r, &o.sn_p0, &o.sn_ldw, &o.sn_ldf, &o.sn_level, &o.sn_parent,
                  &o.sn_sub, &o.sn_child_rank})
    v->resize(NS);
  o.sn_rows_off.resize(NS);
  o.sn_foff.resize(NS);
  o.asm_ptr.resize(NS + 1);
  o.rel_off.resize(NS + 1);
  o.asm_ptr[0] = 0;
  o.rel_off[0] = 0;
  // pass 2 (parallel over subdomains): fill
  std::atomic<int> next2{0};
  auto fill = [&]() {
    for (int s; (s = next2.fetch_add(1)) < nsub;) {
      SubResult& r = res[s];
      const int sn0 = (int)o_sn[s];
      o.sub_n[s] = 3 * r.n_nodes;
      o.sub_base[s] = o_loc[s];
      o.sub_sn0[s] = sn0;
      o.sub_sn1[s] = (int)o_sn[s + 1];
      const int32_t* gn = nodes.data() + ptr[s];
      int64_t t = o_loc[s];
      for (int a : r.order)
        for (int c = 0; c < 3; ++c, ++t) {
          o.gmap[t] = 3 * gn[a] + c;
          o.lidx[t] = 3 * a + c;
        }
      int p0 = 0;
      int64_t roff = o_rows[s], aoff = o_asm[s], loff = o_rel[s], foff = o_f[s];
      std::vector<int> nchild(r.sns.size(), 0);
      for (size_t k = 0; k < r.sns.size(); ++k) {
        const int64_t g = sn0 + (int64_t)k;
        const int w = 3 * (int)r.sns[k].members.size(), rr = 3 * (int)r.st[k].size();
        o.sn_w[g] = w;
        o.sn_r[g] = rr;
        o.sn_p0[g] = p0;
        o.sn_ldw[g] = rr + (rr & 1);
        o.sn_ldf[g] = w + (w & 1);
        o.sn_level[g] = r.level[k];
        o.sn_parent[g] = r.sns[k].parent >= 0 ? sn0 + r.sns[k].parent : -1;
        o.sn_sub[g] = s;
        int rank = 0;
        if (r.sns[k].parent >= 0) rank = nchild[r.sns[k].parent]++;
        o.sn_child_rank[g] = rank;
        o.sn_rows_off[g] = roff;
        for (int q : r.st[k])
          for (int c = 0; c < 3; ++c) o.rows[roff++] = 3 * q + c;
        o.sn_foff[g] = foff;
        foff += sn_rows_doubles(rr) + (int64_t)o.sn_ldw[g] * w + (int64_t)o.sn_ldf[g] * w;
        p0 += w;
        std::copy(r.ae[k].begin(), r.ae[k].end(), o.asm_e.begin() + aoff);
        std::copy(r.au[k].begin(), r.au[k].end(), o.asm_u.begin() + aoff);
        std::copy(r.av[k].begin(), r.av[k].end(), o.asm_v.begin() + aoff);
        aoff += (int64_t)r.ae[k].size();
        o.asm_ptr[g + 1] = aoff;
        std::copy(r.rel[k].begin(), r.rel[k].end(), o.rel.begin() + loff);
        loff += (int64_t)r.rel[k].size();
        o.rel_off[g + 1] = loff;
      }
      r = SubResult();   // free
    }
  };
  {
    std::vector<std::thread> th2;
    for (unsigned t = 0; t + 1 < nth; ++t) th2.emplace_back(fill);
    fill();
    for (auto& t : th2) t.join();
  }
  for (int64_t g = 0; g < NS; ++g) {
    o.max_w = std::max(o.max_w, o.sn_w[g]);
    o.max_r = std::max(o.max_r, o.sn_r[g]);
    o.n_levels = std::max(o.n_levels, o.sn_level[g] + 1);
    o.max_children = std::max(o.max_children, o.sn_child_rank[g] + 1);
  }
  for (int s = 0; s < nsub; ++s) o.max_n = std::max(o.max_n, o.sub_n[s]);
  const int64_t foff = o_f[nsub];
  o.factor_doubles = foff;
  o.shape = shape;
  o.xg1 = sn_pick_xg(nsub, nsm, o.max_n, o.max_r, shape, o.max_w, xg_mode);
  o.chunk_doubles = sn_pick_chunk(nsub, nsm, o.max_n, o.max_r, shape, o.max_w, o.xg1);
  const double t2 = now();
  // TMA chunk schedule: forward = (W_S, rows, F_SS^-1) per S in postorder,
  // backward = (rows, W_S) per S in reverse postorder; W/F chunks are whole
  // columns of at most SN_CHUNK_DOUBLES.
  auto push = [&](int sn, int kind, int64_t off, int bytes, int c0, int nc, bool last,
                  bool rows_prefix = false) {
    SnChunk ch;
    ch.off = off;
    // thread-group size for the rows of this part: TG = pow2 >= max(64, ceil(h/8)),
    // so a thread holds up to 4 row pairs and the remaining threads take other
    // columns.  The floor 64 (r02; r01: 32) halves the column groups of the
    // small parts -- fewer partial sums to reduce at each part end: cfg3
    // contact / grain apply 1.834 / 1.270 -> 1.789 / 1.256 ms; 128 (G <= 2)
    // 1.875 / 1.292, 256 2.25 / 1.47 (HPLMM_SN_TGMIN = log2 floor)
    const int h = (kind == SN_F_FWD) ? o.sn_w[sn] : o.sn_r[sn];
    static const int lg0 = getenv("HPLMM_SN_TGMIN") ? atoi(getenv("HPLMM_SN_TGMIN")) : 6;
    static const int hdiv = getenv("HPLMM_SN_TGDIV") ? atoi(getenv("HPLMM_SN_TGDIV")) : 8;
    int lg = lg0;
    while ((1 << lg) < (h + hdiv - 1) / hdiv && lg < 9) ++lg;
    ch.bytes = bytes | ((lg - 5) << 24);
    ch.info = c0 | ((nc - 1) << 12) | (kind << 24) | (last ? SN_INFO_LAST : 0) |
              (rows_prefix ? SN_INFO_ROWS : 0);
    ch.p0 = o.sn_p0[sn];
    ch.w = o.sn_w[sn];
    ch.r = o.sn_r[sn];
    ch.sub = o.sn_sub[sn];
    o.chunks.push_back(ch);
  };
  // W_S / F_SS^-1 as whole-column chunks; a W part may take the supernode's row
  // list (stored right before W_S) into its first chunk (returns true then):
  // 21% of the chunks at cfg3 were row lists of ~0.6 KB, each a ring slot and a
  // consumer round trip of its own (HPLMM_SN_PACK=0: separate row chunks)
  static const bool pack_rows = !(getenv("HPLMM_SN_PACK") && getenv("HPLMM_SN_PACK")[0] == '0');
  auto cols = [&](int sn, int kind, int64_t off0, int ld, int ncols_total, int64_t rows_at = -1,
                  int rd = 0) {
    int c0 = 0;
    bool packed = false;
    if (rows_at >= 0 && pack_rows) {
      const int per1 = (o.chunk_doubles - rd) / ld;
      if (per1 >= 1) {
        const int nc = std::min(per1, ncols_total);
        push(sn, kind, rows_at, (rd + nc * ld) * 8, 0, nc, nc == ncols_total, true);
        c0 = nc;
        packed = true;
      }
    }
    const int per = std::max(1, o.chunk_doubles / ld);
    for (; c0 < ncols_total; c0 += per) {
      int nc = std::min(per, ncols_total - c0);
      push(sn, kind, off0 + (int64_t)c0 * ld, nc * ld * 8, c0, nc, c0 + nc == ncols_total);
    }
    return packed;
  };
  for (auto* v : {&o.sn_fcb, &o.sn_fce, &o.sn_bcb, &o.sn_bce}) v->assign(NS, 0);
  for (int s = 0; s < nsub; ++s) {
    int64_t fb = 0;
    o.sub_fc0.push_back((int64_t)o.chunks.size());
    for (int k = o.sub_sn0[s]; k < o.sub_sn1[s]; ++k) {
      const int w = o.sn_w[k], r = o.sn_r[k];
      o.sn_fcb[k] = (int64_t)o.chunks.size();
      const int64_t rows_at = o.sn_foff[k], w_at = rows_at + sn_rows_doubles(r);
      const int64_t f_at = w_at + (int64_t)o.sn_ldw[k] * w;
      if (r > 0) {
        if (!cols(k, SN_W_FWD, w_at, o.sn_ldw[k], w, rows_at, (int)sn_rows_doubles(r)))
          push(k, SN_ROWS_FWD, rows_at, (int)(8 * sn_rows_doubles(r)), 0, 1, true);
      }
      cols(k, SN_F_FWD, f_at, o.sn_ldf[k], w);
      o.sn_fce[k] = (int64_t)o.chunks.size();
      fb += 8 * (2 * sn_rows_doubles(r) + 2 * (int64_t)o.sn_ldw[k] * w + (int64_t)o.sn_ldf[k] * w);
    }
    o.sub_fc1.push_back((int64_t)o.chunks.size());
    o.sub_bc0.push_back((int64_t)o.chunks.size());
    for (int k = o.sub_sn1[s] - 1; k >= o.sub_sn0[s]; --k) {
      const int r = o.sn_r[k];
      o.sn_bcb[k] = o.sn_bce[k] = (int64_t)o.chunks.size();
      if (r == 0) continue;
      if (pack_rows && (o.chunk_doubles - sn_rows_doubles(r)) / o.sn_ldw[k] >= 1) {
        cols(k, SN_W_BWD, o.sn_foff[k] + sn_rows_doubles(r), o.sn_ldw[k], o.sn_w[k], o.sn_foff[k],
             (int)sn_rows_doubles(r));
      } else {
        push(k, SN_ROWS_BWD, o.sn_foff[k], (int)(8 * sn_rows_doubles(r)), 0, 1, true);
        cols(k, SN_W_BWD, o.sn_foff[k] + sn_rows_doubles(r), o.sn_ldw[k], o.sn_w[k]);
      }
      o.sn_bce[k] = (int64_t)o.chunks.size();
    }
    o.sub_bc1.push_back((int64_t)o.chunks.size());
    o.sub_fbytes.push_back(fb);
  }
  if (dbg) {
    double bw = 0, bf = 0, br = 0;
    for (int64_t g = 0; g < NS; ++g) {
      bw += 2.0 * 8 * o.sn_ldw[g] * o.sn_w[g];
      bf += 8.0 * o.sn_ldf[g] * o.sn_w[g];
      br += 2.0 * 8 * sn_rows_doubles(o.sn_r[g]);
    }
    fprintf(stderr, "hplmm sn_analyse: solve bytes W (fwd+bwd) %.3f GB, F_SS^-1 %.3f GB, rows %.3f GB\n",
            bw / 1e9, bf / 1e9, br / 1e9);
    int64_t nk[5] = {0, 0, 0, 0, 0}, bk[5] = {0, 0, 0, 0, 0}, small = 0;
    for (const SnChunk& c : o.chunks) {
      const int kind = (c.info >> 24) & 7;
      nk[kind]++;
      bk[kind] += c.bytes & 0xffffff;
      small += (c.bytes & 0xffffff) < 8192;
    }
    fprintf(stderr, "hplmm sn_analyse: %lld supernodes, %zu chunks (W fwd %lld / %.1f KB avg, F %lld / %.1f KB, "
            "W bwd %lld / %.1f KB, rows fwd %lld / %.2f KB, rows bwd %lld / %.2f KB), %lld chunks < 8 KB\n",
            (long long)NS, o.chunks.size(), (long long)nk[0], bk[0] / 1024.0 / std::max<int64_t>(nk[0], 1),
            (long long)nk[1], bk[1] / 1024.0 / std::max<int64_t>(nk[1], 1), (long long)nk[2],
            bk[2] / 1024.0 / std::max<int64_t>(nk[2], 1), (long long)nk[3],
            bk[3] / 1024.0 / std::max<int64_t>(nk[3], 1), (long long)nk[4],
            bk[4] / 1024.0 / std::max<int64_t>(nk[4], 1), (long long)small);
  }
  if (dbg)
    fprintf(stderr, "hplmm sn_analyse: %d subdomains, %u threads: per-subdomain %.3f s, concat %.3f s, "
            "schedule %.3f s\n", nsub, nth, t1 - t0, t2 - t1, now() - t2);
  return true;
}

}  // namespace hplmm
