// Host integer setup of libhplmm: mesh numbering, BSR pattern, node classes,
// contact interfaces, contact grids, mortar placement, shape-vector columns.
//
// Every rule here is a reading of PAPER.md written down in DESIGN.md
// ("Readings"); this code is an independent implementation of those rules and
// shares nothing with oracle/.  Compiled with -ffp-contract=off so that the
// mortar-placement potentials (the only floating point here) are the IEEE
// sequence R10 prescribes: sum_j 1.0/sqrt((double)d2), in chosen order.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <thread>
#include <cstring>
#include <numeric>

#include "hplmm_internal.h"

namespace hplmm {

static inline int64_t d2i(const int32_t* a, const int32_t* b) {
  int64_t dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return dx * dx + dy * dy + dz * dz;
}

// sum_{j != skip} 1/||y - x_j||, sequential in the order of X (eq:node_init).
static double potential(const int32_t* y, const std::vector<int32_t>& X, int skip,
                        const int32_t* ijk) {
  double s = 0.0;
  for (size_t j = 0; j < X.size(); ++j) {
    if ((int)j == skip) continue;
    s += 1.0 / std::sqrt((double)d2i(y, ijk + 3 * (int64_t)X[j]));
  }
  return s;
}

// PAPER.md P:135-142 (eq:node_init) with reading R10.
std::vector<int32_t> place_mortars(const int32_t* F, int nF, const int32_t* ijk, int n) {
  int nu = std::min(n, nF);
  std::vector<int32_t> X;
  if (nu == nF) {
    X.assign(F, F + nF);
    return X;
  }
  if (nu == 1) {  // node nearest the centroid: integer |F|^2 d^2, lowest id on ties
    int64_t S[3] = {0, 0, 0};
    for (int a = 0; a < nF; ++a)
      for (int c = 0; c < 3; ++c) S[c] += ijk[3 * (int64_t)F[a] + c];
    int best = -1;
    int64_t bd = 0;
    for (int a = 0; a < nF; ++a) {
      int64_t d = 0;
      for (int c = 0; c < 3; ++c) {
        int64_t t = (int64_t)nF * ijk[3 * (int64_t)F[a] + c] - S[c];
        d += t * t;
      }
      if (best < 0 || d < bd) { best = F[a]; bd = d; }
    }
    X.push_back(best);
    return X;
  }
  // farthest pair, lowest (id_a, id_b) lexicographic (F ascending)
  int ba = -1, bb = -1;
  int64_t bd = -1;
  for (int a = 0; a < nF; ++a)
    for (int b = a + 1; b < nF; ++b) {
      int64_t d = d2i(ijk + 3 * (int64_t)F[a], ijk + 3 * (int64_t)F[b]);
      if (d > bd) { bd = d; ba = F[a]; bb = F[b]; }
    }
  X.push_back(ba);
  X.push_back(bb);
  // greedy Coulomb argmin over unchosen nodes, lowest id on exact ties
  while ((int)X.size() < nu) {
    int arg = -1;
    double val = 0.0;
    for (int a = 0; a < nF; ++a) {
      int y = F[a];
      if (std::find(X.begin(), X.end(), y) != X.end()) continue;
      double v = potential(ijk + 3 * (int64_t)y, X, -1, ijk);
      if (arg < 0 || v < val) { arg = y; val = v; }
    }
    X.push_back(arg);
  }
  // sweeps in ascending mortar index; move only on > 1e-12 relative gain
  for (int sweep = 0; sweep < 20; ++sweep) {
    bool moved = false;
    for (int i = 0; i < nu; ++i) {
      double cur = potential(ijk + 3 * (int64_t)X[i], X, i, ijk);
      int arg = -1;
      double val = 0.0;
      for (int a = 0; a < nF; ++a) {
        int y = F[a];
        bool other = false;
        for (int j = 0; j < nu; ++j)
          if (j != i && X[j] == y) { other = true; break; }
        if (other) continue;
        double v = potential(ijk + 3 * (int64_t)y, X, i, ijk);
        if (arg < 0 || v < val) { arg = y; val = v; }
      }
      if (val < cur * (1.0 - 1e-12)) { X[i] = arg; moved = true; }
    }
    if (!moved) break;
  }
  return X;
}

bool host_setup(const hplmm_problem* p, const hplmm_options* opt, HostSetup& hs,
                std::string& err) {
  if (!p || !opt || p->nx <= 0 || p->ny <= 0 || p->nz <= 0 || !p->solid || !p->E ||
      !p->grain || !p->node_dirichlet || !p->node_u || !p->node_f || p->n_grains <= 0) {
    err = "hplmm_create: invalid problem";
    return false;
  }
  if (opt->n_mortar < 1 || opt->contact_h < 0 || opt->restart < 1 || opt->restart > 512 ||
      opt->max_iter < 1 || opt->n_st < 1 || opt->n_st > 64 || !(opt->beta > 0) ||
      (opt->smoother != 0 && opt->smoother != 1) ||
      (opt->operator_kind != 0 && opt->operator_kind != 1) ||
      (opt->local_factor != 0 && opt->local_factor != 1) ||
      (opt->coarse_solver != 0 && opt->coarse_solver != 1) ||
      (opt->mortar_kind < 0 || opt->mortar_kind > 2) ||
      (opt->sn_shape != 0 && opt->sn_shape != 8 && opt->sn_shape != 16) ||
      opt->sn_split < -1 || opt->sn_split > 3 ||
      (opt->host_loop != 0 && opt->host_loop != 1) || opt->rhs_block < 0 || opt->rhs_block > 4) {
    err = "hplmm_create: invalid options (n_mortar>=1, contact_h>=0, 1<=restart<=512, 1<=n_st<=64, "
          "smoother/local_factor/coarse_solver/operator_kind in {0,1}, mortar_kind in {0,1,2}, sn_shape in {0,8,16}, sn_split in -1..3, host_loop in {0,1}, rhs_block in 0..4)";
    return false;
  }
  hs.opt = *opt;
  const int nx = p->nx, ny = p->ny, nz = p->nz;
  hs.nx = nx; hs.ny = ny; hs.nz = nz; hs.nu = p->nu; hs.n_grains = p->n_grains;
  const int64_t nvox = (int64_t)nx * ny * nz;
  const int LX = nx + 1, LY = ny + 1, LZ = nz + 1;
  const int64_t nlat = (int64_t)LX * LY * LZ;
  hs.solid.assign(p->solid, p->solid + nvox);
  hs.E.assign(p->E, p->E + nvox);
  hs.grain.assign(p->grain, p->grain + nvox);
  for (int64_t v = 0; v < nvox; ++v) {
    if (hs.solid[v] && (hs.grain[v] < 0 || hs.grain[v] >= p->n_grains)) {
      err = "hplmm_create: solid voxel with grain id outside [0,n_grains)";
      return false;
    }
    if (hs.solid[v] && !(hs.E[v] > 0)) {
      err = "hplmm_create: solid voxel with E <= 0";
      return false;
    }
  }
  auto vox = [&](int i, int j, int k) -> int64_t {
    if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz) return -1;
    int64_t v = i + (int64_t)nx * (j + (int64_t)ny * k);
    return hs.solid[v] ? v : -1;
  };

  static const bool dbg = getenv("HPLMM_DEBUG") != nullptr;
  auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double tph = now();
  auto phase = [&](const char* name) {
    if (!dbg) return;
    const double t = now();
    fprintf(stderr, "hplmm host setup: %-18s %.3f s\n", name, t - tph);
    tph = t;
  };
  // ---- mesh: solid nodes in ascending lattice key (R3) -------------------
  hs.lat_id.assign(nlat, -1);
  for (int k = 0; k < LZ; ++k)
    for (int j = 0; j < LY; ++j)
      for (int i = 0; i < LX; ++i) {
        bool any = false;
        for (int a = 0; a < 8 && !any; ++a)
          any = vox(i - 1 + (a & 1), j - 1 + ((a >> 1) & 1), k - 1 + ((a >> 2) & 1)) >= 0;
        if (!any) continue;
        int64_t key = i + (int64_t)LX * (j + (int64_t)LY * k);
        hs.lat_id[key] = (int32_t)hs.node_key.size();
        hs.node_key.push_back(key);
        hs.node_ijk.push_back(i); hs.node_ijk.push_back(j); hs.node_ijk.push_back(k);
      }
  const int N = (int)hs.node_key.size();
  hs.n_nodes = N;
  hs.dir.resize(N);
  hs.u_D.resize(3 * (size_t)N);
  hs.f.resize(3 * (size_t)N);
  for (int q = 0; q < N; ++q) {
    int64_t key = hs.node_key[q];
    hs.dir[q] = p->node_dirichlet[key] ? 1 : 0;
    for (int c = 0; c < 3; ++c) {
      hs.u_D[3 * (size_t)q + c] = p->node_u[3 * key + c];
      hs.f[3 * (size_t)q + c] = p->node_f[3 * key + c];
    }
  }

  phase("mesh");
  // ---- pattern: p~q iff they share a solid voxel; D rows keep only the
  //      diagonal, free rows drop D columns (R4) ---------------------------
  // two passes over node ranges in parallel (row lengths, then fill); the
  // result is independent of the thread count
  hs.row_ptr.assign(N + 1, 0);
  hs.drow_ptr.assign(N + 1, 0);
  auto neighbours = [&](int q, int32_t* nb) -> int {
    const int32_t* x = &hs.node_ijk[3 * (size_t)q];
    int cnt = 0;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int i = x[0] + dx, j = x[1] + dy, k = x[2] + dz;
          if (i < 0 || j < 0 || k < 0 || i >= LX || j >= LY || k >= LZ) continue;
          int r = hs.lat_id[i + (int64_t)LX * (j + (int64_t)LY * k)];
          if (r < 0) continue;
          // share a voxel: the voxel spanning min..min+1 in each axis is solid
          bool share = false;
          int vi0 = std::min(x[0], i), vj0 = std::min(x[1], j), vk0 = std::min(x[2], k);
          int ei = (dx == 0) ? 2 : 1, ej = (dy == 0) ? 2 : 1, ek = (dz == 0) ? 2 : 1;
          for (int a = 0; a < ek && !share; ++a)
            for (int b = 0; b < ej && !share; ++b)
              for (int c = 0; c < ei && !share; ++c)
                share = vox(vi0 - (dx == 0 ? c : 0), vj0 - (dy == 0 ? b : 0),
                            vk0 - (dz == 0 ? a : 0)) >= 0;
          if (share) nb[cnt++] = r;
        }
    std::sort(nb, nb + cnt);   // lattice-scan order is already ascending; kept for clarity
    return cnt;
  };
  const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  auto parallel = [&](auto&& body) {
    std::vector<std::thread> th;
    const int per = (N + (int)nth - 1) / (int)nth;
    for (unsigned t = 0; t < nth; ++t) {
      const int q0 = (int)t * per, q1 = std::min(N, q0 + per);
      if (q0 < q1) th.emplace_back([&, q0, q1] { body(q0, q1); });
    }
    for (auto& t : th) t.join();
  };
  parallel([&](int q0, int q1) {
    int32_t nb[27];
    for (int q = q0; q < q1; ++q) {
      const int cnt = neighbours(q, nb);
      int nf = 0, nd = 0;
      if (hs.dir[q]) {
        nf = 1;
      } else {
        for (int t = 0; t < cnt; ++t) (hs.dir[nb[t]] ? nd : nf)++;
      }
      hs.row_ptr[q + 1] = nf;
      hs.drow_ptr[q + 1] = nd;
    }
  });
  for (int q = 0; q < N; ++q) {
    hs.row_ptr[q + 1] += hs.row_ptr[q];
    hs.drow_ptr[q + 1] += hs.drow_ptr[q];
  }
  hs.col_idx.resize(hs.row_ptr[N]);
  hs.dcol.resize(hs.drow_ptr[N]);
  parallel([&](int q0, int q1) {
    int32_t nb[27];
    for (int q = q0; q < q1; ++q) {
      int32_t* cf = hs.col_idx.data() + hs.row_ptr[q];
      int32_t* cd = hs.dcol.data() + hs.drow_ptr[q];
      if (hs.dir[q]) {
        *cf = q;
        continue;
      }
      const int cnt = neighbours(q, nb);
      for (int t = 0; t < cnt; ++t) {
        if (hs.dir[nb[t]]) *cd++ = nb[t];
        else *cf++ = nb[t];
      }
    }
  });

  phase("pattern");
  // ---- node classes (R6) -------------------------------------------------
  hs.node_class.assign(N, CLS_GRAIN);
  hs.node_owner.assign(N, -1);
  hs.node_iface.assign(N, -1);
  std::vector<int32_t> pair0(N, -1), pair1(N, -1);
  for (int q = 0; q < N; ++q) {
    const int32_t* x = &hs.node_ijk[3 * (size_t)q];
    int gs[8], ng = 0;
    for (int a = 0; a < 8; ++a) {
      int64_t v = vox(x[0] - 1 + (a & 1), x[1] - 1 + ((a >> 1) & 1), x[2] - 1 + ((a >> 2) & 1));
      if (v >= 0) gs[ng++] = hs.grain[v];
    }
    std::sort(gs, gs + ng);
    ng = (int)(std::unique(gs, gs + ng) - gs);
    if (hs.dir[q]) {
      hs.node_class[q] = CLS_DIRICHLET;
      hs.node_owner[q] = gs[0];
    } else if (ng >= 2) {
      hs.node_class[q] = CLS_IFACE;
      pair0[q] = gs[0];
      pair1[q] = gs[1];
    } else {
      hs.node_owner[q] = gs[0];
    }
  }

  phase("node classes");
  // ---- interfaces: connected components per pair (R7) --------------------
  struct Comp { int32_t g1, g2, first; std::vector<int32_t> nodes; };
  std::vector<Comp> comps;
  std::vector<uint8_t> seen(N, 0);
  std::vector<int32_t> stack;
  for (int q = 0; q < N; ++q) {
    if (hs.node_class[q] != CLS_IFACE || seen[q]) continue;
    Comp c{pair0[q], pair1[q], q, {}};
    stack.assign(1, q);
    seen[q] = 1;
    while (!stack.empty()) {
      int a = stack.back();
      stack.pop_back();
      c.nodes.push_back(a);
      for (int e = hs.row_ptr[a]; e < hs.row_ptr[a + 1]; ++e) {
        int b = hs.col_idx[e];
        if (!seen[b] && hs.node_class[b] == CLS_IFACE && pair0[b] == c.g1 && pair1[b] == c.g2) {
          seen[b] = 1;
          stack.push_back(b);
        }
      }
    }
    std::sort(c.nodes.begin(), c.nodes.end());
    comps.push_back(std::move(c));
  }
  std::stable_sort(comps.begin(), comps.end(), [](const Comp& a, const Comp& b) {
    if (a.g1 != b.g1) return a.g1 < b.g1;
    if (a.g2 != b.g2) return a.g2 < b.g2;
    return a.first < b.first;
  });
  hs.iface_ptr.assign(1, 0);
  for (size_t c = 0; c < comps.size(); ++c) {
    hs.iface_pair.push_back(comps[c].g1);
    hs.iface_pair.push_back(comps[c].g2);
    for (int a : comps[c].nodes) {
      hs.iface_nodes.push_back(a);
      hs.node_iface[a] = (int32_t)c;
    }
    hs.iface_ptr.push_back((int32_t)hs.iface_nodes.size());
  }
  const int NC = (int)comps.size();

  phase("interfaces");
  // ---- grain-interior sets I_g (R18) -------------------------------------
  hs.grain_ptr.assign(p->n_grains + 1, 0);
  for (int q = 0; q < N; ++q)
    if (hs.node_class[q] != CLS_IFACE) hs.grain_ptr[hs.node_owner[q] + 1]++;
  for (int g = 0; g < p->n_grains; ++g) hs.grain_ptr[g + 1] += hs.grain_ptr[g];
  hs.grain_nodes.assign(hs.grain_ptr.back(), 0);
  {
    std::vector<int32_t> fill(hs.grain_ptr.begin(), hs.grain_ptr.end() - 1);
    for (int q = 0; q < N; ++q)
      if (hs.node_class[q] != CLS_IFACE) hs.grain_nodes[fill[hs.node_owner[q]]++] = q;
  }

  phase("grain sets");
  // ---- contact grids: Chebyshev dilation by h, non-D nodes (R8) ----------
  const int h = opt->contact_h;
  hs.contact_ptr.assign(1, 0);
  {
    std::vector<std::vector<int32_t>> zs(NC);
    std::atomic<int> next{0};
    auto work = [&]() {
      std::vector<int32_t> stamp(N, -1);
      for (int c; (c = next.fetch_add(1)) < NC;) {
        std::vector<int32_t>& zeta = zs[c];
        for (int e = hs.iface_ptr[c]; e < hs.iface_ptr[c + 1]; ++e) {
          const int32_t* x = &hs.node_ijk[3 * (size_t)hs.iface_nodes[e]];
          for (int dz = -h; dz <= h; ++dz)
            for (int dy = -h; dy <= h; ++dy)
              for (int dx = -h; dx <= h; ++dx) {
                int i = x[0] + dx, j = x[1] + dy, k = x[2] + dz;
                if (i < 0 || j < 0 || k < 0 || i >= LX || j >= LY || k >= LZ) continue;
                int r = hs.lat_id[i + (int64_t)LX * (j + (int64_t)LY * k)];
                if (r < 0 || hs.dir[r] || stamp[r] == c) continue;
                stamp[r] = c;
                zeta.push_back(r);
              }
        }
        std::sort(zeta.begin(), zeta.end());
      }
    };
    const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t + 1 < nth; ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    for (int c = 0; c < NC; ++c) {
      hs.contact_nodes.insert(hs.contact_nodes.end(), zs[c].begin(), zs[c].end());
      hs.contact_ptr.push_back((int32_t)hs.contact_nodes.size());
    }
  }

  phase("contact grids");
  // ---- mortar placement (eq:node_init, R9, R10) --------------------------
  // interfaces are independent: placed in parallel, concatenated in order
  // (each placement is sequential and deterministic, so the result is too)
  hs.mortar_ptr.assign(1, 0);
  {
    std::vector<std::vector<int32_t>> Xs(NC);
    std::atomic<int> next{0};
    auto work = [&]() {
      for (int c; (c = next.fetch_add(1)) < NC;)
        Xs[c] = place_mortars(&hs.iface_nodes[hs.iface_ptr[c]], hs.iface_ptr[c + 1] - hs.iface_ptr[c],
                              hs.node_ijk.data(), opt->n_mortar);
    };
    const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t + 1 < nth; ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    for (int c = 0; c < NC; ++c) {
      hs.mortar_nodes.insert(hs.mortar_nodes.end(), Xs[c].begin(), Xs[c].end());
      hs.mortar_ptr.push_back((int32_t)hs.mortar_nodes.size());
    }
  }

  phase("mortar placement");
  // ---- shape-vector column sets (R14, structural option B) ---------------
  hs.gcols_ptr.assign(1, 0);
  hs.giface_ptr.assign(1, 0);
  std::vector<int32_t> mark(NC, -1), ifs;
  for (int g = 0; g < p->n_grains; ++g) {
    ifs.clear();
    for (int e = hs.grain_ptr[g]; e < hs.grain_ptr[g + 1]; ++e) {
      int q = hs.grain_nodes[e];
      if (hs.node_class[q] != CLS_GRAIN) continue;
      for (int t = hs.row_ptr[q]; t < hs.row_ptr[q + 1]; ++t) {
        int c = hs.node_iface[hs.col_idx[t]];
        if (c >= 0 && mark[c] != g) { mark[c] = g; ifs.push_back(c); }
      }
    }
    std::sort(ifs.begin(), ifs.end());
    for (int c : ifs) {
      hs.giface.push_back(c);
      for (int k = 3 * hs.mortar_ptr[c]; k < 3 * hs.mortar_ptr[c + 1]; ++k) hs.gcols.push_back(k);
    }
    hs.giface_ptr.push_back((int32_t)hs.giface.size());
    hs.gcols_ptr.push_back((int32_t)hs.gcols.size());
  }
  return true;
}

}  // namespace hplmm
