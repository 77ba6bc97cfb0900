// Internal declarations of libhplmm (not part of the ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hplmm.h"

namespace hplmm {

enum NodeClass : int32_t { CLS_GRAIN = 0, CLS_IFACE = 1, CLS_DIRICHLET = 2 };

// Integer (host) setup: everything that must be bit-exact with the oracle.
struct HostSetup {
  // problem copy
  int nx = 0, ny = 0, nz = 0;
  double nu = 0.0;
  int n_grains = 0;
  std::vector<uint8_t> solid;     // [nz][ny][nx]
  std::vector<double> E;          // [nz][ny][nx]
  std::vector<int32_t> grain;     // [nz][ny][nx]
  hplmm_options opt{};

  // mesh (R3)
  int n_nodes = 0;
  std::vector<int64_t> node_key;  // lattice key i + (nx+1)(j + (ny+1)k)
  std::vector<int32_t> node_ijk;  // 3 per node
  std::vector<int32_t> lat_id;    // lattice -> node id or -1
  std::vector<uint8_t> dir;       // Dirichlet flag per node
  std::vector<double> u_D, f;     // 3 per node

  // A^ pattern with Dirichlet couplings removed (R4) + removed D-couplings of
  // free rows (for the RHS lift)
  std::vector<int32_t> row_ptr, col_idx;
  std::vector<int32_t> drow_ptr, dcol;

  // decomposition (R6, R7, R18, R8)
  std::vector<int32_t> node_class, node_owner, node_iface;
  std::vector<int32_t> iface_pair;                 // 2 per interface
  std::vector<int32_t> iface_ptr, iface_nodes;
  std::vector<int32_t> contact_ptr, contact_nodes;
  std::vector<int32_t> grain_ptr, grain_nodes;     // I_g node lists (class G or D)

  // mortars (eq:node_init, R9, R10) and shape-vector columns (R14)
  std::vector<int32_t> mortar_ptr, mortar_nodes;   // per interface, placement order
  std::vector<int32_t> gcols_ptr, gcols;           // mortar DOF columns per grain
  std::vector<int32_t> giface_ptr, giface;         // interfaces per grain (sorted)

  int n_ifaces() const { return (int)iface_ptr.size() - 1; }
  int n_mortar_nodes() const { return mortar_ptr.empty() ? 0 : mortar_ptr.back(); }
};

// Builds every integer artifact; returns false and sets err on bad input.
bool host_setup(const hplmm_problem* prob, const hplmm_options* opt, HostSetup& hs,
                std::string& err);

// Mortar placement (R10) on one interface node list, exposed for tests.
std::vector<int32_t> place_mortars(const int32_t* F, int nF, const int32_t* node_ijk, int n);

}  // namespace hplmm
