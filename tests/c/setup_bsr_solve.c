/* Plain C client of include/hplmm.h (no ctypes, no Python): the north star's
 * hplmm_setup(A in 3x3-block CSR, subdomain partition, material and BC data)
 * followed by hplmm_solve(b, tol) -> x, iterations, residual history.
 *
 * usage: setup_bsr_solve DIR [tol]
 * DIR holds raw little-endian arrays written by the test harness from the
 * ORACLE (tests/test_c_client.py): dims.txt = "nx ny nz n_grains n_nodes nnzb
 * nu", solid.u8, E.f64, grain.i32, dir.u8, node_u.f64, node_f.f64 (voxel /
 * lattice arrays of hplmm_problem), row_ptr.i32, col_idx.i32, val.f64,
 * node_ijk.i32 (the oracle's BSR A^), b.f64 (the oracle's b^).
 * Writes DIR/x.f64 and DIR/hist.f64 and prints one line
 * "status S iterations I converged C relres R hist_len H".  A failing call
 * prints "status S <message>" and exits with code 3. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hplmm.h"

static void* slurp(const char* dir, const char* name, size_t* bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "rb");
  if (!f) { fprintf(stderr, "cannot open %s\n", path); exit(2); }
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  void* p = malloc(n > 0 ? (size_t)n : 1);
  if (n > 0 && fread(p, 1, (size_t)n, f) != (size_t)n) { fprintf(stderr, "short read %s\n", path); exit(2); }
  fclose(f);
  if (bytes) *bytes = (size_t)n;
  return p;
}

static void spill(const char* dir, const char* name, const void* p, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "wb");
  if (!f || fwrite(p, 1, bytes, f) != bytes) { fprintf(stderr, "cannot write %s\n", path); exit(2); }
  fclose(f);
}

int main(int argc, char** argv) {
  if (argc < 2) { fprintf(stderr, "usage: %s DIR [tol]\n", argv[0]); return 2; }
  const char* dir = argv[1];
  const double tol = argc > 2 ? atof(argv[2]) : 1e-8;
  int nx, ny, nz, ng, nn;
  long long nnzb;
  double nu;
  {
    char path[4096];
    snprintf(path, sizeof path, "%s/dims.txt", dir);
    FILE* f = fopen(path, "r");
    if (!f || fscanf(f, "%d %d %d %d %d %lld %lf", &nx, &ny, &nz, &ng, &nn, &nnzb, &nu) != 7) {
      fprintf(stderr, "bad dims.txt\n");
      return 2;
    }
    fclose(f);
  }
  hplmm_problem geom;
  geom.nx = nx; geom.ny = ny; geom.nz = nz;
  geom.solid = (const uint8_t*)slurp(dir, "solid.u8", NULL);
  geom.E = (const double*)slurp(dir, "E.f64", NULL);
  geom.nu = nu;
  geom.grain = (const int32_t*)slurp(dir, "grain.i32", NULL);
  geom.n_grains = ng;
  geom.node_dirichlet = (const uint8_t*)slurp(dir, "dir.u8", NULL);
  geom.node_u = (const double*)slurp(dir, "node_u.f64", NULL);
  geom.node_f = (const double*)slurp(dir, "node_f.f64", NULL);
  hplmm_bsr A;
  A.n_nodes = nn;
  A.nnzb = nnzb;
  A.row_ptr = (const int32_t*)slurp(dir, "row_ptr.i32", NULL);
  A.col_idx = (const int32_t*)slurp(dir, "col_idx.i32", NULL);
  A.val = (const double*)slurp(dir, "val.f64", NULL);
  A.node_ijk = (const int32_t*)slurp(dir, "node_ijk.i32", NULL);
  double* b = (double*)slurp(dir, "b.f64", NULL);

  hplmm_options opt;
  hplmm_default_options(&opt);
  hplmm_handle* h = NULL;
  hplmm_status s = hplmm_setup_bsr(&A, &geom, &opt, 0, NULL, &h);
  if (s != HPLMM_OK) {
    printf("status %d %s\n", (int)s, hplmm_last_error());
    return 3;
  }
  const int n = 3 * nn;
  double* x = (double*)calloc((size_t)n, sizeof(double));
  double hist[1024];
  hplmm_report rep;
  s = hplmm_solve(h, b, tol, x, &rep, hist, 1024, NULL);
  if (s < 0) {
    printf("status %d %s\n", (int)s, hplmm_last_error());
    hplmm_destroy(h);
    return 3;
  }
  spill(dir, "x.f64", x, (size_t)n * sizeof(double));
  spill(dir, "hist.f64", hist, (size_t)rep.hist_len * sizeof(double));
  printf("status %d iterations %d converged %d relres %.6e hist_len %d fine_operator %d\n", (int)s,
         rep.iterations, rep.converged, rep.final_true_relres, rep.hist_len, rep.fine_operator);
  hplmm_destroy(h);
  free(x);
  free(b);
  return 0;
}
