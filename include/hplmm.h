/* hplmm.h -- C ABI of the B200-native hPLMM-preconditioned GMRES solver.
 *
 * Method: arXiv 2509.19777 (Khan & Mehmani), "High-order Multiscale
 * Preconditioner for Elasticity of Arbitrary Structures".  Citations are
 * PAPER.md line numbers (P:<line>) plus the LaTeX equation label.  Readings
 * R1..R24 where the paper is silent are listed in DESIGN.md ("Readings").
 *
 * The library solves the fine Q1-hex FEM elasticity system
 *     A^ x^ = b^                                   (eq:ls_all)
 * with right-preconditioned GMRES(restart) (R22) whose preconditioner is
 *     M^-1 = M_G^-1 + M_L^-1 (I - A^ M_G^-1)       (eq:multi_precond)
 *     M_G^-1 = P^ (P^T A^ P^)^-1 P^T,  P^ = W Q P  (eq:mg_struct/eq:WQP)
 *     M_L = M_CG = M_zeta^-1 + M_g^-1 (I - A^ M_zeta^-1)
 *                                                  (eq:local_smoother_CG)
 * on one CUDA device (sm_100a).  All arithmetic is fp64 (R1).
 *
 * Conventions (all entry points)
 *  - Return value: hplmm_status; negative = error (message via
 *    hplmm_last_error(), thread-local, valid until the next call on this
 *    thread), 0 = OK, positive = a non-fatal outcome (NOT_CONVERGED).
 *  - Pointers marked "host or device" are classified with
 *    cudaPointerGetAttributes; device pointers must live on the handle's
 *    device.  Every input is borrowed for the call only (copied if kept).
 *    Outputs are caller-allocated with the stated length.
 *  - A handle owns all device memory it allocates; hplmm_destroy frees it.
 *    A handle is not thread-safe; distinct handles are independent.
 *  - Streams: every GPU entry point takes a cudaStream_t (0 = legacy default
 *    stream) passed as void* so this header needs no CUDA include.  Calls are
 *    synchronous with respect to the host on return unless stated.
 *  - There is no CPU fallback: GPU entry points fail with HPLMM_ERR_CUDA when
 *    no device is usable.
 */
#ifndef HPLMM_H
#define HPLMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HPLMM_OK = 0,
  HPLMM_NOT_CONVERGED = 1,        /* solve hit max_iter; x and history written  */
  HPLMM_ERR_ARG = -1,             /* bad argument / size / null pointer         */
  HPLMM_ERR_CUDA = -2,            /* CUDA runtime error (incl. no device)       */
  HPLMM_ERR_OOM = -3,             /* device allocation failed                   */
  HPLMM_ERR_SINGULAR_LOCAL = -4,  /* non-positive pivot in a grain/contact-grid
                                     factorisation; report.err_index = subdomain */
  HPLMM_ERR_SINGULAR_COARSE = -5, /* non-positive pivot in the coarse matrix S  */
  HPLMM_ERR_NONFINITE = -6,       /* NaN/Inf in the GMRES residual estimate     */
  HPLMM_ERR_STATE = -7            /* call out of order (e.g. solve before setup) */
} hplmm_status;

/* Voxel problem (§2; Cartesian decomposition §3.1).
 * All arrays are HOST arrays, x fastest: voxel arrays [nz][ny][nx], node
 * (lattice) arrays [nz+1][ny+1][nx+1] (x3 for vectors, component fastest). */
typedef struct {
  int32_t nx, ny, nz;            /* voxels                                          */
  const uint8_t *solid;          /* 1 = solid voxel (one Q1 hex element)      */
  const double *E;               /* Young's modulus per voxel (read where solid)    */
  double nu;                     /* uniform Poisson ratio (eq:stiff_iso via R2)     */
  const int32_t *grain;          /* grain id per voxel in [0,n_grains), -1 = void   */
  int32_t n_grains;
  const uint8_t *node_dirichlet; /* 1 = all 3 components prescribed (R4)            */
  const double *node_u;          /* prescribed displacement (used where dirichlet)  */
  const double *node_f;          /* consistent external nodal force                 */
} hplmm_problem;

typedef struct {
  int32_t n_mortar;   /* n: mortar nodes per interface (R9, default 4)             */
  double beta;        /* Gaussian mortar spread (eq:gauss; default 4.0)      */
  int32_t contact_h;  /* contact-grid Chebyshev dilation h in nodes (R8); <0 invalid */
  int32_t restart;    /* GMRES restart m (R22, default 50; 1..512)                  */
  int32_t max_iter;   /* total Arnoldi steps cap (default 300)               */
  int32_t n_st;       /* smoother stages of eq:local_smoother, 1..64:
                         M_L^-1 = sum_i M_l^-1 prod_{j<i} (I - A^ M_l^-1),
                         evaluated as t_1 = r, u_i = M_l^-1 t_i,
                         t_{i+1} = t_i - A^ u_i (R28).  default 1            */
  int32_t coarse_refine; /* 1 = one step of iterative refinement of the coarse
                            solve y = S^-1 r with S kept resident (residual
                            ~(kappa u)^2 instead of ~kappa u); default 0        */
  int32_t local_factor;  /* exact local solves of M_zeta and M_g (eq:Mg_Mz; the
                            paper's precomputed LU):
                            0 = explicit dense inverse of every subdomain block
                                (packed 64x64 lower tiles, one symmetric
                                mat-vec per apply);
                            1 = supernodal block-LDL^T factor on a geometric
                                nested-dissection ordering (W_S = F_RS F_SS^-1,
                                F_SS^-1; forward + backward sweep per apply,
                                ~4x fewer bytes, needed for cfg4/cfg5).
                            default 1                                          */
  int32_t coarse_solver; /* coarse mortar-block solve y = S^-1 r (eq:mg_struct,
                            P:741 "direct solver"):
                            0 = explicit S^-1 (packed lower tiles) applied by one
                                symmetric mat-vec (default; half the bytes of
                                two triangular sweeps, no dependency chain);
                            1 = Cholesky factor S = L L^T applied by a forward
                                and a backward triangular solve               */
  int32_t mortar_kind;   /* mortar functions: 0 = Gaussian (eq:gauss,
                            the paper's choice, default); 1 = Algebraic
                            (eq:algebra, built by the Remark's constrained
                            interface solves on A^{c}_{c}; reading R25);
                            2 = Algebraic on the interface surface: the same
                            constrained solves on eq:algebra discretised over
                            the voxel faces shared by the pair's grains
                            (tangential strain, Q1) + a translation-free tie
                            (reading R29; partition of unity exact)        */
  int32_t smoother;      /* base smoother M_l of eq:local_smoother:
                            0 = contact-grain M_CG (eq:local_smoother_CG, the
                                paper's choice with n_st = 1; default);
                            1 = ILU(0) of A^ (paper: n_st = 6):
                                scalar ILU(0) in the natural DOF order on the
                                pattern of every stored 3x3 block (R26), held
                                as block ILU(0) factors in A^'s BSR layout;
                                contact-grid factors are not built        */
  int32_t operator_kind; /* how the solve applies A^ (GMRES, eq:multi_precond,
                            eq:local_smoother_CG):
                            0 = element-by-element from the voxel data,
                                sum_e E_e K0 x_e over each node's voxels with
                                R4's identity Dirichlet rows (default; used
                                only when A^ is the library's own assembly --
                                after hplmm_set_matrix the stored blocks are
                                used);
                            1 = the stored BSR blocks (TMA-streamed SpMV)    */
  int32_t sn_shape;      /* launch shape of the supernodal local solves
                            (local_factor = 1): 0 = automatic (8 consumer warps
                            x 2 CTAs per SM when a batch has >= 2 subdomains per
                            CTA or may share subdomains between CTAs (sn_split
                            >= 0), else 16 x 1; default), 8 = force 8 x 2, 16 =
                            force 16 x 1 (a shape the subdomains do not fit
                            falls back to automatic).  Same operator A_s^-1;
                            only the summation order of the group reductions
                            differs (parity tests run both shapes)          */
  int32_t sn_split;      /* subtree-parallel supernodal solves: a batch with too
                            few subdomains to load the CTAs evenly shares its
                            largest subdomains between teams of up to 2^L CTAs
                            (the top L levels of the nested-dissection tree are
                            cut; the members exchange the separators' x rows).
                            0 = automatic, L <= 3 (default; the cuts are
                            chosen by a modelled makespan and a batch that
                            gains < 5% keeps one CTA per subdomain), -1 = off,
                            1..3 = forced: every subdomain, largest first, is
                            cut as deep as its tree allows (<= L levels) while
                            CTAs last (tests, experiments).  Same
                            operator A_s^-1: only the order in which the
                            subtrees' updates of a separator are added differs */
  int32_t host_loop;     /* how hplmm_solve drives GMRES (R22):
                            0 = device-resident (default): the whole solve --
                                every Arnoldi step, Givens update, stop test and
                                restart cycle -- is one CUDA-graph launch (two
                                nested WHILE conditional nodes) and one host
                                synchronisation; used with smoother = 0 and
                                coarse_solver = 0 while profiling is off (else
                                the host loop runs);
                            1 = host-driven loop: one pinned D2H of the
                                Hessenberg column and one synchronisation per
                                Arnoldi step, Givens on the host            */
  int32_t rhs_block;     /* hplmm_solve_many: right-hand sides solved together.
                            0 = automatic (default): blocks of 4, unless the
                            one-RHS local solves form CTA teams (sn_split: a
                            batch with few subdomains) -- the block solves do
                            not, and one team solve per column is then faster
                            (cfg2, 4 load cases: 0.109 s vs 0.127 s);
                            2..4 = blocks of that width; 1 = one hplmm_solve
                            per column.  A block runs lockstep GMRES(m): each
                            column keeps its own Arnoldi process, correction
                            columns (eq:col_cg, R15) and stop test, while
                            every operator application streams its matrix
                            data once for the whole block (the supernodal
                            local factors, P^_B; NEXT #2).
                            Blocks need local_factor = 1, smoother = 0,
                            n_st = 1                                        */
} hplmm_options;

typedef struct {
  /* sizes */
  int32_t n_nodes;        /* FEM nodes (DOF = 3 n_nodes, R3)                        */
  int64_t nnzb;           /* 3x3 blocks of A^ after Dirichlet removal               */
  int32_t n_grains;       /* grain grids N^g                                        */
  int32_t n_interfaces;   /* contact interfaces N^c = contact grids N^zeta          */
  int32_t n_mortar_dofs;  /* N^o_m = 3 N^m                                          */
  int32_t n_coarse;       /* N^o_m + number of correction columns (after set_rhs)   */
  int64_t local_bytes;    /* bytes of the local operators (packed inverse tiles, or
                             supernodal factors)                                  */
  int64_t coarse_bytes;   /* bytes of the packed coarse inverse tiles               */
  int64_t prolong_nnz;    /* stored entries of P^_B (grain blocks + Q^o)            */
  /* solve outcome */
  int32_t iterations;     /* total Arnoldi steps                                    */
  int32_t converged;
  int32_t hist_len;       /* entries written to hist                                */
  int32_t err_index;      /* failing subdomain for SINGULAR_LOCAL, else -1          */
  double final_true_relres; /* ||b - A x|| / ||b|| at exit                          */
  /* timings (s), CUDA events on the call's stream                                 */
  double t_host_setup_s;  /* integer setup (hplmm_create)                           */
  double t_assemble_s;
  double t_setup_local_s; /* ~T_ML: grain + contact-grid inversions                 */
  double t_setup_coarse_s;/* ~T_MG: mortars, P^_B, S, coarse inversion              */
  double t_rhs_s;         /* per-RHS correction columns (set_rhs)                   */
  double t_solve_s;       /* GMRES (T_sol)                                          */
  double t_update_s;      /* last hplmm_update_moduli (assembly + refactorisation)  */
  int64_t kernel_launches;/* kernels launched by the last solve                      */
  int32_t fine_operator;  /* A^ applied by the solve: 0 element-by-element, 1 BSR   */
  int32_t sn_shape_grain;   /* consumer warps per CTA of the grain / contact-grid    */
  int32_t sn_shape_contact; /* supernodal solves in use (8: 8 x 2 CTAs/SM, 16: 16 x 1;
                               0 = not built)                                      */
  int32_t sn_teams_grain;   /* grains / contact grids shared by a team of CTAs      */
  int32_t sn_teams_contact; /* (sn_split), and the CTAs of the largest team         */
  int32_t sn_team_max;
  int32_t sn_xg_grain;      /* 1: the batch's one-RHS solves keep x in the CTA's     */
  int32_t sn_xg_contact;    /* global-memory slice (subdomains too large for two
                               CTAs per SM with x in shared memory), 0: x in
                               shared memory                                      */
} hplmm_report;

typedef struct hplmm_handle hplmm_handle;

/* The fine matrix A^ of eq:ls_all in 3x3-block CSR (BSR), node-major
 * DOFs 3 p + c (R3).  Every array is HOST or DEVICE memory (classified per
 * pointer) and borrowed for the call.
 *   row_ptr  int32[n_nodes + 1]  block-row offsets, row_ptr[0] = 0
 *   col_idx  int32[nnzb]         block columns, strictly ascending in a row
 *   val      double[9 nnzb]      each block row-major (entry (a, b) of block e at
 *                                val[9 e + 3 a + b])
 *   node_ijk int32[3 n_nodes]    lattice coordinates (i, j, k) of node p, or NULL
 *                                (then the R3 numbering is assumed)           */
typedef struct {
  int32_t n_nodes;
  int64_t nnzb;
  const int32_t *row_ptr;
  const int32_t *col_idx;
  const double *val;
  const int32_t *node_ijk;
} hplmm_bsr;

/* Default options: n=4, beta=4, h=1, restart=50, max_iter=300, n_st=1,
 * coarse_refine=0, sn_split=0, rhs_block=0. */
void hplmm_default_options(hplmm_options *opt);

/* Host-only integer setup (no GPU work; bit-exact vs the oracle):
 * mesh numbering (R3), BSR pattern with Dirichlet couplings removed (R4),
 * node classes (R6), interfaces (R7), grain-interior sets (R18), contact grids
 * (R8), mortar placement (eq:node_init, R10), shape-vector column sets (R14).
 * Copies everything it needs from `prob`.  opt = NULL: the defaults. */
hplmm_status hplmm_create(const hplmm_problem *prob, const hplmm_options *opt,
                          hplmm_handle **out);

/* GPU assembly of A^ values and b^ (R2, R4) into handle-owned device
 * memory.  Selects device `device` for the handle (cudaSetDevice). */
hplmm_status hplmm_assemble(hplmm_handle *h, int32_t device, void *stream);

/* hplmm_setup(A in 3x3-block CSR, subdomain partition, material and BC data)
 * of the north star, in one call: the problem A^ x^ = b^ (eq:ls_all)
 * on the voxel geometry `geom` (grain labels per voxel = the subdomain partition
 * of §3.1; Dirichlet flags = the BC data of eq:BC P:53-61; E, nu only
 * for mortar_kind = 2, which builds its interface operators from them) with
 * the CALLER's matrix A.  Runs hplmm_create (integer setup from geom),
 * checks that A's node numbering (node_ijk, if given) and block pattern are
 * the ones the geometry defines (R3: nodes in lattice-key order; R4:
 * Dirichlet couplings removed, identity-pattern Dirichlet rows) -- the
 * decomposition (R6-R8, R14) is defined on that pattern --, binds `device`,
 * uploads A's values and runs hplmm_setup with them.  The solve then applies
 * the stored blocks (operator_kind 1).  A must be SPD on the non-Dirichlet
 * DOFs (SINGULAR_LOCAL / SINGULAR_COARSE otherwise).  On success *out is a
 * handle ready for hplmm_solve / hplmm_apply; on error *out = NULL and nothing
 * is leaked.  ERR_ARG names the first mismatching row / node. */
hplmm_status hplmm_setup_bsr(const hplmm_bsr *A, const hplmm_problem *geom,
                             const hplmm_options *opt, int32_t device, void *stream,
                             hplmm_handle **out);

/* The library's own assembly of A^ and b^ (R2-R4) returned to the
 * host: *A (and its arrays) and *b (n_dof doubles) are allocated by the
 * library and released with hplmm_free_bsr.  Runs on `device`. */
hplmm_status hplmm_assemble_bsr(const hplmm_problem *prob, int32_t device, hplmm_bsr **A,
                                double **b);
void hplmm_free_bsr(hplmm_bsr *A, double *b);

/* Replace the values of A^ (nnzb*9 doubles, row-major 3x3 blocks in the
 * handle's pattern, host or device) -- used to parity-test later stages on an
 * externally supplied matrix.  Must precede hplmm_setup. */
hplmm_status hplmm_set_matrix(hplmm_handle *h, const double *val, void *stream);

/* GPU numeric setup, timed separately from the solve (north_star (6)):
 * Gaussian mortar weights (eq:gauss), inverses (local_factor 0) or
 * supernodal factors (local_factor 1) of every grain block A^{g}_{g} and
 * contact-grid block A^[zeta,zeta] (T_ML), shape vectors
 * B = -A_g^-1 Abar^g_m Q^o (eq:col_pk, R14), S = P_B^T A^ P_B (eq:mg_struct,
 * R16) and its inverse (R17).  Errors: SINGULAR_LOCAL (report.err_index via
 * hplmm_get_report), SINGULAR_COARSE, OOM. */
hplmm_status hplmm_setup(hplmm_handle *h, void *stream);

/* Reuse of M_G across a perturbed A^ (reading R30):
 * "the coefficient matrix remains unchanged (load steps) or is perturbed only
 * slightly (local cracks), in which case the M_G of hPLMM can be reused".
 * E: nx*ny*nz new Young's moduli (HOST, [z][y][x] as hplmm_problem.E; read
 * where solid, must be > 0 there); geometry, grains, boundary data and nu are
 * the handle's.  Re-assembles A^ and b^ on the GPU and refactorises every
 * grain block and contact-grid block numerically (the symbolic analysis,
 * factor layout, work lists and solve graph of hplmm_setup are kept), so the
 * residual operator, M_g, M_zeta and -- at the next hplmm_set_rhs /
 * hplmm_solve -- the correction columns (eq:col_cg) follow the new matrix,
 * while M_G keeps the P^_B and S^-1 built by hplmm_setup from the original
 * one.  GMRES then solves the NEW system; only its iteration count feels the
 * older coarse space (a local perturbation costs a few iterations; a global
 * one can stall GMRES -- then set up again).  Cost: report.t_update_s (cfg3:
 * 0.21 s vs 1.26 s for hplmm_setup).  The updated b^ is hplmm_export(RHS).  Needs local_factor = 1,
 * smoother = 0 and the library's own assembly (not hplmm_setup_bsr /
 * hplmm_set_matrix).  Errors: STATE, ARG (E <= 0 in a solid voxel),
 * SINGULAR_LOCAL (report.err_index). */
hplmm_status hplmm_update_moduli(hplmm_handle *h, const double *E, void *stream);

/* "Otherwise, M_G must be updated periodically": rebuild M_G for the
 * handle's CURRENT A^ (after hplmm_update_moduli) -- shape vectors
 * (eq:col_pk) with the current grain factors, S = P^_B^T A^ P^_B
 * (eq:mg_struct, R16) and S^-1 (R17) -- without repeating the integer setup,
 * the symbolic analysis or the local factorisations.  After
 * hplmm_update_moduli + hplmm_refresh_coarse the handle applies the same M^-1
 * as a fresh hplmm_setup on the new moduli.  Time in report.t_setup_coarse_s
 * (cfg3: ~0.6 s).  Needs the default configuration: local_factor = 1,
 * smoother = 0, coarse_solver = 0, coarse_refine = 0, Gaussian mortars (their
 * weights are geometric; the Algebraic ones depend on A^).  Errors: STATE,
 * SINGULAR_COARSE. */
hplmm_status hplmm_refresh_coarse(hplmm_handle *h, void *stream);

/* Per-RHS correction columns c^g = A_g^-1 b^g (eq:col_cg) for grains with
 * b[I_g] != 0 (R15), D_c[g] = b^g . c^g (R16).  b: n_dof doubles, host or
 * device.  hplmm_solve calls it itself; needed before hplmm_apply(MG/MINV). */
hplmm_status hplmm_set_rhs(hplmm_handle *h, const double *b, void *stream);

/* Solve A^ x = b to ||b - A^x||/||b|| < tol (R22).  b, x: n_dof doubles, host
 * or device (x is overwritten, x0 = 0).  hist: host array of hist_cap doubles
 * receiving the per-step Arnoldi estimates (may be NULL).  report may be NULL.
 * Returns OK, NOT_CONVERGED (x = last iterate) or an error.  b = 0 => x = 0. */
hplmm_status hplmm_solve(hplmm_handle *h, const double *b, double tol, double *x,
                         hplmm_report *report, double *hist, int32_t hist_cap,
                         void *stream);

/* Multi-RHS reuse (the paper's economic argument, P:743,
 * P:819): solve A^ X = B for nrhs right-hand sides with one setup -- the
 * local factors and S^-1 are reused, only the correction columns (eq:col_cg,
 * R15) are built per column.  Columns are solved in blocks of
 * hplmm_options.rhs_block (lockstep GMRES, batched operator applications:
 * each column's iterates are those of its own hplmm_solve).  B, X: nrhs x
 * n_dof doubles, column-contiguous (column i at B + i n_dof), host or
 * device.  reports: nrhs entries or NULL (t_solve_s: the column's block).
 * Returns the worst status over the columns (an error stops at that block). */
hplmm_status hplmm_solve_many(hplmm_handle *h, int32_t nrhs, const double *B, double tol,
                              double *X, hplmm_report *reports, void *stream);

typedef enum {
  HPLMM_OP_SPMV = 0,   /* out = A^ in, by the solve's operator (operator_kind;
                          before hplmm_setup: the stored blocks)               */
  HPLMM_OP_MG = 1,     /* out = M_G^-1 in        (needs set_rhs)                */
  HPLMM_OP_MZETA = 2,  /* out = M_zeta^-1 in     (eq:Mg_Mz)                      */
  HPLMM_OP_MGRAIN = 3, /* out = M_g^-1 in        (eq:Mg_Mz, R18)                 */
  HPLMM_OP_MCG = 4,    /* out = M_CG^-1 in       (eq:local_smoother_CG)          */
  HPLMM_OP_MINV = 5,   /* out = M^-1 in          (eq:multi_precond; set_rhs)     */
  HPLMM_OP_RESTRICT = 6,/* out[n_coarse] = P^T in                               */
  HPLMM_OP_PROLONG = 7, /* out[n_dof] = P^ in, in has n_coarse entries          */
  HPLMM_OP_COARSE = 8,  /* out[N_m] = S^-1 in[N_m]: the coarse mortar-block solve  */
  HPLMM_OP_MILU = 9,    /* out = U^-1 L^-1 in: one ILU(0) apply (smoother = 1)     */
  HPLMM_OP_ML = 10,     /* out = M_L^-1 in: n_st stages of the base smoother
                           (eq:local_smoother)                                   */
  HPLMM_OP_SPMV_BSR = 11 /* out = A^ in from the stored BSR blocks, whatever
                           operator_kind (HPLMM_OP_SPMV uses the solve's
                           operator); for operator parity                      */
} hplmm_op;

/* One application of an operator (parity entry point).  in/out: host or
 * device; lengths n_dof unless stated. */
hplmm_status hplmm_apply(hplmm_handle *h, int32_t op, const double *in, double *out,
                         void *stream);

/* Block application of a local operator to ncols (1..4) vectors at once --
 * the batched form hplmm_solve_many uses:
 * the supernodal factors of the contact grids / grains stream once per block
 * (k_sn_solve with NRHS = 2 or 4 columns) instead of once per vector.
 * op: HPLMM_OP_MZETA, HPLMM_OP_MGRAIN or HPLMM_OP_MCG (the operators that do
 * not depend on the right-hand side; eq:Mg_Mz, eq:local_smoother_CG), or
 * HPLMM_OP_SPMV (A^ by the solve's operator: the element-by-element operator
 * applied to the block in one launch, eq:ls_all).  Column
 * c of in / out is in + c ldin / out + c ldout (ldin, ldout >= n_dof), host or
 * device; out[c] equals hplmm_apply(op, in[c]) up to the summation order of
 * the group reductions.  Needs local_factor = 1 (supernodal) and smoother = 0
 * (else HPLMM_ERR_STATE); ncols outside 1..4 or a bad op: HPLMM_ERR_ARG. */
hplmm_status hplmm_apply_many(hplmm_handle *h, int32_t op, int32_t ncols, const double *in,
                              int64_t ldin, double *out, int64_t ldout, void *stream);

typedef enum {
  HPLMM_ART_NODE_KEY = 0,     /* int64[n_nodes] lattice key of each node (R3)   */
  HPLMM_ART_ROW_PTR = 1,      /* int32[n_nodes+1]                               */
  HPLMM_ART_COL_IDX = 2,      /* int32[nnzb]                                    */
  HPLMM_ART_NODE_CLASS = 3,   /* int32[n_nodes] 0=grain-interior 1=interface 2=Dirichlet */
  HPLMM_ART_NODE_IFACE = 4,   /* int32[n_nodes] interface id or -1              */
  HPLMM_ART_NODE_OWNER = 5,   /* int32[n_nodes] owning grain or -1 (interface)  */
  HPLMM_ART_IFACE_PTR = 6,    /* int32[N^c+1] CSR over interface node lists     */
  HPLMM_ART_IFACE_NODES = 7,  /* int32[...] ascending nodes of each interface   */
  HPLMM_ART_CONTACT_PTR = 8,  /* int32[N^c+1]                                   */
  HPLMM_ART_CONTACT_NODES = 9,/* int32[...] ascending nodes of each contact grid */
  HPLMM_ART_MORTAR_PTR = 10,  /* int32[N^c+1] CSR over mortar nodes             */
  HPLMM_ART_MORTAR_NODES = 11,/* int32[N^m] mortar node ids in placement order  */
  HPLMM_ART_GRAIN_COLS_PTR = 12, /* int32[N^g+1] CSR over shape-vector columns  */
  HPLMM_ART_GRAIN_COLS = 13,  /* int32[...] ascending mortar DOF columns (R14)  */
  HPLMM_ART_VAL = 14,         /* double[nnzb*9] values of A^ (after assemble)   */
  HPLMM_ART_RHS = 15,         /* double[n_dof] b^ (after assemble)              */
  HPLMM_ART_S = 16,           /* double[N_m*N_m] coarse mortar block S (setup)  */
  HPLMM_ART_MORTAR_W = 17,    /* double[sum 9 |F_c| nu_c] mortar blocks M^{c} (3|F_c| x 3nu_c,
                                 row 3f+d, column 3i+gamma), row-major per interface */
  HPLMM_ART_ILU = 18          /* double[nnzb*9] block ILU(0) factor in A^'s BSR layout
                                 (smoother = 1): L_IK (K<I), A~_IJ (J>I), A~_II^-1 */
} hplmm_artifact;

/* Copy an artifact to the host buffer `buf` of `cap` BYTES; *len receives the
 * element count (call with buf=NULL to query).  ERR_STATE if not yet built. */
hplmm_status hplmm_export(hplmm_handle *h, int32_t artifact, void *buf, int64_t cap,
                          int64_t *len);

/* Sizes / timings gathered so far. */
hplmm_status hplmm_get_report(hplmm_handle *h, hplmm_report *report);

/* Profiling of the dominant kernels (supernodal local solves, packed SYMV tiles
 * of the local / coarse inverses, ILU(0) sweeps, fine operator; classes as in
 * hplmm_kernel_stats): when enabled, CUDA events are recorded around each such
 * launch on the launch stream (this adds event records to the timed path --
 * keep it off for headline timings).  reset != 0 clears the accumulated
 * statistics. */
hplmm_status hplmm_profile(hplmm_handle *h, int32_t enable, int32_t reset);

/* Statistics of kernel class `kernel` (0 = grain SYMV tiles, 1 = contact-grid
 * SYMV tiles, 2 = coarse SYMV tiles, 3 = grain supernodal solve, 4 =
 * contact-grid supernodal solve, 5 = ILU(0) apply = forward + backward sweep,
 * 6 = element-by-element fine operator, 7 = stored-block BSR SpMV; for 6 / 7
 * tile_bytes = the algorithmic bytes of one y = A^ x apply):
 * total device ms and launch count since the last reset; tile_bytes = factor
 * bytes one launch streams. */
hplmm_status hplmm_kernel_stats(hplmm_handle *h, int32_t kernel, double *total_ms,
                                int64_t *launches, int64_t *tile_bytes);

void hplmm_destroy(hplmm_handle *h);
const char *hplmm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HPLMM_H */
