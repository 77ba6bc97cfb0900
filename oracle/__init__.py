"""CPU oracle for the hPLMM-preconditioned GMRES path (arXiv 2509.19777).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path
(``paper_2509_19777_b200/``) may import, call, link or execute anything under
``oracle/``; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs do.  The oracle shares no code with
the CUDA path; the only shared module is ``workloads`` (seeded inputs, no
method arithmetic).

Plain, slow, obviously-correct fp64 NumPy/SciPy code, following PAPER.md step
by step.  Citations use ``P:<line>`` for PAPER.md lines and the LaTeX label of
the equation; readings where the paper is silent are SURVEY.md §8(c)'s R1-R24
(restated in DESIGN.md "Readings").

Modules
  fem     Q1 element matrix, mesh numbering, assembly, Dirichlet BCs
  decomp  node classes, contact interfaces, contact grids (§3.1)
  mortar  mortar-node placement and Gaussian mortars (eq:node_init, eq:gauss)
  hplmm   Q^o, P^ = WQP, coarse operator, M_G, M_zeta, M_g, M_CG, M
          (eq:reduced_defs .. eq:Mg_Mz, eq:multi_precond)
  gmres   right-preconditioned GMRES(50) with CGS2 + Givens (R22)

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` except the GMRES iteration COUNT, which the paper
cannot pin (its datasets are absent): "parity unpinned" for the iteration
count only (DESIGN.md §Oracle pins).
"""
