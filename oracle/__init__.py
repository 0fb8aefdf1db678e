"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation (numpy/scipy, fp64) of
what the B200 hot path computes, written from the paper (PAPER.md, arXiv
1009.4975) and the readings listed in DESIGN.md / SURVEY.md §8(c).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything from here.
The product package ``paper_1009_4975_b200`` never imports it, and this
package imports nothing from the product (shared: only ``inputs/``, which
holds no method arithmetic).

Modules
-------
mesh     2:1 balance (C10), canonical numbering (C2-C5), hanging-node
         constraints (C6, Eq. 6), fixed DOFs (C7), consistent
         loads (C8), filter neighbourhoods (C9).
fe       element stiffness by Gauss quadrature, SIMP (Eq. 2), assembled K,
         constraint matrix C, projected operator A (Eq. 8) and rhs, recovery
         (Eq. 9), compliance (Eq. 1).
solve    textbook Jacobi-PCG (PAPER.md:511-523 rescaling reading), CG on the
         explicitly rescaled system, dense direct solve.
topopt   sensitivities, Sigmund/Stainko filter
         (Eqs. 3-5) and the DENS variant, brute-force twins.
oc       OC design update with the bisection on the volume multiplier
         (reading R18) and the Fig. 1 loop with
         p-continuation (reading R19).
amr      the dynamic AMR strategy: adaptation trigger,
         marking with r_amr, the two compatibility sweeps, refine/derefine
         with density transfer (readings R21-R23), and Fig. 1 with AMR.
sample   one-by-one evaluation of rows of A, sensitivities and filter outputs
         for full-size configurations (parity on sampled outputs).

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
(closed forms, invariants, brute force, paper numbers).  The synthetic
refinement rule R lives in ``inputs/`` (input generation, not method).
"""
