"""Plain fp64 CPU oracle for FB-LTS (arXiv 2405.10505) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()``, ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs and ``scripts/cfl_scan.py`` (which writes the stored time steps of
``configs/dt.json`` from oracle calls only) may import this package.  The product path
(``paper_2405_10505_b200``) never imports it, and this package never imports the
product path: they share no code (only the seeded input generators in
``inputs/``, which hold none of the method's arithmetic).

It is a literal, slow, numpy transcription of PAPER.md:
  * ``trisk``   -- TRiSK operators Psi_i (eq. trisk_thickness),
                   Phi^fast (eq. fast_terms) and the slow terms
                   (eq. nonlinear_swe, eq. trisk_vorticity P:L1044-1060,
                   eq. splitting);
  * ``fbrk32``  -- global FB-RK(3,2) (eq. fbrk32), split and unsplit,
                   plus classical RK4 as a convergence reference;
  * ``lts``     -- LTS region labelling and the four FB-LTS phases
                    in the original mesh order, with explicit region
                   masks and NaN outside every phase's extent;
  * ``diagnostics`` -- mass, absolute vorticity (Theorems 1-2),
                   RMS error (eq. rmse), Courant numbers (eq. cfl).

Every reading of an ambiguous passage follows SURVEY.md section 8(c) c.4 and is
listed in DESIGN.md.  Canonical evaluation order (so that a faithful GPU
implementation can agree bit for bit): every sum is sequential in stored slot
order starting from +0.0; expressions are evaluated left to right exactly as
written in the functions below; no fused multiply-add (numpy never contracts).

Parity status: every function is pinned by tests in tests/test_oracle_*.py
(see DESIGN.md "Oracle pins").  Nothing here is "parity unpinned" except the
conventions listed in DESIGN.md (q-hat, edge thickness, KE quadrature closures),
which no printed value in the paper fixes.
"""
