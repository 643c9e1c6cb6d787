"""fp64 CPU oracle of the NAT Helmholtz boundary-integral hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product (``paper_2506_06190_b200``) imports,
links or executes this package; only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may.  It shares no
code, table or constant generator with the CUDA path; the only thing both sides use
is ``nat_inputs`` (seeded input arrays, no arithmetic of the method).

Plain, slow, obviously correct: NumPy in float64 / complex128, each function following
the passage of ``PAPER.md`` it cites (``P:n`` = line n) and, where the paper is silent,
the reading recorded in ``DESIGN.md`` §3 (taken from SURVEY.md §8(c)).

Modules
  kernel     G, dG/dn_y
  geometry   a1 mesh preparation
  quadrature triangle rules, subdivision, polar self term
  nearlist   a2 near list, brute force           ("adjacent or identical elements")
  bem        a4+a5 collocation assembly, a6 matvec (Eq. BM with beta = 0)
  gmres      a7 unrestarted GMRES (MGS)
  philox     Philox4x32-10 counter RNG            (Salmon et al. SC'11)
  mc         a8 sampling, a9/a10 MC system       (Eq. BIE / SYS / DISK)
  radiate    a11 exterior representation formula (coefficient 1)
  listeners  a12 listener shell grid
  analytic   closed forms used only as pins      (sphere solutions, eigenvalues)

Parity status per function is listed in DESIGN.md §3 ("pinned by"); the MC sample
realisation and the modal Neumann fields are "parity unpinned" pointwise (statistical
pins only), as stated there.
"""
