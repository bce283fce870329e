"""CPU oracle for the EpiRK/Krylov hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain NumPy (plus ``scipy.linalg.expm`` for the
small dense exponential, exactly as the reference does), the algorithm of the
reference package ``expmhd`` (``/root/reference/pkg/src/expmhd``) for the four
pieces of the hot path:

* ``oracle.stencil``  — the 2.5D resistive-MHD right-hand side
  (reference ``mhd.py:99-285``), bit-for-bit: same operation order, no FMA;
* ``oracle.jvp``      — the forward-difference Jacobian action
  (reference ``fdjac.py:19-49``);
* ``oracle.krylov_cpu`` — Arnoldi with modified Gram–Schmidt plus one
  re-orthogonalisation pass, the residual surrogate, multi-scale phi
  evaluation and the augmented-operator phi combination with adaptive substeps
  (reference ``krylov.py:127-383``, ``phifuncs.py:65-107``);
* ``oracle.epirk_cpu`` — the EPIRK4 / EPIRK5P1 steps and the fixed and
  adaptive drivers that call the path (reference ``epirk.py:134-411``).

Who may use it: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg — as the checker or as the timed
CPU baseline, never as the thing measured or shipped.  The product package
``paper_1604_02614_b200`` never imports this package.

Pinning: ``tests/golden/make_golden.py`` imports the unmodified reference from
``/root/reference/pkg/src`` (available only in the build container) and writes
the fixtures under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks
this restatement against them (bitwise for the RHS and Jv, to round-off for
the Krylov and EpiRK layers whose BLAS summation order is not fixed).

Third-party arithmetic on the path (not vendored in the reference): numpy
2.3.5 (OpenBLAS ``ddot``/``dgemv`` through ``np.dot``/``@``) and scipy 1.18.1
(``scipy.linalg.expm``, Al-Mohy & Higham 2009 Padé scaling and squaring).
"""
