"""CPU oracle for the exact-gradient evaluation of arXiv 2104.12282 (ONSG).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or run
anything in this package.  The CUDA product path (``paper_2104_12282_b200``)
never imports it, and this package never imports the product path: the two
share no code.  The only shared module is the seeded input generator
``paper_2104_12282_b200/inputs.py``, which holds none of the method's
arithmetic.

Plain, slow, obviously correct fp64 NumPy/SciPy, following the paper's
definitions in the paper's order:

* ``grid``   numbering, element->DOF map, BC presets         ("K(z)u - f = 0")
* ``fem``    KE by 2x2x2 Gauss quadrature of B^T C B, SIMP, sparse assembly, matrix-free
             element loop, fixed DOFs as identity rows/cols
* ``solve``  direct sparse solve (the plain definition u = K^-1 f) and textbook
             Jacobi-PCG
* ``sens``   compliance f^T u (Eq. 4), sensitivity Eq. 5
* ``filt``   density filter P as an explicit sparse matrix; P x, P^T v, dv = P^T 1
                                                             
* ``oc``     optimality-criteria update, canonical bisection
* ``loop``   one exact-gradient evaluation and the SIMP loop (Eq. 2, 133-138 Alg. 1)
* ``twoscale`` block averaging and BC restriction of the coarse path
* ``mg``     Galerkin multigrid hierarchy and MG-preconditioned CG (SURVEY f2,
             reading R5) - pinned by linear reproduction of P, the coarse rigid-body null
             space and agreement with the direct solve

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): KE closed-form entries and
spectrum, rigid-body null space, patch test, golden tiny compliances,
Euler-Bernoulli/Timoshenko refinement, finite-difference sensitivities, the
homogeneity identity, filter closed forms, OC invariants, PCG toy systems.
Functions without an independent pin say "parity unpinned" in their docstring.
"""
