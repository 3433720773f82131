"""CPU oracle for the split-step propagation path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy/scipy (plus one plain-C file), the algorithm
of the reference package `ctapsim` (arXiv:1309.2451) for exactly the hot path
that paper_1309_2451_b200 re-implements on the B200.  It is the checker, never
the product: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
/ `--impl reference` arm may import it.  The product package never imports
anything from here and fails loudly when libctap.so is missing.

Pinning: every function is checked against golden vectors produced by running
the reference itself in the build container (tests/golden/make_golden.py,
fixtures in tests/golden/*.npz, test tests/test_oracle_golden.py).

Third-party arithmetic the reference delegates (named with pinned versions,
see DESIGN.md §Oracle):
  * 3D FFT: scipy.fft.fftn/ifftn (pocketfft) -- scipy 1.18.1 in this image;
    the reference pins only scipy>=1.10 (pkg/pyproject.toml:12).
  * phase factors: numpy complex exp -- numpy 2.3.5.
  * potential: numba 0.65 JIT of magfield._potential_kernel; restated here in
    C (oracle/potential.c), which is bit-identical to the numba kernel.
"""
