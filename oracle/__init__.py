"""CPU oracle for the batched power-flow hot path -- TEST INFRASTRUCTURE ONLY.

A plain numpy/scipy restatement of the reference package's algorithm
(arxiv 2605.14103, `acpflow`, pkg/src/acpflow/*.py), each function citing the
reference file:line it follows. It exists to *check* the CUDA path, never to
be it: only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
``--impl reference`` arm may import it. The product package
(paper_2605_14103_b200) never imports this module and has no CPU fallback.

Parity status: PINNED. tests/test_oracle_golden.py checks this restatement
against golden vectors produced by running the real reference in the build
container (tools/make_golden.py -> tests/golden/*.npz): identical Newton /
fixed-point flags and iteration counts, states within 1e-10.

Third-party arithmetic the reference delegates (and this restatement uses
the same way): LAPACK getrf/getrs via scipy.linalg.lu_factor/lu_solve,
scipy sparse CSR products, numpy Philox4x64-10.
"""
