"""CPU oracle for the per-histogram compress/decompress hot path.

TEST INFRASTRUCTURE ONLY.  This package is a plain numpy + C restatement
of the reference (`/root/reference/pkg/src/mlk`, arXiv 2212.10733) used as
the parity checker for the B200 path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it; the product package
``paper_2212_10733_b200`` never does.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference in
the build container (compiled Cython backend, ``OPENBLAS_NUM_THREADS=1``)
and commits its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this restatement against them.
"""
