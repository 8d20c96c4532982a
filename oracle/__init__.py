"""CPU oracle for the CVA / PCA hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference ``undertext`` hot path
(``/root/reference/pkg/src/undertext``): scatter, regularized generalized
eigensolve, unsupervised PCA covariance, per-pixel projection and the full-range
uint8 stretch.  It exists to *check* the B200 implementation, never to stand in
for it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
  ``--impl reference`` arm may import it;
* the product package ``paper_1612_06457_b200`` never imports it and fails loudly
  when its CUDA library is missing.

Parity pinning: every function here is checked bit-for-bit (or to 1e-12 where a
BLAS reduction order may differ between machines) against golden vectors that
``tests/golden/make_golden.py`` produced by importing and running the real
reference in the build container (``tests/golden/*.npz``).  See DESIGN.md §3.
"""

from .cva_pca import (  # noqa: F401
    OracleError,
    OracleNumericError,
    assemble,
    cpu_cva_pipeline,
    cpu_pca_pipeline,
    fit_cva,
    fit_lda,
    fit_pca_unsupervised,
    gen_eig_sym,
    linear_to_codes,
    nearest_rank,
    normalize_stack,
    rescale_percentile,
    rescale_training_range,
    project,
    regularize,
    rescale_full,
    round_half_away,
    scatter,
    sign_normalize,
    standardize,
)
