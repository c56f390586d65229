"""Module alias for the reference's ``specdens.matrix`` (matrix.py:1-331).

The operator types live in ``operators.py`` and the test-matrix generator in
``workloads.py``; this module re-exports them under the reference's module
name so ``from specdens.matrix import ...`` call sites keep working.
"""

from .operators import (  # noqa: F401
    DEFAULT_INTERVAL_MARGIN,
    DEFAULT_LANCZOS_STEPS,
    MappedOperator,
    MatvecCounter,
    SparseSymmetricMatrix,
    StencilOperator,
    apply_spectral_map,
    as_operator,
    estimate_spectral_interval,
    load_matrix_market,
    save_matrix_market,
)
from .workloads import DEFAULT_BUMPS, generate_modified_laplacian_2d  # noqa: F401
