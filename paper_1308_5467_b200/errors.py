"""Exception types of the reference (specdens/errors.py:1-9), re-declared.

If the reference package is importable in the same process its classes are
reused, so ``except specdens.NumericalFailure`` catches errors raised here.
"""

try:  # pragma: no cover - depends on the environment
    from specdens.errors import NumericalFailure, OracleCapExceeded  # type: ignore
except Exception:  # the reference is not installed (e.g. on the GPU box)

    class NumericalFailure(RuntimeError):
        """A computation produced non-finite or otherwise unusable numbers."""

    class OracleCapExceeded(RuntimeError):
        """A dense reference computation was requested above its size cap."""


__all__ = ["NumericalFailure", "OracleCapExceeded"]
