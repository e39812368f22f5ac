"""Exception types of the drop-in, same names and hierarchy as the reference
(/root/reference/pkg/src/fuzzdepth/errors.py:9-30) so callers catching the
reference's exceptions keep working.

When the reference package is importable, its classes are re-used so that
`except fuzzdepth.ValidationError` catches errors raised here too.
"""
from __future__ import annotations

try:  # pragma: no cover - depends on the caller's environment
    from fuzzdepth.errors import (  # type: ignore[import-not-found]
        DegenerateEnsembleError,
        FuzzdepthError,
        GridMismatchError,
        ManifestError,
        ValidationError,
        VolumeFormatError,
    )
except Exception:  # the reference is not installed: define the same hierarchy

    class FuzzdepthError(Exception):
        """Base class for every deliberate error of the depth path."""

    class ValidationError(FuzzdepthError):
        """Input violates a documented precondition (range, shape, config)."""

    class GridMismatchError(FuzzdepthError):
        """Two objects that must share a grid do not."""

    class DegenerateEnsembleError(FuzzdepthError):
        """The ensemble cannot support the statistic (e.g. all-zero mean mask)."""

    class VolumeFormatError(FuzzdepthError):
        """A volume container is corrupt or unsupported (kept for API parity)."""

    class ManifestError(FuzzdepthError):
        """An ensemble manifest is malformed (kept for API parity)."""


__all__ = [
    "FuzzdepthError",
    "ValidationError",
    "GridMismatchError",
    "DegenerateEnsembleError",
    "VolumeFormatError",
    "ManifestError",
]
