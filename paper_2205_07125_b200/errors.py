"""Exception contract of the drop-in API.

Mirrors ``neurocomm/errors.py:4-19``: every error a caller can trigger is a
``ValueError`` subclass, so ``except ValueError`` in reference-facing code
keeps working.  Native failures (CUDA errors, exchange watchdog timeouts)
surface as ``RuntimeError`` through :mod:`._native`.
"""

from __future__ import annotations


class SpecificationError(ValueError):
    """A configuration value is outside its documented range (errors.py:4)."""


class ParseError(ValueError):
    """Malformed data file; ``line`` is the 1-based offending line (errors.py:8-15)."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


class MissingBridgeError(ValueError):
    """An inter-group demand has no bridge for its group pair (errors.py:18-19)."""
