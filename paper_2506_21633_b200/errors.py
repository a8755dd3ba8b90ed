"""Exception hierarchy of the drop-in (mirrors sarsplat/validation.py:12-33).

The classes have the reference's names and bases so callers' ``except``
clauses keep working when they switch packages.
"""
from __future__ import annotations


class SarsplatError(Exception):
    """Base class for all package-specific errors."""


class InvalidParameterError(SarsplatError, ValueError):
    """An input value violates a documented precondition."""


class DegenerateProjectionError(SarsplatError, ArithmeticError):
    """A projected 2D covariance is singular or indefinite."""


class NumericalError(SarsplatError, ArithmeticError):
    """A non-finite value appeared mid-computation."""


class StateError(SarsplatError, RuntimeError):
    """An operation was called without the forward state it requires."""


class DivergenceError(SarsplatError, RuntimeError):
    """Training produced non-finite losses twice in a row."""


class DeviceError(SarsplatError, RuntimeError):
    """A CUDA launch or runtime failure inside libsdgr."""
