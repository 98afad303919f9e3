"""Exception hierarchy of the drop-in API.

Mirrors the reference's error contract (``pkg/src/treesmpc/errors.py:4-26``):
malformed documents raise :class:`ParseError`, invariant violations raise
:class:`ValidationError` carrying the full list of violations, shape mismatches
raise :class:`DimensionError`.  Native status codes from ``libtsmpc`` are mapped
onto the same classes (see ``_native.py``); device faults raise
:class:`DeviceError`.
"""

from __future__ import annotations


class TreeSmpcError(Exception):
    """Root of every error raised by this package."""


class ParseError(TreeSmpcError):
    """An input document could not be decoded (bad JSON, missing keys, shapes)."""


class ValidationError(TreeSmpcError):
    """Input decoded but breaks a model/tree/config invariant.

    ``violations`` holds every failed check, in the order they were found.
    """

    def __init__(self, violations):
        items = [violations] if isinstance(violations, str) else list(violations)
        self.violations = items
        super().__init__("; ".join(items))


class DimensionError(TreeSmpcError):
    """Two operands disagree in shape."""


class DeviceError(TreeSmpcError):
    """The CUDA path failed (no device, launch failure, out of memory)."""


__all__ = ["TreeSmpcError", "ParseError", "ValidationError", "DimensionError",
           "DeviceError"]
