"""Exception taxonomy of holoquant (reference proj/include/holoquant/errors.hpp).

Names and meanings are the reference's so call sites read the same:
ShapeError (errors.hpp:10-13), ValueError (15-18), ContractError (20-23),
FormatError with .fault/.offset (37-55), PlanError (58-60).  Each also
derives from the closest Python builtin.
"""
from __future__ import annotations

import builtins
import enum


class HoloquantError(Exception):
    """Base of every error raised by this package."""


class ShapeError(HoloquantError, builtins.ValueError):
    """Dimension / length mismatch."""


class ValueError(HoloquantError, builtins.ValueError):  # noqa: A001 - mirrors holoquant::ValueError
    """Numeric contract violation (e.g. spline evaluated at non-finite x)."""


class ContractError(HoloquantError, RuntimeError):
    """Misuse of an API contract (undersized workspace, bad tables)."""


class PlanError(HoloquantError, RuntimeError):
    """Memory-plan arithmetic overflow or degenerate header."""


class CudaError(HoloquantError, RuntimeError):
    """Device failure (no reference counterpart)."""


class FormatFault(enum.IntEnum):
    """holoquant::FormatFault (errors.hpp:37-45), same order."""
    BadMagic = 0
    BadVersion = 1
    BadEndianness = 2
    BadHeader = 3
    Truncated = 4
    IndexOutOfRange = 5
    BadQuantParam = 6


class FormatError(HoloquantError, RuntimeError):
    """Malformed SKAN file; carries the fault kind and byte offset."""

    def __init__(self, fault: FormatFault, offset: int, msg: str):
        super().__init__(msg)
        self.fault = fault
        self.offset = offset


def from_status(status: int, msg: str, offset: int = 0, fault: int = -1) -> HoloquantError:
    if status == 1:
        return ShapeError(msg)
    if status == 2:
        return ValueError(msg)
    if status == 3:
        return ContractError(msg)
    if status == 4:
        return FormatError(FormatFault(fault), offset, msg)
    if status == 5:
        return PlanError(msg)
    return CudaError(msg)
