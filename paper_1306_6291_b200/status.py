"""The per-matrix status byte (include/symdiag_b200.h) and its mapping back
to the reference's branch enum and exception taxonomy.

Bits 0-3 = outcome code, bit 4/5 = selected sign of phi2/phi3 is -1,
bit 6 = near_tie, bit 7 = polished.  Error codes are the exceptions
`diagonalize3` lets escape.
"""

from __future__ import annotations

import numpy as np

CODE_MASK = 0x0F
GENERIC, ALREADY_DIAGONAL_2D, DOUBLE_ROOT, TRIPLE_ROOT = 0, 1, 2, 3
STAGE_DEGENERATE_EIGENVALUES, STAGE_BOTH_F_ZERO = 6, 7
ERR_FIRST = 8
(ERR_NONFINITE_INPUT, ERR_P_NEGATIVE, ERR_ACOS_SLACK, ERR_DOMAIN_EXCURSION,
 ERR_NOT_DOUBLE_ROOT, ERR_ANGLE_OF_ZERO, ERR_MATH_DOMAIN, ERR_OVERFLOW) = range(8, 16)
FLAG_S2_NEG, FLAG_S3_NEG, FLAG_NEAR_TIE, FLAG_POLISHED = 0x10, 0x20, 0x40, 0x80

CODE_NAMES = {
    GENERIC: "Generic", ALREADY_DIAGONAL_2D: "AlreadyDiagonal2D",
    DOUBLE_ROOT: "DoubleRoot", TRIPLE_ROOT: "TripleRoot",
    STAGE_DEGENERATE_EIGENVALUES: "DegenerateEigenvalues",
    STAGE_BOTH_F_ZERO: "BothFVectorsZero",
    ERR_NONFINITE_INPUT: "NonFiniteInput", ERR_P_NEGATIVE: "ValueError(p negative)",
    ERR_ACOS_SLACK: "ValueError(arccos slack)", ERR_DOMAIN_EXCURSION: "DomainExcursion",
    ERR_NOT_DOUBLE_ROOT: "NotDoubleRoot", ERR_ANGLE_OF_ZERO: "AngleOfZeroVector",
    ERR_MATH_DOMAIN: "ValueError(math domain error)", ERR_OVERFLOW: "OverflowError",
}


def code(status):
    return np.asarray(status) & CODE_MASK


def is_error(status):
    return code(status) >= ERR_FIRST


def signs(status):
    """Selected (sign2, sign3) per row as int arrays of +-1."""
    s = np.asarray(status)
    return (np.where(s & FLAG_S2_NEG, -1, 1), np.where(s & FLAG_S3_NEG, -1, 1))


def near_tie(status):
    return (np.asarray(status) & FLAG_NEAR_TIE) != 0


def polished(status):
    return (np.asarray(status) & FLAG_POLISHED) != 0


def exception_for(code_value: int, where: str = ""):
    """The exception instance the reference raises for an error code."""
    from . import core, eig3
    c = int(code_value) & CODE_MASK
    msg = f"{CODE_NAMES.get(c, c)}{(' in ' + where) if where else ''}"
    if c == ERR_NONFINITE_INPUT:
        return core.NonFiniteInput(msg)
    if c == ERR_P_NEGATIVE:
        return ValueError("p is negative beyond rounding tolerance")
    if c == ERR_ACOS_SLACK:
        return ValueError("arccos argument out of range beyond slack")
    if c == ERR_DOMAIN_EXCURSION:
        return eig3.DomainExcursion(msg)
    if c == ERR_NOT_DOUBLE_ROOT:
        return eig3.NotDoubleRoot("repeated and distinct eigenvalues coincide")
    if c == ERR_ANGLE_OF_ZERO:
        return core.AngleOfZeroVector("angle_of requires a nonzero vector")
    if c == ERR_MATH_DOMAIN:
        return ValueError("math domain error")
    if c == ERR_OVERFLOW:
        return OverflowError(34, "Numerical result out of range")
    if c == STAGE_DEGENERATE_EIGENVALUES:
        return eig3.DegenerateEigenvalues(msg)
    if c == STAGE_BOTH_F_ZERO:
        return eig3.BothFVectorsZero("matrix is diagonal with two equal entries")
    return None


def raise_for(code_value: int, where: str = ""):
    exc = exception_for(code_value, where)
    if exc is not None:
        raise exc
