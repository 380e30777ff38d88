"""Plain-text matrix files, byte-compatible with the reference's serializer.

Written from the format statement in SPEC.md:125 (the reference implements it in
``logmpoly/matcore.py:362-431``): a size line ``n``, then ``n`` lines of ``n``
whitespace-separated decimal scalars; a complex scalar is one token ``<re><sign><im>i``;
reals carry 17 significant digits so every double round-trips exactly.  Lines that are
blank or whose first non-blank character is ``#`` carry no data.  Byte equality with the
reference's writer is pinned by ``tests/golden/matio_ref*.txt``.

Grammar used by the reader (one token)::

    real    := python float literal (what ``float()`` accepts)
    complex := NUM SIGN UNUM "i"        NUM = [sign] digits[.digits][e[sign]digits]

Anything else -- or a file whose row / column counts disagree with its size line -- raises
``SchemeFormatError`` (a ``ValueError``); non-finite values are rejected like ``as_square``.
"""
import re

import numpy as np

from .exceptions import SchemeFormatError

_UNUM = r"(?:\d+(?:\.\d*)?|\.\d+)(?:[eE][+-]?\d+)?"
_COMPLEX = re.compile(rf"^(?P<re>[+-]?{_UNUM})(?P<im>[+-]{_UNUM})[iI]$")


def _text_of(x, is_complex):
    if is_complex:
        z = complex(x)
        return "%.17g%+.17gi" % (z.real, z.imag)
    return "%.17g" % float(x)


def _value_of(token):
    if token[-1] in "iI":
        m = _COMPLEX.match(token)
        if m is None:
            raise SchemeFormatError(f"cannot read complex scalar {token!r}")
        return complex(float(m.group("re")), float(m.group("im")))
    try:
        return float(token)
    except ValueError:
        raise SchemeFormatError(f"cannot read scalar {token!r}") from None


def _checked(M):
    M = np.asarray(M)
    if M.ndim != 2 or M.shape[0] < 1 or M.shape[0] != M.shape[1]:
        raise ValueError(f"matrix must be square, got shape {M.shape}")
    if not np.isfinite(M).all():
        raise ValueError("matrix has non-finite entries")
    return M.astype(np.complex128) if np.iscomplexobj(M) else M.astype(np.float64)


def format_matrix(A):
    """Serialize one square matrix (size line, then one line per row, trailing newline)."""
    M = _checked(A)
    cplx = np.iscomplexobj(M)
    out = [f"{M.shape[0]}"]
    out.extend(" ".join(_text_of(v, cplx) for v in row) for row in M)
    out.append("")
    return "\n".join(out)


def _data_lines(text):
    for raw in text.splitlines():
        s = raw.strip()
        if s and not s.startswith("#"):
            yield s


def parse_matrix(text):
    """Read the text form back (inverse of ``format_matrix``; exact for doubles)."""
    lines = _data_lines(text)
    head = next(lines, None)
    if head is None:
        raise SchemeFormatError("no data in matrix text")
    if not head.isdigit():
        raise SchemeFormatError(f"first data line must be the size n, got {head!r}")
    n = int(head)
    if n == 0:
        raise SchemeFormatError("matrix size must be at least 1")
    entries = []
    for r in range(n):
        line = next(lines, None)
        if line is None:
            raise SchemeFormatError(f"size line says {n} rows, text ends after {r}")
        toks = line.split()
        if len(toks) != n:
            raise SchemeFormatError(f"row {r} has {len(toks)} entries, size line says {n}")
        entries.append([_value_of(t) for t in toks])
    vals = np.array(entries)
    return _checked(vals)


def write_matrix(path, A):
    text = format_matrix(A)
    with open(path, "w") as fh:
        fh.write(text)


def read_matrix(path):
    with open(path) as fh:
        return parse_matrix(fh.read())
