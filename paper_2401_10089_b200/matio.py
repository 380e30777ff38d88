"""Plain-text matrix I/O in the reference's format (``logmpoly/matcore.py:362-431``).

Format: first non-comment line holds n, then n rows of n whitespace-separated scalars;
blank lines and lines starting with ``#`` are ignored.  Reals are written with 17
significant digits (``%.17g``, round-trip exact); complex entries as ``re+imi``.  Malformed
input raises ``SchemeFormatError`` (a ``ValueError``), as in the reference.
"""
import numpy as np

from .exceptions import SchemeFormatError


def _fmt(x):
    if np.iscomplexobj(x):
        z = complex(x)
        return f"{z.real:.17g}{z.imag:+.17g}i"
    return f"{float(x):.17g}"


def _token(tok):
    t = tok.strip()
    if t[-1:] in ("i", "I"):
        body = t[:-1]
        # the imaginary part starts at the last sign that is not an exponent sign
        cut = next((k for k in range(len(body) - 1, 0, -1) if body[k] in "+-" and body[k - 1] not in "eE"), -1)
        if cut <= 0:
            raise SchemeFormatError(f"malformed complex token: {tok!r}")
        try:
            return complex(float(body[:cut]), float(body[cut:]))
        except ValueError as exc:
            raise SchemeFormatError(f"malformed complex token: {tok!r}") from exc
    try:
        return float(t)
    except ValueError as exc:
        raise SchemeFormatError(f"malformed scalar token: {tok!r}") from exc


def _square(A):
    A = np.asarray(A)
    if A.ndim != 2 or A.shape[0] != A.shape[1] or A.shape[0] < 1:
        raise ValueError(f"matrix must be square, got shape {A.shape}")
    if not np.all(np.isfinite(A)):
        raise ValueError("matrix has non-finite entries")
    return A.astype(np.complex128 if np.iscomplexobj(A) else np.float64)


def format_matrix(A):
    """Text form of a square matrix (matcore.py:393-401)."""
    A = _square(A)
    rows = [" ".join(_fmt(x) for x in row) for row in A]
    return "\n".join([str(A.shape[0])] + rows) + "\n"


def parse_matrix(text):
    """Inverse of ``format_matrix`` (matcore.py:404-421)."""
    lines = [ln for ln in text.splitlines() if ln.strip() and not ln.lstrip().startswith("#")]
    if not lines:
        raise SchemeFormatError("empty matrix file")
    try:
        n = int(lines[0].strip())
    except ValueError as exc:
        raise SchemeFormatError(f"bad dimension line: {lines[0]!r}") from exc
    if n < 1 or len(lines) < n + 1:
        raise SchemeFormatError(f"expected {n} rows, found {len(lines) - 1}")
    rows = []
    for ln in lines[1:n + 1]:
        toks = ln.split()
        if len(toks) != n:
            raise SchemeFormatError(f"expected {n} entries per row, got {len(toks)}")
        rows.append([_token(t) for t in toks])
    vals = np.array(rows)
    return _square(vals if np.iscomplexobj(vals) else vals.astype(np.float64))


def write_matrix(path, A):
    with open(path, "w") as fh:
        fh.write(format_matrix(A))


def read_matrix(path):
    with open(path) as fh:
        return parse_matrix(fh.read())
