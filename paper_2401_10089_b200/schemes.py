"""Evaluation schemes of the degree-optimal graph polynomial (the reference's ``GraphScheme``
surface, logmpoly/schemes.py:31-126 and 240-321), host side.

A scheme with k products: P1 = I, P2 = X, P_{j+2} = (sum_i lhs[j][i] P_i)(sum_i rhs[j][i] P_i)
for j = 0..k-1 (row j has j + 2 coefficients), output z(X) = sum_i out[i] P_i (k + 2
coefficients).  ``eval_degopt`` (primitives.py) evaluates any such scheme with k <= 9 on the
GPU (lgm_eval_degopt_scheme_f64); the shipped ones are ``builtin_scheme(k)``.

Text format (what the reference's save_scheme writes and load_scheme reads): ``#`` comment
lines, ``key value`` header lines (k, m_order, degree, radius, target), then a line ``H``
followed by the k lhs rows, ``G`` and the k rhs rows, ``y`` and the output row; doubles with 17
significant digits so a write / read round trip is exact.
"""
import math
from dataclasses import dataclass, field

from . import constants as C
from .exceptions import SchemeFormatError


@dataclass(frozen=True)
class SchemeMeta:
    order_label: str = ""
    degree: int = 0
    target: str = "neglog1m"
    radius: float = 0.0
    provenance: str = ""

    @property
    def order(self):
        label = self.order_label[:-1] if self.order_label.endswith("+") else self.order_label
        return int(label) if label else 0


@dataclass(frozen=True)
class GraphScheme:
    lhs: tuple
    rhs: tuple
    out: tuple
    meta: SchemeMeta = field(default_factory=SchemeMeta)

    def __post_init__(self):
        k = len(self.lhs)
        shape_ok = len(self.rhs) == k and len(self.out) == k + 2
        if not shape_ok:
            raise SchemeFormatError(f"scheme shape: {k} lhs rows, {len(self.rhs)} rhs rows, "
                                    f"{len(self.out)} output coefficients (want k, k, k + 2)")
        for j in range(k):
            if len(self.lhs[j]) != j + 2 or len(self.rhs[j]) != j + 2:
                raise SchemeFormatError(f"product {j + 1}: lhs / rhs rows need {j + 2} coefficients")
        if any(not math.isfinite(v) for row in (*self.lhs, *self.rhs, self.out) for v in row):
            raise SchemeFormatError("non-finite scheme coefficient")

    @property
    def mults(self):
        return len(self.lhs)

    @property
    def degree(self):
        return 2 ** self.mults

    @property
    def is_normalized(self):
        """P3 = X^2 exactly: the one-product saving with a known first product applies."""
        return tuple(self.lhs[0]) == (0.0, 1.0) and tuple(self.rhs[0]) == (0.0, 1.0)

    def flat(self):
        """lhs rows, rhs rows, out: the coefficient layout of the C ABI."""
        return [float(v) for row in (*self.lhs, *self.rhs, self.out) for v in row]


def _g17(x):
    return "%.17g" % x


def save_scheme(scheme, comment=""):
    text = ["# logmpoly evaluation-scheme coefficients"]
    text += [f"# {c}" for c in (comment or scheme.meta.provenance).splitlines()]
    text += [f"k {scheme.mults}",
             f"m_order {scheme.meta.order_label or scheme.degree}",
             f"degree {scheme.meta.degree or scheme.degree}",
             f"radius {_g17(scheme.meta.radius)}",
             f"target {scheme.meta.target}"]
    for tag, rows in (("H", scheme.lhs), ("G", scheme.rhs), ("y", (scheme.out,))):
        text.append(tag)
        text += [" ".join(_g17(v) for v in row) for row in rows]
    return "\n".join(text) + "\n"


def load_scheme(text):
    data = [s for s in (ln.strip() for ln in text.splitlines()) if s and s[0] != "#"]
    pos = 0
    header = {}
    while pos < len(data) and data[pos].split()[0] not in ("H", "G", "y"):
        key, _, value = data[pos].partition(" ")
        if not value.strip():
            raise SchemeFormatError(f"header line without a value: {data[pos]!r}")
        header[key] = value.strip()
        pos += 1
    if "k" not in header or not header["k"].lstrip("-").isdigit():
        raise SchemeFormatError("header needs an integer 'k'")
    k = int(header["k"])

    def block(tag, lengths):
        nonlocal pos
        if pos >= len(data) or data[pos] != tag:
            raise SchemeFormatError(f"block {tag!r} expected")
        pos += 1
        rows = []
        for want in lengths:
            if pos >= len(data):
                raise SchemeFormatError(f"block {tag!r} ends early")
            toks = data[pos].split()
            if len(toks) != want:
                raise SchemeFormatError(f"block {tag!r}: a row of {want} coefficients expected, got {len(toks)}")
            try:
                rows.append(tuple(float(t) for t in toks))
            except ValueError:
                raise SchemeFormatError(f"block {tag!r}: unreadable coefficient") from None
            pos += 1
        return tuple(rows)

    lhs = block("H", [j + 2 for j in range(k)])
    rhs = block("G", [j + 2 for j in range(k)])
    (out,) = block("y", [k + 2])
    meta = SchemeMeta(order_label=header.get("m_order", ""), degree=int(header.get("degree", 2 ** k)),
                      target=header.get("target", "neglog1m"), radius=float(header.get("radius", 0.0)))
    return GraphScheme(lhs=lhs, rhs=rhs, out=out, meta=meta)


def read_scheme(path):
    with open(path) as fh:
        return load_scheme(fh.read())


def write_scheme(path, scheme, comment=""):
    with open(path, "w") as fh:
        fh.write(save_scheme(scheme, comment))


_BUILTIN = {}


def builtin_scheme(k):
    """Shipped scheme with k products (constants.SCHEMES): k = 1..5 the reference's files, k = 6..9
    generated by the reference's fit_minmax (data/scheme_k*.txt, tools/gen_schemes.py)."""
    k = int(k)
    if k not in _BUILTIN:
        if not 1 <= k <= len(C.SCHEMES):
            raise ValueError(f"no built-in scheme with k={k}")
        lhs, rhs, out = C.SCHEMES[k - 1]
        _BUILTIN[k] = GraphScheme(lhs=tuple(map(tuple, lhs)), rhs=tuple(map(tuple, rhs)), out=tuple(out),
                                  meta=SchemeMeta(order_label=str(C.ORDER[k - 1]), degree=2 ** k))
    return _BUILTIN[k]


__all__ = ["GraphScheme", "SchemeMeta", "builtin_scheme", "load_scheme", "read_scheme", "save_scheme",
           "write_scheme"]
