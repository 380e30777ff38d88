"""GraphScheme surface on the host (schemes.py:31-126, 240-321): the coefficient-file format
round trip, the shape / finiteness checks and the shipped schemes."""
import os

import numpy as np
import pytest

import paper_2401_10089_b200 as lp
from paper_2401_10089_b200 import constants as C

DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2401_10089_b200", "data")


def test_builtin_schemes_match_frozen_tables_and_files():
    for k in range(1, C.K_MAX + 1):
        s = lp.builtin_scheme(k)
        assert s.mults == k and s.degree == 2 ** k and s.is_normalized
        lhs, rhs, out = C.SCHEMES[k - 1]
        assert s.flat() == [float(v) for row in (*lhs, *rhs, out) for v in row]
    for k in range(6, C.K_MAX + 1):  # the generated files parse to the frozen coefficients
        f = lp.read_scheme(os.path.join(DATA, f"scheme_k{k}.txt"))
        assert f.flat() == lp.builtin_scheme(k).flat()
    with pytest.raises(ValueError):
        lp.builtin_scheme(C.K_MAX + 1)


def test_save_load_round_trip_bitwise(tmp_path):
    rng = np.random.default_rng(3)
    k = 4
    s = lp.GraphScheme(lhs=tuple(tuple(rng.standard_normal(j + 2)) for j in range(k)),
                       rhs=tuple(tuple(rng.standard_normal(j + 2)) for j in range(k)),
                       out=tuple(rng.standard_normal(k + 2)),
                       meta=lp.SchemeMeta(order_label="7+", degree=16, radius=0.123456789012345678))
    text = lp.save_scheme(s, comment="round trip")
    t = lp.load_scheme(text)
    assert t.flat() == s.flat() and t.meta.order == 7 and t.meta.radius == s.meta.radius
    p = tmp_path / "s.txt"
    lp.write_scheme(str(p), s)
    assert lp.read_scheme(str(p)).flat() == s.flat()


@pytest.mark.parametrize("text", [
    "k 1\nH\n0 1\nG\n0 1\n",                 # missing y
    "k 1\nH\n0 1 2\nG\n0 1\ny\n0 1 0.5\n",   # wrong row length
    "H\n0 1\nG\n0 1\ny\n0 1 0.5\n",          # no k
    "k 1\nH\n0 x\nG\n0 1\ny\n0 1 0.5\n",     # unreadable token
    "k 2\nH\n0 1\nG\n0 1\ny\n0 1 0.5\n",     # truncated block
])
def test_load_rejects_malformed(text):
    with pytest.raises(lp.SchemeFormatError):
        lp.load_scheme(text)


def test_scheme_checks():
    with pytest.raises(lp.SchemeFormatError):
        lp.GraphScheme(lhs=((0.0, 1.0),), rhs=((0.0, 1.0),), out=(0.0, 1.0))
    with pytest.raises(lp.SchemeFormatError):
        lp.GraphScheme(lhs=((0.0, float("nan")),), rhs=((0.0, 1.0),), out=(0.0, 1.0, 0.5))
    assert not lp.GraphScheme(lhs=((0.5, 1.0),), rhs=((0.0, 1.0),), out=(0.0, 1.0, 0.5)).is_normalized
