"""Golden text for the matrix I/O format, written by the reference's own serializer.

    python tests/golden/make_matio_golden.py      (needs /root/reference; run in the build container)

Writes tests/golden/matio_ref.txt = logmpoly.matcore.format_matrix(M) (matcore.py:393-401) for a
fixed 5x5 matrix with awkward values (signed zero, subnormal, huge/tiny exponents, integers,
irrationals), and tests/golden/matio_ref_complex.txt for a 2x2 complex matrix.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_reference  # noqa: E402


def matrices():
    M = np.array([[1.0, -0.0, 5e-324, 1.7976931348623157e308, -2.5],
                  [np.pi, -np.e, 1e-300, 123456789.0, 0.1],
                  [1.0 / 3.0, 2.0 / 3.0, -1e-17, 7.0, -8.0],
                  [np.sqrt(2.0), 1e22, 1e-22, -0.5, 0.0],
                  [6.02214076e23, -1.602176634e-19, 299792458.0, 9.1093837015e-31, 1.0]])
    Z = np.array([[1 + 2j, -0.5 - 1e-20j], [3.25e-7 + 0j, -1e300 + 1e-300j]])
    return M, Z


if __name__ == "__main__":
    mc, _, _ = load_reference()
    M, Z = matrices()
    with open(os.path.join(HERE, "matio_ref.txt"), "w") as fh:
        fh.write(mc.format_matrix(M))
    with open(os.path.join(HERE, "matio_ref_complex.txt"), "w") as fh:
        fh.write(mc.format_matrix(Z))
    print("wrote matio_ref.txt, matio_ref_complex.txt")
