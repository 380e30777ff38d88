"""B200-native batched FP64 matrix logarithm (arXiv 2401.10089, inverse scaling-and-squaring
with computation-graph polynomials).  Public surface mirrors the reference ``logmpoly``
package (``pkg/src/logmpoly/__init__.py:55,60-75``): ``logm(A, opts) -> (L, LogmReport)``.
"""
