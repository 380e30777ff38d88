"""CPU oracle for the batched matrix-logarithm hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from this package, and only as the
checker or the timed CPU baseline.  The product (``paper_2401_10089_b200``) never
imports it and has no CPU fallback.

Contents
--------
``oracle.primitives``  numpy/scipy restatement of the reference primitives the path
                       calls (matcore / sqrtm / schemes), each citing the reference
                       file:line it follows.
``oracle.driver``      the restated Algorithm 1; the
                       reference's own ``logmpoly/driver.py`` is missing
                       (``logmpoly/__init__.py:55``), so this restatement *is* the
                       contract.  It is written over a pluggable primitive set so
                       that ``tests/golden/make_golden.py`` can run the very same
                       driver over the reference's own primitives (imported from
                       /root/reference in the build container) and pin this
                       restatement to them bit-for-bit.

Pinning: see ``tests/test_oracle_golden.py`` (restated primitives and driver vs the
fixtures generated from the reference primitives, plus the SPEC known-answer
examples).  The end-to-end (s, k) selection logic itself has no reference code to
pin against (the driver file is absent); it is pinned to SPEC.md:429-502 and
PAPER.md:724-840 only, as SURVEY.md section 8(c) records.
"""
