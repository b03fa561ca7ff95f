"""ORACLE - test infrastructure only.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import anything in this directory, and only as the checker / the
reference arm; the product package ``paper_2408_07436_b200`` never does.

Contents:
  port.py       numpy restatement of the reference's evaluate path (each
                function cites pkg/src/kifmm3d file:line)
  hot.c         C restatement of the reference's _hot.pyx loops
  build_ref.py  compiles the unmodified reference package with Cython into
                _ref/kifmm3d (a .so-only namespace package)
  Makefile      builds _build/libkifmm_oracle.so from hot.c

Parity pinning: tests/test_oracle_golden.py checks the restatement against
golden vectors the reference itself produced (tests/golden/make_golden.py).
"""

import os
import sys

REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "kifmm3d"))


def import_reference():
    """Import the Cython-compiled unmodified reference package (kifmm3d)."""
    if not reference_available():
        raise ImportError("oracle/_ref/kifmm3d is not built (python oracle/build_ref.py)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import kifmm3d.engine  # noqa: F401
    import kifmm3d
    return kifmm3d
