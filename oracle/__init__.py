"""ORACLE — test infrastructure only (see orc.c header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The product path (paper_2506_09198_b200) never imports it.
"""
from .orc import Oracle, build_oracle, LIB_PATH  # noqa: F401
