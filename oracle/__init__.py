"""Seven-League float64 CPU oracle.  TEST INFRASTRUCTURE ONLY: importable by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs, never by the
product package (see oracle/sl7_oracle.py header)."""
from .sl7_oracle import *  # noqa: F401,F403
