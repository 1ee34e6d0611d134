"""Test-infrastructure oracles for the SerRGG hot path.

ORACLE ONLY — imported by tests/, ``__graft_entry__.smoke()`` and bench.py's
reference / cpu_baseline legs, never by the product package.

* :mod:`oracle.oracle` — ctypes wrapper over ``librgg_oracle.so``, our plain-C
  restatement of the reference algorithm (``rgg_oracle.c``).
* :mod:`oracle.ref` — ctypes wrapper over ``_ref/librgg_ref.so``, the unmodified
  reference library compiled from ``/root/reference/proj/src`` plus
  ``ref_shim.cpp``.
"""
