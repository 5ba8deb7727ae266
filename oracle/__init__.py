"""oracle/ — TEST INFRASTRUCTURE ONLY.

Two CPU checkers for the B200 path, loaded through ctypes:

* ``RefSystem`` wraps ``oracle/_ref/libhexsem_ref.so``: the UNMODIFIED
  reference library (hexsem, /root/reference/proj/src) compiled by
  ``oracle/Makefile`` with the Eigen-API shim in ``oracle/eigen_shim``.
* ``OracleSystem`` wraps ``oracle/_ref/libhexsem_oracle.so``: the plain C++
  restatement of the reference algorithm in ``oracle/hexsem_oracle.cpp``
  (each function cites the reference file:line it follows).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.
The product (``paper_1506_05996_b200``) never does.
"""
from .ctypes_oracle import (  # noqa: F401
    RefSystem,
    OracleSystem,
    OracleFmaSystem,
    oracle_fma_available,
    RefConfig,
    ref_available,
    ref_read_mesh,
    ref_write_mesh,
    ref_solve_heat,
    oracle_available,
    ref_gll,
    ref_pencil,
    oracle_gll,
    oracle_pencil,
    words_model,
    flops_model,
    fine_ops_model,
    fine_words_model,
    splitmix_vector,
)
