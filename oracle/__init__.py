"""TEST INFRASTRUCTURE ONLY.

CPU oracle of the reference (`gcnpart`) GCN training path: a fp64 numpy
restatement (gcn_oracle.py) plus C kernels (oracle.c, built by the Makefile
into oracle/_build/liboracle.so).  Importable only by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg —
never by the product package, which has no CPU fallback.
"""
