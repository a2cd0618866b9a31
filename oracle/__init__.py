"""TEST INFRASTRUCTURE ONLY — CPU oracle for the BLWS partial-SVT hot path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs. See oracle/blws_oracle.hpp and DESIGN.md §3.
"""
