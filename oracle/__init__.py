"""CPU oracle for the Schwinger-model HMC hot path — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs.  See schwinger_oracle.py for the restated algorithms and the
reference file:line each one follows.
"""
