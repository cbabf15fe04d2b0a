"""CPU oracle package — TEST INFRASTRUCTURE ONLY (see oracle/oracle.h).
Importable only from tests/, __graft_entry__.smoke() and bench.py."""
