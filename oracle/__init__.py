"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference hot path
(ssg_oracle.c via oracle.py) and the reference package build (oracle/_ref).
Importable by tests/, __graft_entry__.smoke() and bench.py's CPU legs only."""
