"""CPU oracle for the soft-snake step — TEST INFRASTRUCTURE ONLY (see
softsnake_oracle.c). Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline / --impl reference leg may import this package."""
