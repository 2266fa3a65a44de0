"""ORACLE — test infrastructure only (see oracle/oracle.hpp). Loaded by tests/, smoke() and
bench.py's CPU-baseline / --impl reference legs; never by the product path."""
