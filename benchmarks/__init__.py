"""Per-config benchmark legs for bench.py (--config c2..c5); C1 lives in bench.py."""
