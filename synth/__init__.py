"""Seeded synthetic input generators shared by tests, bench.py and smoke() (no method arithmetic)."""
