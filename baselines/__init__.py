"""Reported CPU baselines for bench.py (never on the product path)."""
