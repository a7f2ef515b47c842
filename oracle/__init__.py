"""Test infrastructure: CPU oracle for parity checks (never imported by the product)."""
