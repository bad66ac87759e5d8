"""Seeded counter-based input generators (host and device); no GEMM arithmetic."""
