"""Test infrastructure: CPU oracle for the PaSTiLa hot path (see pastila_oracle.py).

Never imported by the product package ``paper_2401_13680_b200``.
"""
