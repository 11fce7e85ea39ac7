"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and
bench.py.  This package holds NO arithmetic of the method (no contraction, SVD,
truncation or split): only the record codec (records.py) and the seeded input
generators (gen.py) — complex Gaussian site tensors with p random mantissa bits
and Haar-random unitaries orthonormalised at p+32 bits (SURVEY.md §8(d)
"Synthetic inputs")."""
from . import records  # noqa: F401
