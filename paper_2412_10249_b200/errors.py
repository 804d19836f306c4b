"""Exception types of the reference API (linops.py:19-20)."""


class DimensionMismatch(ValueError):
    """Vector length does not match an operator dimension."""
