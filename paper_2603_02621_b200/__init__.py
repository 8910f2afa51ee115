"""B200-native segmented double-sieve Goldbach verifier (arXiv 2603.02621 hot path).

Importing the package loads libgb.so (built in-tree by __graft_entry__.build());
there is no CPU fallback.
"""
from . import gb  # noqa: F401  (loads libgb.so or raises ImportError)
from .gb import decode_result  # noqa: F401

__all__ = ["gb", "decode_result"]
