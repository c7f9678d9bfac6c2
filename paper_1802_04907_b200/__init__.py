"""B200-native low-precision IHT (arXiv 1802.04907): the hot path of Algorithm 1.

The product is libiht.so (CUDA for sm_100a behind the C ABI in include/iht.h);
``paper_1802_04907_b200.iht`` is its thin Python binding.  This package never
imports ``oracle`` (the CPU test oracle) and has no CPU fallback.
"""
from . import _lib  # noqa: F401

__version__ = "0.1.0"
