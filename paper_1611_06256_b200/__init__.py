"""B200-native GA3C hot path (arXiv 1611.06256) behind the reference qac API.

The product is the C ABI library libga3c_b200.so (include/ga3c.h): sm_100a
kernels for the predictor forward, the trainer's A3C loss/backward, RMSProp,
n-step returns and action sampling, plus the C++ host pipeline.  This package
holds the in-tree build and its Python bindings:
  _abi   -- ctypes binding of the C ABI (fails loudly if the .so is missing)
  qac    -- reference-shaped API (nnet/returns names and error behaviour)
"""
from . import _abi  # noqa: F401  (raises ImportError without the built library)
from . import qac  # noqa: F401

__all__ = ["_abi", "qac"]
