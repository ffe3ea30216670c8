"""colo-b200: sm_100a implementation of the colosim (arXiv 2503.01066) admission hot path.

The compute lives in ``libcolo_b200.so`` (C-ABI: ``include/colo_abi.h``);
``colosim`` mirrors the reference's C++ API on top of it.
"""
from . import _lib, colosim
from ._lib import ColoError, ColoInvalidArgument, ColoValidationError, lib

__all__ = ["_lib", "lib", "colosim", "ColoError", "ColoInvalidArgument", "ColoValidationError"]
