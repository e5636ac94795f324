"""B200-native SGML solve path (arXiv 1703.07206) behind the reference's API.

The product is ``lib/libsgml_b200.so``: hand-written sm_100a fp64 kernels
plus the C++ engine, exposed through the C-ABI in ``include/sgml_b200.h``.
This package mirrors the reference's ``sgml`` C++ API in Python over that
C-ABI.  There is no CPU fallback.
"""
from ._capi import LIB_PATH, SgmlError, device_count, header_symbols, kernel_error  # noqa: F401
from .api import *  # noqa: F401,F403
from .api import Work  # noqa: F401
from .problems import *  # noqa: F401,F403

__version__ = "0.1.0"
