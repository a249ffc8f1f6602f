"""B200-native hot path of DuetServe (arXiv 2511.04791): thin Python binding of libduet.so.

Every step of the path runs in libduet.so (C++ host code + sm_100a kernels); this module
only marshals arguments (ctypes) with the C names of ``include/duet.h``.  There is no CPU
fallback: if the library is missing, importing the binding raises.
"""
from ._native import *  # noqa: F401,F403
from ._native import lib, DuetError  # noqa: F401
