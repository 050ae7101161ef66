"""B200-native NNEinFact multiplicative-update sweep (arxiv 2602.02759).

The compute path is libnef.so (C ABI in include/nef.h, sm_100a kernels in csrc/); this
package is only its ctypes binding (``nef``).  Importing fails loudly if the library is not
built -- there is no CPU fallback.
"""
from . import nef  # noqa: F401
from .nef import NefError, Plan  # noqa: F401
