"""B200-native correlator-contraction engine (arXiv:2511.02257 hot path).

The product is libcc.so (include/cc.h): host C++ schedulers and planner, sm_100a
contraction kernels, the executor.  `cc` is its thin ctypes binding.  Importing this
package without a built libcc.so raises ImportError (no fallback path exists).
"""
from .cc import Context, CCError, cc_version, cc_scratch_bytes  # noqa: F401
from . import cc  # noqa: F401
