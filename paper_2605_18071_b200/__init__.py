"""B200-native (sm_100a) decode-step hot path of KVDrive (arxiv 2605.18071).

The product is ``libkvd.so`` (CUDA kernels + C ABI, ``include/kvd.h``); this
package is its thin Python binding (argument marshalling only).  There is no
CPU fallback: if the library is missing the import of ``kvd`` fails loudly.
"""
from .kvd import (KVDError, KVCache, Config, Stats, POLICY, lib, LIB_PATH)  # noqa: F401

__all__ = ["KVDError", "KVCache", "Config", "Stats", "POLICY", "lib", "LIB_PATH"]
