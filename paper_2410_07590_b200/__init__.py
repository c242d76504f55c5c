"""B200-native TurboRAG prefill engine (arxiv 2410.07590).

The product is libtkv_b200.so (sm_100a CUDA kernels + C++ host engine behind include/tkv.h).
`turbokv` mirrors the reference's C++ API over that C ABI. Importing this package never
falls back to CPU code: `turbokv.lib()` raises if the library is not built.
"""
from . import turbokv  # noqa: F401

__all__ = ["turbokv"]
