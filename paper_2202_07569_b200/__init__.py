"""B200-native server answer of constant-weight PIR (arXiv 2202.07569).

The hot path (``process_query``: query expansion -> constant-weight equality ->
payload inner product -> relinearisation) runs as hand-written sm_100a CUDA in
``libcwgpu.so`` behind the C ABI of ``include/cwgpu.h``; this package is the thin
host-side binding plus the seeded workload definitions.
"""
from . import configs
from .cwgpu import (OP_ARITH, OP_FOLKLORE, Client, Context, CudaError, HeError, Keys, StateError,
                    load_client_library, load_library)

__all__ = ["configs", "Context", "Client", "Keys", "HeError", "CudaError", "StateError", "load_library", "load_client_library",
           "OP_FOLKLORE", "OP_ARITH"]
