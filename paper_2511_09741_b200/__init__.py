"""B200-native TawPipe (arXiv 2511.09741) training step: DBS + GWPS + CCO over NCCL, sm_100a kernels.

The product is ``libtawpipe.so`` (C ABI in include/tawpipe.h); ``tawpipe.py`` is its ctypes binding.
"""
from .tawpipe import (BF16, FP32, GWPS, LITERAL, NO_CCO, RING, ModelDims, Session, TawpipeError, bootstrap, lib,  # noqa: F401
                      pack_full_model)
