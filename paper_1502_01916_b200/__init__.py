"""B200-native batch decoder for the Group formats of arXiv 1502.01916.

The product is libgc.so (include/gc.h): sm_100a CUDA kernels for Group-Simple,
Group-Scheme (10 variants), Group-AFOR and Group-PFD decoding, fused with the d-gap
prefix sum, plus a multi-threaded host encoder.  `gc` is the thin ctypes binding.
"""
from . import gc  # noqa: F401
from .gc import (GROUP_AFOR, GROUP_PFD, GROUP_SCHEME, GROUP_SIMPLE, DeviceBatch,  # noqa: F401
                 HostBatch, checksum, decode, decode_dgaps, decode_host, encode_batch,
                 gsc_variant, read_device_status, to_device, workspace_size)
