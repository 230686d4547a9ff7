"""B200-native HieraSparse hot path: hierarchical 2:4 KV compression and
Trans-Both sparse attention (arxiv 2604.16864) behind a C ABI
(include/hierasparse_b200.h) with sm_100a kernels in csrc/."""
from .errors import ConfigError, CudaError, DataError, IoError  # noqa: F401

__all__ = ["ConfigError", "DataError", "IoError", "CudaError"]
