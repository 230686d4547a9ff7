"""Error taxonomy of the reference (errors.hpp:10-25) on the Python side."""


class ConfigError(ValueError):
    """Invalid caller-supplied arguments or configuration (std::invalid_argument)."""


class DataError(RuntimeError):
    """A well-formed call over corrupt or inconsistent data (std::runtime_error)."""


class IoError(RuntimeError):
    """Filesystem and stream failures."""


class CudaError(RuntimeError):
    """A CUDA runtime or launch failure inside the native library."""
