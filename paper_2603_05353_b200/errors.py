"""Exception hierarchy of the drop-in API (reference errors.py:1-10).

Argument/shape/budget problems raise ConfigurationError (the reference's CLI
exit code 2); corrupt on-disk data raises DataFormatError (exit code 3).  A
failing CUDA launch inside the native library raises NativeError.
"""


class ChunkKVError(Exception):
    """Base class for all library errors."""


class ConfigurationError(ChunkKVError):
    """Invalid configuration, arguments, or request shapes."""


class DataFormatError(ChunkKVError):
    """Corrupt, truncated, or incompatible on-disk data."""


class NativeError(ChunkKVError):
    """The sm_100a native library reported a CUDA failure or is unavailable."""
