"""Exception types of the drop-in, mirroring the reference (errors.py:4-22).

Same names, same base classes, same meaning, so code written against the
reference's exceptions behaves identically:

* ``ConfigurationError`` -- a combination that can never run (weak route on a
  monoid without inverse, unknown names, no GPU kernel for a monoid); the
  reference CLI maps it to exit code 2.
* ``UsageError`` (also a ``ValueError``) -- malformed extents / boxes / data.
* ``VerificationError`` -- output did not match the oracle (exit code 1).
* ``DeviceError`` -- new here: a CUDA failure inside the native library, or
  the native library is missing.  There is no CPU fallback.
"""


class ExsumError(Exception):
    """Base class for all errors raised by this package."""


class ConfigurationError(ExsumError):
    """An algorithm/monoid/parameter combination that can never run."""


class UsageError(ExsumError, ValueError):
    """Malformed inputs: bad coordinates, extents, boxes, or data."""


class VerificationError(ExsumError):
    """Output did not match the reference oracle."""


class DeviceError(ExsumError, RuntimeError):
    """CUDA failure in the native library, or the library is not built."""
