"""Operator descriptors: the reference's monoid plug-in surface.

The reference selects the operator through the ``MonoidOps`` instance bound to
a ``Tensor`` (monoid.py:30-106): ``name``, ``dtype``, ``identity``,
``commutative`` and ``has_inverse`` drive every algorithm.  Here the same
attributes select a CUDA kernel instantiation; the scalar ``combine`` /
``subtract`` are kept for API parity (and for tests), but no bulk arithmetic
ever runs on the host -- the device library does all of it.

Instances (same names as the reference):

=========  ===================  ===========  ============  ==========
name       reference            dtype        identity      inverse
=========  ===================  ===========  ============  ==========
add-i64    IntAddOps :130-164   int64        0             yes (wraps)
add-f64    FloatAddOps :167-204 float64      0.0           yes
add-f32    (new)   float32      0.0           yes
max-i64    IntMaxOps :207-232   int64        INT64_MIN     no
mod-add:m  ModAddOps :235-286   int64        0             yes (mod m)
=========  ===================  ===========  ============  ==========

Any object with ``name``/``dtype`` matching one of these (for example the
reference's own monoid instances, or its ``InstrumentedMonoid`` wrapper, which
is unwrapped through ``.inner`` like bench.py:128 does) is accepted.
"""

from __future__ import annotations

import numpy as np

from .errors import ConfigurationError


class MonoidOps:
    name = "abstract"
    dtype = np.dtype(np.int64)
    identity = 0
    commutative = True
    has_inverse = False
    op = None  # device operator code: "add" or "max"

    def combine(self, a, b):
        raise NotImplementedError

    def subtract(self, a, b):
        raise ConfigurationError(f"monoid {self.name!r} has no inverse")

    # -- bulk kernels (monoid.py:66-104): in place, on the GPU (pieces.py) -------
    def combine_into(self, dst, src):
        from . import pieces

        pieces.combine_into(self, dst, src)

    def rcombine_into(self, dst, src):
        from . import pieces

        pieces.rcombine_into(self, dst, src)

    def subtract_into(self, dst, src):
        from . import pieces

        pieces.subtract_into(self, dst, src)

    def rsubtract_scalar(self, total, dst):
        from . import pieces

        pieces.rsubtract_scalar(self, total, dst)

    def accumulate(self, arr, axis, reverse=False):
        from . import pieces

        pieces.accumulate(self, arr, axis, reverse)

    def fold(self, arr):
        from . import pieces

        return pieces.fold(self, arr)

    def __repr__(self):
        return f"{type(self).__name__}({self.name})"


class IntAddOps(MonoidOps):
    """64-bit integer addition (wraps mod 2^64, like numpy)."""

    name = "add-i64"
    dtype = np.dtype(np.int64)
    identity = 0
    has_inverse = True
    op = "add"

    def combine(self, a, b):
        return _wrap64(int(a) + int(b))

    def subtract(self, a, b):
        return _wrap64(int(a) - int(b))


class FloatAddOps(MonoidOps):
    """Float64 addition."""

    name = "add-f64"
    dtype = np.dtype(np.float64)
    identity = 0.0
    has_inverse = True
    op = "add"

    def combine(self, a, b):
        return a + b

    def subtract(self, a, b):
        return a - b


class Float32AddOps(FloatAddOps):
    """Float32 addition (not a reference monoid; BASELINE configs 3-4 need it)."""

    name = "add-f32"
    dtype = np.dtype(np.float32)
    identity = np.float32(0.0)

    def combine(self, a, b):
        return np.float32(np.float32(a) + np.float32(b))

    def subtract(self, a, b):
        return np.float32(np.float32(a) - np.float32(b))


class IntMaxOps(MonoidOps):
    """64-bit integer maximum; identity is the most negative int64."""

    name = "max-i64"
    dtype = np.dtype(np.int64)
    identity = int(np.iinfo(np.int64).min)
    has_inverse = False
    op = "max"

    def combine(self, a, b):
        return a if a >= b else b


MOD_ADD_MAX_MODULUS = 2**31  # monoid.py:27: keeps raw int64 partial sums overflow-free


class ModAddOps(MonoidOps):
    """Addition modulo m (2 <= m <= 2**31), values canonicalized to [0, m)
    by every combine (monoid.py:235-286)."""

    dtype = np.dtype(np.int64)
    identity = 0
    has_inverse = True
    op = "mod-add"

    def __init__(self, modulus: int):
        if not isinstance(modulus, (int, np.integer)) or isinstance(modulus, bool):
            raise ConfigurationError("mod-add modulus must be an integer")
        modulus = int(modulus)
        if not 2 <= modulus <= MOD_ADD_MAX_MODULUS:
            raise ConfigurationError(
                f"mod-add modulus must be in [2, {MOD_ADD_MAX_MODULUS}], got {modulus}"
            )
        self.modulus = modulus
        self.name = f"mod-add:{modulus}"

    def combine(self, a, b):
        return (int(a) + int(b)) % self.modulus

    def subtract(self, a, b):
        return (int(a) - int(b)) % self.modulus


def _wrap64(v: int) -> int:
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= 1 << 63 else v


MONOIDS = {cls.name: cls for cls in (IntAddOps, FloatAddOps, Float32AddOps, IntMaxOps)}
MONOID_CHOICES = tuple(MONOIDS) + ("mod-add:<m>",)


def resolve_monoid(name: str) -> MonoidOps:
    """Name -> monoid instance (monoid.py:362-385): add-i64, add-f64, add-f32,
    max-i64 or mod-add:<m>."""
    if isinstance(name, str) and name.startswith("mod-add:"):
        text = name.split(":", 1)[1]
        try:
            modulus = int(text)
        except ValueError:
            raise ConfigurationError(f"bad mod-add modulus: {text!r}") from None
        return ModAddOps(modulus)
    cls = MONOIDS.get(name)
    if cls is None:
        raise ConfigurationError(
            f"unknown monoid {name!r}; choose from {', '.join(MONOID_CHOICES)}"
        )
    return cls()


def unwrap(ops):
    """Strip instrumentation wrappers (InstrumentedMonoid.inner, bench.py:128)."""
    seen = 0
    while hasattr(ops, "inner") and seen < 8:
        ops = ops.inner
        seen += 1
    return ops


def device_operator(ops):
    """(dtype, op, has_inverse) for the device library, or ConfigurationError --
    before any work.  For mod-add the modulus is ``modulus_of(ops)``."""
    base = unwrap(ops)
    name = getattr(base, "name", None)
    if isinstance(name, str) and name.startswith("mod-add:"):
        modulus_of(base)  # validates like ModAddOps.__init__
        if np.dtype(getattr(base, "dtype", np.int64)) != np.dtype(np.int64):
            raise ConfigurationError(f"monoid {name!r} must be int64")
        return np.dtype(np.int64), "mod-add", True
    cls = MONOIDS.get(name)
    if cls is None:
        raise ConfigurationError(
            f"monoid {name!r} has no B200 kernel; supported: {', '.join(MONOID_CHOICES)}"
        )
    dtype = np.dtype(getattr(base, "dtype", cls.dtype))
    if dtype != cls.dtype:
        raise ConfigurationError(f"monoid {name!r} with dtype {dtype} has no B200 kernel")
    return cls.dtype, cls.op, cls.has_inverse


def modulus_of(ops) -> int:
    """The modulus of a mod-add monoid (0 for the others), validated."""
    base = unwrap(ops)
    name = getattr(base, "name", "")
    if not (isinstance(name, str) and name.startswith("mod-add:")):
        return 0
    m = getattr(base, "modulus", None)
    if m is None:
        try:
            m = int(name.split(":", 1)[1])
        except ValueError:
            raise ConfigurationError(f"bad mod-add modulus in {name!r}") from None
    m = int(m)
    if not 2 <= m <= MOD_ADD_MAX_MODULUS:
        raise ConfigurationError(f"mod-add modulus must be in [2, {MOD_ADD_MAX_MODULUS}], got {m}")
    return m
