"""Host-side exact arithmetic types of the `hardround` API.

Restates the value semantics of /root/reference/pkg/src/hardround/fixedpoint.py
(UFrac 36-90, DivisionMode 26-33, frac_div 103-131, MPInt 140-305) so that
callers of the reference can pass the same objects here.  Only the semantics
matter for the device path: UFrac raws become u64 words, MPInt values become
two's complement limbs (slices.py), and MPInt's overflow rule -- every result
must satisfy |x| < 2^(32*limbs) -- is what the host checks before handing a
slice to the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from fractions import Fraction

DEFAULT_WORD_BITS = 64
LIMB_BITS = 32
_SUBTRACTIVE_CHUNK = 4096


class DivisionMode(Enum):
    """Quotient strategy of the classic walk (fixedpoint.py:26-33); in the
    searches it changes only the classic iteration accounting."""

    SUBTRACTIVE = "sub"
    HARDWARE = "hw"
    HYBRID = "hybrid"


# wire codes (include/hrb200.h HRB_MODE_*; lowerbound.py:80-85)
MODE_CODE = {DivisionMode.SUBTRACTIVE: 0, DivisionMode.HYBRID: 1, DivisionMode.HARDWARE: 2}


@dataclass(frozen=True, slots=True, order=True)
class UFrac:
    """raw / 2^width in [0, 1), width in {32, 64}."""

    raw: int
    width: int = DEFAULT_WORD_BITS

    def __post_init__(self) -> None:
        if self.width not in (32, 64):
            raise ValueError(f"word width must be 32 or 64, got {self.width}")
        if not 0 <= self.raw < (1 << self.width):
            raise ValueError(f"raw value {self.raw} out of range for width {self.width}")

    @classmethod
    def from_fraction(cls, value, width: int = DEFAULT_WORD_BITS) -> "UFrac":
        """floor(frac(value) * 2^width) for an exact rational value."""
        q = Fraction(value)
        num, den = q.numerator % q.denominator, q.denominator
        return cls((num << width) // den, width)

    @classmethod
    def from_rational(cls, num: int, den: int, width: int = DEFAULT_WORD_BITS) -> "UFrac":
        return cls.from_fraction(Fraction(num, den), width)

    def to_fraction(self) -> Fraction:
        return Fraction(self.raw, 1 << self.width)

    def __float__(self) -> float:
        return self.raw / float(1 << self.width)

    def _same(self, other: "UFrac") -> None:
        if self.width != other.width:
            raise ValueError("mixed word widths")

    def __add__(self, other: "UFrac") -> "UFrac":
        self._same(other)
        return UFrac((self.raw + other.raw) % (1 << self.width), self.width)

    def __sub__(self, other: "UFrac") -> "UFrac":
        self._same(other)
        return UFrac((self.raw - other.raw) % (1 << self.width), self.width)

    def __repr__(self) -> str:
        return f"UFrac({self.raw}/2^{self.width})"


def frac_add_mod1(x: UFrac, y: UFrac) -> UFrac:
    return x + y


def frac_sub_mod1(x: UFrac, y: UFrac) -> UFrac:
    return x - y


def _quotient(q: int, p: int, mode: DivisionMode) -> int:
    if p <= 0:
        raise ZeroDivisionError("division by zero-length fraction")
    if mode is DivisionMode.SUBTRACTIVE:
        k = 0
        while q >= p:
            q -= p
            k += 1
            if k == _SUBTRACTIVE_CHUNK:
                return k + q // p
        return k
    if mode is DivisionMode.HYBRID:
        return 0 if q < p else 1 + (q - p) // p
    return q // p


def frac_div(q: UFrac, p: UFrac, mode: DivisionMode = DivisionMode.HARDWARE) -> tuple[int, UFrac]:
    """q = k p + r with 0 <= r < p; identical (k, r) in every mode."""
    q._same(p)
    k = _quotient(q.raw, p.raw, mode)
    return k, UFrac(q.raw - k * p.raw, q.width)


class MPOverflowError(OverflowError):
    """A fixed-limb result did not fit (never wrapped silently)."""


class MPInt:
    """Signed integer bounded to `limb_count` 32-bit limbs of magnitude.

    Stored as a Python int; every constructor and operation enforces
    |value| < 2^(32 * limb_count), the overflow rule of the reference's
    sign-magnitude limbs."""

    __slots__ = ("_v", "_n")

    def __init__(self, limbs, negative: bool = False):
        limbs = tuple(limbs)
        if not limbs:
            raise ValueError("MPInt needs at least one limb")
        mag = 0
        for i, limb in enumerate(limbs):
            if not 0 <= limb < (1 << LIMB_BITS):
                raise ValueError(f"limb {limb} out of 32-bit range")
            mag |= limb << (LIMB_BITS * i)
        self._v = -mag if negative else mag
        self._n = len(limbs)

    @classmethod
    def _raw(cls, value: int, n: int, what: str | None = None) -> "MPInt":
        # the reference's messages: from_int "<v> needs <b> bits, have <B>",
        # mp_add "addition carry out of top limb", mp_mul "product exceeds
        # limb budget" (fixedpoint.py:136-137, 239, 291, 300)
        if abs(value) >> (LIMB_BITS * n):
            raise MPOverflowError(what or f"{value} needs {abs(value).bit_length()} bits, have {LIMB_BITS * n}")
        obj = cls.__new__(cls)
        obj._v = value
        obj._n = n
        return obj

    @classmethod
    def from_int(cls, value: int, limb_count: int) -> "MPInt":
        return cls._raw(int(value), limb_count)

    @property
    def limb_count(self) -> int:
        return self._n

    @property
    def limbs(self) -> tuple[int, ...]:
        mag = abs(self._v)
        return tuple((mag >> (LIMB_BITS * i)) & 0xFFFFFFFF for i in range(self._n))

    @property
    def negative(self) -> bool:
        return self._v < 0

    def to_int(self) -> int:
        return self._v

    def _other(self, other) -> int:
        if isinstance(other, MPInt):
            if other._n != self._n:
                raise ValueError("mixed limb counts")
            return other._v
        if isinstance(other, int):
            return MPInt._raw(other, self._n)._v
        return NotImplemented

    def __neg__(self) -> "MPInt":
        return MPInt._raw(-self._v, self._n)

    _ADD = "addition carry out of top limb"
    _MUL = "product exceeds limb budget"

    def __add__(self, other):
        o = self._other(other)
        return NotImplemented if o is NotImplemented else MPInt._raw(self._v + o, self._n, self._ADD)

    __radd__ = __add__

    def __sub__(self, other):
        o = self._other(other)
        return NotImplemented if o is NotImplemented else MPInt._raw(self._v - o, self._n, self._ADD)

    def __rsub__(self, other):
        o = self._other(other)
        return NotImplemented if o is NotImplemented else MPInt._raw(o - self._v, self._n, self._ADD)

    def __mul__(self, other):
        o = self._other(other)
        return NotImplemented if o is NotImplemented else MPInt._raw(self._v * o, self._n, self._MUL)

    __rmul__ = __mul__

    def __eq__(self, other) -> bool:
        if isinstance(other, MPInt):
            return self._v == other._v
        if isinstance(other, int):
            return self._v == other
        return NotImplemented

    def __hash__(self) -> int:
        return hash(self._v)

    def __repr__(self) -> str:
        return f"MPInt({self._v}, limbs={self._n})"


def mp_add(a: MPInt, b: MPInt) -> MPInt:
    return a + b


def mp_mul(a: MPInt, b: MPInt) -> MPInt:
    return a * b


def as_int(c) -> int:
    """Coefficient (MPInt or int) as a Python int."""
    return c.to_int() if isinstance(c, MPInt) else int(c)
