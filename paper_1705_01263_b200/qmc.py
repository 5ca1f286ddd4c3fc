"""Host-side QMC tables for the device sampler.

Mirrors the public API of the reference module `lumenwave.qmc`
(`qmc.py:17-29`): prime bases, Faure digit scrambling, the exact radical
inverse, the strength-reduced divider, global sample enumeration and the
fixed dimension layout.  The per-sample evaluation runs on the GPU
(`csrc/lw_qmc.cuh`); everything here builds the tables it consumes and the
exact big-integer evaluation that defines the expected bits.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

__all__ = [
    "ScrambledBase",
    "FastDivisor",
    "primes",
    "faure_permutation",
    "scrambled_base",
    "radical_inverse",
    "prepare_fast_divisor",
    "fast_divide",
    "global_sample_index",
    "DimensionTable",
]

_MASK64 = (1 << 64) - 1


def primes(count: int) -> np.ndarray:
    """The first `count` primes (qmc.py:34-52)."""
    if count <= 0:
        return np.zeros(0, dtype=np.int64)
    limit = 16
    while True:
        is_p = np.ones(limit + 1, dtype=bool)
        is_p[:2] = False
        is_p[4::2] = False
        for k in range(3, int(limit**0.5) + 1, 2):
            if is_p[k]:
                is_p[k * k :: 2 * k] = False
        found = np.nonzero(is_p)[0]
        if found.size >= count:
            return found[:count].astype(np.int64)
        limit *= 2


@lru_cache(maxsize=None)
def _faure(base: int) -> tuple:
    """Faure's recursive permutation (qmc.py:55-69), built bottom-up.

    sigma_2 = (0, 1).  For even b, sigma_b lists 2*sigma_{b/2} followed by
    2*sigma_{b/2}+1.  For odd b, the middle value c=b//2 is inserted at
    position c of sigma_{b-1} after shifting every entry >= c up by one.
    """
    if base < 1:
        raise ValueError("base must be >= 1")
    if base == 1:
        return (0,)
    if base == 2:
        return (0, 1)
    if base & 1:
        mid = base >> 1
        lower = np.asarray(_faure(base - 1), dtype=np.int64)
        lower = lower + (lower >= mid)
        return tuple(np.insert(lower, mid, mid).tolist())
    half = np.asarray(_faure(base >> 1), dtype=np.int64)
    return tuple(np.concatenate([2 * half, 2 * half + 1]).tolist())


def faure_permutation(base: int) -> np.ndarray:
    """Digit permutation for `base`; sigma(0)=0, base 2 is the identity (qmc.py:72-80)."""
    return np.array(_faure(int(base)), dtype=np.int64)


@dataclass(frozen=True)
class ScrambledBase:
    """Prime base with its digit permutation (qmc.py:83-94)."""

    base: int
    permutation_digits: np.ndarray

    def __post_init__(self):
        perm = np.asarray(self.permutation_digits, dtype=np.int64)
        ok = perm.shape == (self.base,) and np.array_equal(np.sort(perm), np.arange(self.base))
        if not ok:
            raise ValueError("permutation_digits must be a bijection on 0..base-1")
        object.__setattr__(self, "permutation_digits", perm)


@lru_cache(maxsize=None)
def scrambled_base(base: int) -> ScrambledBase:
    return ScrambledBase(int(base), faure_permutation(base))


def radical_inverse(base, index: int) -> float:
    """Exact scrambled radical inverse in [0, 1) (qmc.py:112-135).

    Digits are permuted in integer arithmetic and the final ratio is rounded
    once by Python's correctly rounded int/int division, so this is the
    ground truth the device sampler must reproduce bit for bit.
    """
    sb = scrambled_base(base) if isinstance(base, (int, np.integer)) else base
    index = int(index)
    if index < 0 or index >> 64:
        raise ValueError("index must fit in 64 bits")
    b = sb.base
    if b == 2:
        rev = int(format(index, "064b")[::-1], 2)
        return rev / (1 << 64)
    perm = sb.permutation_digits.tolist()
    num, den = 0, 1
    while index:
        index, digit = divmod(index, b)
        num = num * b + perm[digit]
        den *= b
    return num / den


@dataclass(frozen=True)
class FastDivisor:
    """Magic-number unsigned division by a constant (qmc.py:138-164)."""

    divisor: int
    magic: int
    shift: int
    add: bool


def prepare_fast_divisor(divisor: int, bits: int = 64) -> FastDivisor:
    """Round-up magic for `bits`-wide unsigned operands.

    bits=64 reproduces the reference's tables; bits=32 gives the 32-bit
    variant the device uses while the sample index fits in 32 bits.
    """
    divisor = int(divisor)
    if divisor < 2:
        raise ValueError("divisor must be >= 2")
    if divisor & (divisor - 1) == 0:
        return FastDivisor(divisor, 0, divisor.bit_length() - 1, False)
    ell = (divisor - 1).bit_length()
    m = -(-(1 << (bits + ell)) // divisor)
    if m >> bits == 0:
        return FastDivisor(divisor, m, ell, False)
    return FastDivisor(divisor, m - (1 << bits), ell - 1, True)


def fast_divide(d: FastDivisor, n: int, bits: int = 64) -> int:
    """floor(n / d.divisor) from the magic constants (qmc.py:171-182)."""
    n = int(n)
    if n < 0 or n >> bits:
        raise ValueError(f"n must fit in {bits} bits")
    if d.magic == 0:
        return n >> d.shift
    hi = (d.magic * n) >> bits
    if d.add:
        return (((n - hi) >> 1) + hi) >> d.shift
    return hi >> d.shift


def global_sample_index(pixel_id: int, iteration: int, pixel_count: int) -> int:
    """Sample index enumerated over the full screen (qmc.py:185-196)."""
    if pixel_id < 0 or pixel_id >= pixel_count:
        raise ValueError("pixel_id out of range")
    index = int(iteration) * int(pixel_count) + int(pixel_id)
    if index >> 64:
        raise OverflowError("sample index exceeds 64 bits")
    return index


# Fixed dimension layout (qmc.py:241-271)
DIM_AA_X = 0
DIM_AA_Y = 1
DIM_TIME = 2
DIM_WAVELENGTH = 3
EYE_BOUNCE_BASE = 4
BOUNCE_STRIDE = 8
OFF_BSDF_U = 0
OFF_BSDF_V = 1
OFF_NEE_U = 2
OFF_NEE_V = 3
OFF_ROULETTE = 4
OFF_VOLUME = 5
OFF_PHASE_U = 6
OFF_PHASE_V = 7
LIGHT_HEAD_DIMS = 6
LIGHT_SELECT = 0
LIGHT_POS_U = 1
LIGHT_POS_V = 2
LIGHT_AIM_U = 3
LIGHT_AIM_V = 4


class DimensionTable:
    """Per-dimension bases, scrambling tables and dividers (qmc.py:274-315).

    Attributes used by the device: `bases`, `perm_flat`, `perm_offset`
    (the reference's kernel inputs) plus `magic`/`shift`/`add` (64-bit) and
    `magic32`/`shift32`/`add32` (32-bit) division tables.
    """

    def __init__(self, max_depth: int):
        self.max_depth = int(max_depth)
        self.light_base = EYE_BOUNCE_BASE + BOUNCE_STRIDE * self.max_depth
        self.ndims = self.light_base + LIGHT_HEAD_DIMS + BOUNCE_STRIDE * self.max_depth
        self.bases = primes(self.ndims)
        perms = [faure_permutation(b) for b in self.bases.tolist()]
        sizes = np.array([len(p) for p in perms], dtype=np.int64)
        self.perm_offset = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
        self.perm_flat = np.concatenate(perms).astype(np.int64) if perms else np.zeros(0, np.int64)
        d64 = [prepare_fast_divisor(b, 64) for b in self.bases.tolist()]
        d32 = [prepare_fast_divisor(b, 32) for b in self.bases.tolist()]
        self.magic = np.array([d.magic for d in d64], dtype=np.uint64)
        self.shift = np.array([d.shift for d in d64], dtype=np.int64)
        self.add = np.array([int(d.add) for d in d64], dtype=np.int64)
        self.magic32 = np.array([d.magic for d in d32], dtype=np.uint64)
        self.shift32 = np.array([d.shift for d in d32], dtype=np.int64)
        self.add32 = np.array([int(d.add) for d in d32], dtype=np.int64)

    def eye_bounce_dim(self, bounce: int, offset: int) -> int:
        return EYE_BOUNCE_BASE + BOUNCE_STRIDE * bounce + offset

    def light_bounce_dim(self, bounce: int, offset: int) -> int:
        return self.light_base + LIGHT_HEAD_DIMS + BOUNCE_STRIDE * bounce + offset

    def sample(self, dim: int, index: int) -> float:
        """Exact evaluation; the device kernels reproduce these bits."""
        return radical_inverse(int(self.bases[dim]), index)
