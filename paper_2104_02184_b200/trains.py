"""Packed pulse-train format <-> the reference's PulseTrains.

The reference stores trains as one uint8 per (slot, line), slot-major, with
separate int signs (proj/include/xbarsim/pulsed.hpp:31-50).  The B200 path
packs one uint32 per (sample, line): bits 0..bl-1 are the slots, bit 31 is
the sign (1 = negative).  A line with sign 0 carries no bits (its
probability is 0), so the packing is lossless for coincidence counting.
"""
from __future__ import annotations

import numpy as np

SIGN_BIT = np.uint32(0x80000000)


def pack(bits: np.ndarray, signs: np.ndarray) -> np.ndarray:
    """bits [bl][lines] (0/1), signs [lines] (-1/0/+1) -> words [lines]."""
    bits = np.asarray(bits, dtype=np.uint32)
    bl = bits.shape[0]
    if bl > 31:
        raise ValueError("packed trains hold at most 31 slots")
    shifts = np.arange(bl, dtype=np.uint32)[:, None]
    words = np.bitwise_or.reduce(bits << shifts, axis=0) if bl else np.zeros(bits.shape[1],
                                                                              np.uint32)
    words = words.astype(np.uint32)
    words[np.asarray(signs) < 0] |= SIGN_BIT
    return words


def unpack(words: np.ndarray, bl: int):
    """words [lines] -> (bits [bl][lines] uint8, signs [lines] int32 in {-1,+1})."""
    words = np.asarray(words, dtype=np.uint32)
    shifts = np.arange(bl, dtype=np.uint32)[:, None]
    bits = ((words[None, :] >> shifts) & 1).astype(np.uint8)
    signs = np.where(words & SIGN_BIT, -1, 1).astype(np.int32)
    return bits, signs


def coincidences(xw: np.ndarray, dw: np.ndarray) -> np.ndarray:
    """Brute-force coincidence counts [rows][cols] of one sample's words."""
    m = np.uint32(0x7FFFFFFF)
    c = (dw[:, None] & xw[None, :]) & m
    # popcount on uint32
    c = c - ((c >> 1) & 0x55555555)
    c = (c & 0x33333333) + ((c >> 2) & 0x33333333)
    c = (c + (c >> 4)) & 0x0F0F0F0F
    return ((c * 0x01010101) & 0xFFFFFFFF) >> 24
