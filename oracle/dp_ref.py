"""Restatement of the data-parallel lane encoding (TEST INFRASTRUCTURE ONLY):
a W-bit quire value split into 60-bit digits + a NaR lane, summed across
ranks as int64, carry-normalised mod 2^W.  Mirrors csrc/dp.cu for the CPU
(gloo) multi-process tests."""
from __future__ import annotations


def lane_count(W: int) -> int:
    return (W + 59) // 60


def words_to_lanes(values, nars, W: int):
    L = lane_count(W)
    out = []
    for v, nar in zip(values, nars):
        v &= (1 << W) - 1
        out.append([(v >> (60 * l)) & ((1 << 60) - 1) for l in range(L)] + [1 if nar else 0])
    return out


def lanes_to_words(lanes, W: int):
    L = lane_count(W)
    vals, nars = [], []
    for row in lanes:
        v = sum(int(row[l]) << (60 * l) for l in range(L))
        vals.append(v & ((1 << W) - 1))
        nars.append(int(row[L]) > 0)
    return vals, nars
