"""Philox4x64-10 counter-based generator (oracle copy; TEST INFRASTRUCTURE ONLY).

The paper draws D and S with Matlab's generator and does not fix an
RNG.  Reading R4 fixes Philox4x64-10 (Salmon, Moraes, Dror, Shaw,
"Parallel random numbers: as easy as 1, 2, 3", SC'11) so that the GPU and the
oracle can derive the same D and S independently.

Stream convention (reading R4): word ``w`` of stream ``(k0, k1)`` is word
``w mod 4`` of ``philox4x64_10(ctr=(1 + w//4, 0, 0, 0), key=(k0, k1))``.  This is
exactly what ``numpy.random.Philox(key=[k0, k1]).random_raw()`` returns, so the
bulk generator below is that library routine; ``philox4x64_10`` is the plain
definition, pinned to the published known-answer vectors in
``tests/golden/philox4x64_10_kat.txt``.
"""

import numpy as np

MASK64 = (1 << 64) - 1
# Round multipliers and Weyl key increments of Philox4x64 (Salmon et al. 2011).
PHILOX_M0 = 0xD2E7470EE14C6C93
PHILOX_M1 = 0xCA5A826395121157
PHILOX_W0 = 0x9E3779B97F4A7C15
PHILOX_W1 = 0xBB67AE8584CAA73B


def _mulhilo(a, b):
    p = a * b
    return (p >> 64) & MASK64, p & MASK64


def philox4x64_10(ctr, key):
    """One Philox4x64 block with 10 rounds: 4 counter words, 2 key words -> 4 words.

    Round (Salmon et al. Fig. 2 / Random123 philox4x64round):
        (hi0, lo0) = M0 * c0 ; (hi1, lo1) = M1 * c2
        c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    and the key is bumped by (W0, W1) between rounds.
    """
    c0, c1, c2, c3 = (int(v) & MASK64 for v in ctr)
    k0, k1 = (int(v) & MASK64 for v in key)
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + PHILOX_W0) & MASK64
            k1 = (k1 + PHILOX_W1) & MASK64
        hi0, lo0 = _mulhilo(PHILOX_M0, c0)
        hi1, lo1 = _mulhilo(PHILOX_M1, c2)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return (c0, c1, c2, c3)


def stream_word_py(k0, k1, w):
    """Word ``w`` of stream (k0, k1), straight from the definition (slow)."""
    return philox4x64_10((1 + w // 4, 0, 0, 0), (k0, k1))[w % 4]


def stream_words(k0, k1, count):
    """Words 0..count-1 of stream (k0, k1) as a uint64 array (library routine)."""
    g = np.random.Philox(key=np.array([k0 & MASK64, k1 & MASK64], dtype=np.uint64))
    return g.random_raw(int(count)).astype(np.uint64)
