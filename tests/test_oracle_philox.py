"""Pins for oracle/philox.py: published KAT vectors and the stream convention (R4)."""

import numpy as np

from oracle import philox
from tests.conftest import golden_path


def _kat():
    rows = []
    with open(golden_path("philox4x64_10_kat.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            v = [int(t, 16) for t in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_kat_vectors_pure_python():
    rows = _kat()
    assert len(rows) == 3
    for ctr, key, out in rows:
        assert list(philox.philox4x64_10(ctr, key)) == out


def test_numpy_stream_matches_definition():
    # The bulk generator (numpy library routine) must equal the stream definition
    # word w = philox(ctr=(1 + w//4, 0, 0, 0), key)[w % 4], itself KAT-pinned.
    for k0, k1 in [(0, 0), (0, 1), (12345, 7), (2**64 - 1, 2**63 + 5), (0, 2 * 2999 + 1)]:
        words = philox.stream_words(k0, k1, 23)
        for w in range(23):
            assert int(words[w]) == philox.stream_word_py(k0, k1, w)


def test_stream_prefix_property():
    a = philox.stream_words(3, 4, 1000)
    b = philox.stream_words(3, 4, 37)
    assert np.array_equal(a[:37], b)
