"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
symbol include/blws_cuda.h declares, and its host-side Rng / sampler are
bit-identical to the oracle's (core/rng.hpp:17-90, synth.hpp:23-33)."""
import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "blws_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(blws_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(G):
    lib = ctypes.CDLL(G.LIB_PATH)
    names = _declared()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding covers the whole header
    assert set(names) == set(G.api.SIGNATURES), set(names) ^ set(G.api.SIGNATURES)


def test_rng_bit_identical_to_oracle(G, O):
    for seed in (0, 1, 5489, 0xB10C ^ 0x5BDBEEF):
        rg, ro = G.Rng(seed), O.Rng(seed)
        assert [rg.next_u64() for _ in range(50)] == [ro.next_u64() for _ in range(50)]
        assert [rg.normal() for _ in range(33)] == [ro.normal() for _ in range(33)]
        assert [rg.uniform(-500.0, 500.0) for _ in range(20)] == [ro.uniform(-500.0, 500.0) for _ in range(20)]
        assert [rg.uniform_index(97) for _ in range(20)] == [ro.uniform_index(97) for _ in range(20)]
        sg, so = rg.split(13), ro.split(13)
        assert np.array_equal(sg.gaussian_matrix(7, 5), so.gaussian_matrix(7, 5))


def test_mt19937_64_known_answer(G):
    r = G.Rng(5489)
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042  # C++ [rand.predef]


def test_sample_distinct_matches_oracle(G, O):
    for n, s, seed in [(6400, 640, 21), (250000, 12500, 1), (10**6, 3 * 10**5, 4)]:
        a = G.sample_distinct(n, s, G.Rng(seed).split(4))
        b = O.sample_distinct(n, s, O.Rng(seed).split(4))
        assert len(a) == s and np.array_equal(a, b)
        assert np.all(np.diff(a) > 0)
