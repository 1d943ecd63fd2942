"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and the host build of the K0 generator reproduces numpy's
SeedSequence/PCG64/choice bits (the reference's sample_rows). No device
compute here."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2507_13681_b200 import _lib
from oracle import seeding as oseed

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "loopserve_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)  # drop comments
    return sorted(set(re.findall(r"(?:^|\n)\s*(?:int|size_t|uint64_t|const char \*)\s*(ls_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/loopserve_b200.h but not exported"
    assert set(names) == set(_lib.SIGNATURES), "ctypes signature table out of sync with the header"


def test_version_and_error_string():
    lib = _lib.lib()
    assert lib.ls_version() == 1
    n = ctypes.c_int32()
    assert lib.ls_sample_size(0, 0.1, 32, ctypes.byref(n)) == -8  # EmptyBlock
    assert b"empty" in lib.ls_last_error()


@pytest.mark.parametrize("n_new,rate,floor", [(1000, 0.1, 32), (5128, 0.1, 32), (10128, 0.1, 32),
                                              (1, 0.1, 32), (2, 0.1, 32), (33, 0.1, 32),
                                              (20000, 0.1, 32), (12000, 0.01, 32), (97, 1.0, 1)])
def test_sample_size_matches_reference_formula(n_new, rate, floor):
    n = ctypes.c_int32()
    assert _lib.lib().ls_sample_size(n_new, rate, floor, ctypes.byref(n)) == 0
    assert n.value == oseed.sample_size(n_new, rate, floor)


def test_host_generator_matches_golden(golden):
    lib = _lib.lib()
    for i, c in enumerate(golden.case("seeds")):
        hs = lib.ls_head_seed_host(c["session_seed"], c["turn"], c["layer"], c["head"])
        assert str(hs) == c["head_seed"]
        ref = golden[f"seeds/{i}/rows"]
        out = np.zeros(len(ref), dtype=np.int32)
        st = lib.ls_sample_rows_host(c["session_seed"], c["turn"], c["layer"], c["head"], c["n_new"],
                                     c["rate"], c["floor"], out.ctypes.data)
        assert st == 0
        assert np.array_equal(out, ref), f"case {i}"


def test_host_generator_matches_numpy_sweep():
    lib = _lib.lib()
    rng = np.random.Generator(np.random.PCG64(2024))
    for _ in range(200):
        seed = int(rng.integers(0, 2 ** 63))
        t, l, h = (int(x) for x in rng.integers(0, 100, size=3))
        n_new = int(rng.choice([int(rng.integers(1, 300)), int(rng.integers(300, 12000))]))
        rate = float(rng.choice([0.1, 0.05, 0.3, 1.0]))
        floor = int(rng.choice([1, 8, 32]))
        hs = oseed.head_seed(seed, t, l, h)
        assert lib.ls_head_seed_host(seed, t, l, h) == hs
        ref = oseed.sample_rows(n_new, rate, floor, hs)
        out = np.zeros(len(ref), dtype=np.int32)
        assert lib.ls_sample_rows_host(seed, t, l, h, n_new, rate, floor, out.ctypes.data) == 0
        assert np.array_equal(out, ref)
