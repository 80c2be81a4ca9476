"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a, loads,
exports every symbol include/argus.h declares, and its host-only helpers agree
with the oracle.  No compute calls (there is no GPU here)."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def argus():
    from paper_2511_06724_b200 import build
    build.build()
    from paper_2511_06724_b200 import argus as a
    return a


def header_symbols():
    with open(os.path.join(ROOT, "include", "argus.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(argus_\w+)\s*\(", src)))


def test_header_symbols_exported(argus):
    decl = header_symbols()
    assert len(decl) >= 15
    assert sorted(argus.SYMBOLS) == decl
    out = subprocess.run(["nm", "-D", "--defined-only", argus.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (argus_\w+)", out))
    assert set(decl) <= exported, set(decl) - exported
    # nothing else leaks from the library
    assert exported == set(decl)


def test_library_is_sm100a(argus):
    out = subprocess.run(["cuobjdump", "--list-elf", argus.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_quota_helper_matches_oracle(argus):
    rng = np.random.default_rng(0)
    for _ in range(300):
        L = int(rng.integers(1, 33))
        N = int(rng.integers(0, 9000))
        f = rng.random(L) * (rng.random(L) < 0.85)
        if f.sum() == 0:
            f[-1] = 0.5
        np.testing.assert_array_equal(argus.argus_quota_from_fractions(f, N), oracle.quota_from_fractions(f, N))
    with pytest.raises(argus.ArgusError):
        argus.argus_quota_from_fractions([0.0, 0.0], 3)
    with pytest.raises(argus.ArgusError):
        argus.argus_quota_from_fractions([np.nan, 1.0], 3)


def test_strerror(argus):
    assert argus.strerror(0) == "ok"
    assert "capacity" in argus.strerror(argus.ARGUS_E_CAPACITY)
    assert "unknown" in argus.strerror(12345)


def test_init_rejects_bad_config_without_touching_gpu(argus):
    from synth import argus_inputs as gen
    p = gen.small_problem("C1", N=4, M=0)
    with pytest.raises(argus.ArgusError) as e:   # d not a multiple of 64
        argus.Router(100, 4, p.opts, np.zeros((256, 104), np.float32), p.b1, p.W2, p.b2, 10, 4)
    assert e.value.code == argus.ARGUS_E_INVALID
    bad = [dict(o) for o in p.opts]
    bad[0]["k_skip"] = 5                          # option 0 must be the full model
    with pytest.raises(argus.ArgusError) as e:
        argus.Router(768, 4, bad, p.W1, p.b1, p.W2, p.b2, 10, 4)
    assert e.value.code == argus.ARGUS_E_INVALID
    bad = [dict(o) for o in p.opts]
    bad[2]["p_th_qpm"] = 1.0                      # p_th must be non-decreasing (slow -> fast)
    with pytest.raises(argus.ArgusError):
        argus.Router(768, 4, bad, p.W1, p.b1, p.W2, p.b2, 10, 4)
    W1 = p.W1.copy()
    W1[3, 7] = np.inf
    with pytest.raises(argus.ArgusError):
        argus.Router(768, 4, p.opts, W1, p.b1, p.W2, p.b2, 10, 4)


def test_product_never_imports_oracle():
    """The CUDA path shares no code with the oracle and never loads it."""
    pkg = os.path.join(ROOT, "paper_2511_06724_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "argus_oracle" not in src and "liboracle" not in src, f
    lib = os.path.join(pkg, "libargus.so")
    if os.path.exists(lib):
        out = subprocess.run(["ldd", lib], capture_output=True, text=True).stdout
        assert "oracle" not in out
