"""CPU checks of the C-ABI library: it loads, exports every symbol the header
declares, and its host-side logic (pool sizing, argument validation, error
taxonomy) matches the reference without touching a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hierasparse_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2604_16864_b200 import build, capi
    build.build()
    return capi.load()


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"HS_API\s+[\w\s\*]+?\b(hs_\w+)\s*\(", src)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    from paper_2604_16864_b200 import capi
    assert syms == sorted(capi.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.hs_version() == 1


def test_library_is_sm100a_only(lib):
    import subprocess
    from paper_2604_16864_b200 import capi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


@pytest.mark.parametrize("rows,s,sink,window", [
    (131072, 1.0, 0, 0), (65536, 0.75, 0, 0), (4096, 0.5, 64, 100), (48 * 64, 1.0, 1, 9 * 64),
    (1024, 0.3, 64 * 16, 64 * 16), (64, 0.0, 0, 0), (0, 1.0, 0, 0),
])
def test_pool_counts_match_oracle(lib, port, rows, s, sink, window):
    from paper_2604_16864_b200 import hierasparse as hs
    nb, dc, sc, pre, suf = hs.pool_counts(rows, hs.SparsityConfig(s, s, 64, sink, window), s)
    p, q, quota = port.pool_counts(rows, 64, s, sink, window)
    assert (nb, dc, sc, pre, suf) == (rows // 64, rows // 64 - quota, quota, p, q)


def test_pool_counts_errors(lib):
    from paper_2604_16864_b200 import ConfigError
    from paper_2604_16864_b200 import hierasparse as hs
    with pytest.raises(ConfigError):
        hs.pool_counts(100, hs.SparsityConfig(0.5, 0.5, 64), 0.5)      # rows % B
    with pytest.raises(ConfigError):
        hs.pool_counts(128, hs.SparsityConfig(1.5, 0.5, 64), 0.5)      # s_key outside [0, 1]
    with pytest.raises(ConfigError):
        hs.pool_counts(64 * 40000, hs.SparsityConfig(0, 0, 64), 0.0)   # int16 index capacity


def test_cache_bytes(lib):
    from paper_2604_16864_b200 import capi
    c = capi.DeviceCacheC(0, 0, 128, 64, 8, 2048, 0, 2048, None, None, None, None, None)
    vals = [C.c_uint64() for _ in range(5)]
    capi.check(lib.hs_cache_bytes(C.byref(c), *[C.byref(v) for v in vals]))
    idx, den, nnz, meta, sb = (v.value for v in vals)
    # measure_size (compressed_cache.hpp:303-310) per unit x 8 units
    assert (idx, den, nnz, meta) == (8 * 4096, 0, 8 * 16777216, 8 * 2097152)
    assert sb == 8 * 2048 * 4


def test_attention_argument_validation_without_gpu(lib):
    """Workload validation mirrors check_view_pair (attention.hpp:139-156) and
    returns before any device work."""
    from paper_2604_16864_b200 import ConfigError, capi
    k = capi.DeviceCacheC(0, 1, 128, 64, 1, 4, 0, 4, 1, None, 1, 1, None)  # value-grouped in the key slot
    v = capi.DeviceCacheC(0, 1, 128, 64, 1, 4, 0, 4, 1, None, 1, 1, None)
    rc = lib.hs_decode(1, C.byref(k), C.byref(v), None, None, 0, 4, 0.1, 0, 1, None)
    with pytest.raises(ConfigError, match="channel-grouped"):
        capi.check(rc)
    k.axis = 0
    rc = lib.hs_decode(1, C.byref(k), C.byref(v), None, None, 0, 0, 0.1, 0, 1, None)
    with pytest.raises(ConfigError, match="no query rows"):
        capi.check(rc)
    bad = capi.DeviceCacheC(0, 0, 64, 64, 1, 4, 0, 4, 1, None, 1, 1, None)  # head_dim 64 vs 128
    rc = lib.hs_decode(1, C.byref(bad), C.byref(v), None, None, 0, 4, 0.1, 0, 1, None)
    with pytest.raises(ConfigError, match="head dims differ"):
        capi.check(rc)
    odd = capi.DeviceCacheC(0, 0, 130, 64, 1, 4, 0, 4, 1, None, 1, 1, None)  # d not a multiple of 4
    rc = lib.hs_decode(1, C.byref(odd), C.byref(v), None, None, 0, 4, 0.1, 0, 1, None)
    with pytest.raises(ConfigError, match="m_group"):
        capi.check(rc)


def test_closed_form_flop_count_matches_oracle(port):
    """hierasparse.flop_count == flop_and_byte_count (attention.hpp:426-467) on
    random masks, causal and not, with and without a dense tail."""
    import numpy as np
    from oracle.oracle import SparsityConfig
    from paper_2604_16864_b200.hierasparse import flop_count
    rng = np.random.default_rng(4)
    for it in range(60):
        B, d = 16, 32
        nb = 1 + int(rng.integers(0, 12))
        tail = int(rng.integers(0, B)) if it % 3 == 0 else 0
        x = np.zeros((nb * B, d), np.float32)
        kf = rng.integers(0, 2, nb).astype(np.uint8)
        vf = rng.integers(0, 2, nb).astype(np.uint8)
        kc = port.compress_with_flags(x, SparsityConfig(block_size=B), 0, kf)
        vc = port.compress_with_flags(x, SparsityConfig(block_size=B), 1, vf)
        n_kv = nb * B + tail
        causal = bool(it % 2)
        n_q = 1 + int(rng.integers(0, n_kv)) if causal else 1 + int(rng.integers(0, 40))
        want = port.flop_and_byte_count(n_q, d, kc, vc, tail, causal)[0]
        kd = kf if (kc.sparse_count and kc.dense_count) else [int(kc.sparse_count == 0)] * nb
        vd = vf if (vc.sparse_count and vc.dense_count) else [int(vc.sparse_count == 0)] * nb
        assert flop_count(kd, vd, B, d, n_q, tail, causal) == want, it


def test_cpp_header_is_standalone():
    """include/hierasparse_b200.hpp compiles on its own (no reference headers)."""
    import shutil
    import subprocess
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    inc = os.path.join(ROOT, "include")
    src = '#include "hierasparse_b200.hpp"\nint main() { hierasparse::b200::SparsityConfig c; return (int)c.block_size - 64; }\n'
    out = subprocess.run([gxx, "-std=c++17", "-fsyntax-only", "-I", inc, "-I", "/usr/local/cuda/include", "-x", "c++",
                          "-"], input=src, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
