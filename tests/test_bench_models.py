"""CPU checks of bench.py's accounting: the prefill shared-memory model
(268 KB per dense 128x128 tile, 216 KB per 2:4 tile) and the
causal tile counts it is built on."""
import types

import torch

import bench


def _cache(nb, U, sparse):
    idx = torch.full((U, nb), -1 if sparse else 1, dtype=torch.int16)
    return types.SimpleNamespace(index_map=idx)


def _tiles_causal(L):
    n_qt = L // 128
    return n_qt * (n_qt + 1) // 2  # q-tile t sees t + 1 key tiles of 128 keys


def test_smem_model_per_tile_bytes():
    L, U, G = 8192, 2, 4
    nb = L // 64
    for sparse, per_tile in ((False, 268), (True, 216)):
        kc = vc = _cache(nb, U, sparse)
        got = bench.prefill_smem_bytes(kc, vc, L, G)
        assert got == _tiles_causal(L) * U * G * per_tile * 1024, (sparse, got)


def test_smem_model_mixed_between_dense_and_sparse():
    L, U, G = 8192, 1, 1
    nb = L // 64
    kc = _cache(nb, U, True)
    vc = _cache(nb, U, False)  # 2:4 keys, dense values
    got = bench.prefill_smem_bytes(kc, vc, L, G)
    lo = bench.prefill_smem_bytes(_cache(nb, U, True), _cache(nb, U, True), L, G)
    hi = bench.prefill_smem_bytes(_cache(nb, U, False), _cache(nb, U, False), L, G)
    assert lo < got < hi
