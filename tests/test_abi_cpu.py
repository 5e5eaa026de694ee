"""CPU-side checks of the boundary: libkvd.so loads without a GPU, exports every
symbol include/kvd.h declares, and validates configurations synchronously."""
import ctypes

import numpy as np
import os
import re

import pytest

from paper_2605_18071_b200 import KVCache, KVDError, lib
from paper_2605_18071_b200.kvd import EXPORTS, LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "kvd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kvd_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(LIB_PATH)
    decl = header_functions()
    assert len(decl) >= 18
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(EXPORTS) == decl          # the binding covers the whole ABI
    assert lib().kvd_version().startswith(b"kvd")


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


BASE = dict(num_layers=32, num_q_heads=32, num_kv_heads=8, block_tokens=16, max_requests=8, max_context=32768,
            slots_per_segment=2048, max_select=128)


def test_required_bytes_c2_shape():
    dev, host = KVCache.required_bytes(**BASE)
    slots = 32 * 8 * 8 * 2048 * 8192
    summ = 32 * 8 * 8 * 128 * 2048 * 2
    assert host == 0
    assert slots + summ < dev < slots + summ + (1 << 30)


def test_required_bytes_host_backed_alias():
    kw = dict(BASE, max_requests=16, max_context=131072, host_layer_alias=4)
    dev, host = KVCache.required_bytes(**kw)
    assert host == 4 * 16 * 8 * 8192 * 8192          # A=4 host layers of 8 KiB records


@pytest.mark.parametrize("bad", [dict(head_dim=64), dict(num_q_heads=30), dict(block_tokens=3),
                                 dict(num_q_heads=80, num_kv_heads=8), dict(max_select=5000),
                                 dict(policy="mru" if False else 7), dict(max_context=0)])
def test_invalid_configs_rejected(bad):
    kw = dict(BASE)
    kw.update(bad)
    if kw.get("policy") == 7:
        kw.pop("policy")
        from paper_2605_18071_b200.kvd import Config
        cfg = Config(32, 32, 8, 128, 16, 8, 32768, 2048, 128, 4, 64, 7, 0, 0)
        d, h = ctypes.c_size_t(), ctypes.c_size_t()
        assert lib().kvd_required_bytes(ctypes.byref(cfg), ctypes.byref(d), ctypes.byref(h)) == 1
        return
    with pytest.raises(KVDError) as e:
        KVCache.required_bytes(**kw)
    assert e.value.status == "KVD_EINVAL"


def test_no_gpu_create_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(KVDError):
        KVCache(**dict(BASE, num_layers=1, max_requests=1, max_context=4096, slots_per_segment=256, max_select=32))


def test_config_limits_of_this_build():
    """Host-backed caches rank victims on chip (C <= ~27,000 at max_select 128) and the top-k
    cluster holds <= 262,144 blocks per request; both are rejected up front (include/kvd.h)."""
    with pytest.raises(KVDError):
        KVCache.required_bytes(**dict(BASE, max_context=1 << 20, slots_per_segment=40000))
    KVCache.required_bytes(**dict(BASE, max_context=1 << 20, slots_per_segment=16384))   # c4 fits
    KVCache.required_bytes(**dict(BASE, max_context=1 << 20, slots_per_segment=1 << 16))  # resident
    with pytest.raises(KVDError):
        KVCache.required_bytes(**dict(BASE, block_tokens=1, max_context=300000, slots_per_segment=1 << 20))


def test_step_calls_validate_before_launch():
    """Every step call rejects a NULL cache synchronously (nothing launched) and the launch
    counter does not move."""
    L = lib()
    n0 = L.kvd_launch_count()
    q = ctypes.c_void_p(0)
    reqs = (ctypes.c_int32 * 1)(0)
    assert L.kvd_select_topk(None, 0, q, reqs, 1, 8, q, q, q) == 1
    assert L.kvd_resolve_and_fetch(None, 0, reqs, 1, q, 8, 1, q, q) == 1
    assert L.kvd_select_resolve_fetch(None, 0, q, reqs, 1, 8, 1, q, q, q, q) == 1
    assert L.kvd_sparse_decode(None, 0, q, reqs, 1, q, 13, q, q, q) == 1
    assert L.kvd_select_resolve_fetch_heads(None, 0, q, reqs, 1, 0, 1, 8, 1, q, q, q, q) == 1
    assert L.kvd_sparse_decode_heads(None, 0, q, reqs, 1, 0, 1, q, 13, q, q, q) == 1
    assert L.kvd_launch_count() == n0
    assert b"NULL" in L.kvd_last_error() or b"null" in L.kvd_last_error()


def test_window_scaling_planner_matches_oracle_greedy():
    # the product's offline MCKP planner (host code in libkvd) against the oracle's greedy (O11,
    # itself pinned by exhaustive search), on random profile-like instances
    import oracle
    from paper_2605_18071_b200 import kvd
    rng = np.random.default_rng(7)
    for _ in range(50):
        pairs, sizes = int(rng.integers(1, 64)), int(rng.integers(2, 6))
        step = rng.integers(1, 6, size=(pairs, 1)).astype(np.float64)
        cost = step * np.arange(1, sizes + 1)[None, :]
        gains = -np.sort(-rng.random((pairs, sizes - 1)), axis=1) * rng.random((pairs, 1)) * 10
        benefit = np.concatenate([np.zeros((pairs, 1)), np.cumsum(gains, axis=1)], axis=1)
        budget = cost[:, 0].sum() + rng.random() * (cost[:, -1].sum() - cost[:, 0].sum())
        _, ref = oracle.mckp(benefit, cost, budget)
        assert np.array_equal(kvd.plan_window_scaling(benefit, cost, budget), ref)
    with pytest.raises(kvd.KVDError):
        kvd.plan_window_scaling(np.zeros((2, 2)), np.ones((2, 2)), 1.0)
