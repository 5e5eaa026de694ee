"""CPU-side checks of the boundary: libkvd.so loads without a GPU, exports every
symbol include/kvd.h declares, and validates configurations synchronously."""
import ctypes
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
