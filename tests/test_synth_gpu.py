"""The device K/V generator (synth/synth_gpu.cu, used by bench.py) writes exactly
the bytes of the host generator (synth/synth.c) that the oracle tests use."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,l,r,Hkv,n", [(0, 0, 0, 2, 4096), (3, 5, 7, 3, 1000), (1, 2, 9, 1, 17)])
def test_device_generator_is_byte_identical(seed, l, r, Hkv, n):
    K, V = synth.request_kv(seed, l, r, Hkv, n)
    Kd = torch.empty((Hkv, n, 128), dtype=torch.int16, device="cuda")
    Vd = torch.empty_like(Kd)
    synth.request_kv_device(seed, l, r, Hkv, n, Kd, Vd)
    assert np.array_equal(Kd.cpu().numpy().view(np.uint16), K)
    assert np.array_equal(Vd.cpu().numpy().view(np.uint16), V)
