"""Seeded synthetic inputs (keys, values, decode queries) — inputs only.

Shared by the CUDA path (bench, GPU tests) and the oracle tests.  Holds none
of the method's arithmetic; see synth.c for the recipe.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_GPU_SO = os.path.join(_HERE, "libsynth_gpu.so")
_lib = None
_glib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC",
                               "-o", _SO, src, "-lm"])
    return _SO


def build_gpu(force: bool = False) -> str:
    """Device copy of the K/V generator (synth_gpu.cu), sm_100a."""
    src = os.path.join(_HERE, "synth_gpu.cu")
    if force or not os.path.exists(_GPU_SO) or os.path.getmtime(_GPU_SO) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-Xcompiler", "-fPIC", "-shared", "-o", _GPU_SO + ".tmp", src])
        os.replace(_GPU_SO + ".tmp", _GPU_SO)
    return _GPU_SO


def glib():
    global _glib
    if _glib is None:
        build_gpu()
        L = ctypes.CDLL(_GPU_SO)
        L.synth_gpu_segment_kv.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p]
        L.synth_gpu_segment_kv.restype = ctypes.c_int
        _glib = L
    return _glib


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        u64, i64, i32, p = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        L.synth_segment_kv.argtypes = [u64, i64, i64, i64, i64, i32, p, p]
        L.synth_request_kv.argtypes = [u64, i64, i64, i32, i64, i32, p, p]
        L.synth_queries.argtypes = [u64, i64, i64, i64, i32, i32, i64, i64, ctypes.c_double, p]
        L.synth_batch_queries.argtypes = [u64, i64, p, i32, i32, i32, i32, i64, i64, ctypes.c_double, p]
        L.synth_batch_queries_x.argtypes = [u64, i64, i64, p, i32, i32, i32, i32, i64, i64, ctypes.c_double, p]
        L.synth_segment_plan.argtypes = [u64, i64, i64, i64, i64, i32, p, p, p]
        for f in (L.synth_segment_kv, L.synth_request_kv, L.synth_queries, L.synth_batch_queries,
                  L.synth_segment_plan):
            f.restype = None
        _lib = L
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def segment_kv(seed, layer, req, head, n, d=128):
    """K, V of one segment as bf16 bit patterns, token-major [n][d] uint16."""
    K = np.empty((n, d), np.uint16)
    V = np.empty((n, d), np.uint16)
    lib().synth_segment_kv(seed, layer, req, head, n, d, _ptr(K), _ptr(V))
    return K, V


def request_kv(seed, layer, req, Hkv, n, d=128, out_k=None, out_v=None):
    """K, V of all KV heads of one (layer, request): [Hkv][n][d] uint16.

    out_k / out_v may be caller-provided (e.g. pinned torch buffers viewed as
    numpy) so large prefixes are generated in place."""
    K = out_k if out_k is not None else np.empty((Hkv, n, d), np.uint16)
    V = out_v if out_v is not None else np.empty((Hkv, n, d), np.uint16)
    lib().synth_request_kv(seed, layer, req, Hkv, n, d, _ptr(K), _ptr(V))
    return K, V


def request_kv_device(seed, layer, req, Hkv, n, K, V, d=128, stream=None, head0=0):
    """Same bytes as request_kv, generated on the GPU into device torch tensors
    K, V [Hkv][n][d] (int16 / uint16 views of bf16) for KV heads head0 ..
    head0+Hkv-1.  Host computes the per-token topic runs and topic centres; the
    device expands them."""
    import torch
    topic = np.empty(n, np.uint8)
    mu = np.empty((32, d), np.float32)
    keys = np.empty(2, np.uint64)
    dev = K.device
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    for h in range(Hkv):
        lib().synth_segment_plan(seed, layer, req, head0 + h, n, d, _ptr(topic), _ptr(mu), _ptr(keys))
        t_d = torch.from_numpy(topic).to(dev)
        m_d = torch.from_numpy(mu).to(dev)
        rc = glib().synth_gpu_segment_kv(n, d, t_d.data_ptr(), m_d.data_ptr(), int(keys[0]), int(keys[1]),
                                         K[h].data_ptr(), V[h].data_ptr(), s)
        if rc:
            raise RuntimeError(f"synth_gpu_segment_kv: cuda error {rc}")
        torch.cuda.current_stream(dev).synchronize()


def queries(seed, layer, req, head, G, d=128, t0=0, nsteps=1, alpha=0.9):
    """Decode queries of one KV head's G query heads: [nsteps][G][d] uint16."""
    out = np.empty((nsteps, G, d), np.uint16)
    lib().synth_queries(seed, layer, req, head, G, d, t0, nsteps, float(alpha), _ptr(out))
    return out


def batch_queries(seed, layer, reqs, Hkv, G, d=128, t0=0, nsteps=1, alpha=0.9, stream_layer=None):
    """Queries of a batch for one layer: [nsteps][B][Hkv*G][d] uint16.  The queries follow
    the key topics of `layer`; `stream_layer` (default `layer`) keys their random streams, so
    a layer whose keys alias another's (host-layer aliasing) still gets its own queries."""
    reqs = np.ascontiguousarray(np.asarray(reqs, np.int32))
    B = len(reqs)
    out = np.empty((nsteps, B, Hkv * G, d), np.uint16)
    ls = layer if stream_layer is None else stream_layer
    lib().synth_batch_queries_x(seed, layer, ls, _ptr(reqs), B, Hkv, G, d, t0, nsteps, float(alpha), _ptr(out))
    return out


def bf16_bits_to_f32(a):
    """bf16 bit patterns -> float32 values (exact widening)."""
    return (np.asarray(a, np.uint16).astype(np.uint32) << 16).view(np.float32)
