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
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC",
                               "-o", _SO, src, "-lm"])
    return _SO


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
        for f in (L.synth_segment_kv, L.synth_request_kv, L.synth_queries, L.synth_batch_queries):
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


def queries(seed, layer, req, head, G, d=128, t0=0, nsteps=1, alpha=0.9):
    """Decode queries of one KV head's G query heads: [nsteps][G][d] uint16."""
    out = np.empty((nsteps, G, d), np.uint16)
    lib().synth_queries(seed, layer, req, head, G, d, t0, nsteps, float(alpha), _ptr(out))
    return out


def batch_queries(seed, layer, reqs, Hkv, G, d=128, t0=0, nsteps=1, alpha=0.9):
    """Queries of a batch for one layer: [nsteps][B][Hkv*G][d] uint16."""
    reqs = np.ascontiguousarray(np.asarray(reqs, np.int32))
    B = len(reqs)
    out = np.empty((nsteps, B, Hkv * G, d), np.uint16)
    lib().synth_batch_queries(seed, layer, _ptr(reqs), B, Hkv, G, d, t0, nsteps, float(alpha), _ptr(out))
    return out


def bf16_bits_to_f32(a):
    """bf16 bit patterns -> float32 values (exact widening)."""
    return (np.asarray(a, np.uint16).astype(np.uint32) << 16).view(np.float32)
