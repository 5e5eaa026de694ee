"""A small decode run for compute-sanitizer (tests/test_gpu_sanitizer.py): c1 (resident) and
c1-evict (host-backed, 69 slots, evictions) through both call paths, flat and hierarchical index,
with the oracle check of the harness."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gpu_harness import Case  # noqa: E402

for kw in (dict(C=None, fused=False), dict(C=69, fused=False, policy="la"), dict(C=69, fused=True, policy="lru"),
           dict(C=69, fused=True, policy="la", index_ratio=4)):
    c = Case(L=1, B=1, Hq=8, Hkv=2, n=4096, P=16, k=32, seed=3, **kw)
    c.run(steps=3)
print("sanitize case ok")
