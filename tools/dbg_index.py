"""Debug: one step of a small hierarchical-index case, GPU vs oracle, printing where they differ."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle
from gpu_harness import Case

for n, k, fused in [(20000, 32, False), (1 << 20, 128, True)]:
    c = Case(L=1, B=1, Hq=8, Hkv=2, n=n, P=16, k=k, C=4096 if n > 100000 else 200, policy="la", seed=51,
             fused=fused, index_ratio=4)
    c.check_index()
    q = c.queries(0, 0)
    g = c.gpu_layer(0, q, 1)
    o = c.oracle_layer(0, q, 1)
    for h in range(2):
        ref = o[(0, h)]
        nb = len(ref["scores"])
        sc = c.cache.read_scores(0, 0, h, nb)
        diff = np.nonzero(sc.view(np.uint32) != ref["scores"].view(np.uint32))[0]
        print(n, h, "ids equal", np.array_equal(g["ids"][0, h], ref["ids"]), "la diffs", len(diff), diff[:10],
              sc[diff[:5]], ref["scores"][diff[:5]])
        print("  gpu ids", g["ids"][0, h][:12], " ref", ref["ids"][:12])
