"""Phase timelines of the step kernels (experiment build: KVD_BUILD_EXPERIMENTS=1, env KVD_EXP_TRACE=1).

    python tools/exp_trace.py --config c2 [--chain-size 8] [--layers 1]

Runs the bench's Runner to steady state, then one layer of one chain eagerly: the select kernel
(kvd_select_resolve_fetch) and the attention kernel (kvd_sparse_decode) separately synchronised,
and prints per-phase percentiles (us after the first unit's entry) of every CTA / warp."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["KVD_EXP_TRACE"] = "1"

import bench  # noqa: E402


def read(lib, units):
    out = np.zeros((units, 8), np.uint64)
    rc = lib.kvd_exp_read_trace(out.ctypes.data_as(ctypes.c_void_p), units)
    assert rc == 0, lib.kvd_last_error()
    return out


def show(name, tr, phases):
    used = tr[:, 0] > 0
    if not used.any():
        print(f"{name}: no stamps")
        return
    tr = tr[used].astype(np.float64)
    t0 = tr[:, 0].min()
    print(f"{name}: {used.sum()} units")
    for i, ph in enumerate(phases):
        v = tr[:, i]
        v = v[v > 0]
        if len(v) == 0:
            continue
        v = (v - t0) * 1e-3
        print(f"   {ph:12s} min {v.min():7.2f}  p10 {np.percentile(v, 10):7.2f}  p50 {np.percentile(v, 50):7.2f}"
              f"  p90 {np.percentile(v, 90):7.2f}  max {v.max():7.2f} us")


def main():
    import argparse
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--chain-size", type=int, default=0, help="requests per launch (0 = whole batch)")
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    args = bench.parse(["--config", a.config, "--layers", str(a.layers), "--steps", "2", "--warmup", "1"])
    cfg = dict(bench.CONFIGS[a.config])
    cfg["L"] = a.layers
    dev = torch.device("cuda", 0)
    R = bench.Runner(args, cfg, 0, dev)
    from paper_2605_18071_b200 import kvd
    lib = kvd.lib()
    lib.kvd_exp_read_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
    print(lib.kvd_version().decode())
    s = torch.cuda.Stream()
    for _ in range(R.fill):
        R.eager_step(s)
    s.synchronize()
    nb = a.chain_size or R.B
    k = cfg["k"]
    for rep in range(a.reps):
        read(lib, 16384)
        with torch.cuda.stream(s):
            R.q_cur.copy_(R.q_dev[R.row()])
        R.t += 1
        q = R.q_cur[0, :nb]
        R.cache.select_resolve_fetch(0, q, R.reqs[:nb], k, R.t, R.ids[0, :nb], R.attn[0, :nb], stream=s)
        s.synchronize()
        tr = read(lib, 16384)
        show(f"[{rep}] select_kernel ({nb} requests)", tr[:8192],
             ["entry", "after_wait", "keys", "first_digit", "compacted", "threshold", "emitted", "end"])
        if tr[8192:, 0].any():
            show(f"[{rep}] cand_kernel (index stage 2)", tr[8192:],
                 ["entry", "after_wait", "candidates", "la_scores", "scored", "radix", "emitted", "end"])
        R.cache.sparse_decode(0, q, R.reqs[:nb], R.attn[0, :nb], R.W, R.out[0, :nb], R.lse[0, :nb], stream=s)
        s.synchronize()
        show(f"[{rep}] attn_kernel", read(lib, 16384), ["entry", "after_wait", "tile0", "stream_end", "merged"])


if __name__ == "__main__":
    main()
