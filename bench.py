"""bench.py — decode-step throughput of the KVDrive hot path on B200 (libkvd).

One "step" = one decode token for every request of the batch through all L
layers: per layer, kvd_select_resolve_fetch (a1+a2+a3+a4: score kernel, then
one fused top-k + resolve + fetch kernel; --unfused: kvd_select_topk then
kvd_resolve_and_fetch) -> kvd_sparse_decode (a5+a6), layers serially
(DESIGN.md §2).  The per-kernel roofline pass times the three separate calls.  The whole step
is captured once as a CUDA graph and replayed; the decode-step index lives in
device memory (kvd_set_device_step) so every replay is a new step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
    python bench.py --impl reference ...   # the CPU oracle on a bounded sample

Multi-GPU (torchrun, one process per GPU): (request, KV-head) units are
independent through every row, so every rank serves its own
B requests (global batch N*B, weak scaling) with no collective on the decode
path; the only collectives are the timing barrier and the max-over-ranks.

Inputs are seeded synthetic Llama-3.1-8B / Qwen2.5-1M-shaped K/V/queries
(synth/), resident in HBM (or in the pinned host store for the
host-backed configs) before the timed region.  Every step touches far more
than the 126 MB L2 (3.3 GB at c2, 13 GB + host fetches at c3), so no flush is
needed ("l2": "inputs larger than L2").
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np


def ncu_traffic(config, bound, dom):
    """DRAM bytes per ABI call (scaled per segment) from the committed ncu capture, or None."""
    if bound != "hbm":
        return None
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "*_ncu_traffic.json")))
    if not files:
        return None
    try:
        d = json.load(open(files[-1]))
        e = d[config][dom]
        return {"bytes_per_call": e["dram_bytes_per_call"], "segments": e["segments"],
                "source": f"{os.path.basename(files[-1])}: {e['kernels']}"}
    except (KeyError, ValueError, OSError):
        return None


def kvd_launch_count():
    from paper_2605_18071_b200 import kvd
    return int(kvd.lib().kvd_launch_count())

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs: per-rank shapes.
CONFIGS = {
    "c1": dict(chains=1, L=1, B=1, Hq=8, Hkv=2, n=4096, P=16, k=32, C=None, alias=0,
               desc="1 req, 1 layer, 8q/2kv, d128, 4k ctx, block 16, top-k 32, resident"),
    "c2": dict(chains=8, L=32, B=8, Hq=32, Hkv=8, n=32768, P=16, k=128, C=None, alias=0,
               desc="Llama-3.1-8B shapes (32 layers, 32q/8kv, d128) bf16, 32k ctx, batch 8, top-k 2048 tokens, resident"),
    "c3": dict(chains=16, L=32, B=16, Hq=32, Hkv=8, n=131072, P=16, k=128, C=2048, alias=4,
               desc="Llama-3.1-8B shapes, 128k ctx, batch 16, GPU cache 25% of KV (2048 slots/segment), misses "
                    "gathered from pinned host DRAM, top-k 2048 tokens"),
    "c4": dict(chains=4, L=28, B=4, Hq=28, Hkv=4, n=1 << 20, P=16, k=128, C=16384, alias=2,
               desc="Qwen2.5-7B-1M shapes (28 layers, 28q/4kv, d128), 1M ctx, batch 4, GPU cache 25%, host-backed"),
    "c5": dict(chains=16, L=32, B=64, Hq=32, Hkv=8, n=131072, P=16, k=128, C=768, alias=2,
               desc="Llama-3.1-8B shapes, 128k ctx, batch 64, GPU cache 768 slots/segment (9.4%), host-backed"),
}
METRIC = "decode tokens/s at 128k ctx; sparse-attn HBM GB/s % peak; fetch GB/s, 1-8 GPU"
RECORD = 8192           # bytes of one 16-token K||V block record (bf16)
SUMMARY = 256           # bytes of one block summary (128 bf16)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="kvd", choices=["kvd", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--policy", default="la", choices=["lru", "lfu", "la"])
    ap.add_argument("--alpha", type=float, default=0.9)
    ap.add_argument("--alias", type=int, default=None, help="host-layer alias A (layer l uses synthetic layer l %% A)")
    ap.add_argument("--fill", type=int, default=None, help="untimed cache-fill steps before warm-up")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch layer by layer instead of graph replay")
    ap.add_argument("--chains", type=int, default=None,
                    help="micro-batch chains (SFC overlap): the batch is split into this many request groups, "
                         "each run through all layers on its own stream inside the graph")
    ap.add_argument("--shard", default="requests", choices=["requests", "heads"],
                    help="multi-GPU unit assignment: 'requests' = every rank serves its own B requests (weak "
                         "scaling, no collective); 'heads' = the config's B*Hkv units are partitioned over the "
                         "ranks (strong scaling; SURVEY 8.6) and the fp32 outputs are all-gathered each step")
    ap.add_argument("--unfused", action="store_true",
                    help="step through kvd_select_topk + kvd_resolve_and_fetch instead of the fused "
                         "kvd_select_resolve_fetch (same results)")
    ap.add_argument("--layers", type=int, default=None, help="override L (profiling only; not a bench number)")
    ap.add_argument("--cpu-sample-s", type=float, default=12.0, help="target seconds of oracle work")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- algorithmic bytes
def per_segment_bytes(cfg, misses_per_seg=0.0):
    nb = (cfg["n"] + cfg["P"] - 1) // cfg["P"]
    G = cfg["Hq"] // cfg["Hkv"]
    k = cfg["k"]
    p = 1 + (64 + cfg["P"] - 1) // cfg["P"]          # sink block + local blocks (n % P == 0)
    return dict(
        select=SUMMARY * nb + 2 * G * 128 + 8 * k,          # summaries + q + (ids, scores)
        attn=RECORD * (k + p) + 2 * G * 128 + 4 * G * 128 + 4 * G,   # K/V pages + q + o + lse
        fetch=RECORD * misses_per_seg,                     # host link read (and HBM write)
    )


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        self.t.join(1)
        sm = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8 for i in range(4)
                          if r[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ---------------------------------------------------------------- the GPU arm
class Runner:
    def __init__(self, args, cfg, rank, dev):
        import torch
        import synth
        from paper_2605_18071_b200 import KVCache
        self.torch, self.args, self.cfg, self.rank, self.dev = torch, args, cfg, rank, dev
        L, B, Hq, Hkv, n, P, k = (cfg[x] for x in ("L", "B", "Hq", "Hkv", "n", "P", "k"))
        self.G = G = Hq // Hkv
        nb = (n + P - 1) // P
        C = cfg["C"] if cfg["C"] is not None else nb
        A = args.alias if args.alias is not None else cfg["alias"]
        A = A if (A and A < L) else L
        if C < nb and args.alias is None:
            # keep every rank's pinned host store under ~40 % of the box's RAM (all ranks share it)
            world_ = int(os.environ.get("WORLD_SIZE", "1"))
            per_layer = cfg["B"] * cfg["Hkv"] * nb * RECORD
            ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
            A = max(1, min(A, int(0.4 * ram / world_ // per_layer)))
        self.A = A
        self.resident = C >= nb
        from paper_2605_18071_b200 import dist as kdist
        world = int(os.environ.get("WORLD_SIZE", "1"))
        self.mode = getattr(args, "shard", "requests")
        self.h0 = 0
        if self.mode == "heads":
            # strong scaling: this rank owns heads h0..h1-1 of some of the config's B requests
            self.all_parts = kdist.unit_partition(B, Hkv, world)
            self.greqs, self.h0, h1 = kdist.rank_heads(self.all_parts[rank])
            Hkv = h1 - self.h0
            Hq = Hkv * G
            B = len(self.greqs)
        else:
            self.greqs = kdist.rank_requests(rank, world, B)   # synthetic identity of this rank's requests
        self.B, self.Hkv, self.Hq = B, Hkv, Hq                  # this rank's (local) shapes
        self.reqs = list(range(B))
        self.cache = KVCache(num_layers=L, num_q_heads=Hq, num_kv_heads=Hkv, block_tokens=P, max_requests=B,
                             max_context=n, slots_per_segment=C, max_select=k, sink_tokens=4, local_tokens=64,
                             policy=args.policy, host_layer_alias=(0 if self.A == L else self.A), device=dev.index)
        self.W = self.cache.attn_width(k)
        t0 = time.time()
        Kd = torch.empty((Hkv, n, 128), dtype=torch.int16, device=dev)
        Vd = torch.empty_like(Kd)
        for sl in range(self.A):
            for r, gr in zip(self.reqs, self.greqs):
                synth.request_kv_device(args.seed, sl, gr, Hkv, n, Kd, Vd, head0=self.h0)
                for l in range(sl, L, self.A):
                    self.cache.load_prefix(l, r, Kd, Vd, n)
        del Kd, Vd
        torch.cuda.synchronize(dev)
        self.setup_s = time.time() - t0
        # queries for every step of the run, per synthetic layer: [T][L][B][Hq][128]
        self.fill = max(1, args.fill if args.fill is not None else (1 if self.resident else max(4, 2 * C // k)))
        self.T = self.fill + args.warmup + 3 * args.steps + 2
        Hkv_all = cfg["Hkv"]
        qs = [synth.batch_queries(args.seed, sl, self.greqs, Hkv_all, G, t0=0, nsteps=self.T,
                                  alpha=args.alpha)[:, :, self.h0 * G:(self.h0 + Hkv) * G]
              for sl in range(self.A)]
        qh = np.stack([qs[l % self.A] for l in range(L)], axis=1)        # [T][L][B][Hq][128]
        self.q_host = torch.from_numpy(qh.view(np.int16)).pin_memory()
        self.q_dev = self.q_host.to(dev)
        self.q_cur = torch.empty_like(self.q_dev[0])
        self.ids = torch.empty((L, B, Hkv, k), dtype=torch.int32, device=dev)
        self.attn = torch.empty((L, B, Hkv, self.W, 2), dtype=torch.int32, device=dev)
        self.out = torch.empty((L, B, Hq, 128), dtype=torch.float32, device=dev)
        self.lse = torch.empty((L, B, Hq), dtype=torch.float32, device=dev)
        self.out_host = torch.empty_like(self.out, device="cpu").pin_memory()
        self.step_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.t = 0                     # next step index to run (query row)
        m = args.chains if args.chains else cfg.get("chains", 1)
        m = max(1, min(m, B))
        edges = [round(i * B / m) for i in range(m + 1)]
        self.chains = [(edges[i], edges[i + 1]) for i in range(m) if edges[i + 1] > edges[i]]
        self.chain_streams = [torch.cuda.Stream(device=dev) for _ in self.chains]
        self.fused = not args.unfused
        self.launches_per_step = None  # counted by libkvd (kvd_launch_count) over one eager step / the capture

    # one layer of one chain (requests b0..b1-1) through the three ABI calls
    def layer(self, l, s, step=0, chain=None):
        c, k = self.cache, self.cfg["k"]
        b0, b1 = chain if chain else (0, len(self.reqs))
        reqs = self.reqs[b0:b1]
        q = self.q_cur[l, b0:b1]
        if self.fused:   # kvd_select_resolve_fetch: top-k, resolve and fetch with no kernel boundary
            c.select_resolve_fetch(l, q, reqs, k, step, self.ids[l, b0:b1], self.attn[l, b0:b1], stream=s)
        else:
            c.select_topk(l, q, reqs, k, self.ids[l, b0:b1], None, stream=s)
            c.resolve_and_fetch(l, reqs, self.ids[l, b0:b1], k, step, self.attn[l, b0:b1], stream=s)
        c.sparse_decode(l, q, reqs, self.attn[l, b0:b1], self.W, self.out[l, b0:b1], self.lse[l, b0:b1], stream=s)

    def eager_step(self, s):
        torch = self.torch
        with torch.cuda.stream(s):
            self.q_cur.copy_(self.q_dev[self.t], non_blocking=True)
        self.t += 1
        self.cache.set_device_step(None)
        n0 = kvd_launch_count()
        for l in range(self.cfg["L"]):
            self.layer(l, s, step=self.t)
        self.launches_per_step = kvd_launch_count() - n0

    def capture(self, s):
        torch = self.torch
        self.cache.set_device_step(self.step_dev)
        g = torch.cuda.CUDAGraph()
        n0 = kvd_launch_count()
        with torch.cuda.graph(g, stream=s):
            self.step_dev.add_(1)
            # SFC overlap: each request group runs its own chain of layers on its own stream
            # (fork from / join to the capture stream); groups share no state, so the GPU
            # overlaps one chain's host-link gathers with the others' HBM-bound kernels
            for ch, cs in zip(self.chains, self.chain_streams):
                cs.wait_stream(s)
                for l in range(self.cfg["L"]):
                    self.layer(l, cs, chain=ch)
            for cs in self.chain_streams:
                s.wait_stream(cs)
        self.launches_per_step = kvd_launch_count() - n0
        self.graph = g

    def prepare_graph(self, s):
        """Capture the step graph; the device step counter continues from the eager steps."""
        torch = self.torch
        self.step_dev.fill_(self.t)
        torch.cuda.synchronize(self.dev)
        self.capture(s)

    def graph_step(self, s, source="dev"):
        torch = self.torch
        with torch.cuda.stream(s):
            if source == "dev":
                self.q_cur.copy_(self.q_dev[self.t], non_blocking=True)
            else:
                self.q_cur.copy_(self.q_host[self.t], non_blocking=True)
            self.graph.replay()
            if source != "dev":
                self.out_host.copy_(self.out, non_blocking=True)
        self.t += 1


def run_gpu(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2605_18071_b200 import build as kb
    if rank == 0 or not os.path.exists(kb.SO):
        kb.build()
    import synth
    synth.build_gpu()
    cfg = dict(CONFIGS[args.config])
    if args.layers:
        cfg["L"] = args.layers

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    from paper_2605_18071_b200 import dist as kdist

    def max_over_ranks(x):
        return kdist.max_over_ranks(x, dev)

    def sum_over_ranks(x):
        return kdist.sum_over_ranks(x, dev)

    R = Runner(args, cfg, rank, dev)
    s = torch.cuda.Stream(device=dev)
    L, B, Hkv = cfg["L"], R.B, R.Hkv                          # this rank's shapes
    segs_per_layer = B * Hkv
    heads_mode = R.mode == "heads" and world > 1
    # all_gather_into_tensor output: per-rank outputs concatenated along dim 0 ([world*L][B_r][Hq_r][128])
    gathered = (torch.empty((world * R.out.shape[0],) + tuple(R.out.shape[1:]), dtype=R.out.dtype, device=dev)
                if heads_mode else None)

    def gather_outputs():
        # head sharding: the step's per-rank fp32 outputs -> every rank (NCCL over NVLink)
        with torch.cuda.stream(s):
            dist.all_gather_into_tensor(gathered, R.out)
    # cache fill (cold start -> steady state; untimed, parity-checked in tests)
    for _ in range(R.fill):
        R.eager_step(s)
    s.synchronize()
    # capture one step as a CUDA graph (the step index is read on the device)
    if not args.no_graph:
        R.prepare_graph(s)
    step_fn = (lambda: R.eager_step(s)) if args.no_graph else (lambda: R.graph_step(s))

    def run():
        step_fn()
        if heads_mode:
            gather_outputs()
    clk = ClockSampler(local)          # sampled from warm-up through the e2e pass (GPU busy throughout)
    clk.start()
    for _ in range(args.warmup):
        run()
    s.synchronize()
    R.cache.reset_stats()
    # ---- timed region: K steps, device-timed on the launching stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(s)
    for _ in range(args.steps):
        run()
    ev1.record(s)
    ev1.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    st = R.cache.stats()
    ms_max = max_over_ranks(ms)
    # whole-job tokens: requests mode sums every rank's requests; heads mode counts each
    # of the config's requests once (its heads are spread over the ranks)
    tokens = cfg["B"] * args.steps if heads_mode else sum_over_ranks(B * args.steps)
    value = tokens / (ms_max * args.steps * 1e-3)
    hit_rate = st["hits"] / max(1, st["selected"])
    misses_per_seg = st["misses"] / max(1, args.steps * L * segs_per_layer)

    # ---- per-kernel pass: the same steps, each ABI call bracketed by CUDA events on the
    # launching stream.  A GPU spin (torch.cuda._sleep) gates each step so the host has
    # queued every launch before the device starts: the events then see device time only.
    kt = {"select": 0.0, "resolve_fetch": 0.0, "attn": 0.0}
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(L)]
    npk = args.steps
    R.cache.set_device_step(None)
    for _ in range(npk):
        with torch.cuda.stream(s):
            torch.cuda._sleep(20_000_000)            # ~10 ms at 1.965 GHz: covers the host enqueue
            R.q_cur.copy_(R.q_dev[R.t], non_blocking=True)
        R.t += 1
        c = R.cache
        for l in range(L):
            e = evs[l]
            e[0].record(s)
            c.select_topk(l, R.q_cur[l], R.reqs, cfg["k"], R.ids[l], None, stream=s)
            e[1].record(s)
            c.resolve_and_fetch(l, R.reqs, R.ids[l], cfg["k"], R.t, R.attn[l], stream=s)
            e[2].record(s)
            c.sparse_decode(l, R.q_cur[l], R.reqs, R.attn[l], R.W, R.out[l], R.lse[l], stream=s)
            e[3].record(s)
        s.synchronize()
        for l in range(L):
            e = evs[l]
            kt["select"] += e[0].elapsed_time(e[1])
            kt["resolve_fetch"] += e[1].elapsed_time(e[2])
            kt["attn"] += e[2].elapsed_time(e[3])
    nl = npk * L
    per_launch_ms = {key: v / nl for key, v in kt.items()}
    b = per_segment_bytes(cfg, misses_per_seg)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs") or 6650.0
    hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs") else "fallback (B200_PROFILING.md)"
    link = host_link_probe(torch, dev) if not R.resident else None
    kernels = {}
    for key, by in (("select", b["select"]), ("attn", b["attn"])):
        gbs = by * segs_per_layer / (per_launch_ms[key] * 1e-3) / 1e9
        kernels[key] = {"ms_per_launch": per_launch_ms[key], "bytes_per_launch": by * segs_per_layer,
                        "gbs": gbs, "frac_hbm": gbs / hbm_peak}
    fetch_bytes = b["fetch"] * segs_per_layer
    kernels["resolve_fetch"] = {"ms_per_launch": per_launch_ms["resolve_fetch"], "host_bytes_per_launch": fetch_bytes,
                                "host_gbs": fetch_bytes / (per_launch_ms["resolve_fetch"] * 1e-3) / 1e9}
    if link:
        kernels["resolve_fetch"]["frac_host_link"] = kernels["resolve_fetch"]["host_gbs"] / link["gbs"]
    dom = max(per_launch_ms, key=per_launch_ms.get)
    if dom == "resolve_fetch" and link:
        roof = {"kernel": "resolve+gather (a3+a4)", "bound": "host-link", "achieved": kernels[dom]["host_gbs"],
                "peak": link["gbs"], "unit": "GB/s", "frac": kernels[dom]["frac_host_link"],
                "peak_source": "pinned H2D cudaMemcpy probe in this run", "traffic": None}
    else:
        if dom == "resolve_fetch":
            dom = "attn"
        roof = {"kernel": {"select": "score+topk (a1+a2)", "attn": "sparse decode + merge (a5+a6)"}[dom],
                "bound": "hbm", "achieved": kernels[dom]["gbs"], "peak": hbm_peak, "unit": "GB/s",
                "frac": kernels[dom]["frac_hbm"], "peak_source": hbm_src, "traffic": None}
    # traffic: DRAM bytes per launch of the dominant ABI call's kernels from one committed
    # `ncu --set full` capture (profiles/*_ncu_traffic.json, written by tools/ncu_traffic.py);
    # host-link-bound calls have no DRAM equivalent of their algorithmic bytes (null)
    tr = ncu_traffic(args.config, roof["bound"], dom)
    if tr:
        roof["traffic"] = tr["bytes_per_call"] * (segs_per_layer / tr["segments"])
        roof["traffic_source"] = tr["source"]
    # the attention kernel's roofline is always reported (north_star: sparse-attn HBM GB/s % peak)
    roof_attn = {"achieved": kernels["attn"]["gbs"], "peak": hbm_peak, "unit": "GB/s",
                 "frac": kernels["attn"]["frac_hbm"]}

    # ---- e2e: queries H2D from pinned host + result D2H inside the timed region
    e2e = None
    if not args.no_e2e and not args.no_graph:
        R.cache.set_device_step(R.step_dev)
        R.step_dev.fill_(R.t)
        torch.cuda.synchronize(dev)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.steps):
            R.graph_step(s, source="host")
            if heads_mode:
                gather_outputs()
        e1.record(s)
        e1.synchronize()
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        e2e = {"value": tokens / (ems * args.steps * 1e-3), "unit": "tokens/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(R.q_cur.numel() * 2), "d2h_bytes_per_step": int(R.out.numel() * 4)}
    R.cache.check()
    clocks = clk.stop()

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong" if heads_mode else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded; DESIGN.md §4)",
        "config": {"workload": args.config, "desc": cfg["desc"], "global_batch": cfg["B"] if heads_mode else B * world, "seq_len": cfg["n"],
                   "layers": L, "q_heads": cfg["Hq"], "kv_heads": cfg["Hkv"], "block_tokens": cfg["P"],
                   "top_k_blocks": cfg["k"], "slots_per_segment": cfg["C"] or (cfg["n"] // cfg["P"]),
                   "policy": args.policy, "alpha": args.alpha, "host_layer_alias": R.A if not R.resident else None,
                   "fill_steps": R.fill, "graph": not args.no_graph, "chains": len(R.chains), "fused_select_resolve": R.fused, "parallelism": (f"head-shard x{world} + NCCL all-gather" if heads_mode else f"request-shard x{world}"),
                   "l2": "inputs larger than L2 (no flush)"},
        "hit_rate": hit_rate, "misses_per_segment": misses_per_seg,
        "roofline": roof, "roofline_attn": roof_attn, "kernels": kernels,
        "host_link": link, "e2e": e2e, "gpu_launches": R.launches_per_step * args.steps,
        "clocks": clocks, "setup_s": R.setup_s,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, cfg, args.cpu_sample_s)
    if rank == 0:
        print(json.dumps(line), flush=True)
    R.cache.close()
    if world > 1:
        dist.destroy_process_group()


def host_link_probe(torch, dev, nbytes=1 << 30):
    """Pinned host -> HBM cudaMemcpy bandwidth (the host-link denominator)."""
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        d.copy_(h, non_blocking=True)
    e1.record()
    e1.synchronize()
    gbs = 4 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9
    del h, d
    return {"gbs": gbs, "how": "pinned H2D cudaMemcpyAsync, 1 GiB x4"}


# ---------------------------------------------------------------- the CPU oracle (baseline / reference arm)
def cpu_baseline(args, cfg, target_s):
    """Time the oracle (as it stands) on a bounded sample of the same workload:
    whole segments (select O2-O5 + resolve O6 + fetch O7 + attention O8) of one
    layer's decode step, scaled to tokens/s = B / (per-segment time x B*Hkv*L)."""
    import oracle
    import synth
    L, B, Hq, Hkv, n, P, k = (cfg[x] for x in ("L", "B", "Hq", "Hkv", "n", "P", "k"))
    G = Hq // Hkv
    nb = (n + P - 1) // P
    C = cfg["C"] if cfg["C"] is not None else nb
    W = k + 1 + (64 + P - 1) // P + 1
    done, spent, t_all = 0, 0.0, time.time()
    seg = 0
    while spent < target_s and time.time() - t_all < 3 * target_s and seg < B * Hkv:
        r, h = divmod(seg, Hkv)
        K, V = synth.segment_kv(args.seed, 0, r, h, n)
        S = oracle.block_summaries(K, P)          # setup (a0), not timed
        pinned = oracle.pinned_blocks(n, P)
        oc = oracle.SegmentCache(nb, C, pinned)
        q = synth.queries(args.seed, 0, r, h, G, t0=0, nsteps=3, alpha=args.alpha)
        for t in range(3):
            t0 = time.perf_counter()
            oracle.segment_step(oc, q[t], S, K, V, P, k, t + 1, oracle.POLICIES[args.policy], W)
            spent += time.perf_counter() - t0
            done += 1
        seg += 1
    per_seg = spent / max(1, done)
    step_s = per_seg * B * Hkv * L
    return {"value": B / step_s, "unit": "tokens/s", "cores": 1, "kind": "oracle",
            "sample": f"{done} segment-steps ({seg} segments x 3 steps) of layer 0, {spent:.1f} s of oracle work; "
                      f"scaled x{B * Hkv * L} segments/step"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = dict(CONFIGS[args.config])
    import oracle
    oracle.build()
    # K steps of a bounded per-step sample, after W warm-up samples
    per = max(1.0, min(10.0, 60.0 / max(1, args.steps)))
    for _ in range(min(args.warmup, 1)):
        cpu_baseline(args, cfg, 0.5)
    vals = [cpu_baseline(args, cfg, per) for _ in range(args.steps)]
    # one host runs the oracle for the whole job (N*B requests): tokens/s is the per-host rate
    v = float(np.mean([x["value"] for x in vals]))
    B = cfg["B"] * world
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": B / v * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (oracle)",
            "data": "synthetic (seeded; DESIGN.md §4)",
            "config": {"workload": args.config, "desc": cfg["desc"], "global_batch": B, "seq_len": cfg["n"]},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": 1, "kind": "oracle",
                             "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
