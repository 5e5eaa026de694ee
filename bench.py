"""bench.py — decode-step throughput of the KVDrive hot path on B200 (libkvd).

One "step" = one decode token for every request of the batch through all L
layers: per layer, kvd_select_resolve_fetch (a1+a2+a3+a4: one kernel scores the
block summaries, selects the top-k, resolves them against the GPU cache and
copies the misses from pinned host DRAM; --unfused: kvd_select_topk then
kvd_resolve_and_fetch) -> kvd_sparse_decode (a5+a6: split-K attention with the
LSE merge in the same kernel), layers serially.  The whole step
is captured once as a CUDA graph and replayed; the decode-step index lives in
device memory (kvd_set_device_step) so every replay is a new step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
    python bench.py --impl reference ...   # the CPU oracle on a bounded sample

Multi-GPU: one process per GPU (self-launched through torch.distributed.run when
--gpus N > 1 and WORLD_SIZE is unset).  (request, KV-head) units are independent
through every row: "weak" sharding gives every rank its own B
requests; "strong" partitions the config's B*Hkv units over the ranks (whole
requests when N divides B: no collective at all; otherwise head ranges, and one
NCCL all-gather of the step's fp32 outputs).  c4 / c5 default to strong.

Inputs are seeded synthetic Llama-3.1-8B / Qwen2.5-1M-shaped K/V/queries
(synth/), resident in HBM (or in the pinned host store for the
host-backed configs) before the timed region.  Every step touches far more
than the 126 MB L2 (3.3 GB at c2, 13 GB + host fetches at c3), so no flush is
needed ("l2": "inputs larger than L2").

Measurement: the timed region replays the step graph K times
between CUDA events on the launching stream (max over ranks).  The graph's
kernels carry libkvd's device-side kernel timer (kvd_enable_kernel_timer), so
every kernel's launch duration is measured on the path that is timed; the same
graph without the timer is replayed right after as a check.  The roofline is
reported for the resource that binds the step (algorithmic bytes per step of
that resource / ms_per_step) and per kernel (algorithmic bytes per launch /
average launch duration).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs.  B is the config's batch (per rank for weak scaling).
CONFIGS = {
    "c1": dict(chains=1, L=1, B=1, Hq=8, Hkv=2, n=4096, P=16, k=32, C=None, alias=0, shard="weak",
               desc="1 req, 1 layer, 8q/2kv, d128, 4k ctx, block 16, top-k 32, resident"),
    "c2": dict(chains=16, L=32, B=8, Hq=32, Hkv=8, n=32768, P=16, k=128, C=None, alias=0, shard="weak",
               desc="Llama-3.1-8B shapes (32 layers, 32q/8kv, d128) bf16, 32k ctx, batch 8, top-k 2048 tokens, resident"),
    "c3": dict(chains=16, L=32, B=16, Hq=32, Hkv=8, n=131072, P=16, k=128, C=2048, alias=4, shard="weak",
               desc="Llama-3.1-8B shapes, 128k ctx, batch 16, GPU cache 25% of KV (2048 slots/segment), misses "
                    "gathered from pinned host DRAM, top-k 2048 tokens"),
    "c4": dict(chains=16, L=28, B=4, Hq=28, Hkv=4, n=1 << 20, P=16, k=128, C=16384, alias=2, shard="strong",
               desc="Qwen2.5-7B-1M shapes (28 layers, 28q/4kv, d128), 1M ctx, batch 4, GPU cache 25%, host-backed"),
    "c4k": dict(chains=16, L=28, B=4, Hq=28, Hkv=4, n=1 << 20, P=16, k=1024, C=16384, alias=2, shard="strong",
                desc="c4 with top-k 1024 blocks (16384 tokens = 1.56% of 1M, SURVEY 8.2)"),
    "c4h": dict(chains=16, L=28, B=4, Hq=28, Hkv=4, n=1 << 20, P=16, k=128, C=16384, alias=2, shard="strong", index=4,
                desc="c4 with the hierarchical centroid index (k-means over block summaries, 4 blocks per centroid; "
                     "PAPER.md:388-391, DESIGN.md R27)"),
    "c3h": dict(chains=16, L=32, B=16, Hq=32, Hkv=8, n=131072, P=16, k=128, C=2048, alias=4, shard="weak", index=4,
                desc="c3 with the hierarchical centroid index (4 blocks per centroid)"),
    "c3q": dict(chains=16, L=32, B=16, Hq=32, Hkv=8, n=131072, P=16, k=128, C=2048, alias=4, shard="weak",
                summary="minmax", desc="c3 with Quest min/max block summaries (the paper's baseline selection, "
                                       "PAPER.md:211; DESIGN.md R30)"),
    "c5": dict(chains=16, L=32, B=64, Hq=32, Hkv=8, n=131072, P=16, k=128, C=768, alias=2, shard="strong",
               desc="Llama-3.1-8B shapes, 128k ctx, batch 64 partitioned over the GPUs, GPU cache 768 "
                    "slots/segment (9.4%), host-backed"),
}
METRIC = "decode tokens/s at 128k ctx; sparse-attn HBM GB/s % peak; fetch GB/s, 1-8 GPU"
RECORD = 8192           # bytes of one 16-token K||V block record (bf16)
SUMMARY = 256           # bytes of one block summary (128 bf16)
KINDS = ("score", "select", "resolve", "gather", "attn")
KIND_NAMES = {"score": "score_kernel (a1)", "select": "rank_kernel (a2; fused: +a3+a4)",
              "resolve": "resolve_kernel (a3)", "gather": "gather_kernel (a4)", "attn": "attn_kernel (a5+a6)"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="kvd", choices=["kvd", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--policy", default="la", choices=["lru", "lfu", "la"])
    ap.add_argument("--alpha", type=float, default=0.9)
    ap.add_argument("--alias", type=int, default=None, help="host-layer alias A (layer l uses the K/V of layer l %% A)")
    ap.add_argument("--fill", type=int, default=None, help="untimed cache-fill steps before warm-up")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-isolated", action="store_true", help="skip the whole-batch per-kernel roofline pass")
    ap.add_argument("--no-graph", action="store_true", help="launch layer by layer instead of graph replay")
    ap.add_argument("--chains", type=int, default=None,
                    help="micro-batch chains (SFC overlap): the batch is split into this many request groups "
                         "(more chains than requests: one request per chain, its KV heads split into groups), "
                         "each run through all layers on its own stream inside the graph")
    ap.add_argument("--shard", default=None, choices=["weak", "strong"],
                    help="multi-GPU unit assignment (default per config): 'weak' = every rank serves its own B "
                         "requests; 'strong' = the config's B*Hkv units are partitioned over the ranks")
    ap.add_argument("--unfused", action="store_true",
                    help="step through kvd_select_topk + kvd_resolve_and_fetch instead of the fused "
                         "kvd_select_resolve_fetch (same results)")
    ap.add_argument("--layers", type=int, default=None, help="override L (profiling only; not a bench number)")
    ap.add_argument("--cpu-sample-s", type=float, default=6.0, help="target seconds per oracle sample")
    ap.add_argument("--master-port", type=int, default=29531, help="self-launch rendezvous port (N > 1)")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- algorithmic bytes
def per_segment_bytes(cfg, misses_per_seg=0.0, victims=True):
    """Algorithmic bytes per segment per step, by row.  With the
    hierarchical index (R27) select reads the centroids (256 B each, ~nb/ratio) and the member
    summaries of the m chosen centroids (~ratio * m blocks) instead of every block summary."""
    nb = (cfg["n"] + cfg["P"] - 1) // cfg["P"]
    G = cfg["Hq"] // cfg["Hkv"]
    k = cfg["k"]
    ratio = cfg.get("index", 0)
    if cfg.get("summary") == "minmax":
        sel_blocks = 2 * nb                       # minimum and maximum summaries
    elif ratio:
        nc = -(-nb // ratio)
        p_ = 1 + (64 + cfg["P"] - 1) // cfg["P"]
        m = min(nc, max(-(-4 * k // ratio), k + p_))
        sel_blocks = nc + ratio * m               # centroid rows + member rows (expected)
    else:
        sel_blocks = nb
    C = cfg["C"] if cfg["C"] is not None else nb
    p = 1 + (64 + cfg["P"] - 1) // cfg["P"]          # sink block + local blocks (n % P == 0)
    resident = C >= nb
    return dict(
        select=SUMMARY * sel_blocks + 2 * G * 128 + 8 * k,  # summaries (or centroids + members) + q + ids
        # the kernels of the select call: score_kernel streams the summaries and writes fp32 scores;
        # rank_kernel ranks them from L2 and writes the ids
        score=SUMMARY * sel_blocks + 2 * G * 128 + 4 * nb,
        topk=8 * k,
        resolve=4 * k + (0 if resident or not victims else 13 * C + 4 * C),   # table probes + victim scan (LA)
        attn=RECORD * (k + p) + 2 * G * 128 + 4 * G * 128 + 4 * G,   # K/V pages + q + o + lse
        fetch=RECORD * misses_per_seg,                     # host link read (and HBM write)
    )


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(config, kind):
    """Per-launch DRAM / PCIe bytes of one kernel kind from the committed ncu capture
    (profiles/*_ncu_traffic.json, written by tools/ncu_traffic.py), per segment."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_traffic.json")))
    if not files:
        return None
    try:
        d = json.load(open(files[-1]))
        e = d[config][kind]
        e = dict(e)
        e["source"] = os.path.basename(files[-1])
        return e
    except (KeyError, ValueError, OSError):
        return None


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
    def __init__(self, args, cfg, rank, dev, world=None):
        import torch
        import synth
        from paper_2605_18071_b200 import KVCache
        from paper_2605_18071_b200 import dist as kdist
        self.torch, self.args, self.cfg, self.rank, self.dev = torch, args, cfg, rank, dev
        world = world if world is not None else int(os.environ.get("WORLD_SIZE", "1"))
        L, B, Hq, Hkv, n, P, k = (cfg[x] for x in ("L", "B", "Hq", "Hkv", "n", "P", "k"))
        self.G = G = Hq // Hkv
        nb = (n + P - 1) // P
        C = cfg["C"] if cfg["C"] is not None else nb
        self.resident = C >= nb
        # ---- this rank's units
        self.shard = args.shard or cfg.get("shard", "weak")
        self.h0 = 0
        self.gather = False                       # heads split: all-gather the step's outputs
        if self.shard == "strong" and world > 1:
            self.all_parts = kdist.unit_partition(B, Hkv, world)
            self.greqs, self.h0, h1 = kdist.rank_heads(self.all_parts[rank])
            self.gather = not kdist.whole_requests(self.all_parts, Hkv)
            Hkv = h1 - self.h0
            Hq = Hkv * G
            B = len(self.greqs)
        else:
            self.greqs = kdist.rank_requests(rank, world, B) if world > 1 else list(range(B))
        self.B, self.Hkv, self.Hq = B, Hkv, Hq                  # this rank's (local) shapes
        self.reqs = list(range(B))
        # ---- host-layer alias A: the pinned host store holds A layers; layer l's K/V are the
        # synthetic layer l % A's (queries stay per layer: own random streams)
        A = args.alias if args.alias is not None else cfg["alias"]
        A = A if (A and A < L) else L
        if not self.resident and args.alias is None:
            # keep every rank's pinned host store under ~40 % of the box's RAM (all ranks share it)
            per_layer = B * Hkv * nb * RECORD
            ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
            A = max(1, min(A, int(0.4 * ram / world // per_layer)))
        self.A = A
        self.cache = KVCache(num_layers=L, num_q_heads=Hq, num_kv_heads=Hkv, block_tokens=P, max_requests=B,
                             max_context=n, slots_per_segment=C, max_select=k, sink_tokens=4, local_tokens=64,
                             policy=args.policy, host_layer_alias=(0 if self.A == L else self.A), device=dev.index,
                             index_ratio=cfg.get("index", 0), summary_kind=cfg.get("summary", "mean"))
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
        # queries for every step of the run: [T][L][B][Hq][128]; layer l follows the key topics
        # of its K/V (synthetic layer l % A) with its own random streams (stream layer l)
        self.fill = max(1, args.fill if args.fill is not None else (1 if self.resident else max(4, 2 * C // k)))
        # one query row per step of the whole run (fill, warm-up, timed, kernel-timer, isolated and
        # e2e passes): no step replays an earlier step's queries, so no pass sees an artificial hit
        self.T = self.fill + args.warmup + 4 * args.steps + 8
        Hkv_all = cfg["Hkv"]
        qh = np.stack([synth.batch_queries(args.seed, l % self.A, self.greqs, Hkv_all, G, t0=0, nsteps=self.T,
                                           alpha=args.alpha, stream_layer=l)[:, :, self.h0 * G:(self.h0 + Hkv) * G]
                       for l in range(L)], axis=1)
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
        m = max(1, min(m, B * Hkv))
        if m <= B:          # request groups, every KV head
            edges = [round(i * B / m) for i in range(m + 1)]
            self.chains = [(edges[i], edges[i + 1], 0, Hkv) for i in range(m) if edges[i + 1] > edges[i]]
        else:               # one request per chain, its KV heads split into hs groups (head-range calls)
            hs = max(d for d in range(1, Hkv + 1) if Hkv % d == 0 and d <= m // B)
            self.chains = [(b, b + 1, g * (Hkv // hs), Hkv // hs) for b in range(B) for g in range(hs)]
        self.chain_streams = [torch.cuda.Stream(device=dev) for _ in self.chains]
        self.fused = not args.unfused
        self.launches_per_step = None  # counted by libkvd (kvd_launch_count) over one eager step / the capture

    def row(self):
        return self.t % self.T

    # one layer of one chain (requests b0..b1-1) through the ABI calls
    def layer(self, l, s, step=0, chain=None):
        c, k = self.cache, self.cfg["k"]
        b0, b1, h0, nh = chain if chain else (0, len(self.reqs), 0, self.Hkv)
        heads = None if nh == self.Hkv else (h0, nh)     # head-range calls (kvd_*_heads)
        reqs = self.reqs[b0:b1]
        q = self.q_cur[l, b0:b1]
        if self.fused:   # kvd_select_resolve_fetch: score, then top-k + resolve + fetch
            c.select_resolve_fetch(l, q, reqs, k, step, self.ids[l, b0:b1], self.attn[l, b0:b1], stream=s, heads=heads)
        else:
            assert heads is None, "--unfused runs whole-head chains"
            c.select_topk(l, q, reqs, k, self.ids[l, b0:b1], None, stream=s)
            c.resolve_and_fetch(l, reqs, self.ids[l, b0:b1], k, step, self.attn[l, b0:b1], stream=s)
        c.sparse_decode(l, q, reqs, self.attn[l, b0:b1], self.W, self.out[l, b0:b1], self.lse[l, b0:b1], stream=s,
                        heads=heads)

    def eager_step(self, s):
        torch = self.torch
        with torch.cuda.stream(s):
            self.q_cur.copy_(self.q_dev[self.row()], non_blocking=True)
        self.t += 1
        self.cache.set_device_step(None)
        n0 = kvd_launch_count()
        for l in range(self.cfg["L"]):
            for ch in self.chains:                # the graph's launches, serialised on one stream
                self.layer(l, s, step=self.t, chain=ch)
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
        return g

    def prepare_graph(self, s):
        """Capture the step graph; the device step counter continues from the eager steps."""
        torch = self.torch
        self.step_dev.fill_(self.t)
        torch.cuda.synchronize(self.dev)
        self.graph = self.capture(s)

    def graph_step(self, s, source="dev"):
        torch = self.torch
        with torch.cuda.stream(s):
            if source == "dev":
                self.q_cur.copy_(self.q_dev[self.row()], non_blocking=True)
            else:
                self.q_cur.copy_(self.q_host[self.row()], non_blocking=True)
            self.graph.replay()
            if source != "dev":
                self.out_host.copy_(self.out, non_blocking=True)
        self.t += 1


def kvd_launch_count():
    from paper_2605_18071_b200 import kvd
    return int(kvd.lib().kvd_launch_count())


def run_gpu(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2605_18071_b200 import build as kb
    if rank == 0 or not os.path.exists(kb.SO):
        kb.build()
    if world > 1:
        dist.barrier()
    import synth
    synth.build_gpu()
    cfg = dict(CONFIGS[args.config])
    if args.layers:
        cfg["L"] = args.layers
    from paper_2605_18071_b200 import dist as kdist

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    R = Runner(args, cfg, rank, dev, world)
    s = torch.cuda.Stream(device=dev)
    L, B, Hkv = cfg["L"], R.B, R.Hkv                          # this rank's shapes
    segs_per_layer = B * Hkv
    gathered = (torch.empty((world * R.out.shape[0],) + tuple(R.out.shape[1:]), dtype=R.out.dtype, device=dev)
                if R.gather else None)

    def gather_outputs():
        # head sharding: the step's per-rank fp32 outputs -> every rank (NCCL over NVLink)
        with torch.cuda.stream(s):
            dist.all_gather_into_tensor(gathered, R.out)
    # cache fill (cold start -> steady state; untimed, parity-checked in tests)
    for _ in range(R.fill):
        R.eager_step(s)
    s.synchronize()
    step_fn = (lambda: R.eager_step(s)) if args.no_graph else (lambda: R.graph_step(s))

    def run():
        step_fn()
        if R.gather:
            gather_outputs()

    def timed_steps(k):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(k):
            run()
        e1.record(s)
        e1.synchronize()
        barrier()
        return e0.elapsed_time(e1) / k
    # capture the step (the step index is read on the device)
    if not args.no_graph:
        R.prepare_graph(s)
    clk = ClockSampler(local)          # sampled from warm-up through the e2e pass (GPU busy throughout)
    clk.start()
    for _ in range(args.warmup):
        run()
    s.synchronize()
    R.cache.reset_stats()
    # ---- timed region: K steps, device-timed on the launching stream
    ms = timed_steps(args.steps)
    st = R.cache.stats()
    ms_max = kdist.max_over_ranks(ms, dev)
    # whole-job tokens: every rank's requests once (strong mode: a request split over head
    # ranges is counted once)
    tokens_per_step = cfg["B"] if (R.shard == "strong" and world > 1) else kdist.sum_over_ranks(B, dev)
    value = tokens_per_step / (ms_max * 1e-3)
    hit_rate = st["hits"] / max(1, st["selected"])
    misses_per_seg = st["misses"] / max(1, args.steps * L * segs_per_layer)

    # ---- per-kernel launch durations: the same step graph re-captured with libkvd's device-side
    # kernel timer on (kvd_enable_kernel_timer: no event node between the kernels), K steps
    R.cache.enable_kernel_timer(True)
    if not args.no_graph:
        R.prepare_graph(s)
    for _ in range(2):
        run()
    R.cache.enable_kernel_timer(True)             # zero the accumulators (synchronises)
    ms_timer = kdist.max_over_ranks(timed_steps(args.steps), dev)
    kt = R.cache.read_kernel_timer()
    R.cache.enable_kernel_timer(False)
    if not args.no_graph:
        R.prepare_graph(s)                        # the plain graph again (e2e pass)

    # ---- rooflines
    b = per_segment_bytes(cfg, misses_per_seg)
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs") or 6650.0
    hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs") else "fallback (B200_PROFILING.md)"
    link = None if R.resident else host_link_probes(torch, dev)
    misses_per_step = misses_per_seg * L * segs_per_layer
    hbm_bytes_step = L * segs_per_layer * (b["select"] + b["resolve"] + b["attn"]) + RECORD * misses_per_step
    link_bytes_step = RECORD * misses_per_step
    hbm_step = {"achieved": hbm_bytes_step / (ms * 1e-3) / 1e9, "bytes_per_step": hbm_bytes_step}
    hbm_step["frac"] = hbm_step["achieved"] / hbm_peak
    link_step = None
    if link:
        link_step = {"achieved": link_bytes_step / (ms * 1e-3) / 1e9, "bytes_per_step": link_bytes_step,
                     "peak": link["gbs"]}
        link_step["frac"] = link_step["achieved"] / link["gbs"]
    # per kernel (device-timed launches of the timed graph)
    chains = len(R.chains)
    kernels = {}
    for kind in KINDS:
        ns, nl = kt[kind]
        if nl == 0:
            continue
        avg_ms = ns / nl * 1e-6
        segs_per_launch = segs_per_layer * L * args.steps / nl
        e = {"kernel": KIND_NAMES[kind], "launches_per_step": nl / args.steps, "avg_launch_us": avg_ms * 1e3,
             "busy_ms_per_step": ns * 1e-6 / args.steps, "segments_per_launch": segs_per_launch}
        e["busy_share"] = e["busy_ms_per_step"] / ms_timer         # > 1 when launches of chains overlap
        if kind == "score":
            e["hbm_bytes_per_launch"] = b["score"] * segs_per_launch
        elif kind == "select":
            by = b["topk"] + (b["resolve"] if R.fused else 0)
            e["hbm_bytes_per_launch"] = by * segs_per_launch
            e["note"] = "ranks the scores from L2 (4 B per block); HBM bytes: ids (+ resolve)"
            if R.fused and link:
                e["host_bytes_per_launch"] = RECORD * misses_per_seg * segs_per_launch
        elif kind == "attn":
            e["hbm_bytes_per_launch"] = b["attn"] * segs_per_launch
        elif kind == "resolve":
            e["hbm_bytes_per_launch"] = b["resolve"] * segs_per_launch
        elif kind == "gather":
            e["host_bytes_per_launch"] = RECORD * misses_per_seg * segs_per_launch
        if "hbm_bytes_per_launch" in e:
            e["hbm_gbs_per_launch"] = e["hbm_bytes_per_launch"] / (avg_ms * 1e-3) / 1e9
            e["frac_hbm_per_launch"] = e["hbm_gbs_per_launch"] / hbm_peak
        if "host_bytes_per_launch" in e and link:
            e["host_gbs_per_launch"] = e["host_bytes_per_launch"] / (avg_ms * 1e-3) / 1e9
        kernels[kind] = e
    dom = max(kernels, key=lambda k_: kernels[k_]["busy_ms_per_step"]) if kernels else None
    # the binding resource of the step: host link when its step fraction is the larger one
    if link_step and link_step["frac"] >= hbm_step["frac"]:
        roof = {"bound": "host-link", "achieved": link_step["achieved"], "peak": link["gbs"], "unit": "GB/s",
                "frac": link_step["frac"], "scope": "step: host-link bytes of the missed blocks / ms_per_step",
                "peak_source": link["how"]}
        tr = ncu_traffic(args.config, "select")
        roof["traffic"] = (tr["pcie_read_bytes_per_segment"] * segs_per_layer * L
                           if tr and tr.get("pcie_read_bytes_per_segment") is not None else None)
    else:
        roof = {"bound": "hbm", "achieved": hbm_step["achieved"], "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm_step["frac"], "scope": "step: algorithmic HBM bytes (SURVEY 8.5) / ms_per_step",
                "peak_source": hbm_src}
        trs = [ncu_traffic(args.config, kd) for kd in ("select", "attn")]
        roof["traffic"] = (sum(t["dram_bytes_per_segment"] for t in trs) * segs_per_layer * L
                           if all(t and t.get("dram_bytes_per_segment") is not None for t in trs) else None)
    roof["traffic_unit"] = "bytes per step (ncu --set full DRAM/PCIe bytes per segment x segments)"
    if dom:
        dk = kernels[dom]
        roof["dominant_kernel"] = {"kind": dom, "name": dk["kernel"], "avg_launch_us": dk["avg_launch_us"],
                                   "busy_share": dk["busy_share"]}
        if "hbm_gbs_per_launch" in dk:
            roof["dominant_kernel"].update(achieved_gbs=dk["hbm_gbs_per_launch"],
                                           frac_hbm=dk["frac_hbm_per_launch"])
    # north_star's named figure: sparse-attention HBM GB/s as a fraction of peak
    roof_attn = None
    if "attn" in kernels:
        ka = kernels["attn"]
        roof_attn = {"achieved": ka["hbm_gbs_per_launch"], "peak": hbm_peak, "unit": "GB/s",
                     "frac": ka["frac_hbm_per_launch"], "scope": "per launch (device-timed in the timed graph)"}

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
            if R.gather:
                gather_outputs()
        e1.record(s)
        e1.synchronize()
        barrier()
        ems = kdist.max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)
        e2e = {"value": tokens_per_step / (ems * 1e-3), "unit": "tokens/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(R.q_cur.numel() * 2), "d2h_bytes_per_step": int(R.out.numel() * 4)}
    # ---- per-kernel rooflines of whole-batch launches (chains = 1: every kernel serves the rank's
    # whole batch and runs alone), device-timed with the kernel timer on the same step graph
    # structure: the kernels' own achieved bandwidth, free of the chains' concurrency
    iso = None
    if not args.no_graph and not args.no_isolated:
        saved = (R.chains, R.chain_streams)
        R.chains, R.chain_streams = [(0, len(R.reqs), 0, R.Hkv)], [torch.cuda.Stream(device=dev)]
        R.cache.enable_kernel_timer(True)
        R.prepare_graph(s)
        for _ in range(2):
            run()
        R.cache.enable_kernel_timer(True)
        ms_iso = kdist.max_over_ranks(timed_steps(args.steps), dev)
        kti = R.cache.read_kernel_timer()
        R.cache.enable_kernel_timer(False)
        R.chains, R.chain_streams = saved
        R.prepare_graph(s)
        iso = {"ms_per_step": ms_iso, "chains": 1}
        for kind, by in (("score", b["score"]), ("select", b["topk"] + (b["resolve"] if R.fused else 0)),
                         ("attn", b["attn"])):
            ns, nl = kti[kind]
            if nl:
                us = ns / nl * 1e-3
                gbs = by * segs_per_layer / (us * 1e-6) / 1e9
                iso[kind] = {"kernel": KIND_NAMES[kind], "avg_launch_us": us, "segments_per_launch": segs_per_layer,
                             "hbm_bytes_per_launch": by * segs_per_layer, "achieved_gbs": gbs,
                             "frac_hbm": gbs / hbm_peak, "launches_per_step": nl / args.steps}
        if "attn" in iso:
            roof_attn = {"achieved": iso["attn"]["achieved_gbs"], "peak": hbm_peak, "unit": "GB/s",
                         "frac": iso["attn"]["frac_hbm"],
                         "scope": "attention kernel, whole-batch launches (chains = 1), device-timed"}
    R.cache.check()
    clocks = clk.stop()

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong" if (R.shard == "strong" and world > 1) else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded; DESIGN.md §4)",
        "config": {"workload": args.config, "desc": cfg["desc"],
                   "global_batch": tokens_per_step if world > 1 else B, "seq_len": cfg["n"],
                   "layers": L, "q_heads": cfg["Hq"], "kv_heads": cfg["Hkv"], "block_tokens": cfg["P"],
                   "top_k_blocks": cfg["k"], "slots_per_segment": cfg["C"] or (cfg["n"] // cfg["P"]),
                   "policy": args.policy, "alpha": args.alpha, "host_layer_alias": R.A if not R.resident else None,
                   "fill_steps": R.fill, "graph": not args.no_graph, "chains": chains,
                   "fused_select_resolve": R.fused,
                   "parallelism": (f"{R.shard}-shard x{world}" + (" + NCCL all-gather of head outputs" if R.gather
                                                                else ", no collective on the decode path")),
                   "l2": "inputs larger than L2 (no flush)"},
        "hit_rate": hit_rate, "misses_per_segment": misses_per_seg,
        "roofline": roof, "roofline_attn": roof_attn, "hbm_step": hbm_step, "host_link_step": link_step,
        "kernels": kernels, "kernels_isolated": iso, "host_link": link, "e2e": e2e,
        "ms_per_step_with_kernel_timer": ms_timer,
        "gpu_launches": R.launches_per_step * args.steps,
        "clocks": clocks, "setup_s": R.setup_s,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, cfg, args.cpu_sample_s)
    if rank == 0:
        print(json.dumps(line), flush=True)
    R.cache.close()
    if world > 1:
        dist.destroy_process_group()


def host_link_probes(torch, dev, nbytes=1 << 30):
    """The host-link denominator: max of a pinned H2D DMA copy and a zero-copy
    read with the miss gather's own access pattern (kvd_probe_zero_copy), 1 GiB each."""
    from paper_2605_18071_b200 import kvd
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)

    def timed(fn, reps=4):
        fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return reps * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9

    dma = timed(lambda: d.copy_(h, non_blocking=True))
    zc = {}
    for ctas in (148, 296, 592):
        zc[ctas] = timed(lambda: kvd.probe_zero_copy(h, d, nbytes, ctas, s))
    best = max(zc.values())
    del h, d
    return {"gbs": max(dma, best), "dma_gbs": dma, "zero_copy_gbs": best,
            "zero_copy_by_ctas": {str(k): v for k, v in zc.items()},
            "how": "max(pinned H2D cudaMemcpyAsync, zero-copy 16-B loads kvd_probe_zero_copy), 1 GiB x4 each"}


# ---------------------------------------------------------------- the CPU oracle (baseline / reference arm)
class OracleSample:
    """A bounded sample of the workload for the oracle as it stands: `ntasks` whole segment-
    steps runs (select O2-O5 + resolve O6 + attention O8 of one segment of layer 0 for 3 steps
    from a cold cache).  Inputs and summaries (setup, a0) are prepared outside the timed part
    for at most `max_bytes` of K/V; tasks cycle over the prepared segments."""

    def __init__(self, args, cfg, ntasks, max_bytes=3 << 30):
        import oracle
        import synth
        self.oracle = oracle
        L, B, Hq, Hkv, n, P, k = (cfg[x] for x in ("L", "B", "Hq", "Hkv", "n", "P", "k"))
        self.G = Hq // Hkv
        nb = (n + P - 1) // P
        self.C = cfg["C"] if cfg["C"] is not None else nb
        self.W = k + 1 + (64 + P - 1) // P + 1
        self.cfg, self.args, self.k, self.P = cfg, args, k, P
        nseg = max(1, min(ntasks, B * Hkv, max_bytes // (4 * n * 128)))
        self.ntasks = ntasks
        self.segs = []
        for seg in range(nseg):
            r, h = divmod(seg, Hkv)
            K, V = synth.segment_kv(args.seed, 0, r, h, n)
            S = oracle.block_summaries(K, P)
            q = synth.queries(args.seed, 0, r, h, self.G, t0=0, nsteps=3, alpha=args.alpha)
            self.segs.append((K, V, S, q, oracle.pinned_blocks(n, P), nb))

    def run(self, threads):
        """All tasks on `threads` host threads; returns (wall seconds, segment-steps).  The
        oracle's C functions release the GIL (ctypes), so threads run them in parallel."""
        from concurrent.futures import ThreadPoolExecutor
        oracle, pol = self.oracle, self.oracle.POLICIES[self.args.policy]

        def one(i):
            K, V, S, q, pinned, nb = self.segs[i % len(self.segs)]
            oc = oracle.SegmentCache(nb, self.C, pinned)
            for t in range(3):
                oracle.segment_step(oc, q[t], S, K, V, self.P, self.k, t + 1, pol, self.W)
            return 3
        t0 = time.perf_counter()
        if threads <= 1:
            done = sum(one(i) for i in range(self.ntasks))
        else:
            with ThreadPoolExecutor(threads) as ex:
                done = sum(ex.map(one, range(self.ntasks)))
        return time.perf_counter() - t0, done


def cpu_baseline(args, cfg, target_s):
    """The oracle timed on this host's cores: 1 thread and all cores (threads over segments)."""
    cores = cpu_cores()
    L, B, Hkv = cfg["L"], cfg["B"], cfg["Hkv"]
    seg_steps_per_step = B * Hkv * L
    probe = OracleSample(args, cfg, 1)
    w1, n1 = probe.run(1)
    per1 = w1 / n1                                # seconds per segment-step, 1 thread
    n_one = max(1, int(target_s / (3 * per1)))
    n_all = max(cores, int(target_s * cores / (3 * per1)))
    w_one, d_one = OracleSample(args, cfg, n_one).run(1)
    allc = OracleSample(args, cfg, n_all)
    w_all, d_all = allc.run(cores)
    v1 = B / (w_one / d_one * seg_steps_per_step)
    va = B / (w_all / d_all * seg_steps_per_step)
    return {"value": va, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "value_1_thread": v1, "speedup_all_cores": va / v1,
            "sample": f"all cores: {d_all} segment-steps ({n_all} runs of 3 steps over {len(allc.segs)} layer-0 "
                      f"segments) on {cores} threads in {w_all:.1f} s; 1 thread: {d_one} segment-steps in "
                      f"{w_one:.1f} s; each scaled to the {seg_steps_per_step} segment-steps of one decode step "
                      f"(B x Hkv x L)"}


def run_reference(args):
    """--impl reference: the oracle as it stands, on this host's cores.  Each step is one
    bounded sample of the workload (whole segment-steps, threads over segments); ms_per_step
    is that sample's wall time, value extrapolates it to the config's decode tokens/s."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = dict(CONFIGS[args.config])
    import oracle
    oracle.build()
    cores = cpu_cores()
    L, B, Hkv = cfg["L"], cfg["B"], cfg["Hkv"]
    w1, n1 = OracleSample(args, cfg, 1).run(1)
    per_wall = w1 / n1 / cores                    # ~ seconds per segment-step on all cores
    seg_steps_per_step = B * Hkv * L
    # a step = one decode step's worth of segment-steps (B x Hkv x L, in runs of 3 steps), unless
    # that would not fit the budget (whole run within a few minutes): then a proportional sample
    budget = min(8.0, 150.0 / max(1, args.steps + args.warmup))
    ntasks = -(-seg_steps_per_step // 3)
    if ntasks * 3 * per_wall > budget:
        ntasks = max(cores, int(budget / (3 * per_wall)))
    sample = OracleSample(args, cfg, ntasks)
    for _ in range(args.warmup):
        sample.run(cores)
    walls, done = [], 0
    for _ in range(args.steps):
        w, done = sample.run(cores)
        walls.append(w)
    wall = float(np.mean(walls))
    v = B / (wall / done * seg_steps_per_step)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (oracle)",
            "data": "synthetic (seeded; DESIGN.md §4)",
            "config": {"workload": args.config, "desc": cfg["desc"], "global_batch": B, "seq_len": cfg["n"]},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": f"each step: {done} segment-steps ({ntasks} runs of 3 steps over "
                                       f"{len(sample.segs)} layer-0 segments) on {cores} threads, {wall:.2f} s "
                                       f"wall (= ms_per_step); one decode step is {seg_steps_per_step} "
                                       f"segment-steps (B x Hkv x L), value = B / (wall per decode step)"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def self_launch(args):
    """--gpus N > 1 without a torch.distributed environment: launch N ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(args.master_port), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
