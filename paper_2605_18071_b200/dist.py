"""Multi-GPU plumbing for the decode step (host side; torch.distributed only).

SURVEY §8.6 / DESIGN.md §8: every (request, KV head) unit is independent
through select, resolve, fetch and attention, so GPUs never exchange data on
the decode path.  This module only decides which units a rank owns and
reduces the per-rank timings and counts (max of step times, sum of tokens).
Backend-agnostic: NCCL on the B200 box, gloo in the CPU tests.
"""
import torch
import torch.distributed as dist


def rank_requests(rank, world, per_rank):
    """Weak scaling: rank r serves global requests r*per_rank .. (r+1)*per_rank - 1."""
    if not (0 <= rank < world) or per_rank < 1:
        raise ValueError("bad rank / world / per_rank")
    return list(range(rank * per_rank, (rank + 1) * per_rank))


def unit_partition(B, Hkv, world):
    """Strong-scaling partition of B*Hkv (request, KV-head) units over `world` ranks,
    request-major: request sharding when world divides B, else head sharding (each
    rank gets Hkv*B/world consecutive units, i.e. a contiguous head range of one or
    more requests, reading R21).  Returns, per rank, a list of
    (request, head_begin, head_end)."""
    units = B * Hkv
    if units % world:
        raise ValueError(f"{units} units do not split over {world} ranks")
    per = units // world
    out = []
    for r in range(world):
        lo, hi = r * per, (r + 1) * per
        parts = []
        u = lo
        while u < hi:
            req, h = divmod(u, Hkv)
            h_end = min(Hkv, h + (hi - u))
            parts.append((req, h, h_end))
            u += h_end - h
        out.append(parts)
    return out


def rank_heads(parts):
    """(requests, head_begin, head_end) of one rank's unit_partition entry; the head
    range must be the same for every request of the rank (true for c4 and for any
    partition into whole requests)."""
    h0, h1 = parts[0][1], parts[0][2]
    if any((a, b) != (h0, h1) for _, a, b in parts):
        raise ValueError("ranks must own the same head range of each of their requests")
    return [req for req, _, _ in parts], h0, h1


def whole_requests(all_parts, Hkv):
    """True when every rank owns whole requests (all Hkv heads of each): no rank holds a partial
    head range, so no output needs gathering (request sharding)."""
    return all(h0 == 0 and h1 == Hkv for parts in all_parts for _, h0, h1 in parts)


def assemble_heads(gathered, all_parts, B, Hkv, G):
    """Per-rank outputs [world][L][B_r][Hq_r][d] (all_gather_into_tensor of each
    rank's fp32 attention outputs) -> the global [L][B][Hq][d] tensor."""
    world, L, _, _, d = gathered.shape
    out = gathered.new_empty((L, B, Hkv * G, d))
    for r in range(world):
        reqs, h0, h1 = rank_heads(all_parts[r])
        for i, req in enumerate(reqs):
            out[:, req, h0 * G:h1 * G] = gathered[r, :, i, :(h1 - h0) * G]
    return out


def _reduce(x, op, device):
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(x, device="cpu"):
    return _reduce(x, dist.ReduceOp.MAX, device)


def sum_over_ranks(x, device="cpu"):
    return _reduce(x, dist.ReduceOp.SUM, device)
