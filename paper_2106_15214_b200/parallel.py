"""N-column sharding across GPUs (one process per GPU, torch.distributed for
the plumbing, NCCL inside libbnmf for the per-iteration exchange).

Partitioning: rank r owns the column block V[:, n0:n1] and
the matching H[:, n0:n1]; W is replicated.  Columns are independent given W,
so the only exchange per iteration is one allreduce (sum) of the packed
[W numerator F x K | W denominator F x K | objective] partial sums, issued by
libbnmf on its own stream (ncclAllReduce, captured in the iteration graph).
Every rank then applies the identical W update, so W stays bitwise
replicated.  The reference is single-process; nothing here has
a reference counterpart beyond the arithmetic it distributes.

torch.distributed is used only to exchange sizes and the 128-byte NCCL
unique id, and for barriers / max-over-ranks timing in bench.py.
"""

from __future__ import annotations

import numpy as np


def dist_info():
    """(rank, world) of the initialised default process group, else None."""
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover - torch always present in this image
        return None
    if not (dist.is_available() and dist.is_initialized()):
        return None
    return dist.get_rank(), dist.get_world_size()


def balanced_blocks(n, world, align=1):
    """Contiguous column blocks [(n0, n1)] per rank, sizes within `align`."""
    units = (n + align - 1) // align
    out = []
    start = 0
    for r in range(world):
        cnt = units // world + (1 if r < units % world else 0)
        end = min(n, start + cnt * align)
        out.append((start, end))
        start = end
    return out


def allgather_int(x):
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, int(x))
    return out


def column_offsets(n_local):
    """Global column offset of this rank's block and the global N."""
    info = dist_info()
    if info is None:
        return 0, int(n_local)
    rank, _ = info
    counts = allgather_int(n_local)
    return int(sum(counts[:rank])), int(sum(counts))


def allreduce_scalars(values, op="sum"):
    """Allreduce a few host scalars (float64) across ranks."""
    info = dist_info()
    vals = np.asarray(values, dtype=np.float64)
    if info is None:
        return vals
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op={"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN,
                           "max": dist.ReduceOp.MAX}[op])
    return t.cpu().numpy()


def resolve_kappa_global(values, beta, kappa):
    """default_kappa (core.py:176-185) over the union of all shards."""
    if kappa is not None:
        return float(kappa)
    vmin = float(values.min())
    vsum = float(values.sum(dtype=np.float64))
    cnt = float(values.size)
    gmin = allreduce_scalars([vmin], "min")[0]
    gsum, gcnt = allreduce_scalars([vsum, cnt], "sum")
    if 1.0 <= beta <= 2.0 and gmin > 0.0:
        return 0.0
    return 1e-9 * gsum / gcnt


def agree_on_error(local_err):
    """Collective error agreement: if any rank's input checks failed, every
    rank raises (the failing rank its own error, the others a ValueError
    naming the failing ranks), so no rank is left waiting in the next
    collective."""
    info = dist_info()
    if info is None:
        if local_err is not None:
            raise local_err
        return
    rank, world = info
    flags = np.zeros(world)
    flags[rank] = 1.0 if local_err is not None else 0.0
    flags = allreduce_scalars(flags, "sum")
    if local_err is not None:
        raise local_err
    bad = [r for r in range(world) if flags[r] > 0]
    if bad:
        raise ValueError(f"input checks failed on rank(s) {bad}")


def broadcast_uid(make_uid):
    """Rank 0 creates the NCCL unique id (128 bytes); everyone receives it."""
    import torch.distributed as dist
    rank, _ = dist_info()
    obj = [make_uid() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def slice_init(w, h, n0, n_local, n_global):
    """The H columns of this shard from a global init (W is replicated)."""
    h = np.asarray(h)
    if h.shape[1] == n_global:
        return w, h[:, n0:n0 + n_local]
    if h.shape[1] == n_local:
        return w, h
    raise ValueError("init H must have the global or the local column count")
