"""One process per GPU: sharding of the two multi-GPU workloads and their
exchanges.

Batched (BASELINE.json configs[3]): the images are independent, so ranks share
no data on the hot path.  Each rank owns a fixed block of images (weak scaling:
``images_per_rank`` per GPU); the only collective is one all-reduce (SUM) of
the [world * images_per_rank, 4] fp64 per-image result table, where every rank
contributes its own rows and zeros elsewhere -- after it every rank holds every
image's (rate, sse, mse, cost).

Single large image (configs[4]): horizontal strips of pixel rows, one per rank
(``strip_rows``).  Each rank owns the latent rows ceil(r0/2^l) .. ceil(r1/2^l)
of every grid and needs a halo of its neighbours' rows (the window computed by
cc_strip_window from the receptive field).  ``exchange_halos`` is the one data
exchange: grouped point-to-point send/recv (NCCL on GPU, gloo on CPU) of the
contiguous row blocks each rank owns and another's window contains, straight
into the receivers' window buffers.  After it every strip is computed
independently (cc_rd_forward_strip) and the additive (rate, sse, mse, cost)
shares are all-reduced.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class Rank:
    rank: int
    local_rank: int
    world: int


def rank_from_env() -> Rank:
    return Rank(int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
                int(os.environ.get("WORLD_SIZE", "1")))


def owned_images(rank: int, images_per_rank: int):
    """Global image indices rank ``rank`` computes (contiguous block)."""
    return list(range(rank * images_per_rank, (rank + 1) * images_per_rank))


def init(backend: str = "nccl"):
    """Initialise torch.distributed from the torchrun environment (no-op at N=1)."""
    import torch
    import torch.distributed as dist
    r = rank_from_env()
    if r.world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(r.local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", r.local_rank))
        else:
            dist.init_process_group(backend)
    elif backend == "nccl" and torch.cuda.is_available():
        torch.cuda.set_device(r.local_rank)
    return r


def scatter_results(local, rank: int, world: int, images_per_rank: int):
    """Place this rank's [images_per_rank, 4] results into a zeroed global
    [world * images_per_rank, 4] table (same device / dtype)."""
    import torch
    table = torch.zeros((world * images_per_rank, local.shape[1]), dtype=local.dtype, device=local.device)
    table[rank * images_per_rank:(rank + 1) * images_per_rank] = local
    return table


def allreduce_results(table):
    """SUM all-reduce of the per-image result table (NCCL on GPU, gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(table, op=dist.ReduceOp.SUM)
    return table


def barrier():
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def max_over_ranks(value: float, device=None) -> float:
    """Max of a float over ranks (device timing rule: max over ranks)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ strips
def strip_rows(H: int, world: int):
    """Balanced partition of pixel rows [0, H) into ``world`` strips with even
    starts (cc_rd_forward_strip needs r0 even: the x2 upsampling phases pair
    rows (2q, 2q+1))."""
    if world < 1 or 2 * world > H + 1:
        raise ValueError(f"cannot split {H} rows into {world} strips")
    cuts = [0] + [2 * ((k * H) // (2 * world)) for k in range(1, world)] + [H]
    if any(b <= a for a, b in zip(cuts, cuts[1:])):
        raise ValueError(f"empty strip splitting {H} rows into {world}")
    return list(zip(cuts[:-1], cuts[1:]))


class StripLayout:
    """Where each grid's window rows sit in a strip's latent buffer
    (include/ccrd.h: grid l = rows [lo_l, hi_l) x w_l, packed level after
    level).  Pure bookkeeping; no arithmetic of the method."""

    def __init__(self, level_dims, strip):
        self.L = len(level_dims)
        self.w = [w for _, w in level_dims]
        self.h = [h for h, _ in level_dims]
        self.lo = [strip.lo[l] for l in range(self.L)]
        self.hi = [strip.hi[l] for l in range(self.L)]
        self.own_lo = [strip.own_lo[l] for l in range(self.L)]
        self.own_hi = [strip.own_hi[l] for l in range(self.L)]
        self.r0, self.r1 = strip.r0, strip.r1
        self.off = []
        o = 0
        for l in range(self.L):
            self.off.append(o)
            o += (self.hi[l] - self.lo[l]) * self.w[l]
        self.n = o

    def rows(self, l, a, b):
        """Element range [s, e) of global rows [a, b) of grid l in the buffer."""
        assert self.lo[l] <= a <= b <= self.hi[l]
        return self.off[l] + (a - self.lo[l]) * self.w[l], self.off[l] + (b - self.lo[l]) * self.w[l]


def strip_layouts(desc, world: int):
    """cc_strip records + layouts of every rank's strip (each rank computes
    all of them, so both sides of every halo transfer agree without talking)."""
    from . import ccrd
    dims = [(-(-desc.H // (1 << l)), -(-desc.W // (1 << l))) for l in range(desc.L)]
    strips = [ccrd.cc_strip_window(desc, r0, r1) for r0, r1 in strip_rows(desc.H, world)]
    return strips, [StripLayout(dims, st) for st in strips]


def pack_window(full_latents, full_off, layout: StripLayout, owned_only: bool = False, fill=0):
    """Strip buffer from a full packed pyramid (numpy or torch, 1-D):
    window rows (or only the owned rows, the rest = ``fill``)."""
    if hasattr(full_latents, "new_full"):
        buf = full_latents.new_full((layout.n,), fill)
    else:
        import numpy as np
        buf = np.full(layout.n, fill, dtype=full_latents.dtype)
    for l in range(layout.L):
        a, b = (layout.own_lo[l], layout.own_hi[l]) if owned_only else (layout.lo[l], layout.hi[l])
        if b <= a:
            continue
        s, e = layout.rows(l, a, b)
        w = layout.w[l]
        buf[s:e] = full_latents[full_off[l] + a * w: full_off[l] + b * w]
    return buf


def halo_plan(layouts, rank: int):
    """(peer, level, row_lo, row_hi, send?) transfers of ``rank``: rows it owns
    that the peer's window holds (send), rows the peer owns that its own window
    holds (recv).  Deterministic order, identical on both ends."""
    me = layouts[rank]
    plan = []
    for q, other in enumerate(layouts):
        if q == rank:
            continue
        for l in range(me.L):
            a, b = max(other.lo[l], me.own_lo[l]), min(other.hi[l], me.own_hi[l])
            if a < b:
                plan.append((q, l, a, b, True))
            a, b = max(me.lo[l], other.own_lo[l]), min(me.hi[l], other.own_hi[l])
            if a < b:
                plan.append((q, l, a, b, False))
    return plan


def exchange_halos(buf, layouts, rank: int):
    """The halo exchange: one grouped batch of point-to-point
    sends / receives of contiguous row blocks, directly from / into the strip
    buffers (NCCL over NVLink on GPU tensors, gloo on CPU tensors).  Returns
    the number of bytes this rank received."""
    import torch.distributed as tdist
    if not (tdist.is_initialized() and tdist.get_world_size() > 1):
        return 0
    me = layouts[rank]
    ops, nbytes = [], 0
    for q, l, a, b, send in halo_plan(layouts, rank):
        s, e = me.rows(l, a, b)
        view = buf[s:e]
        if send:
            ops.append(tdist.P2POp(tdist.isend, view, q))
        else:
            ops.append(tdist.P2POp(tdist.irecv, view, q))
            nbytes += view.numel() * view.element_size()
    if ops:
        for r in tdist.batch_isend_irecv(ops):
            r.wait()
    return nbytes
