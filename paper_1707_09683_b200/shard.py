"""Multi-GPU driver: one process per GPU, the database sharded by residue
count (lhmm_set_database's LPT tile plan), per-sequence raw scores and pass
bits gathered to rank 0.  The path has no reduction -- only this gather
(BASELINE.json north_star).

Works with any torch.distributed backend: NCCL over NVLink/NVSwitch on the
GPU box, gloo on CPU for the tests.
"""
from __future__ import annotations

import numpy as np


def gather_to_rank0(dist, raw, passed, gidx, n_total, device=None, as_numpy=True,
                    validate=True):
    """Gather each rank's (raw, pass) bytes for its global indices `gidx`
    into full-length arrays on rank 0 (None elsewhere); as_numpy=False keeps
    them as tensors on the gather device.

    raw / passed: uint8 tensors of the shard's local outputs (local order);
    gidx: int64 tensor of the matching global indices.  Shards are padded to
    the largest count so a single gather carries them.
    """
    import torch

    world = dist.get_world_size()
    rank = dist.get_rank()
    dev = raw.device if device is None else device
    n = torch.tensor([raw.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    mx = int(max(int(c) for c in counts))
    # one int64 row of indices + one row of packed (raw | pass << 8) int64
    buf = torch.full((2, max(mx, 1)), -1, dtype=torch.int64, device=dev)
    k = raw.numel()
    buf[0, :k] = gidx.to(dev, torch.int64)
    buf[1, :k] = raw.to(dev, torch.int64) | (passed.to(dev, torch.int64) << 8)
    glist = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, glist, dst=0)
    if rank != 0:
        return None, None
    # scatter into the global arrays where the data lives (device for NCCL)
    allg = torch.cat([g[:, :int(counts[r])] for r, g in enumerate(glist)], dim=1)
    idx, val = allg[0], allg[1]
    if validate and (idx.numel() != n_total or int(torch.unique(idx).numel()) != n_total):
        raise RuntimeError("shards do not partition the database")
    out_raw = torch.zeros(n_total, dtype=torch.uint8, device=dev)
    out_pass = torch.zeros(n_total, dtype=torch.bool, device=dev)
    out_raw[idx] = (val & 0xFF).to(torch.uint8)
    out_pass[idx] = ((val >> 8) & 1).to(torch.bool)
    if as_numpy:
        return out_raw.cpu().numpy(), out_pass.cpu().numpy()
    return out_raw, out_pass


def shard_plan(offsets, rank, world):
    """Global indices shard `rank` of `world` owns (host-only; the same plan
    lhmm_set_database applies)."""
    import ctypes as C

    from . import _native
    from .lanehmm import _check
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = off.size - 1
    cnt = C.c_uint64()
    _check(_native.lib().lhmm_shard_plan(off.ctypes.data_as(_native.u64p), n, rank, world, None,
                                         C.byref(cnt)))
    out = np.zeros(max(cnt.value, 1), dtype=np.uint64)
    _check(_native.lib().lhmm_shard_plan(off.ctypes.data_as(_native.u64p), n, rank, world,
                                         out.ctypes.data_as(_native.u64p), C.byref(cnt)))
    return out[:cnt.value]
