"""Multi-GPU driver: one process per GPU, the database sharded by residue
count (lhmm_set_database's LPT tile plan), per-sequence raw scores and pass
bits gathered to rank 0.  The path has no reduction -- only this gather
(BASELINE.json north_star).

Two gathers:
* PeerOutputs -- the fused one: rank 0's full-length result buffers are
  mapped into every rank through CUDA IPC and each rank's scan kernel stores
  its results there directly (NVLink peer stores), addressed by global
  sequence index (lhmm_scan_device_global).  No separate collective runs.
* gather_to_rank0 -- a torch.distributed gather of (index, raw | pass << 8);
  any backend (NCCL on the box, gloo on CPU for the tests).
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


class PeerOutputs:
    """Rank 0's result buffers for `n_scans` scans of `n_total` sequences,
    mapped into every rank of `dist` through CUDA IPC (handles exchanged with
    broadcast_object_list).  raw(k) / passed(k) are device pointers valid on
    the calling rank; rank 0 reads the results with results(k) after every
    rank's scans are synchronised and a barrier."""

    def __init__(self, dist, scanner, n_total, n_scans=1, comm_device=None):
        """Collective over `dist`: either every rank maps the buffers or every
        rank raises (no rank is left half-configured)."""
        import torch
        self.dist, self.s, self.n, self.k = dist, scanner, int(n_total), int(n_scans)
        nbytes = 2 * self.n * self.k
        self.base, err = None, None
        obj = [None]
        if dist.get_rank() == 0:
            try:
                self.base, handle = scanner.peer_buffer_create(nbytes)
                obj = [handle]
            except Exception as e:  # noqa: BLE001
                err = e
        dist.broadcast_object_list(obj, src=0)
        if dist.get_rank() != 0:
            if obj[0] is None:
                err = RuntimeError("rank 0 could not export its result buffers")
            else:
                try:
                    self.base = scanner.peer_buffer_open(obj[0])
                except Exception as e:  # noqa: BLE001
                    err = e
        dev = comm_device if comm_device is not None else torch.device("cpu")
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            scanner.peer_buffers_release()
            raise RuntimeError(f"fused gather unavailable on some rank ({err or 'peer failure'})")

    def raw(self, k):
        return self.base + 2 * self.n * k

    def passed(self, k):
        return self.base + 2 * self.n * k + self.n

    def mark_unwritten(self):
        """Rank 0: pass bytes to 2 (scans write 0/1) so coverage is checkable."""
        if self.dist.get_rank() == 0:
            self.s.device_fill(self.base, 2, 2 * self.n * self.k)

    def results(self, k):
        """Rank 0: (raw uint8[n], pass bool[n]) of scan k; raises if some
        sequence was not written by any rank."""
        buf = self.s.device_to_host(self.raw(k), 2 * self.n)
        raw, ps = buf[:self.n], buf[self.n:]
        if (ps > 1).any():
            raise RuntimeError("fused gather: %d sequences not written" % int((ps > 1).sum()))
        return raw, ps.astype(bool)

    def close(self):
        self.s.peer_buffers_release()
