"""Multi-GPU driver: one process per GPU, the database sharded by residue
count (lhmm_set_database's LPT tile plan) or as contiguous chunks
(chunk_plan), per-sequence raw scores and pass bits gathered to rank 0.  The
path has no reduction -- only this gather (BASELINE.json north_star;
SURVEY.md §8(e)).

Three gathers:
* BlockGather -- the default: each rank scans into local device buffers and
  copies its contiguous block of results into rank 0's staging buffer (CUDA
  IPC / NVLink peer memory) with ONE bulk copy per scan; rank 0 puts staging
  order into global order with one scatter kernel, or not at all when the
  shards are contiguous ranges of the global order.
* PeerOutputs -- the fused per-sequence form: rank 0's full-length result
  buffers are mapped into every rank and each rank's scan kernel stores every
  result there directly by global index (lhmm_scan_device_global): one remote
  byte store per sequence.
* NcclGather -- the collective fallback: one torch.distributed gather of 2
  bytes (raw, pass) per sequence per scan; the global indices are exchanged
  once at setup.  Any backend (NCCL on the box, gloo on CPU for the tests).
"""
from __future__ import annotations

import numpy as np


class NcclGather:
    """torch.distributed gather of every rank's (raw, pass) bytes to rank 0:
    2 bytes per sequence per call.  The shard sizes and global indices are
    exchanged once here; rank 0 keeps the index map on the gather device."""

    def __init__(self, dist, gidx, n_total, device=None, validate=True):
        import torch
        self.dist, self.n_total = dist, int(n_total)
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        gidx = torch.as_tensor(np.asarray(gidx, dtype=np.int64))
        self.dev = device if device is not None else torch.device("cpu")
        n = torch.tensor([gidx.numel()], dtype=torch.int64, device=self.dev)
        counts = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(counts, n)
        self.counts = [int(c) for c in counts]
        self.mx = max(1, max(self.counts))
        buf = torch.full((self.mx,), -1, dtype=torch.int64, device=self.dev)
        buf[:gidx.numel()] = gidx.to(self.dev)
        glist = [torch.empty_like(buf) for _ in range(self.world)] if self.rank == 0 else None
        dist.gather(buf, glist, dst=0)
        self.index = None
        if self.rank == 0:
            self.index = torch.cat([g[:c] for g, c in zip(glist, self.counts)])
            if validate and (self.index.numel() != self.n_total or
                             int(torch.unique(self.index).numel()) != self.n_total):
                raise RuntimeError("shards do not partition the database")

    def gather(self, raw, passed, as_numpy=True):
        """raw / passed: uint8 tensors of the shard's local outputs (local
        order).  Returns full-length (raw, pass) on rank 0, (None, None)
        elsewhere."""
        import torch
        k = raw.numel()
        buf = torch.zeros((2, self.mx), dtype=torch.uint8, device=self.dev)
        buf[0, :k] = raw.to(self.dev)
        buf[1, :k] = passed.to(self.dev).to(torch.uint8)
        glist = [torch.empty_like(buf) for _ in range(self.world)] if self.rank == 0 else None
        self.dist.gather(buf, glist, dst=0)
        if self.rank != 0:
            return None, None
        allg = torch.cat([g[:, :c] for g, c in zip(glist, self.counts)], dim=1)
        out_raw = torch.zeros(self.n_total, dtype=torch.uint8, device=self.dev)
        out_pass = torch.zeros(self.n_total, dtype=torch.bool, device=self.dev)
        out_raw[self.index] = allg[0]
        out_pass[self.index] = allg[1].to(torch.bool)
        if as_numpy:
            return out_raw.cpu().numpy(), out_pass.cpu().numpy()
        return out_raw, out_pass


def gather_to_rank0(dist, raw, passed, gidx, n_total, device=None, as_numpy=True,
                    validate=True):
    """One-shot NcclGather: full-length (raw, pass) on rank 0, (None, None)
    elsewhere.  raw / passed: uint8 tensors of the shard's local outputs;
    gidx: their global indices."""
    dev = raw.device if device is None else device
    g = NcclGather(dist, gidx.cpu().numpy() if hasattr(gidx, "cpu") else gidx, n_total, dev,
                   validate)
    return g.gather(raw, passed, as_numpy=as_numpy)


def chunk_plan(n_chunks, rank, world):
    """Contiguous chunk ranges per rank: rank r owns chunks
    [r*n/world, (r+1)*n/world) of a database generated (and kept) as n_chunks
    independent, identically distributed pieces -- each rank generates and
    packs only its own chunks, and its shard is a contiguous range of the
    global order (BlockGather needs no permutation)."""
    return range(n_chunks * rank // world, n_chunks * (rank + 1) // world)


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


class BlockGather:
    """Rank 0's staging buffers for `n_scans` scans (raw | pass, n_total bytes
    each), mapped into every rank through CUDA IPC.  push(k, raw, pass) copies
    this rank's contiguous local results into staging at the rank's offset
    (one bulk D2D copy per buffer over NVLink, asynchronous on the scanner's
    stream); after every rank synchronised and a barrier, rank 0 reads the
    results in global order with results(k) -- identity when the shards are
    contiguous ranges of the global order, else one scatter kernel
    (lhmm_scatter_results) through the index map exchanged at setup."""

    def __init__(self, dist, scanner, gidx, n_total, n_scans=1, comm_device=None):
        import torch
        self.dist, self.s, self.n, self.k = dist, scanner, int(n_total), int(n_scans)
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        gidx = np.asarray(gidx, dtype=np.int64)
        self.n_local = int(gidx.size)
        dev = comm_device if comm_device is not None else torch.device("cpu")
        cnt = torch.tensor([self.n_local], dtype=torch.int64, device=dev)
        counts = [torch.zeros_like(cnt) for _ in range(self.world)]
        dist.all_gather(counts, cnt)
        counts = [int(c) for c in counts]
        if sum(counts) != self.n:
            raise RuntimeError("shards do not partition the database")
        self.offset = sum(counts[:self.rank])
        # contiguous shards (chunk_plan) need no permutation on rank 0
        contiguous = bool(self.n_local == 0 or (gidx[0] == self.offset and
                                                np.array_equal(gidx, self.offset +
                                                               np.arange(self.n_local))))
        flag = torch.tensor([1 if contiguous else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        self.identity = bool(int(flag.item()))
        self.index = None
        if not self.identity:
            # the staging-order -> global-order map, once, on rank 0's device
            g = NcclGather(dist, gidx, self.n, dev)
            if self.rank == 0:
                self.index = g.index.to(torch.device("cuda", torch.cuda.current_device()))
                self.final = [(torch.empty(self.n, dtype=torch.uint8, device=self.index.device),
                               torch.empty(self.n, dtype=torch.uint8, device=self.index.device))
                              for _ in range(self.k)]
        self.peer = PeerOutputs(dist, scanner, self.n, n_scans=self.k, comm_device=dev)

    def mark_unwritten(self):
        self.peer.mark_unwritten()

    def push(self, k, raw_ptr, pass_ptr):
        """Copy this rank's local results of scan k (device pointers, n_local
        bytes each) into rank 0's staging block (asynchronous)."""
        if self.n_local:
            self.s.device_copy(self.peer.raw(k) + self.offset, raw_ptr, self.n_local)
            self.s.device_copy(self.peer.passed(k) + self.offset, pass_ptr, self.n_local)

    def finish(self, k):
        """Rank 0, after the ranks' copies landed: staging -> global order."""
        if self.identity or self.rank != 0:
            return
        f = self.final[k]
        self.s.scatter_results(f[0].data_ptr(), f[1].data_ptr(), self.peer.raw(k),
                               self.peer.passed(k), self.index.data_ptr(), self.n)

    def results(self, k):
        """Rank 0: (raw uint8[n], pass bool[n]) of scan k in global order;
        raises if some sequence was not written by any rank."""
        if self.identity:
            return self.peer.results(k)
        self.s.synchronize()
        raw = self.final[k][0].cpu().numpy()
        ps = self.final[k][1].cpu().numpy()
        if (ps > 1).any():
            raise RuntimeError("block gather: %d sequences not written" % int((ps > 1).sum()))
        return raw, ps.astype(bool)

    def close(self):
        self.peer.close()
