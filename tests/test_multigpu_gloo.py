"""The N>1 path on CPU: world-size-2 (and 3) gloo process groups run the shard
plan and the gather-to-rank-0 of per-sequence raw + pass bytes that the
multi-GPU driver uses over NCCL (paper_1707_09683_b200/shard.py).  Per-shard
scores come from the CPU oracle, standing in for the device scan."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    import oracle
    import paper_1707_09683_b200 as P
    from paper_1707_09683_b200.shard import gather_to_rank0, shard_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = P.Rng(2024)
        hmm = rng.random_profile(120)
        db = rng.lognormal_records(1500, 200, 0.6, 2)
        q = oracle.QuantParams(3.0, 120, 3, 20, 20)
        costs = oracle.Oracle().quantize(hmm.match_scores.reshape(-1), q)
        idx = shard_plan(db.offsets, rank, world)
        local = db.subset(idx)
        ora = oracle.Oracle()
        raw = ora.scan_flat(0, costs, local.residues, local.offsets, q, 1)
        lens = np.diff(local.offsets)
        passed = np.array([ora.passes(int(r), int(n), hmm.lambda_, hmm.tau, q, 0, 0.3)
                           for r, n in zip(raw, lens)], dtype=np.uint8)
        out_raw, out_pass = gather_to_rank0(dist, torch.from_numpy(raw), torch.from_numpy(passed),
                                            torch.from_numpy(idx.astype(np.int64)), db.count)
        if rank == 0:
            full = ora.scan_flat(0, costs, db.residues, db.offsets, q, 1)
            ok = np.array_equal(out_raw, full)
            flens = np.diff(db.offsets)
            want_pass = np.array([ora.passes(int(r), int(n), hmm.lambda_, hmm.tau, q, 0, 0.3)
                                  for r, n in zip(full, flens)])
            ok = ok and np.array_equal(out_pass, want_pass)
            with open(result_path, "w") as f:
                f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shard_and_gather_to_rank0(tmp_path, world):
    res = tmp_path / "result.txt"
    mp.spawn(_worker, args=(world, _free_port(), str(res)), nprocs=world, join=True)
    assert res.read_text() == "ok"


def _worker_nccl_gather(rank, world, port, result_path):
    """NcclGather: indices exchanged once, then 2 bytes per sequence per
    gather; contiguous chunk shares (shard.chunk_plan) and LPT shares."""
    import torch
    import torch.distributed as dist

    import oracle
    import paper_1707_09683_b200 as P
    from paper_1707_09683_b200.shard import NcclGather, chunk_plan, shard_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = P.Rng(77)
        hmm = rng.random_profile(90)
        db = rng.lognormal_records(1200, 150, 0.6, 2)
        q = oracle.QuantParams()
        ora = oracle.Oracle()
        costs = ora.quantize(hmm.match_scores.reshape(-1), q)
        full = ora.scan_flat(1, costs, db.residues, db.offsets, q, 1)
        ok = True
        # contiguous shares: 12 chunks of 100 sequences
        mine = chunk_plan(12, rank, world)
        idx_c = np.arange(mine.start * 100, mine.stop * 100, dtype=np.int64)
        for idx in (idx_c, shard_plan(db.offsets, rank, world).astype(np.int64)):
            g = NcclGather(dist, idx, db.count)
            for salt in range(3):  # the same gatherer, several scans
                raw = torch.from_numpy(full[idx] ^ np.uint8(salt))
                ps = torch.from_numpy((full[idx] & 1).astype(np.uint8))
                out_raw, out_pass = g.gather(raw, ps)
                if rank == 0:
                    ok = ok and np.array_equal(out_raw, full ^ np.uint8(salt))
                    ok = ok and np.array_equal(out_pass, (full & 1).astype(bool))
        if rank == 0:
            with open(result_path, "w") as f:
                f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_nccl_gather_two_bytes_per_sequence(tmp_path, world):
    res = tmp_path / "result.txt"
    mp.spawn(_worker_nccl_gather, args=(world, _free_port(), str(res)), nprocs=world, join=True)
    assert res.read_text() == "ok"
