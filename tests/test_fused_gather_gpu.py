"""The fused gather (shard.PeerOutputs + lhmm_scan_device_global): ranks map
rank 0's result buffers through CUDA IPC and their scan kernels store results
there directly by global sequence index.  Two and three processes share the
one GPU of the test box (same-device IPC; on an 8-GPU box the mapping is
NVLink peer memory); the gloo group only exchanges the IPC handle and the
barrier.  Rank 0 checks every byte against the oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    import torch.distributed as dist

    import oracle
    import paper_1707_09683_b200 as P
    from paper_1707_09683_b200.shard import PeerOutputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = P.Rng(4242)
        hmm = rng.random_profile(700)
        db = rng.lognormal_records(6000, 250, 0.6, 2, plant=(hmm, 0.3))
        q = P.QuantParams()
        costs = P.quantize_emissions(hmm, q)
        with P.Scanner(0) as s:
            s.set_profile(costs, q, hmm.lambda_, hmm.tau)
            s.set_database(db, rank, world)
            out = PeerOutputs(dist, s, db.count, n_scans=2)  # gloo: CPU agreement
            out.mark_unwritten()
            dist.barrier()
            for k, (alg, var) in enumerate(((P.Algorithm.Msv, P.Variant.Auto),
                                            (P.Algorithm.Ssv, P.Variant.Fp16x))):
                s.scan_device_global(P.ScanOptions(alg=alg, variant=var, threshold=0.05),
                                     out.raw(k), out.passed(k))
            dist.barrier()
            if rank == 0:
                ora = oracle.Oracle()
                oq = oracle.QuantParams(q.scale, q.base, q.dbias, q.tec, q.tjb)
                ok = True
                for k, alg in enumerate((0, 1)):
                    raw, ps = out.results(k)
                    want = ora.scan_flat(alg, costs.bytes, db.residues, db.offsets, oq)
                    lens = np.diff(db.offsets)
                    wp = np.array([ora.passes(int(r), int(n), hmm.lambda_, hmm.tau, oq, alg, 0.05)
                                   for r, n in zip(want, lens)])
                    ok = ok and np.array_equal(raw, want) and np.array_equal(ps, wp)
                with open(result_path, "w") as f:
                    f.write("ok" if ok else "mismatch")
            dist.barrier()
            out.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_gather_over_ipc(tmp_path, world):
    path = str(tmp_path / "r.txt")
    mp.spawn(_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    assert open(path).read() == "ok"


def _worker_block(rank, world, port, result_path, mode):
    """shard.BlockGather: every rank scans its share into local buffers and
    bulk-copies its block into rank 0's IPC staging buffer; contiguous shares
    (chunk slices: no permutation) and LPT shares (one scatter on rank 0)."""
    import torch
    import torch.distributed as dist

    import oracle
    import paper_1707_09683_b200 as P
    from paper_1707_09683_b200.shard import BlockGather

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = P.Rng(5151)
        hmm = rng.random_profile(300)
        db = rng.lognormal_records(9000, 250, 0.6, 2, plant=(hmm, 0.2))
        q = P.QuantParams()
        costs = P.quantize_emissions(hmm, q)
        torch.cuda.set_device(0)
        with P.Scanner(0) as s:
            s.set_profile(costs, q, hmm.lambda_, hmm.tau)
            if mode == "contiguous":
                lo, hi = db.count * rank // world, db.count * (rank + 1) // world
                local = P.SequenceDB(db.residues[int(db.offsets[lo]):int(db.offsets[hi])],
                                     db.offsets[lo:hi + 1] - db.offsets[lo])
                s.set_database(local)
                gidx = np.arange(lo, hi, dtype=np.int64)
            else:
                s.set_database(db, rank, world)
                gidx = s.shard_indices().astype(np.int64)
            n = len(gidx)
            g = BlockGather(dist, s, gidx, db.count, n_scans=2)
            assert g.identity == (mode == "contiguous")
            g.mark_unwritten()
            dist.barrier()
            bufs = [(torch.empty(max(n, 1), dtype=torch.uint8, device="cuda"),
                     torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")) for _ in range(2)]
            for k, alg in enumerate((P.Algorithm.Msv, P.Algorithm.Ssv)):
                s.scan_device(P.ScanOptions(alg=alg, threshold=0.05), bufs[k][0].data_ptr(),
                              bufs[k][1].data_ptr())
                g.push(k, bufs[k][0].data_ptr(), bufs[k][1].data_ptr())
            s.synchronize()
            dist.barrier()
            if rank == 0:
                for k in range(2):
                    g.finish(k)
                ora = oracle.Oracle()
                oq = oracle.QuantParams(q.scale, q.base, q.dbias, q.tec, q.tjb)
                ok = True
                for k, alg in enumerate((0, 1)):
                    raw, ps = g.results(k)
                    want = ora.scan_flat(alg, costs.bytes, db.residues, db.offsets, oq)
                    lens = np.diff(db.offsets)
                    wp = np.array([ora.passes(int(r), int(m), hmm.lambda_, hmm.tau, oq, alg, 0.05)
                                   for r, m in zip(want, lens)])
                    ok = ok and np.array_equal(raw, want) and np.array_equal(ps, wp)
                with open(result_path, "w") as f:
                    f.write("ok" if ok else "mismatch")
            dist.barrier()
            g.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["contiguous", "lpt"])
@pytest.mark.parametrize("world", [2, 3])
def test_block_gather_over_ipc(tmp_path, world, mode):
    path = str(tmp_path / "r.txt")
    mp.spawn(_worker_block, args=(world, _free_port(), path, mode), nprocs=world, join=True)
    assert open(path).read() == "ok"
