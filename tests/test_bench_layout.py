"""bench.py's database layouts (CPU): chunked databases cover every sequence
exactly once, each rank's share is a contiguous range of the global order,
slices of a single stream reproduce the reference's one-stream set (C2 / C1
as BASELINE defines them), and the reference arm's config equals the b200
arm's for the same run."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1707_09683_b200 as P  # noqa: E402


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "sweep"])
@pytest.mark.parametrize("scaling", ["weak", "strong"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_layout_partitions_the_database(name, scaling, world):
    chunks, share = bench.db_layout(name, scaling, world)
    total = sum(c for _, c in chunks)
    seen = np.zeros(total, np.int32)
    starts = np.cumsum([0] + [c for _, c in chunks])
    prev_end = 0
    for r in range(world):
        for c, lo, hi in share[r]:
            g0, g1 = starts[c] + lo, starts[c] + hi
            assert g0 == prev_end  # contiguous, in rank order
            seen[g0:g1] += 1
            prev_end = g1
    assert (seen == 1).all()
    if name == "c4" and scaling == "strong":
        assert total == 50_000_000


def test_slices_reproduce_the_single_stream_sets():
    api = bench.ProductGen(P)
    parts = [bench.make_inputs(api, "c2", "strong", 3, [r], (48,)) for r in range(3)]
    db = P.Rng(0x5EED).lognormal_records(1_000_000, 290, 0.65, 2)
    assert np.array_equal(np.concatenate([p[0] for p in parts]), db.residues)
    assert [p[2] for p in parts] == [0, 333333, 666666]
    res, off, first, profs = bench.make_inputs(api, "c1", "weak", 1, [0], (200,))
    rng = P.Rng(0xC1)
    hmm = rng.random_profile(200)
    c1 = rng.random_records(10000, 50, 650, plant=(hmm, 0.05))
    assert np.array_equal(res, c1.residues) and np.array_equal(off, c1.offsets)
    assert np.allclose(profs[200][0], hmm.match_scores.reshape(-1))


def test_reference_generators_match_product_generators():
    import oracle
    try:
        ref = oracle.Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")
    a = bench.make_inputs(bench.ProductGen(P), "c4", "weak", 1, [0], (200,))
    b = bench.make_inputs(bench.ReferenceGen(ref, oracle), "c4", "weak", 1, [0], (200,))
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.allclose(a[3][200][0], b[3][200][0])
    cfg_a = bench.workload_config("c4", "weak", "d", (200,), ["msv"], a[1].size - 1,
                                  int(a[1][-1]), 1)
    cfg_b = bench.workload_config("c4", "weak", "d", (200,), ["msv"], b[1].size - 1,
                                  int(b[1][-1]), 1)
    assert cfg_a == cfg_b
