"""examples/scan_fasta.c -- the C ABI used from plain C: profile text + FASTA
or LHMM file in, filter-pipeline results out; checked against the oracle."""
import os
import subprocess

import numpy as np
import pytest

import oracle
import paper_1707_09683_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "bin", "scan_fasta")


def test_example_is_built():
    assert os.path.exists(EXE), "build() compiles examples/*.c"


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["fasta", "lhmm"])
def test_scan_fasta_example_matches_oracle(ora, tmp_path, fmt):
    rng = P.Rng(0xE0E0)
    hmm = rng.random_profile(250)
    db = rng.random_records(3000, 20, 500, plant=(hmm, 0.1))
    db.ids = [f"q{k}" for k in range(db.count)]
    (tmp_path / "p.txt").write_text(P.serialize_profile(hmm))
    if fmt == "fasta":
        path = tmp_path / "db.fa"
        path.write_text(P.to_fasta(db))
        order = np.arange(db.count)
    else:
        path = tmp_path / "db.lhmm"
        bs = P.pack_blocks(db, 6, 32)
        P.write_block_db(bs, str(path))
        pos = {i: k for k, i in enumerate(db.ids)}
        order = np.array([pos[i] for i in bs.db.ids])
    r = subprocess.run([EXE, str(tmp_path / "p.txt"), str(path), "0.05"], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = [ln.split("\t") for ln in r.stdout.strip().splitlines()]
    assert len(lines) == db.count
    q = P.QuantParams()
    costs = P.quantize_emissions(hmm, q)
    oq = oracle.QuantParams(q.scale, q.base, q.dbias, q.tec, q.tjb)
    ssv = ora.scan_flat(1, costs.bytes, db.residues, db.offsets, oq)[order]
    msv = ora.scan_flat(0, costs.bytes, db.residues, db.offsets, oq)[order]
    lens = db.lengths()[order]
    for k, (sid, s_raw, passed, m_raw) in enumerate(lines):
        assert sid == db.ids[int(order[k])]
        assert int(s_raw) == ssv[k]
        want_pass = ora.passes(int(ssv[k]), int(lens[k]), hmm.lambda_, hmm.tau, oq, 1, 0.05)
        assert bool(int(passed)) == bool(want_pass)
        assert (m_raw == "-") if not want_pass else (int(m_raw) == msv[k])
