"""The drop-in proof: the reference's own acceptance suite
(proj/tests/acceptance_main.cpp), linked against the reference library with
src/engine.cpp swapped for paper_1707_09683_b200/dropin/engine_b200.cpp (the
B200 engine behind include/lhmm_b200.h), must pass every criterion the
unmodified reference passes.  Both binaries are built by oracle/Makefile
(`make -C oracle dropin`) where /root/reference exists and travel prebuilt."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B200 = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")
REF = os.path.join(ROOT, "oracle", "_ref", "acceptance_ref")

pytestmark = pytest.mark.gpu


def run(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=1200)
    status = {}
    for line in r.stdout.splitlines():
        m = re.match(r"ACCEPT\[(\d+)\]\s+(\S+)\s*:\s*(PASS|FAIL)", line)
        if m:
            status[int(m.group(1))] = (m.group(2), m.group(3), line)
    return status, r.stdout


def test_reference_acceptance_suite_on_b200_engine():
    got, out = run(B200)
    want, _ = run(REF)
    assert len(got) == 8, out
    for k in range(1, 9):
        # criterion 4 is the reference packer's own balance target (it fails
        # in the unmodified reference too, proj/test_output.txt:11); every
        # other criterion runs through the swapped engine
        assert got[k][1] == want[k][1] or got[k][1] == "PASS", f"{got[k][2]}\nref: {want[k][2]}"
    for k in (1, 2, 3, 5, 6, 7, 8):
        assert got[k][1] == "PASS", got[k][2]
