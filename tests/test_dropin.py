"""The drop-in proof: the reference's own acceptance suite
(proj/tests/acceptance_main.cpp), linked against the reference library with
src/engine.cpp and src/seqdb.cpp swapped for
paper_1707_09683_b200/dropin/{engine,seqdb}_b200.cpp (the B200 engine and
database I/O behind include/lhmm_b200.h), must pass every criterion the
unmodified reference passes; so must the reference's unit tests.  The
binaries are built by oracle/Makefile (`make -C oracle dropin unit`) where
/root/reference exists and travel prebuilt."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B200 = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")
REF = os.path.join(ROOT, "oracle", "_ref", "acceptance_ref")


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


@pytest.mark.gpu
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


# --- the reference's own unit tests (proj/tests/test_*.cpp, built with
# oracle/mini_doctest by `make -C oracle unit`) ---------------------------------
UNIT_REF = os.path.join(ROOT, "oracle", "_ref", "unit_ref")
UNIT_B200 = os.path.join(ROOT, "oracle", "_ref", "unit_b200")


def run_unit(path, *args):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    r = subprocess.run([path, *args], capture_output=True, text=True, timeout=1200)
    m = re.search(r"test cases: (\d+) \| passed: (\d+) \| failed: (\d+)", r.stdout)
    assert m, r.stdout + r.stderr
    return int(m.group(1)), int(m.group(3)), r.stdout + r.stderr


@pytest.mark.gpu
def test_reference_unit_tests_on_b200_engine():
    """test_engine.cpp / test_select.cpp through the B200 engine, every case
    (ReorderMode::PaperWrap included: the kernel's wrap mode)."""
    n, failed, out = run_unit(UNIT_B200, "file=test_engine,test_select")
    assert n >= 20 and failed == 0, out


# the host-only parts (database / profile I/O, oracle, SWAR helpers) need no GPU
def test_reference_unit_tests_host_parts_on_b200_dropin():
    n, failed, out = run_unit(UNIT_B200, "file=test_seqdb,test_profile,test_oracle,test_vwarp")
    assert n >= 40 and failed == 0, out


def test_reference_unit_tests_pass_on_the_reference_itself():
    """The harness check: the unmodified reference passes its own suite."""
    n, failed, out = run_unit(UNIT_REF)
    assert n >= 60 and failed == 0, out
