"""Build-level guards (CPU): the FP16XM / FP16XH forms keep byte scores as
f16 subnormals, so they are exact only if no f16 instruction of the scan
kernels flushes subnormals.  The SASS of the hot instances must not contain
flush-to-zero forms (HADD2.FTZ / HFMA2.FTZ / HMNMX2.FTZ); the runtime probe
(abi.cu subnormal_selfcheck, tests/test_gpu_bench_inputs.py) guards the
device side."""
import glob
import os
import re
import shutil
import subprocess

import pytest

import paper_1707_09683_b200 as P

BUILD = os.path.join(os.path.dirname(P.__file__), "_build")
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


@pytest.mark.parametrize("unit", ["inst_fp16xm_ssv_L8", "inst_fp16xh_msv_L32",
                                  "inst_fp16xm_msv_L16", "inst_fp16x_msv_L1"])
def test_hot_instances_keep_f16_subnormals(unit):
    obj = os.path.join(BUILD, unit + ".cu.o")
    if not os.path.exists(obj) or not os.path.exists(CUOBJDUMP):
        pytest.skip("object or cuobjdump missing (run build first)")
    sass = subprocess.run([CUOBJDUMP, "-sass", obj], capture_output=True, text=True,
                          check=True).stdout
    f16 = re.findall(r"\b(H(?:ADD2|FMA2|MNMX2|MUL2)[.A-Z0-9_]*)", sass)
    assert f16, "no f16 instructions found: the SASS listing changed shape"
    assert not [i for i in f16 if ".FTZ" in i], "flush-to-zero f16 instructions in " + unit


def test_build_flags_have_no_fast_math():
    from paper_1707_09683_b200 import build as B
    flags = " ".join(B.COMMON + B.ARCH)
    assert "fast_math" not in flags and "ftz=true" not in flags
