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


def test_relu_form_of_the_exact_step_is_exact():
    """The two-mode exact step's relu form (lhmm_kernel.cuh relu_step):
    sat(max(x, B) + d) == sat(sat(x - B) + (B + d)) in f16 round-to-nearest,
    for every pair of linear-binade cells x, B (patterns 0x3B01 + v) and
    every dbias (d = dbias / 2048) -- exhaustive, 256 x 256 x 256."""
    import numpy as np
    f = (0x3B01 + np.arange(256, dtype=np.uint16)).astype(np.uint16).view(np.float16)
    X, Bv = f[:, None].astype(np.float32), f[None, :].astype(np.float32)

    def sat(a):  # one f16 op: exact f32 sum, one rounding, clamp to [0, 1]
        return np.clip(a.astype(np.float16), np.float16(0), np.float16(1))

    r = sat(X - Bv).astype(np.float32)
    for dbias in range(256):
        d = np.float32(np.float16(dbias / 2048))
        ref = sat(np.maximum(X, Bv) + d)
        bd = (Bv + d).astype(np.float16).astype(np.float32)  # HADD2, no clamp
        new = sat(r + bd)
        assert np.array_equal(ref.view(np.uint16), new.view(np.uint16)), dbias


def test_relu_form_of_the_negated_exact_step_is_exact():
    """The negated two-mode exact step's relu form (Fp16SatMixed, FORM & 8):
    sat(min(n, nB) - d) == sat((nB - d) - sat(nB - n)) in the f16 subnormal
    domain (byte units of 2^-24), for every cell n, every nB and every dbias d
    -- exhaustive, 256 x 256 x 256."""
    import numpy as np
    unit = np.float32(2.0 ** -24)
    n = (np.arange(256, dtype=np.float32) * unit).astype(np.float16)
    N, NB = n[:, None].astype(np.float32), n[None, :].astype(np.float32)

    def f16(a):  # one f16 op: exact f32 result, one rounding
        return a.astype(np.float16)

    def sat(a):
        return np.clip(f16(a), np.float16(0), np.float16(1))

    r = sat(NB - N).astype(np.float32)
    for d in range(256):
        dd = np.float32(np.float16(d * 2.0 ** -24))
        ref = sat(np.minimum(N, NB) - dd)
        nbd = f16(NB - dd).astype(np.float32)  # HADD2 (no clamp): may be negative
        new = sat(nbd - r)
        assert np.array_equal(ref.view(np.uint16), new.view(np.uint16)), d
