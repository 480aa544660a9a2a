# GPU tests, then the calibration sweep the geometry policy is built from
# (scripts/make_calib.py turns gpurun_out/calib.jsonl into csrc/calib_b200.inc)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 2400 python scripts/calibrate.py --variants ${CALIB_VARIANTS:-fp16,fp16x,dpx16} > gpurun_out/calib.jsonl 2> gpurun_out/calib.err
echo done
