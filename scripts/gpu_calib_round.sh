# GPU tests, then a fresh calibration sweep (fp16 + fp16x + dpx16) for the
# geometry policy, and the headline bench lines.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 1800 python scripts/calibrate.py --variants fp16,fp16x,dpx16 > gpurun_out/calib.jsonl 2> gpurun_out/calib.err
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --workload c3 --steps 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo done
