# GPU tests + calibration of the FP16X points only (merged into the table by
# the caller), + the MSV A/B on C3
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 2400 python scripts/calibrate.py --variants fp16x > gpurun_out/calib_fp16x.jsonl 2> gpurun_out/calib_fp16x.err
for v in fp16 fp16x; do
  timeout 900 python bench.py --workload c3 --steps 5 --variant $v --no-e2e --no-cpu-baseline > gpurun_out/ab_c3_$v.json 2> gpurun_out/ab_c3_$v.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 0 -c 1 -o gpurun_out/prof_msv2405_sat python bench.py --workload c3 --variant fp16x --nseq 200000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_sat.log 2>&1
echo done
