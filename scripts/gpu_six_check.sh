cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_every_instance.py tests/test_gpu_parity.py tests/test_gpu_bench_inputs.py -x -q -k "fp16xm or Mixed or mixed or fp16xrm or Fixed or golden or relaxed or 4096" > gpurun_out/t_six2.log 2>&1; echo rc=$? >> gpurun_out/t_six2.log
for a in "1000 8 63" "400 4 50" "2000 16 63" "900 8 58" "850 8 53" "780 8 48" "1080 8 68" "2405 32 38"; do set -- $a
  echo "M=$1 $(python scripts/one_scan.py --m $1 --alg ssv --variant fp16xm --lanes $2 --rows $3 --reps 4 | tail -1)"; done > gpurun_out/six_one2.txt 2>&1
timeout 1500 python scripts/calibrate.py --variants fp16xm --algs ssv > gpurun_out/calib_xm_ssv_six.jsonl 2>/dev/null
timeout 1500 python scripts/calibrate.py --variants fp16xrm --algs msv --quant nonsat > gpurun_out/calib_xrm_six.jsonl 2>/dev/null
