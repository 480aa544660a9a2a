# Round-2 checks: GPU tests, C1 timing, drop-in acceptance, ncu of the
# FP16XRM kernel, the default bench's launch list (per-piece streaming so the
# streamed e2e kernel does not spin on copy-stream flags under ncu's
# serialisation), sanitizer over the new kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/chk_tests.log 2>&1; echo rc=$? >> gpurun_out/chk_tests.log
python scripts/c1_timing.py 100 > gpurun_out/chk_c1.jsonl 2>&1
./oracle/_ref/acceptance_b200 > gpurun_out/chk_acc.txt 2>&1
./oracle/_ref/dropin_bench harness > gpurun_out/chk_harness.txt 2>&1
for a in "xrm400 --m 400" "xrm2405 --m 2405"; do
  set -- $a; name=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 \
      -o gpurun_out/prof_$name python scripts/one_scan.py "$@" --alg msv --quant nonsat --variant fp16xrm > /dev/null 2>&1
done
LHMM_STREAM_MEM_OPS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/chk_launches.csv python bench.py --steps 2 --warmup 1 --legs none > gpurun_out/chk_ncu_bench.log 2>&1
python scripts/sanitize_driver.py > gpurun_out/chk_sanitize_plain.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $t = memcheck ] && extra="--leak-check full"
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --target-processes all \
      python scripts/sanitize_driver.py > gpurun_out/chk_sanitize_$t.txt 2>&1
  echo "$t rc=$?" >> gpurun_out/chk_sanitize_rc.txt
done
echo done
