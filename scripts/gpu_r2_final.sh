# Round-2 final record: GPU tests, default bench, reference arm, drop-in (C2
# timing, acceptance harness, acceptance suite), launch list of the default
# bench, ncu --set full of the C2 dominant (SSV M=1000) and C3 (MSV M=2405)
# kernels, sanitizer over the kernel forms.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/fin_tests.log 2>&1; echo rc=$? >> gpurun_out/fin_tests.log
tail -2 gpurun_out/fin_tests.log
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
LHMM_DROPIN_TIMING=1 ./oracle/_ref/dropin_bench 1000000 3 > gpurun_out/fin_dropin.json 2> gpurun_out/fin_dropin_timing.txt
./oracle/_ref/dropin_bench harness > gpurun_out/fin_harness.txt 2>&1
./oracle/_ref/acceptance_b200 > gpurun_out/fin_acc_b200.txt 2>&1
LHMM_STREAM_MEM_OPS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/fin_launches.csv python bench.py --steps 2 --warmup 1 --legs none > gpurun_out/fin_ncu_bench.log 2>&1
for a in "c2dom --m 1000 --alg ssv" "c3 --m 2405 --alg msv"; do
  set -- $a; name=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 \
      -o gpurun_out/fin_prof_$name python scripts/one_scan.py "$@" > gpurun_out/fin_ncu_$name.log 2>&1
done
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --target-processes all \
    python scripts/sanitize_driver.py > gpurun_out/fin_sanitize_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/fin_sanitize_memcheck.txt
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --target-processes all \
    python scripts/sanitize_driver.py > gpurun_out/fin_sanitize_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/fin_sanitize_racecheck.txt
echo done
