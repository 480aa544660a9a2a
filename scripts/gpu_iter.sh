# generic GPU iteration: tests, sweep, bench, ncu (pass stages as args)
cd $GRAFT_REPO_ROOT
for stage in "$@"; do
case $stage in
tests) timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt ;;
smoke) timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1 ;;
calib) timeout 1500 python scripts/calibrate.py ${CALIB_ARGS} > gpurun_out/calib.jsonl 2> gpurun_out/calib.err ;;
dropin) (time ./oracle/_ref/acceptance_b200) > gpurun_out/acceptance_b200.txt 2>&1; (time ./oracle/_ref/acceptance_ref) > gpurun_out/acceptance_ref.txt 2>&1 ;;
sweep) timeout 1200 python scripts/sweep.py --variants ${SWEEP_VARIANTS:-fp16,dpx16} --extra-rows ${SWEEP_EXTRA:-1} ${SWEEP_ARGS} > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err ;;
bench) timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err ;;
launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_under_ncu.log 2>&1 ;;
ncu) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-1} -o gpurun_out/prof_${NCU_TAG:-k} python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline ${NCU_BENCH_ARGS} > gpurun_out/ncu_full.log 2>&1 ;;
esac
done
echo done
