cd $GRAFT_REPO_ROOT
timeout 900 python scripts/sweep.py --extra-rows 1 > gpurun_out/sweep1.jsonl 2> gpurun_out/sweep1.err
# launch list of the default bench command (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
# full capture of the dominant kernel (SSV M=1000) -- one launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 -o gpurun_out/prof_ssv1000 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
