# lhmm_scan_streamed_jobs: GPU tests, then C4 (weak, 6.25M env_nr-like per GPU)
# end to end with the upload under every scan (jobs) vs under the first (single)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "streamed" > gpurun_out/jobs_tests.txt 2>&1
tail -3 gpurun_out/jobs_tests.txt
for mode in jobs single; do
  timeout 900 python bench.py --workload c4 --legs verify --steps 5 --no-cpu-baseline --e2e-mode $mode \
    > gpurun_out/jobs_c4_$mode.json 2> gpurun_out/jobs_c4_$mode.err
done
echo done
