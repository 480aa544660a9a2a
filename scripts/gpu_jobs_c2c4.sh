# e2e modes on C2 (3 SSV models) and C4 strong (50M sequences, N=1)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for mode in jobs single jobs single; do
  timeout 900 python bench.py --legs none --steps 10 --no-cpu-baseline --e2e-mode $mode \
    >> gpurun_out/jc2_$mode.json 2>> gpurun_out/jc2_$mode.err
done
timeout 1500 python bench.py --workload c4 --scaling strong --legs verify --steps 3 --no-cpu-baseline \
    > gpurun_out/jc4_strong.json 2> gpurun_out/jc4_strong.err
echo done
