# Full GPU pass: tests, smoke, headline bench lines (C2 default, C3, C1,
# sweep), reference arm, the ncu launch list of the default bench and one
# ncu --set full capture of its dominant kernel.
cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/gpu.txt 2>&1; nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --workload c3 --steps 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload c1 --steps 20 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 1500 python bench.py --workload sweep --steps 3 --no-cpu-baseline > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 -o gpurun_out/prof_c2_dominant python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
