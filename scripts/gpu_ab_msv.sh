# MSV A/B: exact FP16 vs two-mode FP16X on C3 and a model sweep, plus GPU tests
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
for v in fp16 fp16x; do
  timeout 900 python bench.py --workload c3 --steps 5 --variant $v --no-e2e --no-cpu-baseline > gpurun_out/ab_c3_$v.json 2> gpurun_out/ab_c3_$v.err
done
timeout 1200 python scripts/sweep.py --variants fp16,fp16x --algs msv --extra-rows 1 --models 48,200,400,1000,2405 > gpurun_out/ab_sweep.jsonl 2> gpurun_out/ab_sweep.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 0 -c 1 -o gpurun_out/prof_msv2405_sat python bench.py --workload c3 --variant fp16x --nseq 200000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_sat.log 2>&1
echo done
