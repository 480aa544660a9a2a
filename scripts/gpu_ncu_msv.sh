cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
./oracle/_ref/unit_b200 file=test_engine,test_select > gpurun_out/unit_b200.txt 2>&1
for v in fp16 fp16x dpx16; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 0 -c 1 -o gpurun_out/prof_msv2405_$v python bench.py --workload c3 --variant $v --nseq 200000 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$v.log 2>&1
done
echo done
