cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/gpu.txt 2>&1; nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 120 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python -m pytest tests -m gpu -q -rf 2>&1 | tail -60 > gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
