cd $GRAFT_REPO_ROOT
# two ranks sharing the single GPU over gloo: exercises bench.py's N>1 path
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --nseq 200000 > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_2rank_ref.json 2> gpurun_out/bench_2rank_ref.err
echo done
# C4 strong with the streamed-jobs e2e at N=2 (two ranks on one GPU)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --workload c4 --steps 2 --warmup 3 --backend gloo --legs verify --no-cpu-baseline > gpurun_out/bench_2rank_c4.json 2> gpurun_out/bench_2rank_c4.err
echo done2
