cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -20 > gpurun_out/pytest_gpu.txt
for t in "" _t384; do
  LHMM_LIB=$PWD/paper_1707_09683_b200/_lib$t/liblhmm_b200.so timeout 900 python scripts/sweep.py --variants fp16 --extra-rows 0 --models 48,200,400,1000,1500,2405 > gpurun_out/sweep_fp16$t.jsonl 2> gpurun_out/sweep_fp16$t.err
done
echo done
