# A/B side builds (AB_TAGS, e.g. "_mB _mC"; python -m paper_1707_09683_b200.build
# with -D... --tag ...) on the FP16X MSV calibration grid and an MSV bench line
cd $GRAFT_REPO_ROOT
for t in ${AB_TAGS}; do
  export LHMM_LIB=$PWD/paper_1707_09683_b200/_lib$t/liblhmm_b200.so
  timeout 900 python scripts/calibrate.py --variants fp16x,fp16xalt --algs msv --nseq 400000 > gpurun_out/ab$t.jsonl 2> gpurun_out/ab$t.err
  timeout 300 python bench.py --workload c2 --models 48,400,2405 --algs msv --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_bench$t.json 2>> gpurun_out/ab$t.err
done
echo done
