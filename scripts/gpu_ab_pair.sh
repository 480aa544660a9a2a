# A/B of a side build (AB_TAG, built with python -m paper_1707_09683_b200.build
# -D ... --tag AB_TAG) against the main library: GPU tests on the main build,
# then the bench's sweep + C1 legs on both, interleaved twice
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
# the side build is made on the box (AB_DEFS: space-separated -D values)
defs=""; for d in $AB_DEFS; do defs="$defs -D $d"; done
python -m paper_1707_09683_b200.build $defs --tag ${AB_TAG} > gpurun_out/ab_build.log 2>&1 || { tail -5 gpurun_out/ab_build.log; exit 1; }
if [ -z "$AB_SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -rf -x > gpurun_out/ab_pytest_gpu.txt 2>&1
  tail -3 gpurun_out/ab_pytest_gpu.txt
fi
for round in 1 2; do
  for t in main ${AB_TAG}; do
    if [ "$t" = main ]; then unset LHMM_LIB; else export LHMM_LIB=$PWD/paper_1707_09683_b200/_lib$t/liblhmm_b200.so; fi
    timeout 600 python bench.py --legs sweep,c1 --steps 5 --c1-steps 500 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${t}_$round.json 2> gpurun_out/ab_${t}_$round.err
  done
done
unset LHMM_LIB
echo done
