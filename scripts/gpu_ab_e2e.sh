# A/B of a side build (AB_TAG, AB_DEFS; built on the box) against the main
# library on the default bench's headline + e2e (C2), interleaved three times
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
defs=""; for d in $AB_DEFS; do defs="$defs -D $d"; done
python -m paper_1707_09683_b200.build $defs --tag ${AB_TAG} > gpurun_out/ab_build.log 2>&1 || { tail -5 gpurun_out/ab_build.log; exit 1; }
rm -f gpurun_out/abe_*.json
for round in 1 2 3; do
  for t in main ${AB_TAG}; do
    if [ "$t" = main ]; then unset LHMM_LIB; else export LHMM_LIB=$PWD/paper_1707_09683_b200/_lib$t/liblhmm_b200.so; fi
    timeout 600 python bench.py --legs none --steps 20 --no-cpu-baseline >> gpurun_out/abe_$t.json 2>> gpurun_out/abe_$t.err
  done
done
unset LHMM_LIB
echo done
