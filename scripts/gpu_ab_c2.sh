# A/B of side builds (AB_TAGS) on the C2 scans, interleaved: one_scan per
# model per build, three rounds, so drift hits every build alike
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for round in 1 2 3; do
  for t in "" ${AB_TAGS}; do
    if [ -z "$t" ]; then unset LHMM_LIB; name=main; else export LHMM_LIB=$PWD/paper_1707_09683_b200/_lib$t/liblhmm_b200.so; name=$t; fi
    for m in 1000 400; do
      echo "$name M=$m $(python scripts/one_scan.py --m $m --alg ssv --reps 4 | tail -1)" >> gpurun_out/ab_c2.txt
    done
    echo "$name C1 $(python scripts/c1_timing.py 50 2>/dev/null | head -1)" >> gpurun_out/ab_c2.txt
  done
done
echo done
