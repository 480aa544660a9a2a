# A/B of a side build (AB_TAG, AB_DEFS; built on the box) on single instances
# (AB_POINTS: "M alg variant lanes rows" entries separated by ';'), 3 rounds
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
defs=""; for d in $AB_DEFS; do defs="$defs -D $d"; done
python -m paper_1707_09683_b200.build $defs --tag ${AB_TAG} > gpurun_out/ab_build.log 2>&1 || { tail -5 gpurun_out/ab_build.log; exit 1; }
IFS=';' read -ra PTS <<< "$AB_POINTS"
for round in 1 2 3; do
  for t in main ${AB_TAG}; do
    if [ "$t" = main ]; then unset LHMM_LIB; else export LHMM_LIB=$PWD/paper_1707_09683_b200/_lib$t/liblhmm_b200.so; fi
    for pt in "${PTS[@]}"; do set -- $pt
      echo "$t M=$1 $2 $3 L$4 H$5 $(python scripts/one_scan.py --m $1 --alg $2 --variant $3 --lanes $4 --rows $5 --reps 4 | tail -1)"
    done
  done
done > gpurun_out/ab_inst.txt 2>&1
unset LHMM_LIB
echo done
