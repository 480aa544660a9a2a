# A/B of the six-row slot rule: side build with -DLHMM_XM_SIX_MAXPCT=$PCT on
# the box, SSV C2/C5 geometries interleaved with the main build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_1707_09683_b200.build -D LHMM_XM_SIX_MAXPCT=${PCT:-80} --tag _six > gpurun_out/six_build.log 2>&1
for round in 1 2; do
  for t in "" _six; do
    if [ -z "$t" ]; then unset LHMM_LIB; n=main; else export LHMM_LIB=$PWD/paper_1707_09683_b200/_lib$t/liblhmm_b200.so; n=$t; fi
    for a in "1000 8 63" "1000 8 65" "400 4 50" "800 8 50" "2000 16 63" "200 2 50" "100 2 25"; do set -- $a
      echo "$n M=$1 $(python scripts/one_scan.py --m $1 --alg ssv --variant fp16xm --lanes $2 --rows $3 --reps 3 | tail -1)"
    done
  done
done > gpurun_out/six_ab.txt 2>&1
