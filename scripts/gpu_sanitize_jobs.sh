# compute-sanitizer memcheck + racecheck over the sanitizer driver (incl. the
# streamed-jobs path)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/sanitize_driver.py > gpurun_out/sj_plain.txt 2>&1; tail -1 gpurun_out/sj_plain.txt
for t in memcheck racecheck synccheck; do
  extra=""; [ $t = memcheck ] && extra="--leak-check full"
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --target-processes all \
      python scripts/sanitize_driver.py > gpurun_out/sj_$t.txt 2>&1
  echo "$t rc=$?" >> gpurun_out/sj_$t.txt; tail -3 gpurun_out/sj_$t.txt
done
