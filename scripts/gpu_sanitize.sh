# compute-sanitizer over scripts/sanitize_driver.py: memcheck (+ leak check),
# racecheck (shared-memory hazards), synccheck (barrier / warp-sync misuse),
# initcheck (reads of uninitialised device memory); one summary per tool
cd $GRAFT_REPO_ROOT
python scripts/sanitize_driver.py > gpurun_out/sanitize_plain.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $t = memcheck ] && extra="--leak-check full"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --target-processes all \
      python scripts/sanitize_driver.py > gpurun_out/sanitize_$t.txt 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitize_rc.txt
done
echo done
