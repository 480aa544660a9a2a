# Round-2 record run: default bench, reference arm, drop-in C2 bench and the
# acceptance suite on the drop-in, ncu launch list of the default bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/rec_bench.json 2> gpurun_out/rec_bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/rec_ref.json 2> gpurun_out/rec_ref.err
LHMM_DROPIN_TIMING=1 ./oracle/_ref/dropin_bench 1000000 3 > gpurun_out/rec_dropin.json 2> gpurun_out/rec_dropin.err
./oracle/_ref/dropin_bench harness > gpurun_out/rec_harness.txt 2>&1
./oracle/_ref/acceptance_b200 > gpurun_out/rec_acc_b200.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/rec_launches.csv python bench.py --steps 2 --warmup 1 \
    > gpurun_out/rec_ncu_bench.log 2>&1
echo done
