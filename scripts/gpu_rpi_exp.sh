# chunk-budget experiment for two-mode MSV: calibrate FP16X MSV at L=16,32
# against side builds _rA/_rB/_rC (python -m paper_1707_09683_b200.build -D ... --tag ...)
cd $GRAFT_REPO_ROOT
for t in ${RPI_TAGS:-_rA _rB _rC}; do
  LHMM_LIB=$PWD/paper_1707_09683_b200/_lib$t/liblhmm_b200.so timeout 900 python scripts/calibrate.py --variants fp16x --algs msv --lanes 16,32 --nseq 400000 > gpurun_out/rpi$t.jsonl 2> gpurun_out/rpi$t.err
done
echo done
