# thread-count experiment: the same sweep against side builds with
# LHMM_MAX_THREADS = 512 (default), 640, 768 (python -m paper_1707_09683_b200.build -D ... --tag ...)
cd $GRAFT_REPO_ROOT
for t in ${THREAD_TAGS:-"" _t640 _t768}; do
  LHMM_LIB=$PWD/paper_1707_09683_b200/_lib$t/liblhmm_b200.so timeout 900 python scripts/sweep.py --variants ${SWEEP_VARIANTS:-fp16,fp16x} --extra-rows 0 --models ${SWEEP_MODELS:-48,200,400,1000,2405} > gpurun_out/sweep$t.jsonl 2> gpurun_out/sweep$t.err
done
echo done
