# A/B a side build against the main library on both FP16X MSV code forms at
# L=16,32 (AB_TAG names the side build)
cd $GRAFT_REPO_ROOT
timeout 900 python scripts/calibrate.py --variants fp16x,fp16xalt --algs msv --lanes 16,32 --nseq 400000 > gpurun_out/ab_main.jsonl 2> gpurun_out/ab_main.err
LHMM_LIB=$PWD/paper_1707_09683_b200/_lib${AB_TAG}/liblhmm_b200.so timeout 900 python scripts/calibrate.py --variants fp16x,fp16xalt --algs msv --lanes 16,32 --nseq 400000 > gpurun_out/ab_side.jsonl 2> gpurun_out/ab_side.err
echo done
