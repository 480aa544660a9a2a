# A/B of a side build against the main library: GPU tests on the main build,
# then FP16X MSV calibration at L=16,32 on both (AB_TAG names the side build)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 900 python scripts/calibrate.py --variants fp16x --algs msv --lanes 16,32 --nseq 400000 > gpurun_out/ab_main.jsonl 2> gpurun_out/ab_main.err
LHMM_LIB=$PWD/paper_1707_09683_b200/_lib${AB_TAG}/liblhmm_b200.so timeout 900 python scripts/calibrate.py --variants fp16x --algs msv --lanes 16,32 --nseq 400000 > gpurun_out/ab_side.jsonl 2> gpurun_out/ab_side.err
timeout 900 python bench.py --workload c3 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_c3_main.json 2> gpurun_out/ab_c3_main.err
echo done
