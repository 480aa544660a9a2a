# Drop-in (engine.hpp over the C ABI) timing: C2 through lanehmm::scan_database
# with the per-call breakdown, the acceptance harness shape, the acceptance suite
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
LHMM_DROPIN_TIMING=1 ./oracle/_ref/dropin_bench 1000000 3 > gpurun_out/dropin_c2.json 2> gpurun_out/dropin_c2_timing.txt
LHMM_DROPIN_TIMING=1 ./oracle/_ref/dropin_bench harness > gpurun_out/dropin_harness.txt 2>&1
./oracle/_ref/acceptance_b200 > gpurun_out/dropin_acc.txt 2>&1
timeout 600 python -m pytest tests/test_dropin.py -q -x > gpurun_out/dropin_pytest.txt 2>&1
tail -2 gpurun_out/dropin_pytest.txt; cat gpurun_out/dropin_c2.json
