# ncu --set full of single scan_kernel launches for the round-2 kernels:
# FP16XR (relaxed MSV, non-saturating params) at M=2405 (L32 H38) and M=400
# (L4 H50), C3 default (FP16XH L32 H38), C2 dominant (FP16XM SSV L8 H63).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # name, args...
    local name=$1; shift
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 \
        -o gpurun_out/prof_$name python scripts/one_scan.py "$@" > gpurun_out/ncu_$name.log 2>&1
}
run xr2405 --m 2405 --alg msv --quant nonsat --variant fp16xr --lanes 32 --rows 38
run xr400 --m 400 --alg msv --quant nonsat --variant fp16xr --lanes 4 --rows 50
run c3 --m 2405 --alg msv --quant default
run c2dom --m 1000 --alg ssv --quant default
echo done
