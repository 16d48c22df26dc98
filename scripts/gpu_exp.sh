mkdir -p gpurun_out
for v in "" "SUN_CHAIN_HW2=0" "SUN_CHAIN_CLUSTER=0" "SUN_GEMM_CHAIN=0"; do
env $v timeout 900 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py -k cluster_chain -s > gpurun_out/pt_wide_$v.log 2>&1; echo "rc $?" >> gpurun_out/pt_wide_$v.log
done
