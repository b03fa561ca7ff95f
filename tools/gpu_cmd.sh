cd $GRAFT_REPO_ROOT
C2="dict(depth=5, order_equiv=4, backend='blas', precision='f32', sigma_min=1e-6)"
for v in default m8c384 m5c640 m4c896 default m8c384 m5c640 m4c896; do
KIFMM_LIB=$PWD/_variants/lib$v.so timeout 300 python tools/config_times.py 1000000 "$C2" > gpurun_out/var_$v.log 2>&1
echo $v $(grep -h "evaluate\|leaf_pass" gpurun_out/var_$v.log | grep -o "evaluate [0-9.]* ms\|leaf_pass_f32 *[0-9.]* us") >> gpurun_out/variants.log
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
