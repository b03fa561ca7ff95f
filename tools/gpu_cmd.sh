cd $GRAFT_REPO_ROOT
C2="dict(depth=5, order_equiv=4, backend='blas', precision='f32', sigma_min=1e-6)"
for i in 1 2; do for v in default r152 r152m8; do for st in 3 4; do
KIFMM_TMEM_STAGES=$st KIFMM_LIB=$PWD/_variants/lib$v.so timeout 300 python tools/config_times.py 1000000 "$C2" > gpurun_out/var.log 2>&1
echo $v st$st $(grep -h "evaluate\|sweep m2l5" gpurun_out/var.log | grep -o "evaluate [0-9.]* ms\|tmem_f32 *[0-9.]* us") >> gpurun_out/variants.log
done; done; done
