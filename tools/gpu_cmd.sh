cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_paths.py > gpurun_out/check_paths.log 2>&1; cat gpurun_out/check_paths.log
C2="dict(depth=5, order_equiv=4, backend='blas', precision='f32', sigma_min=1e-6)"
rm -f gpurun_out/variants.log
for i in 1 2; do for v in default mma3 mma3ng3; do
  if [ $v == default ]; then L=$PWD/paper_2408_07436_b200/libkifmm_b200.so; else L=$PWD/_variants/lib$v.so; fi
  KIFMM_LIB=$L timeout 300 python tools/config_times.py 1000000 "$C2" > gpurun_out/var.log 2>&1
  echo $v $(grep -h "evaluate\|p2p_mutual\|leaf_pass\|sweep m2l5" gpurun_out/var.log | head -6) >> gpurun_out/variants.log
done; done
cat gpurun_out/variants.log
cat gpurun_out/var.log
