cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mutual" > gpurun_out/r2_t3.log 2>&1
tail -3 gpurun_out/r2_t3.log
C2="dict(depth=5, order_equiv=4, backend='blas', precision='f32', sigma_min=1e-6)"
rm -f gpurun_out/variants.log
for i in 1 2; do for v in default mw2 mw4 direct; do
  if [ $v == default ] || [ $v == direct ]; then L=$PWD/paper_2408_07436_b200/libkifmm_b200.so; else L=$PWD/_variants/lib$v.so; fi
  P2P=mutual; [ $v == direct ] && P2P=direct
  KIFMM_LIB=$L KIFMM_P2P=$P2P timeout 300 python tools/config_times.py 1000000 "$C2" > gpurun_out/var.log 2>&1
  echo $v $(grep -h "evaluate\|p2p_mutual\|l2p_mutual\|leaf_pass" gpurun_out/var.log | head -4) >> gpurun_out/variants.log
done; done
cat gpurun_out/variants.log
