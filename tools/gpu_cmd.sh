# scratch command file for gpurun calls (tools/gpu_cmd.sh); overwritten per experiment
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mutual or evaluate_matches or graph_replay or degenerate or deterministic or separate" > gpurun_out/r2_t3.log 2>&1
tail -5 gpurun_out/r2_t3.log
C2="dict(depth=5, order_equiv=4, backend='blas', precision='f32', sigma_min=1e-6)"
for i in 1 2; do for v in default taillin; do
  if [ $v == default ]; then L=$PWD/paper_2408_07436_b200/libkifmm_b200.so; else L=$PWD/_variants/lib$v.so; fi
  KIFMM_LIB=$L timeout 300 python tools/config_times.py 1000000 "$C2" > gpurun_out/var.log 2>&1
  echo $v $(grep -h "evaluate\|m2l5:m2l_sweep\|p2p_mutual\|l2p_mutual\|leaf_pass" gpurun_out/var.log | head -6) >> gpurun_out/variants.log
done; done
cat gpurun_out/var.log
KIFMM_P2P=direct timeout 300 python tools/config_times.py 1000000 "$C2" > gpurun_out/var_direct.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err
python -c "import json;d=json.loads(open('gpurun_out/r2_bench2.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['kernel_ms'])"
