cd $GRAFT_REPO_ROOT
C2="dict(depth=5, order_equiv=4, backend='blas', precision='f32', sigma_min=1e-6)"
for i in 1 2; do timeout 300 python tools/config_times.py 1000000 "$C2" > gpurun_out/pc.log 2>&1; grep -h "evaluate\|p2m_check\|dense_split" gpurun_out/pc.log | head -3 >> gpurun_out/pcs.log; done
timeout 600 python tools/stress_tmem.py 11 8 > gpurun_out/stress.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
