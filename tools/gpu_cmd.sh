cd $GRAFT_REPO_ROOT
C2="dict(depth=5, order_equiv=4, backend='blas', precision='f32', sigma_min=1e-6)"
timeout 300 python tools/config_times.py 1000000 "$C2" > gpurun_out/c2_v3.log 2>&1
timeout 900 python tools/stress_tmem.py 5 20 > gpurun_out/stress5.log 2>&1
timeout 900 python tools/stress_tmem.py 6 20 > gpurun_out/stress6.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
