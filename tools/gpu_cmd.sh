cd $GRAFT_REPO_ROOT
timeout 300 python tools/bench_gemm.py > gpurun_out/bench_gemm.log 2>&1
KIFMM_GEMM_TS=0 timeout 300 python tools/bench_gemm.py > gpurun_out/bench_gemm_old.log 2>&1
C2="dict(depth=5, order_equiv=4, backend='blas', precision='f32', sigma_min=1e-6)"
timeout 300 python tools/config_times.py 1000000 "$C2" > gpurun_out/c2_gemm.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
