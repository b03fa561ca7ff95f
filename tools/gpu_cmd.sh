cd $GRAFT_REPO_ROOT
C2="dict(depth=5, order_equiv=4, backend='blas', precision='f32', sigma_min=1e-6)"
for i in 1 2 3; do timeout 300 python tools/config_times.py 1000000 "$C2" > gpurun_out/ms.log 2>&1; echo $(grep -h "evaluate" gpurun_out/ms.log | grep -o "evaluate [0-9.]* ms") >> gpurun_out/mss.log; done
timeout 300 python tools/config_times.py 1000000 "dict(depth=5, order_equiv=8, backend='fft', precision='f64')" signed > gpurun_out/ms_c3.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
KIFMM_OVERLAP=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "evaluate_matches" > gpurun_out/gpu_tests_seq.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests_seq.log
