cd $GRAFT_REPO_ROOT
echo "ns2dbg fresh overlap0"; KIFMM_OVERLAP=0 KIFMM_LIB=$PWD/_variants/libns2dbg.so timeout 900 python tools/stress_overlap.py 40 1 > gpurun_out/stress_a.log 2>&1; grep -v "CUDAEvent.h\|^frame" gpurun_out/stress_a.log | grep -E "mismatch|reps|Error|stuck" | head
echo "ns4dbg fresh overlap0"; KIFMM_OVERLAP=0 KIFMM_LIB=$PWD/_variants/libns4dbg.so timeout 900 python tools/stress_overlap.py 60 1 > gpurun_out/stress_b.log 2>&1; grep -v "CUDAEvent.h\|^frame" gpurun_out/stress_b.log | grep -E "mismatch|reps|Error|stuck" | head
echo "default fresh"; timeout 900 python tools/stress_overlap.py 80 1 > gpurun_out/stress_c.log 2>&1; grep -v "CUDAEvent.h\|^frame" gpurun_out/stress_c.log | grep -E "mismatch|reps|Error|stuck" | head
