# time the reference evaluate (c2) under several thread policies
for pol in "OMP_WAIT_POLICY=PASSIVE OPENBLAS_NUM_THREADS=1" "OMP_WAIT_POLICY=ACTIVE OPENBLAS_NUM_THREADS=1" "OMP_WAIT_POLICY=ACTIVE" "OPENBLAS_NUM_THREADS=1"; do
  echo "== $pol"; env $pol timeout 300 python -c "
import os, sys, time; sys.path.insert(0, '.')
import bench
pts, q = bench.inputs()
r = bench.cpu_reference_run(pts, q, steps=2, warmup=1)
print('best', min(r['times']), {k: round(v, 3) for k, v in r['timings'].items()})
" 2>&1 | tail -1; done
