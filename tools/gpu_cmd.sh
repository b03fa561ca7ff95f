cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mutual or out_of_bounds or fresh or evaluate_matches" > gpurun_out/r2_t11.log 2>&1; tail -3 gpurun_out/r2_t11.log
timeout 300 python tools/launch_times.py > gpurun_out/launches_c2.log 2>&1; grep -E "p2p|l2p|m2l5" gpurun_out/launches_c2.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-config3 > gpurun_out/r2_bench11.json 2> gpurun_out/r2_bench11.err
python -c "import json;d=json.loads(open('gpurun_out/r2_bench11.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['e2e']['pageable_value'],d['roofline']['frac'],d['roofline_all']['p2p_mutual_f32']['frac'])"
