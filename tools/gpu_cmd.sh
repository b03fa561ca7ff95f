cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest7.log 2>&1; tail -3 gpurun_out/r2_gputest7.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench7.json 2> gpurun_out/r2_bench7.err
python -c "import json;d=json.loads(open('gpurun_out/r2_bench7.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e'],d['roofline']['frac']);print(d['kernel_ms'])"
