cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest9.log 2>&1; tail -3 gpurun_out/r2_gputest9.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench9.json 2> gpurun_out/r2_bench9.err
python -c "import json;d=json.loads(open('gpurun_out/r2_bench9.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e'],d['roofline']['frac'],d['roofline_all']['p2p_mutual_f32']['frac']);print(d['configs']['c3']['parity'])"
