# quick GPU iteration: build, operator parity, bench without DD legs
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
timeout 600 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_op.log 2>&1; echo "pytest_op rc $?"
tail -3 gpurun_out/pytest_op.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-dd --no-cpu-baseline --no-layered --no-sweep --no-window > gpurun_out/bench_nodd.json 2> gpurun_out/bench_nodd.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_nodd.json')); print(d['value'], d['ms_per_step'], d.get('cufft_reference'), {k: (v['ms'], v['gbs']) for k, v in d['kernels'].items()})"
