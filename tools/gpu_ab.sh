# A/B env switches on the operator: parity with each switch on, then bench all (twice)
# usage: bash tools/gpu_ab.sh VAR=VALUE [VAR=VALUE ...]
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
for v in "$@"; do
  env $v timeout 600 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_ab.log 2>&1; echo "pytest ($v) rc $?"
  tail -3 gpurun_out/pytest_ab.log
done
for rep in 1 2; do
for v in "IE_NONE=0" "$@"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-dd --no-cpu-baseline --no-layered --no-sweep --no-window --no-cufft > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err
  echo "[$v]" $(python -c "import json; d=json.load(open('gpurun_out/bench_ab.json')); print(d['value'], d['ms_per_step'], {k: (v['ms'], v['gbs']) for k, v in d['kernels'].items()})")
done
done
