# build, fused-pass parity, A/B timing of the fused passes (c5, c4h), short bench line
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_op.log 2>&1; echo "pytest_op rc $?"
tail -3 gpurun_out/pytest_op.log
for cfg in c5 c4h; do
  for ab in 1 0; do for de in 1 0; do
    IE_FUSED_AB=$ab IE_FUSED_DE=$de timeout 120 python tools/time_apply.py --config $cfg --steps 30 2>&1 | sed "s/^/AB=$ab DE=$de /"
  done; done
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-dd --no-cpu-baseline --no-layered --no-sweep --no-window > gpurun_out/bench_nodd.json 2> gpurun_out/bench_nodd.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_nodd.json')); print(d['value'], d['ms_per_step'], d['frac_of_hbm_peak'], {k: (v['ms'], v['gbs']) for k, v in d['kernels'].items()})"
