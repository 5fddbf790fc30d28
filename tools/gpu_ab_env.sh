# A/B an environment switch on operator timing: VAR=IE_KC_PIPE bash tools/gpu_ab_env.sh (parity first)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py -q -x -k "not fused" > gpurun_out/p_ab.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/p_ab.log
for rep in 1 2 3; do
  for cfg in c5 c4h; do
    for v in 1 0; do
      env ${VAR:-IE_KC_PIPE}=$v timeout 120 python tools/time_apply.py --config $cfg --steps 40 2>&1 | sed "s/^/${VAR:-IE_KC_PIPE}=$v /"
    done
  done
done
