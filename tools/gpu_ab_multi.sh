# A/B several environment settings on operator timing, interleaved:
#   VARIANTS="IE_KC_FMA=0 IE_KC_FMA=1" CONFIGS="c5 c4h" bash tools/gpu_ab_multi.sh   (parity first)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py -q -x -k "not fused" > gpurun_out/p_ab.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/p_ab.log
for rep in 1 2 3; do
  for cfg in ${CONFIGS:-c5 c4h}; do
    for v in $VARIANTS; do
      env ${v//,/ } timeout 120 python tools/time_apply.py --config $cfg --steps 60 --kernels 2>&1 | sed "s/^/$v /"
    done
  done
done
