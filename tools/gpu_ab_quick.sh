# A/B environment settings on operator timing without the parity run (use gpu_ab_multi.sh before keeping one):
#   VARIANTS="IE_YHINT=0 IE_YHINT=3" CONFIGS="c5 c4h" REPS=3 bash tools/gpu_ab_quick.sh
for rep in $(seq 1 ${REPS:-3}); do
  for cfg in ${CONFIGS:-c5 c4h}; do
    for v in $VARIANTS; do
      env ${v//,/ } timeout 120 python tools/time_apply.py --config $cfg --steps 60 --kernels 2>&1 | grep -v "ms/apply" | sed "s/^/$v /"
    done
  done
done
