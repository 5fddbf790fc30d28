python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
for rep in 1 2; do
for v in "IE_NONE=0" "IE_KNOB=5"; do echo "[$v] $(env $v python tools/time_apply.py --config c4h | tail -1)"; echo "[$v] $(env $v python tools/time_apply.py --config c4h --nrhs 3 | tail -1)"; echo "[$v] $(env $v python tools/time_apply.py --config c3h | tail -1)"; done
echo "[c5] $(python tools/time_apply.py --config c5 | tail -1)"
done
