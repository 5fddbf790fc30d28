python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py -q -x -k "not variants" > gpurun_out/pytest_v.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_v.log
for rep in 1 2 3; do for v in "IE_KC_VARIANT=7" "IE_NONE=0"; do echo "[$v] $(env $v python tools/time_apply.py --config c5 | tail -1)"; done; echo "[c4h] $(python tools/time_apply.py --config c4h | tail -1)"; done
