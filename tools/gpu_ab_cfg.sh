# A/B an env switch on time_apply for several configs (after operator parity with the switch on)
# usage: bash tools/gpu_ab_cfg.sh VAR=VALUE "cfg args" ["cfg args" ...]
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
SW=$1; shift
env $SW timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py -q -x -k "not variants" > gpurun_out/pytest_ab.log 2>&1; echo "pytest ($SW) rc $?"; tail -2 gpurun_out/pytest_ab.log
for rep in 1 2; do for v in "IE_NONE=0" "$SW"; do for a in "$@"; do
  echo "[$v] $a: $(env $v timeout 300 python tools/time_apply.py $a 2>&1 | tail -1)"
done; done; done
