# build + the operator/fullsize/solve GPU tests (a faster subset of tools/gpu_tests.sh)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py tests/test_gpu_solve.py -q -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_q.log
