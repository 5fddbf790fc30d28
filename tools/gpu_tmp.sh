python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x -k "tall" > gpurun_out/pytest_v.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_v.log
