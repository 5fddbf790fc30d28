python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_layered.py -q -x > gpurun_out/pytest_l.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_l.log
