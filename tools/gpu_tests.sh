# build + the GPU test suite (optionally a subset: TESTS="tests/test_gpu_layered.py")
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest ${TESTS:-tests} -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -30 gpurun_out/pytest_gpu.log
