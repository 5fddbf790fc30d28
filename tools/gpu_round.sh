# full GPU test suite (incl. slow full-size c5 parity), smoke, default bench, launch list
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke.log
timeout 1800 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; tail -3 gpurun_out/bench.err
