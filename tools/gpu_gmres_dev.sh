# device-side Arnoldi: parity (solver tests) and A/B timing against the host-recurrence path
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
IE_GMRES_DEVICE=1 timeout 1200 python -m pytest tests/test_gpu_solve.py tests/test_gpu_layered.py tests/test_gpu_layered_physical.py tests/test_gpu_logging.py -x -q -k "not fullsize" > gpurun_out/pytest_solve.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_solve.log
for h in 1 0; do IE_GMRES_DEVICE=$h timeout 300 python tools/gmres_overhead.py c2mod c3h c4h c5 2>&1 | sed "s/^/DEVICE=$h /"; done
