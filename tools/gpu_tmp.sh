L=paper_2306_17537_b200/libie_b200.so
cp build/lib_new.so $L
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x > gpurun_out/pytest_v.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_v.log
for rep in 1 2; do for v in old new; do cp build/lib_$v.so $L; echo "[$v]"; python tools/gmres_overhead.py c5 c4h c3h; done; done
