L=paper_2306_17537_b200/libie_b200.so
cp build/lib_new.so $L
timeout 900 python -m pytest tests/test_gpu_operator.py -q -x -k "not variants" > gpurun_out/pytest_v.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_v.log
for rep in 1 2 3; do for v in old new; do cp build/lib_$v.so $L; for a in "--config c5" "--config c4h"; do echo "[$v] $a: $(timeout 300 python tools/time_apply.py $a 2>&1 | tail -1)"; done; done; done
