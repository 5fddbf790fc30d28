# A/B two prebuilt libraries (build/lib_old.so, build/lib_new.so) on the layered operator
L=paper_2306_17537_b200/libie_b200.so
cp build/lib_new.so $L
timeout 900 python -m pytest tests/test_gpu_layered.py -q -x > gpurun_out/pytest_l.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_l.log
for rep in 1 2; do for v in old new; do cp build/lib_$v.so $L
  for a in "--config c3h --nrhs 3" "--config c3h --nrhs 1" "--config c4h --nrhs 3"; do
    echo "[$v] $a: $(timeout 300 python tools/bench_layered.py $a 2>&1 | tail -1 | cut -c1-200)"
  done
done; done
