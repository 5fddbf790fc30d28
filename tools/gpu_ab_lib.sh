# A/B two builds of the library: the in-tree build (B) against the same sources compiled with
# DEFS (A), e.g.  DEFS="-DIE_FMA8=0" bash tools/gpu_ab_lib.sh   (parity of the in-tree build first)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
mkdir -p /tmp/ablib && rm -f /tmp/ablib/*.o
for s in operator green layered fields krylov api; do
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC $DEFS \
    -c paper_2306_17537_b200/csrc/$s.cu -o /tmp/ablib/$s.o &
done; wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a /tmp/ablib/*.o -o /tmp/ablib/libA.so -lcudart || exit 1
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py -q -x -k "not fused" > gpurun_out/p_ab.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/p_ab.log
for rep in 1 2 3; do
  for cfg in ${CONFIGS:-c5 c4h}; do
    IE_LIB_PATH=/tmp/ablib/libA.so timeout 120 python tools/time_apply.py --config $cfg --steps 60 --kernels 2>&1 | sed "s/^/A /"
    timeout 120 python tools/time_apply.py --config $cfg --steps 60 --kernels 2>&1 | sed "s/^/B /"
  done
done
