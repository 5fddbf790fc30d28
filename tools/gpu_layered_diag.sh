# layered K-C' parity sweep (tools/layered_diag.py) on the current build and, if present, build/lib_old.so
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
echo "== current"; python tools/layered_diag.py 2>&1 | tail -12
if [ -f build/lib_old.so ]; then cp build/lib_old.so paper_2306_17537_b200/libie_b200.so; echo "== old"; python tools/layered_diag.py 2>&1 | tail -12; fi
