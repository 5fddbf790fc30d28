# layered K-C' parity sweep and timing for each prebuilt library build/lib_<name>.so
for f in build/lib_*.so; do cp $f paper_2306_17537_b200/libie_b200.so; echo "== $f"; python tools/layered_diag.py 2>&1 | grep "64) 1\|64) 3\|128) 1"
  for a in "--config c3h --nrhs 1" "--config c3h --nrhs 3"; do echo "$a: $(timeout 300 python tools/bench_layered.py $a 2>&1 | tail -1 | cut -c1-100)"; done; done
