# A/B two prebuilt libraries (build/lib_old.so, build/lib_new.so) on time_apply for several configs
L=paper_2306_17537_b200/libie_b200.so
for rep in 1 2; do
for v in old new; do
  cp build/lib_$v.so $L
  for a in "$@"; do
    echo "[$v] $a: $(timeout 300 python tools/time_apply.py $a 2>&1 | tail -1)"
  done
done
done
