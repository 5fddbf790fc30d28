# A/B two prebuilt libraries (build/lib_old.so, build/lib_new.so) on the bench's per-kernel table
L=paper_2306_17537_b200/libie_b200.so
for rep in 1 2; do for v in old new; do cp build/lib_$v.so $L
timeout 300 python bench.py --steps 20 --warmup 5 --no-dd --no-cpu-baseline --no-layered --no-sweep --no-window --no-cufft > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err
echo "[$v]" $(python -c "import json; d=json.load(open('gpurun_out/bench_ab.json')); print(d['value'], d['ms_per_step'], {k: (v['ms'], v['gbs']) for k, v in d['kernels'].items()})")
done; done
