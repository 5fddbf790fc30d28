# A/B environment switches on the bench command itself (operator legs only), interleaved:
#   VARIANTS="IE_PDL=0 IE_PDL=1" bash tools/gpu_ab_bench.sh   (parity of the default first)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py -q -x -k "not fused" > gpurun_out/p_ab.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/p_ab.log
for rep in 1 2 3; do for v in ${VARIANTS:-IE_REV=0 IE_REV=1}; do
env ${v//,/ } timeout 300 python bench.py --steps 20 --warmup 5 --no-dd --no-cpu-baseline --no-layered --no-sweep --no-window --no-cufft 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d.get('operator_c4_grid') or {}
print('$v', d['ms_per_step'], {k.split()[0]:v['ms'] for k,v in d['kernels'].items()}, 'c4h', c.get('ms_per_apply'))"
done; done
