# A/B IE_REV on the bench command itself (operator leg only), interleaved
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2 3; do for v in 0 1; do
IE_REV=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-dd --no-cpu-baseline --no-layered --no-sweep --no-window --no-cufft 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('IE_REV=$v', d['ms_per_step'], {k.split()[0]:v['ms'] for k,v in d['kernels'].items()})"
done; done
