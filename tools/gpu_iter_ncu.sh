# build, operator parity, bench (no DD), then ncu --set full of one kernel (KREGEX)
bash tools/gpu_iter.sh
python tools/prof_apply.py --config c5 --reps 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_zconv} -s 1 -c 1 \
    -o gpurun_out/prof_kc python tools/prof_apply.py --config c5 --reps 2 > gpurun_out/ncu_kc.log 2>&1
echo "ncu rc $?"
