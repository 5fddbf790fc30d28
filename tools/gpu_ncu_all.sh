# ncu --set full of all five operator kernels of one c5 application (after a plain run exits 0)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
python tools/prof_apply.py --config c5 --reps 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_(x|y|z)' -s 5 -c 5 \
    -o gpurun_out/prof_all python tools/prof_apply.py --config c5 --reps 2 > gpurun_out/ncu_all.log 2>&1
echo "ncu rc $?"
