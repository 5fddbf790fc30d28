# round profile captures: launch list of the bench command and ncu --set full of the hot kernels
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 3 --warmup 3 --no-dd --no-cpu-baseline --no-cufft --no-layered --no-sweep --no-window"
$CMD > gpurun_out/plain_bench.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc $?"
python tools/prof_apply.py --config c5 --reps 2 --gmres 12 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_(x|y|z)|k_mdot|k_maxpy' -s 5 -c 7 \
    -o gpurun_out/prof_full python tools/prof_apply.py --config c5 --reps 2 --gmres 12 > gpurun_out/ncu_full.log 2>&1
echo "full rc $?"
