# round-end validation: full GPU suite, smoke, default bench, then the launch list of the bench command
bash tools/gpu_round.sh
CMD="python bench.py --steps 3 --warmup 3 --no-dd --no-cpu-baseline --no-cufft --no-layered --no-sweep --no-window"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc $?"
