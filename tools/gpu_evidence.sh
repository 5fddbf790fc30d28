# round-2 evidence: reference arm, launch list of the bench command, ncu of K-C' on the physical c3 table
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-dd --no-layered --no-sweep --no-window --no-cpu-baseline --no-cufft > gpurun_out/ncu_launch.log 2>&1; echo "launch rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_zlayer_tma -c 1 -o gpurun_out/ncu_kcprime_c3phys python tools/layered_physical.py --what op > gpurun_out/ncu_kcprime.log 2>&1; echo "kcprime rc $?"
timeout 600 python -m pytest tests/test_gpu_solve.py -q -k "device_side or warm_start" > gpurun_out/pytest_dev.log 2>&1; echo "pytest_dev rc $?"; tail -2 gpurun_out/pytest_dev.log
