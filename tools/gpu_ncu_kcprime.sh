# ncu --set full of the layered K-C' kernel (c3h, 3 RHS, degenerate table), after a plain run exits 0
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
python tools/bench_layered.py --config c3h --nrhs 3 > gpurun_out/plain_l.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_zlayer -s 2 -c 1 \
    -o gpurun_out/prof_kcp python tools/bench_layered.py --config c3h --nrhs 3 --steps 2 > gpurun_out/ncu_kcp.log 2>&1
echo "ncu rc $?"
