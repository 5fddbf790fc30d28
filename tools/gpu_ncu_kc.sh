# ncu --set full of the K-C kernel under the given env switch (c5)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
env $1 python tools/prof_apply.py --config c5 --reps 2 > gpurun_out/plain.log 2>&1 || { echo "plain failed"; exit 1; }
env $1 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_zconv} -s 1 -c 1 \
    -o gpurun_out/prof_kc python tools/prof_apply.py --config c5 --reps 2 > gpurun_out/ncu_kc.log 2>&1
echo "ncu rc $?"
