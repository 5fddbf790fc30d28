# timing probe (results wrong by design): K-B writing / K-D reading its tile contiguously (IE_PROBE=2/4)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
for rep in 1 2 3; do
  for v in 0 2 4 6; do
    IE_PROBE=$v timeout 120 python tools/time_apply.py --config ${CFG:-c5} --steps 60 --kernels 2>&1 | grep K-A | sed "s/^/IE_PROBE=$v /"
  done
done
