# build + fused A/B timing only (parity: tools/gpu_fused.sh)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k fused > gpurun_out/pytest_fused.log 2>&1; echo "pytest_fused rc $?"; tail -2 gpurun_out/pytest_fused.log
for cfg in c5 c4h c3h; do
  for ab in 1 0; do for de in 1 0; do
    IE_FUSED_AB=$ab IE_FUSED_DE=$de timeout 120 python tools/time_apply.py --config $cfg --steps 30 2>&1 | sed "s/^/AB=$ab DE=$de /"
  done; done
done
