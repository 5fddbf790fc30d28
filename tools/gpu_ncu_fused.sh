python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
IE_FUSED_AB=0 IE_FUSED_DE=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_yxinv -c 1 -o gpurun_out/ncu_kde_c5 python tools/time_apply.py --config c5 --steps 2 > gpurun_out/ncu_kde.log 2>&1; echo ncu1 $?
