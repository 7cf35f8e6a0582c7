mkdir -p gpurun_out
WARM_S=0.5 LBFS_GAPS=1 timeout 200 python tools/quick_bfs_time.py 20 6 2>&1 | tail -13 > gpurun_out/s20_gaps.log
WARM_S=0.5 LBFS_TRACE=1 LBFS_SPLIT=1 timeout 200 python tools/quick_bfs_time.py 20 2 2>&1 | grep -v "^\[lbfs\]      split" | tail -20 >> gpurun_out/s20_gaps.log
