mkdir -p gpurun_out
timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1 > gpurun_out/ab_fq.log
timeout 200 python tools/quick_bfs_time.py 20 64 2>&1 | tail -1 >> gpurun_out/ab_fq.log
WARM_S=0.3 LBFS_GAPS=1 timeout 200 python tools/quick_bfs_time.py 24 8 2>&1 | tail -9 | cut -c1-150 >> gpurun_out/ab_fq.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_fq_pytest.log 2>&1
