mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_cp_pytest.log 2>&1
timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1 > gpurun_out/ab_cp.log
timeout 200 python tools/quick_bfs_time.py 20 64 2>&1 | tail -1 >> gpurun_out/ab_cp.log
WARM_S=0.3 LBFS_TRACE=1 timeout 200 python tools/quick_bfs_time.py 24 2 2>&1 | grep "L[0-9]" | grep -o "L[0-9].\{8\}\|compact=.\{8\}" | paste - - >> gpurun_out/ab_cp.log
