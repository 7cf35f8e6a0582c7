mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/cl_pytest.log 2>&1
timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1 > gpurun_out/cl.log
