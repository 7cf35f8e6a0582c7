mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_direction.py -x -q > gpurun_out/do_pytest.log 2>&1
LBFS_DIRECTION=1 timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1 > gpurun_out/do.log
LBFS_DIRECTION=1 timeout 200 python tools/quick_bfs_time.py 20 64 2>&1 | tail -1 >> gpurun_out/do.log
LBFS_DIRECTION=1 WARM_S=0.3 LBFS_TRACE=1 timeout 200 python tools/quick_bfs_time.py 24 2 2>&1 | grep "L[0-9]\|root" | cut -c1-200 >> gpurun_out/do.log
LBFS_DIRECTION=1 timeout 300 python tools/quick_lattice_time.py 4096 2 2>&1 | tail -1 >> gpurun_out/do.log
