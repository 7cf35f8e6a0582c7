mkdir -p gpurun_out
for F in 0 1 0 1; do
echo "FUSE_ALL=$F S24 $(LBFS_FUSE_ALL=$F timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1) S20 $(LBFS_FUSE_ALL=$F timeout 200 python tools/quick_bfs_time.py 20 64 2>&1 | tail -1)" >> gpurun_out/ab_fuse2.log
done
LBFS_FUSE_ALL=1 timeout 900 python -m pytest tests/test_gpu_traversal.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/ab_fuse2_pytest.log 2>&1
