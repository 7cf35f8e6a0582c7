mkdir -p gpurun_out
rm -f gpurun_out/chk.log
V=paper_1604_02844_b200/_native/variants/chk.so
LBFS_LIB=$V timeout 900 python -m pytest tests/test_gpu_traversal.py tests/test_gpu_configs.py tests/test_gpu_direction.py tests/test_distributed.py -m gpu -x -q > gpurun_out/chk_pytest.log 2>&1
for i in $(seq 1 10); do
  echo "HQ run$i $(LBFS_LIB=$V LBFS_FUSE_HQ=1 timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | grep -v '^root' | tail -3 | tr '\n' ' ')" >> gpurun_out/chk.log
done
for i in $(seq 1 6); do
  echo "ALL run$i $(LBFS_LIB=$V LBFS_FUSE_ALL=1 timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | grep -v '^root' | tail -3 | tr '\n' ' ')" >> gpurun_out/chk.log
done
