mkdir -p gpurun_out
rm -f gpurun_out/ab_qrs.log
V=paper_1604_02844_b200/_native/variants/qrs.so
LBFS_LIB=$V timeout 900 python -m pytest tests/test_gpu_traversal.py tests/test_gpu_configs.py tests/test_gpu_direction.py -m gpu -x -q > gpurun_out/ab_qrs_pytest.log 2>&1
for L in "" $V "" $V; do
echo "LIB=$L S24 $(LBFS_LIB=$L timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1) S20 $(LBFS_LIB=$L timeout 200 python tools/quick_bfs_time.py 20 64 2>&1 | tail -1) LAT $(LBFS_LIB=$L timeout 200 python tools/quick_lattice_time.py 4096 1 2>&1 | tail -1)" >> gpurun_out/ab_qrs.log
done
