mkdir -p gpurun_out
rm -f gpurun_out/ab_dense3.log
for M in 2097152 4194304 8388608; do
echo "MIN=$M S20 $(LBFS_DENSE_MIN=$M timeout 200 python tools/quick_bfs_time.py 20 64 2>&1 | tail -1) S22 $(LBFS_DENSE_MIN=$M timeout 200 python tools/quick_bfs_time.py 22 64 2>&1 | tail -1)" >> gpurun_out/ab_dense3.log
done
