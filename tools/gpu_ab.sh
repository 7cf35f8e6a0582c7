mkdir -p gpurun_out
rm -f gpurun_out/ab_init.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_init_pytest.log 2>&1
for i in 1 2 3; do
echo "S24 $(timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1) S20 $(timeout 200 python tools/quick_bfs_time.py 20 64 2>&1 | tail -1)" >> gpurun_out/ab_init.log
done
