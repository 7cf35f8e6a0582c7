mkdir -p gpurun_out
rm -f gpurun_out/ab_fold.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_fold_pytest.log 2>&1
for F in 1 0 1 0; do
echo "FOLD=$F S24 $(LBFS_FOLD_PUBLISH=$F timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1) S20 $(LBFS_FOLD_PUBLISH=$F timeout 200 python tools/quick_bfs_time.py 20 64 2>&1 | tail -1)" >> gpurun_out/ab_fold.log
done
