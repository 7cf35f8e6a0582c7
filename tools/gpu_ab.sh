mkdir -p gpurun_out
rm -f gpurun_out/ab_spec.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_spec_pytest.log 2>&1
for S in 1 0 1 0; do
echo "SPEC=$S S24 $(LBFS_SPEC_FINALIZE=$S timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1) S20 $(LBFS_SPEC_FINALIZE=$S timeout 200 python tools/quick_bfs_time.py 20 64 2>&1 | tail -1)" >> gpurun_out/ab_spec.log
done
