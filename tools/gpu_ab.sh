mkdir -p gpurun_out
rm -f gpurun_out/ab_stab.log
for i in $(seq 1 30); do
  echo "nofuse run$i $(timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1)" >> gpurun_out/ab_stab.log
done
