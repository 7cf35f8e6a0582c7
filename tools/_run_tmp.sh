bash tools/ab_env.sh tools/ab_list.txt > gpurun_out/ab4.log 2>&1; cat gpurun_out/ab4.log
for v in "" dbg1 dbg2 dbg3 dbg4 dbg7; do
  echo "== sweep variant [$v]"
  if [ -n "$v" ]; then export LBFS_LIB=paper_1604_02844_b200/_native/variants/$v.so; fi
  LBFS_TRACE=1 timeout 200 python tools/quick_bfs_time.py 24 3 2>&1 | grep "sweep" | head -3 | cut -c1-60,150-260
done
