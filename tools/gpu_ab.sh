mkdir -p gpurun_out
for V in default c8 c32 default c8; do
  if [ "$V" = default ]; then L=""; else L=paper_1604_02844_b200/_native/variants/$V.so; fi
  echo "VARIANT=$V $(LBFS_LIB=$L timeout 200 python tools/quick_bfs_time.py 24 64 2>&1 | tail -1)" >> gpurun_out/ab_cons.log
  LBFS_LIB=$L WARM_S=0.3 LBFS_TRACE=1 LBFS_SPLIT=1 timeout 200 python tools/quick_bfs_time.py 24 2 2>&1 | grep -B1 "sweep " | grep split | cut -c1-40 >> gpurun_out/ab_cons.log
done
