# A/B: S24 harmonic-mean GTEPS of the default build and each variant .so given
for V in default "$@"; do
  if [ "$V" = default ]; then L=""; else L=paper_1604_02844_b200/_native/variants/$V.so; fi
  echo "VARIANT=$V"; LBFS_LIB=$L timeout 200 python tools/quick_bfs_time.py 24 8 2>&1 | tail -1
done
