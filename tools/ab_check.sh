# correctness A/B: tools/debug_runs.py on each variant .so (default = in-tree build)
S=${S:-12}
for V in default "$@"; do
  if [ "$V" = default ]; then L=""; else L=paper_1604_02844_b200/_native/variants/$V.so; fi
  echo "VARIANT=$V"; LBFS_LIB=$L timeout 100 python tools/debug_runs.py $S 2>&1 | grep -E "bad|Error" | head -3
done
