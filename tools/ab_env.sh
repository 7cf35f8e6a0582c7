# A/B of env settings (one per line in $1, "-" = defaults) on S24 / S20, 16 roots each.
#   bash tools/ab_env.sh tools/ab_list.txt > gpurun_out/ab.log
while IFS= read -r cfg; do
  [ -z "$cfg" ] && continue
  [ "$cfg" = "-" ] && cfg="LBFS_AB_BASE=1"
  echo "== $cfg"
  for s in 24 20; do
    echo -n "S$s: "; env $cfg timeout -k 5 200 python tools/quick_bfs_time.py $s ${NROOTS:-16} 2>&1 | tail -1
  done
done < "$1"
