# A/B of env settings on S24 and S20 (quick_bfs_time harmonic means)
for cfg in "$@"; do echo "== $cfg"; env $cfg python tools/quick_bfs_time.py 24 16 | tail -1; env $cfg python tools/quick_bfs_time.py 20 16 | tail -1; done
