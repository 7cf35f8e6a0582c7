# LBFS_REFRESH sweep on S24 (hub chunks of warp 0 between snapshot refreshes)
for R in ${@:-1 2 3 4}; do echo "REFRESH=$R"; LBFS_REFRESH=$R timeout 200 python tools/quick_bfs_time.py 24 8 2>&1 | tail -1; done
