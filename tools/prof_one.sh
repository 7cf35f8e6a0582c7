# One-BFS ncu capture (--set full) + per-level trace of the current build.
#   bash tools/prof_one.sh TAG [scale] [root_index]
R=${1:-x}; S=${2:-24}; I=${3:-0}
mkdir -p gpurun_out
timeout -k 10 300 python tools/ncu_one_bfs.py $S $I > gpurun_out/${R}_one.log 2>&1 || exit 1
timeout -k 10 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -c 80 \
    -o gpurun_out/${R}_full -f python tools/ncu_one_bfs.py $S $I > gpurun_out/${R}_full.log 2>&1 || echo "full rc=$?"
LBFS_TRACE=1 timeout -k 10 300 python tools/quick_bfs_time.py $S 3 > gpurun_out/${R}_trace_s$S.log 2>&1 || true
