#!/bin/bash
# Profiling evidence for profiles/ (run under gpurun, one GPU):
#  1. plain bench run (must exit 0 before ncu touches the same command)
#  2. launch list: every kernel's device time (cold-cache, serialised)
#  3. one --set full capture of every kernel of one S24 BFS (tools/ncu_one_bfs.py)
#  4. per-level traces (LBFS_TRACE=1) of S24 / S20
set -e
R=${1:-r2}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra-configs"
timeout -k 10 600 $CMD > gpurun_out/${R}_plain.json 2> gpurun_out/${R}_plain.err
timeout -k 10 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_launches.log 2>&1 || echo "launch list rc=$?"
timeout -k 10 300 python tools/ncu_one_bfs.py 24 0 > gpurun_out/${R}_one.log 2>&1
timeout -k 10 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -c 80 \
    -o gpurun_out/${R}_full -f python tools/ncu_one_bfs.py 24 0 > gpurun_out/${R}_full.log 2>&1 || echo "full rc=$?"
LBFS_TRACE=1 timeout -k 10 300 python tools/quick_bfs_time.py 24 3 > gpurun_out/${R}_trace_s24.log 2>&1 || true
LBFS_TRACE=1 timeout -k 10 300 python tools/quick_bfs_time.py 20 3 > gpurun_out/${R}_trace_s20.log 2>&1 || true
echo done
