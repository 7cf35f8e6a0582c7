#!/bin/bash
# Profiling evidence for profiles/ (run under gpurun, one GPU):
#  1. plain bench run (must exit 0 before ncu touches the same command)
#  2. launch list: every kernel's device time (cold-cache, serialised)
#  3. one --set full capture of the expansion + compaction kernels of one BFS
set -e
R=${1:-r1}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --e2e-roots 2 --no-cpu-baseline"
timeout -k 10 600 $CMD > gpurun_out/${R}_plain.json 2> gpurun_out/${R}_plain.err
timeout -k 10 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_launches.log 2>&1
WARM_S=0 timeout -k 10 120 python tools/quick_bfs_time.py 24 1 > gpurun_out/${R}_one.log 2>&1
WARM_S=0 timeout -k 10 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"k_expand|k_compact|k_sweep|k_merge|k_levels|k_resolve|k_finalize|k_init" -c 40 \
    -o gpurun_out/${R}_full python tools/quick_bfs_time.py 24 1 \
    > gpurun_out/${R}_full.log 2>&1
echo done
