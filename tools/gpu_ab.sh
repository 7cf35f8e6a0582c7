mkdir -p gpurun_out
WARM_S=0 timeout -k 10 900 ncu --set full --clock-control none -k regex:"k_levels|k_init|k_finalize" -c 6 -o gpurun_out/r1i_lattice python tools/quick_lattice_time.py 4096 1 > gpurun_out/r1i_lattice.log 2>&1
WARM_S=0 timeout -k 10 900 ncu --set full --clock-control none -k regex:"k_expand|k_compact|k_sweep|k_merge|k_levels|k_resolve|k_finalize|k_init" -c 40 -o gpurun_out/r1i_s20 python tools/quick_bfs_time.py 20 1 > gpurun_out/r1i_s20.log 2>&1
