mkdir -p gpurun_out
LBFS_PART_HEAVY=1 timeout -k 10 600 python bench.py --partitioned --steps 1 --warmup 1 --e2e-roots 2 --no-cpu-baseline > gpurun_out/ph_b1.json 2> gpurun_out/ph_b1.err; echo "rc=$?" >> gpurun_out/ph_b1.err
