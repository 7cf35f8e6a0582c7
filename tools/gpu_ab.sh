mkdir -p gpurun_out
timeout -k 10 900 python bench.py --partitioned --steps 1 --warmup 1 > gpurun_out/part_bench.json 2> gpurun_out/part_bench.err; echo "rc=$?" >> gpurun_out/part_bench.err
