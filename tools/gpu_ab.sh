mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k s27 > gpurun_out/s27_test.log 2>&1; echo "rc=$?" >> gpurun_out/s27_test.log
timeout -k 10 900 python bench.py --scale 27 --steps 1 --warmup 3 > gpurun_out/s27_bench.json 2> gpurun_out/s27_bench.err; echo "rc=$?" >> gpurun_out/s27_bench.err
