mkdir -p gpurun_out
echo "NCCL_DEBUG=$NCCL_DEBUG" > gpurun_out/ph_env.txt
timeout -k 10 600 python bench.py --partitioned --steps 1 --warmup 1 --e2e-roots 2 --no-cpu-baseline > gpurun_out/ph_b2.json 2> gpurun_out/ph_b2.err; echo "rc=$?" >> gpurun_out/ph_b2.err
NCCL_DEBUG=INFO timeout -k 10 600 python bench.py --partitioned --steps 1 --warmup 1 --e2e-roots 2 --no-cpu-baseline > gpurun_out/ph_b3.json 2> gpurun_out/ph_b3.err; echo "rc=$?" >> gpurun_out/ph_b3.err
