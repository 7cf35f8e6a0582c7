set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1c_smi.txt
timeout -k 10 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1c_pytest.log 2>&1; echo "pytest rc=$?"
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1c_smoke.log 2>&1; echo "smoke rc=$?"
timeout -k 10 600 python bench.py > gpurun_out/r1c_bench.json 2> gpurun_out/r1c_bench.err; echo "bench rc=$?"
timeout -k 10 600 python bench.py --impl reference > gpurun_out/r1c_reference.json 2> gpurun_out/r1c_reference.err; echo "ref rc=$?"
bash tools/profile_round.sh r1c; echo "prof rc=$?"
