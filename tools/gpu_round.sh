# Round evidence on one B200 (under gpurun): tests, smoke, both bench arms, profiles.
#   bash tools/gpu_round.sh r2b
R=${1:-r2}
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${R}_smi.txt
timeout -k 10 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$?"
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?"
timeout -k 10 600 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench rc=$?"
timeout -k 10 600 python bench.py --impl reference > gpurun_out/${R}_reference.json 2> gpurun_out/${R}_reference.err; echo "ref rc=$?"
bash tools/profile_round.sh ${R}; echo "prof rc=$?"
tail -3 gpurun_out/${R}_pytest.log; cat gpurun_out/${R}_smoke.log | tail -2; cat gpurun_out/${R}_bench.json
