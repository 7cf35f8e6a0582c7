set -x
mkdir -p gpurun_out
timeout -k 10 1500 python -m pytest tests -m gpu -q > gpurun_out/r1h_pytest.log 2>&1; echo "pytest rc=$?"
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1h_smoke.log 2>&1; echo "smoke rc=$?"
timeout -k 10 600 python bench.py > gpurun_out/r1h_bench.json 2> gpurun_out/r1h_bench.err; echo "bench rc=$?"
timeout -k 10 600 python bench.py --impl reference > gpurun_out/r1h_reference.json 2> gpurun_out/r1h_reference.err; echo "ref rc=$?"
bash tools/profile_round.sh r1h; echo "prof rc=$?"
