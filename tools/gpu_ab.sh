set -x
mkdir -p gpurun_out
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1k_smoke.log 2>&1; echo "smoke rc=$?"
timeout -k 10 600 python bench.py > gpurun_out/r1k_bench.json 2> gpurun_out/r1k_bench.err; echo "bench rc=$?"
timeout -k 10 600 python bench.py --impl reference > gpurun_out/r1k_reference.json 2> gpurun_out/r1k_reference.err; echo "ref rc=$?"
bash tools/profile_round.sh r1k; echo "prof rc=$?"
