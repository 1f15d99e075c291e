# HEAD, 1 GPU: what the driver runs at round end (GPU tests, smoke, default bench)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/hf_tests.txt 2>&1; tail -1 gpurun_out/hf_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/hf_bench.json 2> gpurun_out/hf_bench.err; tail -c 300 gpurun_out/hf_bench.json
