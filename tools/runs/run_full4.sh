timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/gpu_tests_full.txt 2>&1; tail -15 gpurun_out/gpu_tests_full.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 1500 gpurun_out/bench_default.json
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
