# HEAD validation on one B200: GPU tests, smoke, default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/h1_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/h1_tests.txt 2>&1; tail -5 gpurun_out/h1_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h1_smoke.txt 2>&1; tail -2 gpurun_out/h1_smoke.txt
timeout 600 python bench.py > gpurun_out/h1_bench.json 2> gpurun_out/h1_bench.err; tail -c 600 gpurun_out/h1_bench.json
