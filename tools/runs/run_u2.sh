# 1 GPU: two-shot with 2 packets per lane for NR > 4 -- parity (virtual tests) and bench N=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x --timeout 600 -k "all_reduce or wrap or graph or smoke" > gpurun_out/u2_tests.txt 2>&1; tail -1 gpurun_out/u2_tests.txt
for i in 1 2; do
timeout 600 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 2 > gpurun_out/u2_n1.json 2> gpurun_out/u2_n1.err; python -c "import json; d=json.loads(open('gpurun_out/u2_n1.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['step_ms_min'], d['step_ms_median'])"
done
