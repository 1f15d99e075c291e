# 1 GPU, final state: GPU tests, smoke, default bench, ncu launch list + ncu --set full of the bench's dominant kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/z_tests.txt 2>&1; tail -1 gpurun_out/z_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err; python -c "import json; d=json.loads(open('gpurun_out/z_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'])"
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z_launches.csv $CMD > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/z_launches.csv "# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised): $CMD" > gpurun_out/z_launches.txt; head -6 gpurun_out/z_launches.txt
ncu --set full --clock-control none --import-source on -k regex:ar_twoshot_dyn -s 3 -c 1 -o gpurun_out/z_ar $CMD > /dev/null 2>&1
ncu -i gpurun_out/z_ar.ncu-rep --page raw --csv > gpurun_out/z_ar_raw.csv 2>/dev/null; python tools/ncu_summary.py gpurun_out/z_ar_raw.csv
ncu -i gpurun_out/z_ar.ncu-rep --page details --csv > gpurun_out/z_ar_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
