timeout 300 python -m pytest tests/test_gpu_virtual.py -q -x -k "bn or smoke" --timeout 200 2>&1 | tail -2
timeout 300 python tools/bench_bn.py --out gpurun_out/bn_f32.json > gpurun_out/bn_f32.txt 2>&1; cat gpurun_out/bn_f32.txt
timeout 300 python tools/bench_bn.py --dtype bf16 --out gpurun_out/bn_bf16.json > gpurun_out/bn_bf16.txt 2>&1; cat gpurun_out/bn_bf16.txt
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2"
$CMD > gpurun_out/p_plain.json 2> gpurun_out/p_plain.err && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv $CMD > /tmp/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ar_twoshot_dyn -s 3 -c 1 -o /tmp/prof_ar_dyn_n1 $CMD > /tmp/ncu_full.log 2>&1; echo ncu_rc=$?
ncu -i /tmp/prof_ar_dyn_n1.ncu-rep --page raw --csv > gpurun_out/prof_ar_dyn_n1_raw.csv 2>&1
ncu -i /tmp/prof_ar_dyn_n1.ncu-rep --page details --csv > gpurun_out/prof_ar_dyn_n1_details.csv 2>&1
ls -la /tmp/prof_ar_dyn_n1.ncu-rep; du -sh gpurun_out
