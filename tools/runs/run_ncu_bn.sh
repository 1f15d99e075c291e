NCU=/usr/local/cuda/bin/ncu
for dt in f32 bf16; do
timeout 600 $NCU -k regex:bn_partial_nhwc -s 2 -c 1 --set full --import-source on --clock-control none -o /tmp/ncu_bn_$dt python tools/bench_bn.py --only 256x64 --dtype $dt --iters 3 > gpurun_out/ncu_bn_$dt.log 2>&1
$NCU -i /tmp/ncu_bn_$dt.ncu-rep --page raw --csv > gpurun_out/ncu_bn_${dt}_raw.csv 2>/dev/null
$NCU -i /tmp/ncu_bn_$dt.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_bn_${dt}_sass.csv 2>/dev/null
done
