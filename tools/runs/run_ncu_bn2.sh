# ncu --set full of the fused BN statistics kernel (forward = launch 0, backward = launch 4 of bench_bn --iters 1), 1 GPU
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
for skip in 0 4; do
timeout 600 $NCU -k regex:bn_stats_fused -s $skip -c 1 --set full --import-source on --clock-control none -o gpurun_out/ncu_bn_$skip python tools/bench_bn.py --only 128x128 --dtype f32 --iters 1 > gpurun_out/ncu_bn_$skip.log 2>&1
$NCU -i gpurun_out/ncu_bn_$skip.ncu-rep --page raw --csv > gpurun_out/ncu_bn_${skip}_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/ncu_bn_${skip}_raw.csv
done
rm -f gpurun_out/ncu_bn_*.ncu-rep
