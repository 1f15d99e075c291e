# ncu --set full of the fused BN statistics kernel (forward, backward) on the largest SN-GAN layer, 1 GPU
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
for which in "0" "1"; do
timeout 600 $NCU -k "regex:bn_stats_fused<float, $which" -s 1 -c 1 --set full --import-source on --clock-control none -o gpurun_out/ncu_bn_$which python tools/bench_bn.py --only 128x128 --dtype f32 --iters 1 > gpurun_out/ncu_bn_$which.log 2>&1
$NCU -i gpurun_out/ncu_bn_$which.ncu-rep --page raw --csv > gpurun_out/ncu_bn_${which}_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/ncu_bn_${which}_raw.csv
done
